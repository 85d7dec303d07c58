#!/bin/bash
# Build sweep-kernel tiling variants for A/B timing on the GPU box:
#   tools/build_variants.sh tag:THREADS:INNER:OB:MINB ...
# -> build/variants/<tag>/libmltune_b200.so (select with MLTUNE_B200_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1506_00842_b200/csrc
for spec in "$@"; do
  IFS=: read tag thr inner ob minb <<< "$spec"
  out=$ROOT/build/variants/$tag
  mkdir -p $out
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Xcompiler -fvisibility=hidden -I$ROOT/include -DMLT_THREADS=$thr -DMLT_INNER=$inner -DMLT_OB=$ob \
    -DMLT_MINB=$minb -Xptxas -v -o $out/libmltune_b200.so $SRC/abi.cu $SRC/predict.cu $SRC/select.cu \
    $SRC/sweep.cu $SRC/train.cu 2> $out/ptxas.txt &
done
wait
for spec in "$@"; do
  IFS=: read tag rest <<< "$spec"
  echo "$tag: $(grep -A1 'k_sweepILi3' $ROOT/build/variants/$tag/ptxas.txt | grep -o 'Used [0-9]* registers' | head -1) $(grep -A1 'k_sweepILi3' $ROOT/build/variants/$tag/ptxas.txt | grep -o '[0-9]* bytes spill stores' | head -1)"
done
