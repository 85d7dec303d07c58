#!/bin/bash
# Build sweep-kernel variants for A/B timing on the GPU box:
#   tools/build_variants.sh tag:THREADS:INNER:OB:MINB[:DEF=V,DEF=V...] ...
# -> variants/<tag>/libmltune_b200.so (select with MLTUNE_B200_LIB=...)
# Only the core translation units are rebuilt with the variant's defines; the
# benchmark-kernel objects come from the regular build (make -C .../csrc first).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1506_00842_b200/csrc
BENCH_OBJS=$(ls $ROOT/build/bench_*.o)
for spec in "$@"; do
  IFS=: read tag thr inner ob minb extra <<< "$spec"
  out=$ROOT/variants/$tag
  mkdir -p $out
  defs="-DMLT_THREADS=$thr -DMLT_INNER=$inner -DMLT_OB=$ob -DMLT_MINB=$minb"
  for d in ${extra//,/ }; do defs="$defs -D$d"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Xcompiler -fvisibility=hidden -I$ROOT/include $defs -Xptxas -v -o $out/libmltune_b200.so $SRC/abi.cu $SRC/host_format.cu $SRC/host_rng.cu \
    $SRC/predict.cu $SRC/select.cu $SRC/surrogate.cu $SRC/sweep.cu $SRC/train.cu $BENCH_OBJS 2> $out/ptxas.txt &
done
wait
for spec in "$@"; do
  IFS=: read tag rest <<< "$spec"
  echo "$tag: $(grep -A1 'k_sweepILi3' $ROOT/variants/$tag/ptxas.txt | grep -o 'Used [0-9]* registers' | head -1) $(grep -A1 'k_sweepILi3' $ROOT/variants/$tag/ptxas.txt | grep -o '[0-9]* bytes spill stores' | head -1)"
done
