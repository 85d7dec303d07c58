python -m pytest tests/test_gpu_bench_kernels.py -x -q 2>&1 | tail -2
for c in "32 16 4 4 0 1 1 1 1" "32 8 1 4 0 1 1 0 1" "32 8 1 8 0 1 1 0 1" "64 4 1 8 0 1 0 0 1" "32 16 1 4 0 0 1 0 1" "128 2 1 16 0 1 1 0 1" "32 4 1 16 0 1 1 0 1" "64 8 1 4 0 1 1 0 1" "32 8 1 4 0 0 0 0 1" "32 8 2 4 0 1 1 0 1"; do python tools/bench_kernel_probe.py conv $c; done
