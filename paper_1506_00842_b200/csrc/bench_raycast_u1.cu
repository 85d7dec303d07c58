// bench_raycast_u1.cu — raycasting kernel instances with ray-loop unroll factor 1
// (all 32 memory-placement / interleaving combinations).
#include "bench_raycast_kern.cuh"

MLT_RAY_INSTANTIATE(1)
