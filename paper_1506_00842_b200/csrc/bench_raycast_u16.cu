// bench_raycast_u16.cu — raycasting kernel instances with ray-loop unroll factor 16
// (all 32 memory-placement / interleaving combinations).
#include "bench_raycast_kern.cuh"

MLT_RAY_INSTANTIATE(16)
