// bench_stereo_p1.cu — stereo kernel instances for memory-placement combos 2 and 3
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(2)
MLT_STEREO_INSTANTIATE(3)
