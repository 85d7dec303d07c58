// bench_stereo_p0.cu — stereo kernel instances for memory-placement combos 0 and 1
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(0)
MLT_STEREO_INSTANTIATE(1)
