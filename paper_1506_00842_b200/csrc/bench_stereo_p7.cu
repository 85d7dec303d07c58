// bench_stereo_p7.cu — stereo kernel instances for memory-placement combos 14 and 15
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(14)
MLT_STEREO_INSTANTIATE(15)
