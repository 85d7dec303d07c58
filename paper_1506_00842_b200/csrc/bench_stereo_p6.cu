// bench_stereo_p6.cu — stereo kernel instances for memory-placement combos 12 and 13
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(12)
MLT_STEREO_INSTANTIATE(13)
