// bench_stereo_p3.cu — stereo kernel instances for memory-placement combos 6 and 7
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(6)
MLT_STEREO_INSTANTIATE(7)
