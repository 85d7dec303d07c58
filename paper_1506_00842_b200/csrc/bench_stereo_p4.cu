// bench_stereo_p4.cu — stereo kernel instances for memory-placement combos 8 and 9
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(8)
MLT_STEREO_INSTANTIATE(9)
