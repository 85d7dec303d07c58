// bench_stereo_p2.cu — stereo kernel instances for memory-placement combos 4 and 5
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(4)
MLT_STEREO_INSTANTIATE(5)
