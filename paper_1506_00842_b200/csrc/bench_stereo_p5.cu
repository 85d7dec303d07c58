// bench_stereo_p5.cu — stereo kernel instances for memory-placement combos 10 and 11
// (flags = img_left<<3 | img_right<<2 | local_left<<1 | local_right).
#include "bench_stereo_kern.cuh"

MLT_STEREO_INSTANTIATE(10)
MLT_STEREO_INSTANTIATE(11)
