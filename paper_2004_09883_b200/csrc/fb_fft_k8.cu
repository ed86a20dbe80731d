// FFT pass kernels for line lengths 2^{8, 9} (see fb_fft_kern.cuh)
#include "fb_fft_kern.cuh"

namespace fb {
FB_FFT_INSTANTIATE_L(8)
FB_FFT_INSTANTIATE_L(9)
}  // namespace fb
