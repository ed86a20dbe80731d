// FFT pass kernels for line lengths 2^{13, 14} (see fb_fft_kern.cuh)
#include "fb_fft_kern.cuh"

namespace fb {
FB_FFT_INSTANTIATE_L(13)
FB_FFT_INSTANTIATE_L(14)
}  // namespace fb
