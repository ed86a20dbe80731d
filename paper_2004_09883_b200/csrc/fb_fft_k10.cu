// FFT pass kernels for line lengths 2^{10} (see fb_fft_kern.cuh)
#include "fb_fft_kern.cuh"

namespace fb {
FB_FFT_INSTANTIATE_L(10)
}  // namespace fb
