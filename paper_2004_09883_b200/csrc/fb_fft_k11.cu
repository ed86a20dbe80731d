// FFT pass kernels for line lengths 2^{11} (see fb_fft_kern.cuh)
#include "fb_fft_kern.cuh"

namespace fb {
FB_FFT_INSTANTIATE_L(11)
}  // namespace fb
