// FFT pass kernels for line lengths 2^{0, 1, 2, 3, 4, 5, 6, 7} (see fb_fft_kern.cuh)
#include "fb_fft_kern.cuh"

namespace fb {
FB_FFT_INSTANTIATE_L(0)
FB_FFT_INSTANTIATE_L(1)
FB_FFT_INSTANTIATE_L(2)
FB_FFT_INSTANTIATE_L(3)
FB_FFT_INSTANTIATE_L(4)
FB_FFT_INSTANTIATE_L(5)
FB_FFT_INSTANTIATE_L(6)
FB_FFT_INSTANTIATE_L(7)
}  // namespace fb
