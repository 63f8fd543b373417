// serve.cu -- RGB8 quantisation of rendered frames on the device (SURVEY.md
// §8(f) row 4: the consumers of the view-batched forward).
//
// Reference: dataset.py:33-38 quantize_u8 -- np.rint(np.clip(img, 0, 1) *
// 255).astype(np.uint8), the one conversion every output path shares (PNG
// frames, trajectory.py:27-29; the render service payload, service.py:106-107).
// Evaluated in fp64 like numpy: clip, times 255, round half to even (rint).
#include "ssg_common.cuh"

namespace ssg {

template <typename T>
__global__ void k_quantize_u8(const T *__restrict__ src, int64_t n, uint8_t *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = fmin(fmax((double)src[i], 0.0), 1.0);
        dst[i] = (uint8_t)rint(x * 255.0);
    }
}

}  // namespace ssg

extern "C" int ssg_quantize_u8(const void *src, int32_t src_is_f64, int64_t n_values, uint8_t *dst, void *stream) {
    using namespace ssg;
    if (n_values < 0 || (n_values > 0 && (!src || !dst))) return SSG_ERR_INVALID_ARGUMENT;
    if (n_values == 0) return SSG_OK;
    const int64_t blocks64 = (n_values + 255) / 256;
    const unsigned blocks = (unsigned)(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
    if (src_is_f64)
        k_quantize_u8<double><<<blocks, 256, 0, (cudaStream_t)stream>>>((const double *)src, n_values, dst);
    else
        k_quantize_u8<float><<<blocks, 256, 0, (cudaStream_t)stream>>>((const float *)src, n_values, dst);
    return check_launch("k_quantize_u8");
}
