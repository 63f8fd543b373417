// ply.cu -- PLY vertex payload -> device SoA scene.
//
// Reference: scene.py:222-313 (load_ply): a binary little-endian vertex
// element whose properties are read by name and converted to fp64.  Here the
// host parses the header (ply.py) and uploads the raw payload once; this
// kernel unpacks it into the device scene layout (ssg_scene: mu, log_scale,
// rot fp64; sh, opacity_logits, beta, dir fp32).  A CTA stages 64 vertex
// records in shared memory with coalesced loads and then converts one
// destination component per thread: every property type of scene.py:210-216,
// absent optional fields read as 0 (skew_*, dir_*), opacity2 defaults to
// opacity (scene.py:297-298; the host passes opacity's slot for it).
#include <string.h>

#include "ssg_common.cuh"

namespace ssg {

constexpr int kPlyVerts = 64, kPlyThreads = 256;

__device__ __forceinline__ double ply_read(const unsigned char *p, int type) {
    switch (type) {
        case SSG_PLY_F32: { float v; memcpy(&v, p, 4); return (double)v; }
        case SSG_PLY_F64: { double v; memcpy(&v, p, 8); return v; }
        case SSG_PLY_I8: return (double)*(const int8_t *)p;
        case SSG_PLY_U8: return (double)*p;
        case SSG_PLY_I16: { int16_t v; memcpy(&v, p, 2); return (double)v; }
        case SSG_PLY_U16: { uint16_t v; memcpy(&v, p, 2); return (double)v; }
        case SSG_PLY_I32: { int32_t v; memcpy(&v, p, 4); return (double)v; }
        case SSG_PLY_U32: { uint32_t v; memcpy(&v, p, 4); return (double)v; }
        default: return 0.0;  // absent field
    }
}

struct PlyMap {
    int32_t off[18 + 48];
    int32_t type[18 + 48];
};

__global__ void __launch_bounds__(kPlyThreads) k_ply_unpack(const unsigned char *__restrict__ payload, int64_t n,
                                                            int32_t stride, int32_t ncomp, PlyMap map, int K,
                                                            ssg_params out) {
    extern __shared__ __align__(16) unsigned char s_rec[];
    const int64_t v0 = (int64_t)blockIdx.x * kPlyVerts;
    const int nv = (int)(n - v0 < kPlyVerts ? n - v0 : kPlyVerts);
    const size_t bytes = (size_t)nv * stride;
    const unsigned char *src = payload + (size_t)v0 * stride;
    if ((stride & 3) == 0 && (((uintptr_t)src) & 3) == 0) {
        const uint32_t *s4 = reinterpret_cast<const uint32_t *>(src);
        uint32_t *d4 = reinterpret_cast<uint32_t *>(s_rec);
        for (size_t q = threadIdx.x; q < bytes / 4; q += blockDim.x) d4[q] = s4[q];
    } else {
        for (size_t q = threadIdx.x; q < bytes; q += blockDim.x) s_rec[q] = src[q];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nv * ncomp; idx += blockDim.x) {
        const int v = idx / ncomp, c = idx - v * ncomp;
        const int64_t i = v0 + v;
        const int t = map.type[c];
        const double x = t < 0 ? 0.0 : ply_read(s_rec + (size_t)v * stride + map.off[c], t);
        // component order: mu 0-2, log_scale 3-5, rot 6-9, logits 10-11,
        // beta 12-14, dir 15-17, sh 18.. (coefficient-major, then RGB)
        if (c < 3) out.mu[3 * i + c] = x;
        else if (c < 6) out.log_scale[3 * i + c - 3] = x;
        else if (c < 10) out.rot[4 * i + c - 6] = x;
        else if (c < 12) out.opacity_logits[2 * i + c - 10] = (float)x;
        else if (c < 15) out.beta[3 * i + c - 12] = (float)x;
        else if (c < 18) out.dir[3 * i + c - 15] = (float)x;
        else out.sh[(size_t)i * 3 * K + (c - 18)] = (float)x;
    }
}

}  // namespace ssg

extern "C" int ssg_ply_unpack(const uint8_t *payload, int64_t n, int32_t stride, const int32_t *offsets,
                              const int32_t *types, int32_t sh_coeffs, const ssg_params *out, void *stream) {
    using namespace ssg;
    if (!offsets || !types || !out || n < 0 || stride < 1 || sh_coeffs < 1 || sh_coeffs > 16 ||
        out->sh_coeffs != sh_coeffs || (n > 0 && !payload))
        return SSG_ERR_INVALID_ARGUMENT;
    if ((size_t)stride * kPlyVerts > 200 * 1024) return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    const int ncomp = 18 + 3 * sh_coeffs;
    PlyMap map;
    for (int c = 0; c < ncomp; c++) {
        map.off[c] = offsets[c];
        map.type[c] = types[c];
        if (types[c] >= 0 && (offsets[c] < 0 || offsets[c] >= stride)) return SSG_ERR_INVALID_ARGUMENT;
    }
    const size_t smem = (size_t)stride * kPlyVerts;
    static DeviceOnce attr_once;  // function attributes are per device
    const cudaError_t e = attr_once.run(
        [](int) { return cudaFuncSetAttribute(k_ply_unpack, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    if (e != cudaSuccess) { set_error("cudaFuncSetAttribute(ply)", e); return SSG_ERR_CUDA; }
    const unsigned blocks = (unsigned)((n + kPlyVerts - 1) / kPlyVerts);
    k_ply_unpack<<<blocks, kPlyThreads, smem, (cudaStream_t)stream>>>(payload, n, stride, ncomp, map, sh_coeffs,
                                                                        *out);
    return check_launch("k_ply_unpack");
}
