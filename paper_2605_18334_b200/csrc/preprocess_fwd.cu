// preprocess_fwd.cu -- K1: per-primitive EWA projection of 3D skew Gaussians.
//
// Replaces project_scene (reference projection.py:151-235) together with the
// per-primitive half of bin_arrays (raster/tiles.py:49-57: tile rectangle and
// count).  One thread per primitive, fp64 registers, coalesced row loads of
// the SoA scene.  Compiled with --fmad=false: the depth, mean2d and radius
// bits decide the instance lists, which must equal the reference's exactly,
// so no contraction may change an intermediate rounding (the reference's
// own fused op, the BLAS dot of projection.py:160, is spelled out with
// explicit __fma_rn in project_geometry).
#include "ssg_common.cuh"

namespace ssg {

#ifndef SSG_PF_MINB
#define SSG_PF_MINB 4
#endif

template <int DEG>
__global__ void __launch_bounds__(256, SSG_PF_MINB)
k_preprocess_forward(ssg_scene sc, ssg_camera cam, ssg_prim_buffers out, int ntx, int nty) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool fb = false;
    if (i < sc.n) {
        double mu[3], ls[3], q4[4], eta[3];
        float logit[2];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            mu[j] = sc.mu[3 * i + j];
            ls[j] = sc.log_scale[3 * i + j];
            eta[j] = (double)sc.beta[3 * i + j] + (double)sc.dir[3 * i + j];
        }
#pragma unroll
        for (int j = 0; j < 4; j++) q4[j] = sc.rot[4 * i + j];
        logit[0] = sc.opacity_logits[2 * i];
        logit[1] = sc.opacity_logits[2 * i + 1];

        Proj P;
        project_geometry(cam, mu, ls, q4, logit, eta, P);
        fb = P.fallback;

        // colour (projection.py:217-223): view direction (fp64), SH in fp32
        // (the colour only feeds the fp32 blend: ~1e-7 relative), +0.5,
        // floor at 0.  The (K,3) row is 16-byte aligned: float4 loads.
        double dv0 = mu[0] - cam.campos[0], dv1 = mu[1] - cam.campos[1], dv2 = mu[2] - cam.campos[2];
        double dn = sqrt(dv0 * dv0 + dv1 * dv1 + dv2 * dv2);
        double dns = dn > 1e-12 ? dn : 1.0;
        float basis[16];
        sh_basis_f(DEG, (float)(dv0 / dns), (float)(dv1 / dns), (float)(dv2 / dns), basis);
        float col[3] = {0.0f, 0.0f, 0.0f};
        if constexpr ((3 * K) % 4 == 0) {
            const float4 *shp4 = reinterpret_cast<const float4 *>(sc.sh + (size_t)i * (3 * K));
#pragma unroll
            for (int q = 0; q < 3 * K / 4; q++) {
                const float4 v = __ldg(shp4 + q);
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; u++) col[(4 * q + u) % 3] = fmaf(basis[(4 * q + u) / 3], e[u], col[(4 * q + u) % 3]);
            }
        } else {
            const float *shp = sc.sh + (size_t)i * (3 * K);
#pragma unroll
            for (int k = 0; k < K; k++)
#pragma unroll
                for (int c = 0; c < 3; c++) col[c] = fmaf(basis[k], __ldg(shp + 3 * k + c), col[c]);
        }

        ssg_splat s;
        s.mean_x = P.mean2d[0];
        s.mean_y = P.mean2d[1];
        s.conic_a = (float)P.inv_dil[0];
        s.conic_b = (float)P.inv_dil[1];
        s.conic_c = (float)P.inv_dil[3];
        s.skew_x = (float)P.skew[0];
        s.skew_y = (float)P.skew[1];
        s.o1 = (float)(P.sig[0] * P.comp);
        s.o2 = (float)(P.sig[1] * P.comp);
        s.r = fmaxf(col[0] + 0.5f, 0.0f);
        s.g = fmaxf(col[1] + 0.5f, 0.0f);
        s.b = fmaxf(col[2] + 0.5f, 0.0f);
        // fp64 twin of the blend inputs + the fp32 alpha error band
        ssg_splat64 e;
        e.conic_a = P.inv_dil[0];
        e.conic_b = P.inv_dil[1];
        e.conic_c = P.inv_dil[3];
        e.skew_x = P.skew[0];
        e.skew_y = P.skew[1];
        e.o1 = P.sig[0] * P.comp;   // projection.py:209-210
        e.o2 = P.sig[1] * P.comp;
        e.comp = P.comp;
        s.band0 = alpha_band(e.conic_a, e.conic_b, e.conic_c, e.skew_x, e.skew_y, e.o1, e.o2, &s.band1);
        // 64-byte records as four 16-byte stores each
        const int4 *src = reinterpret_cast<const int4 *>(&s);
        int4 *dst = reinterpret_cast<int4 *>(out.splat + i);
#pragma unroll
        for (int j = 0; j < 4; j++) dst[j] = src[j];
        const int4 *src64 = reinterpret_cast<const int4 *>(&e);
        int4 *dst64 = reinterpret_cast<int4 *>(out.splat64 + i);
#pragma unroll
        for (int j = 0; j < 4; j++) dst64[j] = src64[j];

        // tile rectangle and count (tiles.py:49-57)
        uint64_t rect;
        out.tile_count[i] = tile_rect(P.mean2d[0], P.mean2d[1], P.radius, P.valid, ntx, nty, rect);
        out.tile_rect[i] = rect;
        out.valid[i] = (uint8_t)P.valid;
        out.depth[i] = P.t[2];
        out.radius[i] = P.radius;
        // depth > near > 0 for valid primitives: the IEEE bits are monotone
        out.depth_key[i] = P.valid ? (uint64_t)__double_as_longlong(P.t[2]) : ~0ull;
    }
    // n_skew_fallback counts every primitive (projection.py:234)
    unsigned ballot = __ballot_sync(0xffffffffu, fb);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(out.n_skew_fallback, __popc(ballot));
}

}  // namespace ssg

extern "C" int ssg_preprocess_forward(const ssg_scene *scene, const ssg_camera *cam,
                                      const ssg_prim_buffers *out, void *stream) {
    using namespace ssg;
    if (!scene || !cam || !out) return SSG_ERR_INVALID_ARGUMENT;
    if (cam->width > SSG_MAX_IMAGE_DIM || cam->height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    if (cam->width < 1 || cam->height < 1) return SSG_ERR_INVALID_ARGUMENT;
    if (scene->sh_degree < 0 || scene->sh_degree > 3 ||
        scene->sh_coeffs != (scene->sh_degree + 1) * (scene->sh_degree + 1))
        return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(out->n_skew_fallback, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) { set_error("memset fallback", e); return SSG_ERR_CUDA; }
    if (scene->n == 0) return SSG_OK;
    int ntx = (cam->width + SSG_TILE - 1) / SSG_TILE, nty = (cam->height + SSG_TILE - 1) / SSG_TILE;
    unsigned blocks = (unsigned)((scene->n + 255) / 256);
    switch (scene->sh_degree) {
        case 0: k_preprocess_forward<0><<<blocks, 256, 0, st>>>(*scene, *cam, *out, ntx, nty); break;
        case 1: k_preprocess_forward<1><<<blocks, 256, 0, st>>>(*scene, *cam, *out, ntx, nty); break;
        case 2: k_preprocess_forward<2><<<blocks, 256, 0, st>>>(*scene, *cam, *out, ntx, nty); break;
        default: k_preprocess_forward<3><<<blocks, 256, 0, st>>>(*scene, *cam, *out, ntx, nty); break;
    }
    return check_launch("k_preprocess_forward");
}

namespace ssg {
// ------------------------------------------------------------ view batch
// K1 over a batch of up to SSG_MAX_BATCH_VIEWS cameras of one scene (the
// config-4 trajectory batch; the reference renders such batches one
// render_forward at a time, trajectory.py:12-31).  One thread per primitive
// reads the primitive's 304 bytes once for the whole batch instead of once
// per view: the geometry into registers, the view-independent part of the
// projection (world_geometry: rotation, Sigma_world, sigmoids, Sigma eta)
// computed once, the SH row staged into shared memory by cp.async (the
// block's rows are one contiguous range: fully coalesced 16-byte copies,
// landing while view 0's geometry runs).  Per view it runs view_geometry
// and the SH dot product with the same operation sequence as
// k_preprocess_forward, so every output is bit-identical to the
// single-view kernel's.  valid / depth / radius may be NULL per view
// (introspection-only outputs a throughput batch skips).
constexpr int kMvThreads = 128;
#ifndef SSG_MV_MINB
#define SSG_MV_MINB 1
#endif

// padded smem row stride (floats) of a 3K-float SH row: conflict-free
// LDS.128 when 3K % 4 == 0 (an odd number of 16-byte units per row), an odd
// stride for scalar rows
__host__ __device__ constexpr int mv_sh_stride(int K3) {
    return (K3 % 4 == 0) ? ((K3 / 4) % 2 == 0 ? K3 + 4 : K3) : K3;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct MvArgs {
    ssg_camera cam[SSG_MAX_BATCH_VIEWS];
    ssg_prim_buffers out[SSG_MAX_BATCH_VIEWS];
    int ntx[SSG_MAX_BATCH_VIEWS], nty[SSG_MAX_BATCH_VIEWS];
    int nv;
};

template <int DEG>
__global__ void __launch_bounds__(kMvThreads, SSG_MV_MINB)
k_preprocess_forward_views(ssg_scene sc, const __grid_constant__ MvArgs a) {
    constexpr int K = (DEG + 1) * (DEG + 1), K3 = 3 * K, S = mv_sh_stride(K3);
    extern __shared__ __align__(16) float s_sh[];  // [kMvThreads][S]
    const int64_t base = (int64_t)blockIdx.x * kMvThreads;
    const int rows = (int)(sc.n - base < kMvThreads ? sc.n - base : kMvThreads);
    const int tid = threadIdx.x;
    // stage the block's SH rows (one contiguous range of rows * K3 floats)
    if constexpr (K3 % 4 == 0) {
        const float *src = sc.sh + base * K3;
        for (int e = tid; e < rows * (K3 / 4); e += kMvThreads) {
            const int r = e / (K3 / 4), c = e - r * (K3 / 4);
            cp_async16(s_sh + r * S + 4 * c, src + 4 * (int64_t)e);
        }
    } else {
        const float *src = sc.sh + base * K3;
        for (int e = tid; e < rows * K3; e += kMvThreads) {
            const int r = e / K3, c = e - r * K3;
            cp_async4(s_sh + r * S + c, src + e);
        }
    }
    const int64_t i = base + tid;
    const bool live = tid < rows;
    double mu[3] = {0.0, 0.0, 0.0};
    Proj P;
    if (live) {
        double ls[3], q4[4], eta[3];
        float logit[2];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            mu[j] = sc.mu[3 * i + j];
            ls[j] = sc.log_scale[3 * i + j];
            eta[j] = (double)sc.beta[3 * i + j] + (double)sc.dir[3 * i + j];
        }
#pragma unroll
        for (int j = 0; j < 4; j++) q4[j] = sc.rot[4 * i + j];
        logit[0] = sc.opacity_logits[2 * i];
        logit[1] = sc.opacity_logits[2 * i + 1];
        world_geometry(ls, q4, logit, eta, P);
    }
    bool staged = false;
    for (int v = 0; v < a.nv; v++) {
        const ssg_camera &cam = a.cam[v];
        const ssg_prim_buffers &out = a.out[v];
        bool fb = false;
        if (live) view_geometry(cam, mu, P);
        if (!staged) {  // block-uniform: the SH rows have landed
            cp_async_wait_all();
            __syncthreads();
            staged = true;
        }
        if (live) {
            fb = P.fallback;
            double dv0 = mu[0] - cam.campos[0], dv1 = mu[1] - cam.campos[1], dv2 = mu[2] - cam.campos[2];
            double dn = sqrt(dv0 * dv0 + dv1 * dv1 + dv2 * dv2);
            double dns = dn > 1e-12 ? dn : 1.0;
            float basis[16];
            sh_basis_f(DEG, (float)(dv0 / dns), (float)(dv1 / dns), (float)(dv2 / dns), basis);
            float col[3] = {0.0f, 0.0f, 0.0f};
            const float *row = s_sh + tid * S;
            if constexpr (K3 % 4 == 0) {
#pragma unroll
                for (int q = 0; q < K3 / 4; q++) {
                    const float4 v4 = *reinterpret_cast<const float4 *>(row + 4 * q);
                    const float e[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        col[(4 * q + u) % 3] = fmaf(basis[(4 * q + u) / 3], e[u], col[(4 * q + u) % 3]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; k++)
#pragma unroll
                    for (int c = 0; c < 3; c++) col[c] = fmaf(basis[k], row[3 * k + c], col[c]);
            }
            ssg_splat s;
            s.mean_x = P.mean2d[0];
            s.mean_y = P.mean2d[1];
            s.conic_a = (float)P.inv_dil[0];
            s.conic_b = (float)P.inv_dil[1];
            s.conic_c = (float)P.inv_dil[3];
            s.skew_x = (float)P.skew[0];
            s.skew_y = (float)P.skew[1];
            s.o1 = (float)(P.sig[0] * P.comp);
            s.o2 = (float)(P.sig[1] * P.comp);
            s.r = fmaxf(col[0] + 0.5f, 0.0f);
            s.g = fmaxf(col[1] + 0.5f, 0.0f);
            s.b = fmaxf(col[2] + 0.5f, 0.0f);
            ssg_splat64 e;
            e.conic_a = P.inv_dil[0];
            e.conic_b = P.inv_dil[1];
            e.conic_c = P.inv_dil[3];
            e.skew_x = P.skew[0];
            e.skew_y = P.skew[1];
            e.o1 = P.sig[0] * P.comp;
            e.o2 = P.sig[1] * P.comp;
            e.comp = P.comp;
            s.band0 = alpha_band(e.conic_a, e.conic_b, e.conic_c, e.skew_x, e.skew_y, e.o1, e.o2, &s.band1);
            const int4 *src = reinterpret_cast<const int4 *>(&s);
            int4 *dst = reinterpret_cast<int4 *>(out.splat + i);
#pragma unroll
            for (int j = 0; j < 4; j++) dst[j] = src[j];
            const int4 *src64 = reinterpret_cast<const int4 *>(&e);
            int4 *dst64 = reinterpret_cast<int4 *>(out.splat64 + i);
#pragma unroll
            for (int j = 0; j < 4; j++) dst64[j] = src64[j];
            uint64_t rect;
            out.tile_count[i] = tile_rect(P.mean2d[0], P.mean2d[1], P.radius, P.valid, a.ntx[v], a.nty[v], rect);
            out.tile_rect[i] = rect;
            if (out.valid) out.valid[i] = (uint8_t)P.valid;
            if (out.depth) out.depth[i] = P.t[2];
            if (out.radius) out.radius[i] = P.radius;
            out.depth_key[i] = P.valid ? (uint64_t)__double_as_longlong(P.t[2]) : ~0ull;
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, fb);
        if ((tid & 31) == 0 && ballot) atomicAdd(out.n_skew_fallback, __popc(ballot));
    }
}

template <int DEG>
static int launch_views(const ssg_scene &sc, const MvArgs &a, cudaStream_t st) {
    constexpr int K3 = 3 * (DEG + 1) * (DEG + 1);
    const size_t smem = sizeof(float) * (size_t)kMvThreads * mv_sh_stride(K3);
    static DeviceOnce attr_once;  // function attributes are per device
    const cudaError_t e = attr_once.run([smem](int) {
        return cudaFuncSetAttribute(k_preprocess_forward_views<DEG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    });
    if (e != cudaSuccess) { set_error("cudaFuncSetAttribute(preprocess views)", e); return SSG_ERR_CUDA; }
    const unsigned blocks = (unsigned)((sc.n + kMvThreads - 1) / kMvThreads);
    k_preprocess_forward_views<DEG><<<blocks, kMvThreads, smem, st>>>(sc, a);
    return check_launch("k_preprocess_forward_views");
}

}  // namespace ssg

extern "C" int ssg_preprocess_forward_views(const ssg_scene *scene, const ssg_camera *cams,
                                            const ssg_prim_buffers *outs, int32_t n_views, void *stream) {
    using namespace ssg;
    if (!scene || !cams || !outs || n_views < 1 || n_views > SSG_MAX_BATCH_VIEWS) return SSG_ERR_INVALID_ARGUMENT;
    if (scene->sh_degree < 0 || scene->sh_degree > 3 ||
        scene->sh_coeffs != (scene->sh_degree + 1) * (scene->sh_degree + 1))
        return SSG_ERR_INVALID_ARGUMENT;
    MvArgs a;
    a.nv = n_views;
    cudaStream_t st = (cudaStream_t)stream;
    for (int v = 0; v < n_views; v++) {
        const ssg_camera &c = cams[v];
        if (c.width > SSG_MAX_IMAGE_DIM || c.height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
        if (c.width < 1 || c.height < 1) return SSG_ERR_INVALID_ARGUMENT;
        const ssg_prim_buffers &o = outs[v];
        if (!o.splat || !o.splat64 || !o.depth_key || !o.tile_count || !o.tile_rect || !o.n_skew_fallback)
            return SSG_ERR_INVALID_ARGUMENT;
        a.cam[v] = c;
        a.out[v] = o;
        a.ntx[v] = (c.width + SSG_TILE - 1) / SSG_TILE;
        a.nty[v] = (c.height + SSG_TILE - 1) / SSG_TILE;
        cudaError_t e = cudaMemsetAsync(o.n_skew_fallback, 0, sizeof(int32_t), st);
        if (e != cudaSuccess) { set_error("memset fallback", e); return SSG_ERR_CUDA; }
    }
    if (scene->n == 0) return SSG_OK;
    if (scene->sh_degree > 0 && ((uintptr_t)scene->sh & 15) != 0 && (3 * scene->sh_coeffs) % 4 == 0)
        return SSG_ERR_INVALID_ARGUMENT;  // 16-byte cp.async needs aligned rows
    switch (scene->sh_degree) {
        case 0: return launch_views<0>(*scene, a, st);
        case 1: return launch_views<1>(*scene, a, st);
        case 2: return launch_views<2>(*scene, a, st);
        default: return launch_views<3>(*scene, a, st);
    }
}

// Screen records from caller fp64 arrays (the plugin slot's inputs,
// raster/_core.pyx:169-177): the fp32 splat (+ its alpha band) and the fp64
// twin the threshold path reads.
namespace ssg {
__global__ void k_pack_splats(int64_t n, const double *__restrict__ mean2d, const double *__restrict__ conic,
                              const double *__restrict__ skew2d, const double *__restrict__ opair,
                              const double *__restrict__ color, ssg_splat *__restrict__ splat,
                              ssg_splat64 *__restrict__ splat64) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ssg_splat64 e;
    e.conic_a = conic[3 * i];
    e.conic_b = conic[3 * i + 1];
    e.conic_c = conic[3 * i + 2];
    e.skew_x = skew2d[2 * i];
    e.skew_y = skew2d[2 * i + 1];
    e.o1 = opair[2 * i];
    e.o2 = opair[2 * i + 1];
    e.comp = 0.0;
    ssg_splat s;
    s.mean_x = mean2d[2 * i];
    s.mean_y = mean2d[2 * i + 1];
    s.conic_a = (float)e.conic_a;
    s.conic_b = (float)e.conic_b;
    s.conic_c = (float)e.conic_c;
    s.skew_x = (float)e.skew_x;
    s.skew_y = (float)e.skew_y;
    s.o1 = (float)e.o1;
    s.o2 = (float)e.o2;
    s.r = (float)color[3 * i];
    s.g = (float)color[3 * i + 1];
    s.b = (float)color[3 * i + 2];
    s.band0 = alpha_band(e.conic_a, e.conic_b, e.conic_c, e.skew_x, e.skew_y, e.o1, e.o2, &s.band1);
    splat[i] = s;
    splat64[i] = e;
}
}  // namespace ssg

extern "C" int ssg_pack_splats(int64_t n, const double *mean2d, const double *conic, const double *skew2d,
                               const double *opair, const double *color, ssg_splat *splat, ssg_splat64 *splat64,
                               void *stream) {
    using namespace ssg;
    if (n < 0 || (n > 0 && (!mean2d || !conic || !skew2d || !opair || !color || !splat || !splat64)))
        return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    k_pack_splats<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, mean2d, conic, skew2d, opair,
                                                                               color, splat, splat64);
    return check_launch("k_pack_splats");
}
