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
