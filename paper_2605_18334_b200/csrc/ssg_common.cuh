// ssg_common.cuh -- shared device code for the sm_100a skew-splat kernels.
//
// Reference semantics (pkg/src/skewsplat/...):
//   constants            kernel_math.py:17-20, raster/_core.pyx:24-29, tiles.py:16
//   per-primitive math   projection.py:151-235 (project_scene), scene.py:66-96,
//                        projection.py:97-123 (_project_eta), sh.py:25-109
// All preprocess math runs in fp64 registers: the depth and the tile
// rectangle decide the (bit-exact) instance lists.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/ssg_b200.h"

namespace ssg {
// One-time setup that belongs to a device (function attributes, __constant__
// uploads, occupancy-derived grid sizes): run once per device ordinal, under
// a mutex so concurrent first calls from several host threads are safe.
struct DeviceOnce {
    std::mutex mu;
    bool done[64] = {};
    // fn() -> cudaError_t runs on the calling thread's current device
    template <class F>
    cudaError_t run(F &&fn) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
        std::lock_guard<std::mutex> lock(mu);
        if (done[dev]) return cudaSuccess;
        e = fn(dev);
        if (e == cudaSuccess) done[dev] = true;
        return e;
    }
};
}  // namespace ssg

#define SSG_ALPHA_MAX 0.99f          // kernel_math.py:17
#define SSG_ALPHA_SKIP (1.0f / 255.0f) // kernel_math.py:18
#define SSG_T_STOP 1e-4f             // kernel_math.py:19
#define SSG_BETA_CLAMP 20.0          // kernel_math.py:20
#define SSG_SQRT1_2 0.70710678118654752f
#define SSG_TWO_OVER_SQRT_PI 1.12837916709551257f
#define SSG_LOG2E 1.44269504088896341f

namespace ssg {

void set_error(const char *what, cudaError_t e);
int check_launch(const char *what);

// ------------------------------------------------------------------ SH
__device__ __forceinline__ void sh_basis(int deg, double x, double y, double z, double *out) {
    // sh.py:25-54
    out[0] = 0.28209479177387814;
    if (deg < 1) return;
    out[1] = -0.4886025119029199 * y;
    out[2] = 0.4886025119029199 * z;
    out[3] = -0.4886025119029199 * x;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    out[4] = 1.0925484305920792 * xy;
    out[5] = -1.0925484305920792 * yz;
    out[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    out[7] = -1.0925484305920792 * xz;
    out[8] = 0.5462742152960396 * (xx - yy);
    if (deg < 3) return;
    out[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    out[10] = 2.890611442640554 * xy * z;
    out[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    out[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    out[14] = 1.445305721320277 * z * (xx - yy);
    out[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
}

// fp32 twin of sh_basis for the colour of the forward splat record
__device__ __forceinline__ void sh_basis_f(int deg, float x, float y, float z, float *out) {
    out[0] = 0.28209479177387814f;
    if (deg < 1) return;
    out[1] = -0.4886025119029199f * y;
    out[2] = 0.4886025119029199f * z;
    out[3] = -0.4886025119029199f * x;
    if (deg < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    out[4] = 1.0925484305920792f * xy;
    out[5] = -1.0925484305920792f * yz;
    out[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    out[7] = -1.0925484305920792f * xz;
    out[8] = 0.5462742152960396f * (xx - yy);
    if (deg < 3) return;
    out[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    out[10] = 2.890611442640554f * xy * z;
    out[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    out[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    out[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    out[14] = 1.445305721320277f * z * (xx - yy);
    out[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// ------------------------------------------------------ projection (fp64)
// Everything project_scene computes for one primitive that the forward and
// backward kernels need (projection.py:41-79 minus what can be rebuilt).
struct Proj {
    bool valid;
    double t[3];
    double tz;
    double mean2d[2];
    double J00, J02, J11, J12;
    double gate0, gate1;
    double T[6];       // Tmat = J R_w2c (2x3)
    double Sig[9];     // sigma_world
    double Rq[9];
    double qn[4], qnorm;
    double scale[3];
    double cov[4];     // cov_raw
    double inv_raw[4];
    double inv_dil[4];
    double det_raw, dd;
    double comp, radius;
    double sig[2];
    double eta[3], w[3], u[2], v[2], r;
    double pe;         // eta . Sigma eta (projection.py:103)
    bool fallback, clip0, clip1;
    double skew[2];
};

// The view-independent half of a primitive's projection: scene.py:66-96
// (normalised quaternion, rotation, Sigma_world = R S S^T R^T), the
// opacity sigmoids (kernel_math.py:158-165) and the camera-free part of
// _project_eta (w = Sigma eta, p = eta . w; projection.py:101-103).  A view
// batch computes it once per primitive (k_preprocess_forward_views); every
// operation is the one project_geometry performs, so the bits agree.
__device__ __forceinline__ void world_geometry(const double ls[3], const double q4[4], const float logit[2],
                                               const double eta[3], Proj &P) {
    double nrm = sqrt(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
    double w = q4[0] / nrm, x = q4[1] / nrm, y = q4[2] / nrm, z = q4[3] / nrm;
    P.qn[0] = w; P.qn[1] = x; P.qn[2] = y; P.qn[3] = z; P.qnorm = nrm;
    P.Rq[0] = 1 - 2 * (y * y + z * z);
    P.Rq[1] = 2 * (x * y - w * z);
    P.Rq[2] = 2 * (x * z + w * y);
    P.Rq[3] = 2 * (x * y + w * z);
    P.Rq[4] = 1 - 2 * (x * x + z * z);
    P.Rq[5] = 2 * (y * z - w * x);
    P.Rq[6] = 2 * (x * z - w * y);
    P.Rq[7] = 2 * (y * z + w * x);
    P.Rq[8] = 1 - 2 * (x * x + y * y);
#pragma unroll
    for (int j = 0; j < 3; j++) P.scale[j] = exp(ls[j]);
    double M[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) M[3 * a + b] = P.Rq[3 * a + b] * P.scale[b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            P.Sig[3 * a + b] = M[3 * a] * M[3 * b] + M[3 * a + 1] * M[3 * b + 1] + M[3 * a + 2] * M[3 * b + 2];
    // kernel_math.py:158-165
#pragma unroll
    for (int j = 0; j < 2; j++) {
        double l = (double)logit[j];
        double sgm;
        if (l >= 0) sgm = 1.0 / (1.0 + exp(-l));
        else { double ex = exp(l); sgm = ex / (1.0 + ex); }
        P.sig[j] = sgm;
    }
    // _project_eta (projection.py:97-123), camera-free part
#pragma unroll
    for (int j = 0; j < 3; j++) P.eta[j] = eta[j];
#pragma unroll
    for (int a = 0; a < 3; a++)
        P.w[a] = P.Sig[3 * a] * eta[0] + P.Sig[3 * a + 1] * eta[1] + P.Sig[3 * a + 2] * eta[2];
    P.pe = eta[0] * P.w[0] + eta[1] * P.w[1] + eta[2] * P.w[2];
}

// The camera-dependent half (projection.py:151-210 and the rest of
// _project_eta, projection.py:102, 104-121); needs world_geometry's fields.
__device__ __forceinline__ void view_geometry(const ssg_camera &cam, const double mu[3], Proj &P) {
    const double *R = cam.R;
    // projection.py:160 -- numpy/BLAS bits: fma(m2,R2,fma(m1,R1,m0*R0)) + t
#pragma unroll
    for (int c = 0; c < 3; c++)
        P.t[c] = __dadd_rn(__fma_rn(mu[2], R[3 * c + 2], __fma_rn(mu[1], R[3 * c + 1], __dmul_rn(mu[0], R[3 * c]))),
                           cam.t[c]);
    double depth = P.t[2];
    P.valid = depth > cam.near_plane;
    double tz = P.valid ? depth : 1.0;
    P.tz = tz;
    double limx = __dmul_rn(1.3, cam.tan_fovx), limy = __dmul_rn(1.3, cam.tan_fovy);
    double txz = __ddiv_rn(P.t[0], tz), tyz = __ddiv_rn(P.t[1], tz);
    P.gate0 = fabs(txz) <= limx ? 1.0 : 0.0;
    P.gate1 = fabs(tyz) <= limy ? 1.0 : 0.0;
    double txc = __dmul_rn(fmin(fmax(txz, -limx), limx), tz);
    double tyc = __dmul_rn(fmin(fmax(tyz, -limy), limy), tz);
    double tz2 = __dmul_rn(tz, tz);
    P.J00 = __ddiv_rn(cam.fx, tz);
    P.J02 = __ddiv_rn(__dmul_rn(-cam.fx, txc), tz2);
    P.J11 = __ddiv_rn(cam.fy, tz);
    P.J12 = __ddiv_rn(__dmul_rn(-cam.fy, tyc), tz2);
#pragma unroll
    for (int c = 0; c < 3; c++) {
        P.T[c] = __dadd_rn(__dmul_rn(P.J00, R[c]), __dmul_rn(P.J02, R[6 + c]));
        P.T[3 + c] = __dadd_rn(__dmul_rn(P.J11, R[3 + c]), __dmul_rn(P.J12, R[6 + c]));
    }
    double TS[6];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            TS[3 * a + b] = P.T[3 * a] * P.Sig[b] + P.T[3 * a + 1] * P.Sig[3 + b] + P.T[3 * a + 2] * P.Sig[6 + b];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++)
            P.cov[2 * a + b] = TS[3 * a] * P.T[3 * b] + TS[3 * a + 1] * P.T[3 * b + 1] + TS[3 * a + 2] * P.T[3 * b + 2];
    double cd0 = P.cov[0] + cam.s, cd1 = P.cov[1], cd2 = P.cov[2], cd3 = P.cov[3] + cam.s;
    P.det_raw = P.cov[0] * P.cov[3] - P.cov[1] * P.cov[2];
    double det_dil = cd0 * cd3 - cd1 * cd2;
    bool dok = det_dil > 1e-300;
    P.valid = P.valid && dok;
    P.dd = dok ? det_dil : 1.0;
    P.inv_dil[0] = cd3 / P.dd;
    P.inv_dil[3] = cd0 / P.dd;
    P.inv_dil[1] = -cd1 / P.dd;
    P.inv_dil[2] = -cd2 / P.dd;
    P.comp = sqrt((P.det_raw > 0.0 ? P.det_raw : 0.0) / P.dd);
    double mid = 0.5 * (cd0 + cd3);
    double disc = mid * mid - det_dil;
    double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);
    P.radius = 3.0 * sqrt(lam > 0.0 ? lam : 0.0);
    // projection.py:207 -- unclamped ratio, no contraction
    P.mean2d[0] = __dadd_rn(__dmul_rn(cam.fx, txz), cam.cx);
    P.mean2d[1] = __dadd_rn(__dmul_rn(cam.fy, tyz), cam.cy);
    // _project_eta (projection.py:102, 104-121)
#pragma unroll
    for (int a = 0; a < 2; a++) P.u[a] = P.T[3 * a] * P.w[0] + P.T[3 * a + 1] * P.w[1] + P.T[3 * a + 2] * P.w[2];
    bool ok = P.det_raw > 1e-300;
    double d = ok ? P.det_raw : 1.0;
    if (ok) {
        P.inv_raw[0] = P.cov[3] / d;
        P.inv_raw[3] = P.cov[0] / d;
        P.inv_raw[1] = -P.cov[1] / d;
        P.inv_raw[2] = -P.cov[2] / d;
    } else {
        P.inv_raw[0] = P.inv_raw[1] = P.inv_raw[2] = P.inv_raw[3] = 0.0;
    }
    P.v[0] = P.inv_raw[0] * P.u[0] + P.inv_raw[1] * P.u[1];
    P.v[1] = P.inv_raw[2] * P.u[0] + P.inv_raw[3] * P.u[1];
    double qq = P.pe - (P.u[0] * P.v[0] + P.u[1] * P.v[1]);
    double radicand = 1.0 + qq;
    P.fallback = (!ok) || (radicand <= 0.0);
    P.r = sqrt(P.fallback ? 1.0 : radicand);
    double s0 = P.fallback ? 0.0 : P.v[0] / P.r;
    double s1 = P.fallback ? 0.0 : P.v[1] / P.r;
    P.clip0 = fabs(s0) > SSG_BETA_CLAMP;
    P.clip1 = fabs(s1) > SSG_BETA_CLAMP;
    P.skew[0] = fmin(fmax(s0, -SSG_BETA_CLAMP), SSG_BETA_CLAMP);
    P.skew[1] = fmin(fmax(s1, -SSG_BETA_CLAMP), SSG_BETA_CLAMP);
}

// projection.py:151-210 and _project_eta projection.py:97-123.
// `mu`, `ls`, `q` fp64; `eta` = beta + dir (evaluated in fp64 from the fp32
// inputs), logits fp32.
__device__ __forceinline__ void project_geometry(const ssg_camera &cam, const double mu[3],
                                                 const double ls[3], const double q4[4],
                                                 const float logit[2], const double eta[3],
                                                 Proj &P) {
    world_geometry(ls, q4, logit, eta, P);
    view_geometry(cam, mu, P);
}

// ------------------------------------------------------------- tile rect
// raster/tiles.py:49-57: r = ceil(radius); [floor((m-r)/16), floor((m+r)/16)+1)
// clipped to the grid, evaluated in fp64 exactly as numpy does (no products,
// so no contraction can change it).  Returns the packed rect and the count.
__device__ __forceinline__ uint32_t tile_rect(double mx, double my, double radius, bool valid,
                                              int ntx, int nty, uint64_t &packed) {
    double r = ceil(radius);
    double fx0 = floor((mx - r) / 16.0), fx1 = floor((mx + r) / 16.0) + 1.0;
    double fy0 = floor((my - r) / 16.0), fy1 = floor((my + r) / 16.0) + 1.0;
    int x0 = (int)fmin(fmax(fx0, 0.0), (double)ntx);
    int x1 = (int)fmin(fmax(fx1, 0.0), (double)ntx);
    int y0 = (int)fmin(fmax(fy0, 0.0), (double)nty);
    int y1 = (int)fmin(fmax(fy1, 0.0), (double)nty);
    int nx = valid ? max(x1 - x0, 0) : 0;
    int ny = valid ? max(y1 - y0, 0) : 0;
    packed = (uint64_t)x0 | ((uint64_t)x1 << 16) | ((uint64_t)y0 << 32) | ((uint64_t)y1 << 48);
    return (uint32_t)(nx * ny);
}

// --------------------------------------------------------- blend math
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// erfc(x) for x >= 0 with ~1e-7 relative error everywhere (Chebyshev-fitted
// exp form, one rcp + one ex2).  The reference erf (raster/_core.pyx:57-74)
// is near-exact fp64; this keeps the *relative* error of E = 1 + erf(z) =
// erfc(-z) small even deep in the lower tail, which the alpha-skip test
// depends on.
__device__ __forceinline__ float erfc_pos(float x) {
    float t = fast_rcp(fmaf(0.5f, x, 1.0f));
    float p = fmaf(t, 0.17087277f, -0.82215223f);
    p = fmaf(t, p, 1.48851587f);
    p = fmaf(t, p, -1.13520398f);
    p = fmaf(t, p, 0.27886807f);
    p = fmaf(t, p, -0.18628806f);
    p = fmaf(t, p, 0.09678418f);
    p = fmaf(t, p, 0.37409196f);
    p = fmaf(t, p, 1.00002368f);
    p = fmaf(t, p, -1.26551223f);
    return t * fast_exp2((p - x * x) * SSG_LOG2E);
}

// E = 1 + erf(z) (raster/_core.pyx:137).  Skew-free splats never get here
// (the callers take the warp-uniform E = 1 path, erf(0) == 0 exactly as in
// kernel_math.py:79-80); a pixel with z == 0 of a skewed splat gets
// 1 - 3e-8 instead of 1, far below the fp32 blend tolerance.
__device__ __forceinline__ float skew_E(float z) {
    const float y = erfc_pos(fabsf(z));
    return z > 0.0f ? 2.0f - y : y;
}

// ------------------------------------------- fp64 reference alpha (rare path)
// raster/_core.pyx:33-35: the 33 Maclaurin coefficients (-1)^n / (n! (2n+1)),
// generated by the reference's own recurrence (fact *= n in fp64) and written
// out exactly (hex), so the table is bit-identical to the reference's.
static __constant__ double kRefErfCoef[33] = {
    0x1.0000000000000p+0,  -0x1.5555555555555p-2,  0x1.999999999999ap-4,   -0x1.8618618618618p-6,
    0x1.2f684bda12f68p-8,  -0x1.8d3018d3018d3p-11, 0x1.c01c01c01c01cp-14,  -0x1.bbd779334ef0bp-17,
    0x1.87a00187a0018p-20, -0x1.3777c55568ccdp-23, 0x1.c2e3054870b38p-27,  -0x1.2b67310aa9f3ap-30,
    0x1.6f448e13e85e1p-34, -0x1.a289ee7e40f74p-38, 0x1.bd577e658d020p-42,  -0x1.bc6250fb14231p-46,
    0x1.a173a167fba4dp-50, -0x1.7271cbe5863ecp-54, 0x1.377c2110f2083p-58,  -0x1.f1b4073b34a68p-63,
    0x1.7abd72258fb6ep-67, -0x1.13246abce1bddp-71, 0x1.7e6b81382cd42p-76,  -0x1.fd6bebd65107ap-81,
    0x1.45c0a838efe59p-85, -0x1.909c9de3a31c5p-90, 0x1.da7460554e5dap-95,  -0x1.0eef30fa10d2cp-99,
    0x1.2ac65385f79acp-104, -0x1.3e81bb5701ac5p-109, 0x1.4899fcdef0a8ep-114, -0x1.486eea20c2656p-119,
    0x1.3e53defc4e233p-124};
#define SSG_REF_SQRT1_2 0.7071067811865476           // raster/_core.pyx:27
#define SSG_REF_TWO_OVER_SQRT_PI 1.1283791670955126  // raster/_core.pyx:28
#define SSG_REF_SQRT_PI 1.7724538509055159           // raster/_core.pyx:29

// c_erf (raster/_core.pyx:57-74), operation for operation (no contraction).
static __device__ __noinline__ double ref_erf(double x) {
    const double ax = fabs(x);
    double y;
    if (ax <= 2.0) {
        const double u = __dmul_rn(ax, ax);
        double poly = 0.0;
        for (int k = 32; k >= 0; k--) poly = __dadd_rn(__dmul_rn(poly, u), kRefErfCoef[k]);
        y = __dmul_rn(__dmul_rn(SSG_REF_TWO_OVER_SQRT_PI, ax), poly);
    } else if (ax < 6.5) {
        double t = 0.0;
        for (int k = 48; k > 0; k--) t = __ddiv_rn(__dmul_rn(0.5, (double)k), __dadd_rn(ax, t));
        y = __dsub_rn(1.0, __ddiv_rn(__ddiv_rn(exp(-__dmul_rn(ax, ax)), SSG_REF_SQRT_PI), __dadd_rn(ax, t)));
    } else {
        y = 1.0;
    }
    return x < 0.0 ? -y : y;
}

// One pixel-instance pair of the reference blend in fp64 (raster/_core.pyx:
// 129-139 forward, :265-305 backward quantities) from the fp64 splat inputs:
// dx = px - mx with px = col + 0.5, power, z, E = 1 + erf(z), o = mix_opacity,
// G = exp(power), A = o G E (pre-clamp alpha).  skip = power > 0 (the
// reference skips before any erf, :133-135).  no_skew evaluates the skew
// term as zero (the plain-3DGS regression kernel).  Used only on the exact
// (redo) path, for pixels whose fp32 evaluation met an uncertain decision.
// erf is CUDA's (<= 2 ulp): like c_erf (ref_erf above, exposed through
// ssg_erf_probe) it is accurate to a few fp64 ulps, so alpha agrees with the
// reference's to ~1e-15 relative and a decision could differ only for an
// alpha that close to a threshold; c_erf's continued fraction (|z| > 2)
// would cost 48 fp64 divisions per pair.
struct RefPair {
    double dx, dy, power, z, E, o, G, A;
    bool skip;
};
static __device__ __noinline__ RefPair ref_pair(double pxc, double pyc, double mx, double my, const ssg_splat64 &e,
                                                bool no_skew) {
    RefPair r;
    r.dx = __dsub_rn(pxc, mx);
    r.dy = __dsub_rn(pyc, my);
    const double q = __dadd_rn(__dmul_rn(__dmul_rn(e.conic_a, r.dx), r.dx), __dmul_rn(__dmul_rn(e.conic_c, r.dy), r.dy));
    r.power = __dsub_rn(__dmul_rn(-0.5, q), __dmul_rn(__dmul_rn(e.conic_b, r.dx), r.dy));
    r.skip = r.power > 0.0;
    const double sx = no_skew ? 0.0 : e.skew_x, sy = no_skew ? 0.0 : e.skew_y;
    r.z = __dmul_rn(__dadd_rn(__dmul_rn(sx, r.dx), __dmul_rn(sy, r.dy)), SSG_REF_SQRT1_2);
    r.E = __dadd_rn(1.0, erf(r.z));
    r.o = __dmul_rn(0.5, __dadd_rn(__dadd_rn(e.o1, e.o2), __dmul_rn(__dsub_rn(e.o1, e.o2), __dsub_rn(r.E, 1.0))));
    r.G = exp(r.power);
    r.A = __dmul_rn(__dmul_rn(r.o, r.G), r.E);
    return r;
}

// Relative error bound of the blend's fp32 pre-clamp alpha against ref_pair
// for one primitive, as a function of the pair's Gaussian exponent:
// |A_fp32 / A_ref - 1| <= g0 + g1 |power|, valid wherever a decision can
// turn on it (|power| <= ln 510 < 6.3 and z >= -2.05, i.e. A >= 1/255 is
// reachable).  The full band g0 + 6.3 g1 serves the 1/255 skip test; the
// per-pair value bounds the transmittance error (high-alpha pairs sit near
// the centre, where |power| is small).  With eps = 2^-24, lambda_min/max the
// conic's eigenvalues, |d| <= c_d sqrt|power| (c_d = sqrt(2/lambda_min)) the
// pixel offset and sqrt|p| <= (1 + |p|)/2:
//  * power arithmetic: conic rounded to fp32 plus ~5 roundings over
//    |a| dx^2 + |c| dy^2 + 2|b dx dy| <= kappa * 2|power|, kappa =
//    (max(a,c) + |b|) / lambda_min  ->  8 eps kappa |p|;
//  * pixel offset: the tile-local fp32 mean (|m| <= |d| + 16.5) and
//    dx = px - m round by eps (|m| + |dx|) per axis; |grad power| <=
//    sqrt(2 lambda_max |p|)  ->  1.5 sqrt2 eps sqrt(2 lambda_max |p|) (2|d| + 16.5);
//  * skew factor E = erfc(-z): the z error (skew rounding, offsets) times
//    d ln E / dz <= 4.5 on z >= -2.05, plus the fp32 mix of o1, o2
//    (<= 4 eps omax / omin, cancellation);
//  * exp2 (2^-22) and its argument rounding (eps |power| log2e, into g1),
//    the o * G * E products: 6e-7; the skew factor's fast erfc (Chebyshev
//    fit, rcp + exp2 with argument (power - z^2) log2e): 2e-6 more.
// Returns g0 and writes g1 (both 1 for a degenerate conic: always uncertain).
__device__ __forceinline__ float alpha_band(double a, double b, double c, double sx, double sy, double o1, double o2,
                                            float *slope) {
    const double eps = 5.9604644775390625e-08, r2 = 1.4142135623730951;
    const double det = a * c - b * b;
    if (!(a > 0.0) || !(c > 0.0) || !(det > 0.0)) {
        *slope = 1.0f;
        return 1.0f;
    }
    const double half_tr = 0.5 * (a + c), disc = sqrt(0.25 * (a - c) * (a - c) + b * b);
    const double lmax = half_tr + disc, lmin = det / lmax;
    const double kappa = (fmax(a, c) + fabs(b)) / lmin;
    const double cd = sqrt(2.0 / lmin), gradc = sqrt(2.0 * lmax);
    double g0 = 6e-7, g1 = 8.0 * eps * kappa + 1.5 * eps;
    g1 += 1.5 * r2 * eps * gradc * 2.0 * cd;                 // offset x |d|: linear in |p|
    const double h = 1.5 * r2 * eps * gradc * 16.5;          // offset x tile: sqrt|p|
    g0 += 0.5 * h;
    g1 += 0.5 * h;
    if (sx != 0.0 || sy != 0.0) {
        const double s1 = fabs(sx) + fabs(sy);
        g0 += 2e-6 + 4.5 * (s1 * eps * 16.5 / r2 + 4.0 * eps);
        const double k = 4.5 * s1 * eps * 5.0 * cd / r2;     // sqrt|p| part
        g0 += 0.5 * k;
        g1 += 0.5 * k;
        const double omin = fmin(o1, o2), omax = fmax(o1, o2);
        g0 += omin > 0.0 ? 4.0 * eps * omax / omin : 1.0;
    }
    *slope = g1 < 1.0 ? (float)g1 : 1.0f;
    return g0 < 1.0 ? (float)g0 : 1.0f;
}

// 32-bit shared-window loads: keeps the address arithmetic out of the
// generic (cluster-aware) path the compiler otherwise rematerialises per use.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

}  // namespace ssg
