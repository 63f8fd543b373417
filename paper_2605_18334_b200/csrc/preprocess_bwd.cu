// preprocess_bwd.cu -- K8: chain screen-space gradients back to primitive
// parameters, plus the densification statistics g_uv and g_z.
//
// Reference: projection.py:255-379 (projection_backward), with
// _project_eta_vjp projection.py:126-148, _quat_backward projection.py:382-420
// and sh_basis_grad sh.py:57-103.  Like the reference's backward, the
// forward geometry is recomputed (not cached) from the scene; one thread per
// primitive, fp64 registers, fp32 outputs.
#include "ssg_common.cuh"

namespace ssg {

// sum_k w[k] * d basis_k / d dir  (sh.py:57-103 contracted with w), without
// materialising the (K,3) basis-gradient table.
__device__ __forceinline__ void sh_dot_grad(int deg, double x, double y, double z, const double *w,
                                            double *g) {
    const double C1 = 0.4886025119029199;
    g[0] = -C1 * w[3];
    g[1] = -C1 * w[1];
    g[2] = C1 * w[2];
    if (deg < 2) return;
    const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                 C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    g[0] += C20 * y * w[4] + C22 * (-2.0 * x) * w[6] + C23 * z * w[7] + C24 * (2.0 * x) * w[8];
    g[1] += C20 * x * w[4] + C21 * z * w[5] + C22 * (-2.0 * y) * w[6] + C24 * (-2.0 * y) * w[8];
    g[2] += C21 * y * w[5] + C22 * (4.0 * z) * w[6] + C23 * x * w[7];
    if (deg < 3) return;
    const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                 C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                 C36 = -0.5900435899266435;
    const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    g[0] += C30 * 6.0 * xy * w[9] + C31 * yz * w[10] + C32 * (-2.0 * xy) * w[11] + C33 * (-6.0 * xz) * w[12] +
            C34 * (4.0 * zz - 3.0 * xx - yy) * w[13] + C35 * (2.0 * xz) * w[14] + C36 * (3.0 * xx - 3.0 * yy) * w[15];
    g[1] += C30 * (3.0 * xx - 3.0 * yy) * w[9] + C31 * xz * w[10] + C32 * (4.0 * zz - xx - 3.0 * yy) * w[11] +
            C33 * (-6.0 * yz) * w[12] + C34 * (-2.0 * xy) * w[13] + C35 * (-2.0 * yz) * w[14] + C36 * (-6.0 * xy) * w[15];
    g[2] += C31 * xy * w[10] + C32 * (8.0 * yz) * w[11] + C33 * (6.0 * zz - 3.0 * xx - 3.0 * yy) * w[12] +
            C34 * (8.0 * xz) * w[13] + C35 * (xx - yy) * w[14];
}

// fp32 twin of sh_dot_grad (the SH chain runs in fp32, like the forward colour)
__device__ __forceinline__ void sh_dot_grad_f(int deg, float x, float y, float z, const float *w,
                                              float *g) {
    const float C1 = 0.4886025119029199f;
    g[0] = -C1 * w[3];
    g[1] = -C1 * w[1];
    g[2] = C1 * w[2];
    if (deg < 2) return;
    const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
                 C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
    g[0] += C20 * y * w[4] + C22 * (-2.0f * x) * w[6] + C23 * z * w[7] + C24 * (2.0f * x) * w[8];
    g[1] += C20 * x * w[4] + C21 * z * w[5] + C22 * (-2.0f * y) * w[6] + C24 * (-2.0f * y) * w[8];
    g[2] += C21 * y * w[5] + C22 * (4.0f * z) * w[6] + C23 * x * w[7];
    if (deg < 3) return;
    const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
                 C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                 C36 = -0.5900435899266435f;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    g[0] += C30 * 6.0f * xy * w[9] + C31 * yz * w[10] + C32 * (-2.0f * xy) * w[11] + C33 * (-6.0f * xz) * w[12] +
            C34 * (4.0f * zz - 3.0f * xx - yy) * w[13] + C35 * (2.0f * xz) * w[14] + C36 * (3.0f * xx - 3.0f * yy) * w[15];
    g[1] += C30 * (3.0f * xx - 3.0f * yy) * w[9] + C31 * xz * w[10] + C32 * (4.0f * zz - xx - 3.0f * yy) * w[11] +
            C33 * (-6.0f * yz) * w[12] + C34 * (-2.0f * xy) * w[13] + C35 * (-2.0f * yz) * w[14] + C36 * (-6.0f * xy) * w[15];
    g[2] += C31 * xy * w[10] + C32 * (8.0f * yz) * w[11] + C33 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * w[12] +
            C34 * (8.0f * xz) * w[13] + C35 * (xx - yy) * w[14];
}

#ifndef SSG_PB_MINB
#define SSG_PB_MINB 4
#endif

// Geometry part of one primitive: every output but d_sh; the geometric
// d_mu is returned (the SH chain adds its view-direction term).
__device__ __forceinline__ void prep_geom(const ssg_scene &sc, const ssg_camera &cam, const ssg_grad_buffers &gr,
                                          int64_t i, float *dmu_out) {
    const float4 *sg4 = reinterpret_cast<const float4 *>(gr.screen + 12 * i);
    const float4 s0 = sg4[0], s1 = sg4[1], s2 = sg4[2];
    const bool zero = s0.x == 0.0f && s0.y == 0.0f && s0.z == 0.0f && s0.w == 0.0f && s1.x == 0.0f &&
                      s1.y == 0.0f && s1.z == 0.0f && s1.w == 0.0f && s2.x == 0.0f && s2.y == 0.0f &&
                      s2.z == 0.0f && s2.w == 0.0f;
    if (zero) {  // no instance touched a pixel with dL != 0: every output is 0
#pragma unroll
        for (int j = 0; j < 3; j++) dmu_out[j] = gr.d_log_scale[3 * i + j] = gr.d_eta[3 * i + j] = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; j++) gr.d_rot[4 * i + j] = 0.0f;
        gr.d_opacity_logits[2 * i] = gr.d_opacity_logits[2 * i + 1] = 0.0f;
        gr.g_uv[i] = 0.0f;
        gr.g_z[i] = 0.0f;
        return;
    }
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

    if (!P.valid) {  // zero_invalid, projection.py:368-379; g_z -> 0 (:349)
#pragma unroll
        for (int j = 0; j < 3; j++) dmu_out[j] = gr.d_log_scale[3 * i + j] = gr.d_eta[3 * i + j] = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; j++) gr.d_rot[4 * i + j] = 0.0f;
        gr.d_opacity_logits[2 * i] = gr.d_opacity_logits[2 * i + 1] = 0.0f;
        gr.g_uv[i] = 0.0f;
        gr.g_z[i] = 0.0f;
        return;
    }
    const double dm0 = s0.x, dm1 = s0.y;
    const double dc0 = s0.z, dc1 = s0.w, dc2 = s1.x;
    const double dsk0 = s1.y, dsk1 = s1.z;
    const double dop0 = s1.w, dop1 = s2.x;
    const double fx = cam.fx, fy = cam.fy, tz = P.tz;
    const double *R = cam.R;

    // opacity pair (projection.py:278-281)
    gr.d_opacity_logits[2 * i] = (float)(dop0 * P.comp * P.sig[0] * (1.0 - P.sig[0]));
    gr.d_opacity_logits[2 * i + 1] = (float)(dop1 * P.comp * P.sig[1] * (1.0 - P.sig[1]));
    const double d_comp = dop0 * P.sig[0] + dop1 * P.sig[1];

    // conic -> cov_dil: G_dil = -C Gc C (:283-289)
    const double *C = P.inv_dil;
    const double Gc[4] = {dc0, 0.5 * dc1, 0.5 * dc1, dc2};
    double CG[4], Gdil[4], Graw[4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) CG[2 * a + b] = C[2 * a] * Gc[b] + C[2 * a + 1] * Gc[2 + b];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) Gdil[2 * a + b] = -(CG[2 * a] * C[b] + CG[2 * a + 1] * C[2 + b]);
    // comp = sqrt(det_raw / det_dil) (:291-295)
    const double half_comp = P.det_raw > 0.0 ? 0.5 * P.comp * d_comp : 0.0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        Graw[j] = half_comp * P.inv_raw[j];
        Gdil[j] -= half_comp * P.inv_dil[j];
    }
    // skew VJP (:297-303, projection.py:126-148)
    double g0 = P.clip0 ? 0.0 : dsk0, g1 = P.clip1 ? 0.0 : dsk1;
    if (P.fallback) g0 = g1 = 0.0;
    const double r3 = P.r * P.r * P.r;
    const double s_q = -(g0 * P.v[0] + g1 * P.v[1]) / (2.0 * r3);
    const double gv0 = g0 / P.r, gv1 = g1 / P.r;
    double gM[4];
    gM[0] = gv0 * P.u[0] - s_q * (P.u[0] * P.u[0]);
    gM[1] = gv0 * P.u[1] - s_q * (P.u[0] * P.u[1]);
    gM[2] = gv1 * P.u[0] - s_q * (P.u[1] * P.u[0]);
    gM[3] = gv1 * P.u[1] - s_q * (P.u[1] * P.u[1]);
    const double *Mi = P.inv_raw;
    const double gu0 = (Mi[0] * gv0 + Mi[1] * gv1) - 2.0 * s_q * P.v[0];
    const double gu1 = (Mi[2] * gv0 + Mi[3] * gv1) - 2.0 * s_q * P.v[1];
    double MgM[4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) MgM[2 * a + b] = Mi[2 * a] * gM[b] + Mi[2 * a + 1] * gM[2 + b];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) Graw[2 * a + b] += -(MgM[2 * a] * Mi[b] + MgM[2 * a + 1] * Mi[2 + b]);
    double gw[3];
#pragma unroll
    for (int b = 0; b < 3; b++) gw[b] = P.T[b] * gu0 + P.T[3 + b] * gu1;
    double geta[3];
#pragma unroll
    for (int b = 0; b < 3; b++)
        geta[b] = (P.Sig[b] * gw[0] + P.Sig[3 + b] * gw[1] + P.Sig[6 + b] * gw[2]) + 2.0 * s_q * P.w[b];
#pragma unroll
    for (int j = 0; j < 4; j++) Graw[j] += Gdil[j];  // (:306)

    // cov_raw = T Sig T^T (:308-312)
    const double Gsym[4] = {2.0 * Graw[0], Graw[1] + Graw[2], Graw[2] + Graw[1], 2.0 * Graw[3]};
    double TS[6], GT[6], GrT[6], GSig[9];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            TS[3 * a + b] = P.T[3 * a] * P.Sig[b] + P.T[3 * a + 1] * P.Sig[3 + b] + P.T[3 * a + 2] * P.Sig[6 + b];
    const double gu[2] = {gu0, gu1};
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) GT[3 * a + b] = Gsym[2 * a] * TS[b] + Gsym[2 * a + 1] * TS[3 + b] + gu[a] * P.w[b];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) GrT[3 * a + b] = Graw[2 * a] * P.T[b] + Graw[2 * a + 1] * P.T[3 + b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            GSig[3 * a + b] = P.T[a] * GrT[b] + P.T[3 + a] * GrT[3 + b] + (gw[a] * eta[b] + s_q * (eta[a] * eta[b]));
    // T = J R_w2c -> G_J = G_T R^T (:315)
    double GJ[6];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int k = 0; k < 3; k++) GJ[3 * a + k] = GT[3 * a] * R[3 * k] + GT[3 * a + 1] * R[3 * k + 1] + GT[3 * a + 2] * R[3 * k + 2];
    // Sigma = (Rq S)(Rq S)^T (:317-325)
    double GM[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 3; k++) acc += (GSig[3 * a + k] + GSig[3 * k + a]) * (P.Rq[3 * k + b] * P.scale[b]);
            GM[3 * a + b] = acc;
        }
#pragma unroll
    for (int j = 0; j < 3; j++) {
        double gs = P.Rq[j] * GM[j] + P.Rq[3 + j] * GM[3 + j] + P.Rq[6 + j] * GM[6 + j];
        gr.d_log_scale[3 * i + j] = (float)(gs * P.scale[j]);
    }
    // _quat_backward (projection.py:382-420) with G_R = G_M * scale
    {
        const double w = P.qn[0], x = P.qn[1], y = P.qn[2], z = P.qn[3];
        const double dRw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
        const double dRx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
        const double dRy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
        const double dRz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
        double d[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 9; j++) {
            const double GR = GM[j] * P.scale[j % 3];
            d[0] += GR * 2.0 * dRw[j];
            d[1] += GR * 2.0 * dRx[j];
            d[2] += GR * 2.0 * dRy[j];
            d[3] += GR * 2.0 * dRz[j];
        }
        const double inner = P.qn[0] * d[0] + P.qn[1] * d[1] + P.qn[2] * d[2] + P.qn[3] * d[3];
#pragma unroll
        for (int j = 0; j < 4; j++) gr.d_rot[4 * i + j] = (float)((d[j] - P.qn[j] * inner) / P.qnorm);
    }
    // J -> camera-space position (:327-347)
    const double tz2 = tz * tz, tz3 = tz * tz * tz;
    double dt0 = P.gate0 * (-fx / tz2) * GJ[2];
    double dt1 = P.gate1 * (-fy / tz2) * GJ[5];
    const double txc = -P.J02 * tz2 / fx, tyc = -P.J12 * tz2 / fy;
    const double kx = P.gate0 > 0 ? 2.0 : 1.0, ky = P.gate1 > 0 ? 2.0 : 1.0;
    double dt2 = (-fx / tz2) * GJ[0] + (-fy / tz2) * GJ[4];
    dt2 += kx * fx * txc / tz3 * GJ[2];
    dt2 += ky * fy * tyc / tz3 * GJ[5];
    dt0 += dm0 * fx / tz;
    dt1 += dm1 * fy / tz;
    dt2 += -dm0 * fx * P.t[0] / tz2 - dm1 * fy * P.t[1] / tz2;
    gr.g_z[i] = (float)fabs(dt2);                                           // :349
    const double u0 = dm0 * (cam.width / 2.0), u1 = dm1 * (cam.height / 2.0);
    gr.g_uv[i] = (float)sqrt(u0 * u0 + u1 * u1);                            // :350-351
    double dmu[3];
#pragma unroll
    for (int j = 0; j < 3; j++) dmu[j] = dt0 * R[j] + dt1 * R[3 + j] + dt2 * R[6 + j];  // :353

#pragma unroll
    for (int j = 0; j < 3; j++) {
        dmu_out[j] = (float)dmu[j];
        gr.d_eta[3 * i + j] = (float)geta[j];                               // :365-366
    }
}


// Outputs of a primitive whose 12 screen gradients are all zero: every
// gradient is 0 (no instance touched a pixel with dL != 0, or the primitive
// is invalid: zero_invalid, projection.py:368-379).
template <int ROW>
__device__ __forceinline__ void zero_outputs(const ssg_grad_buffers &gr, int64_t i) {
#pragma unroll
    for (int j = 0; j < 3; j++) gr.d_mu[3 * i + j] = gr.d_log_scale[3 * i + j] = gr.d_eta[3 * i + j] = 0.0f;
#pragma unroll
    for (int j = 0; j < 4; j++) gr.d_rot[4 * i + j] = 0.0f;
    gr.d_opacity_logits[2 * i] = gr.d_opacity_logits[2 * i + 1] = 0.0f;
    gr.g_uv[i] = 0.0f;
    gr.g_z[i] = 0.0f;
    float *row = gr.d_sh + (size_t)i * ROW;
    if (ROW % 4 == 0 && (((uintptr_t)row) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < ROW / 4; q++) reinterpret_cast<float4 *>(row)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
#pragma unroll
        for (int q = 0; q < ROW; q++) row[q] = 0.0f;
    }
}

// One kernel for the whole projection backward.  Only primitives with a
// non-zero screen gradient need the chain (off-screen and occluded ones are
// zero-filled), and they are scattered through the index range, so a warp
// owns kPbSpan consecutive primitives and compacts its active ones:
//   scan    the screen gradients of the whole span, all loads in flight at
//           once; inactive primitives are zero-filled, the active ones'
//           offsets listed in shared memory in index order
//   batches of 32 listed primitives, every lane busy:
//     stage   their SH coefficient rows (3K floats each) into shared memory
//             with asynchronous copies (no register round trip)
//     lanes   the fp64 geometry chain of the lane's primitive (prep_geom),
//             then the SH part (projection.py:355-363, sh.py:25-109): d_sh =
//             basis (x) dcolor on the unclamped channels, written back
//             through the same staging, and the view-direction term folded
//             into d_mu before its single store
//     store   the d_sh rows, one row per step (coalesced)
#ifndef SSG_PB_SPAN
#define SSG_PB_SPAN 128
#endif
constexpr int kPbSpan = SSG_PB_SPAN;
constexpr int kPbIt = kPbSpan / 32;

__device__ __forceinline__ void cp_async4(float *dst_smem, const float *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst_smem)), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int DEG>
__global__ void __launch_bounds__(128, SSG_PB_MINB)
k_preprocess_backward(ssg_scene sc, ssg_camera cam, ssg_grad_buffers gr, int zero_inactive) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    constexpr int ROW = 3 * K;                 // floats per primitive
    __shared__ __align__(16) float tile[4][32 * ROW];
    __shared__ int32_t list[4][kPbSpan];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t p0 = ((int64_t)blockIdx.x * 4 + warp) * kPbSpan;
    if (p0 >= sc.n) return;
    const int span = sc.n - p0 < kPbSpan ? (int)(sc.n - p0) : kPbSpan;
    float *t = tile[warp];
    int32_t *q = list[warp];

    // scan: activity of the span's primitives
    int nact = 0;
    {
        float4 g[kPbIt][3];
#pragma unroll
        for (int k = 0; k < kPbIt; k++) {
            const int o = 32 * k + lane;
            const float4 *sg4 = reinterpret_cast<const float4 *>(gr.screen + 12 * (p0 + (o < span ? o : 0)));
            g[k][0] = sg4[0];
            g[k][1] = sg4[1];
            g[k][2] = sg4[2];
        }
#pragma unroll
        for (int k = 0; k < kPbIt; k++) {
            const int o = 32 * k + lane;
            const float4 a = g[k][0], b = g[k][1], c = g[k][2];
            const bool act = o < span && (a.x != 0.0f || a.y != 0.0f || a.z != 0.0f || a.w != 0.0f || b.x != 0.0f ||
                                          b.y != 0.0f || b.z != 0.0f || b.w != 0.0f || c.x != 0.0f ||
                                          c.y != 0.0f || c.z != 0.0f || c.w != 0.0f);
            const uint32_t m = __ballot_sync(0xffffffffu, act);
            if (act) q[nact + __popc(m & lt)] = o;
            if (zero_inactive && o < span && !act) zero_outputs<ROW>(gr, p0 + o);
            nact += __popc(m);
        }
    }
    __syncwarp();

    for (int b0 = 0; b0 < nact; b0 += 32) {
        const int nb = nact - b0 < 32 ? nact - b0 : 32;
        // stage the batch's SH rows (asynchronous copies, one wait)
        for (int r = 0; r < nb; r++) {
            const float *src = sc.sh + (size_t)(p0 + q[b0 + r]) * ROW;
            for (int c = lane; c < ROW; c += 32) cp_async4(t + r * ROW + c, src + c);
        }
        cp_async_wait_all();
        __syncwarp();
        if (lane < nb) {
            const int64_t i = p0 + q[b0 + lane];
            float dmu[3] = {0.0f, 0.0f, 0.0f};
            prep_geom(sc, cam, gr, i, dmu);  // fp64 geometry
            const float *sh = t + lane * ROW;
            const float *sg = gr.screen + 12 * i;
            const float dcol[3] = {sg[9], sg[10], sg[11]};
            // the forward's fp32 colour (preprocess_fwd.cu), recomputed bit for
            // bit so the clamp mask of projection.py:221-223 / :356 is the forward's
            const double dv0 = sc.mu[3 * i] - cam.campos[0], dv1 = sc.mu[3 * i + 1] - cam.campos[1],
                         dv2 = sc.mu[3 * i + 2] - cam.campos[2];
            const double dn = sqrt(dv0 * dv0 + dv1 * dv1 + dv2 * dv2);
            const double dns = dn > 1e-12 ? dn : 1.0;
            const float x = (float)(dv0 / dns), y = (float)(dv1 / dns), z = (float)(dv2 / dns);
            float basis[16];
            sh_basis_f(DEG, x, y, z, basis);
            float col[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int k = 0; k < K; k++)
#pragma unroll
                for (int c = 0; c < 3; c++) col[c] = fmaf(basis[k], sh[3 * k + c], col[c]);
            float dcc[3];
#pragma unroll
            for (int c = 0; c < 3; c++) dcc[c] = (col[c] + 0.5f > 0.0f) ? dcol[c] : 0.0f;
            float w[16];
#pragma unroll
            for (int k = 0; k < K; k++) w[k] = sh[3 * k] * dcc[0] + sh[3 * k + 1] * dcc[1] + sh[3 * k + 2] * dcc[2];
            float dd[3] = {0.0f, 0.0f, 0.0f};
            if (DEG > 0) sh_dot_grad_f(DEG, x, y, z, w, dd);
            float *out = t + lane * ROW;  // this lane's own row: safe to overwrite now
#pragma unroll
            for (int k = 0; k < K; k++)
#pragma unroll
                for (int c = 0; c < 3; c++) out[3 * k + c] = basis[k] * dcc[c];
            if (DEG > 0) {
                const float inner = x * dd[0] + y * dd[1] + z * dd[2];
                const float rdn = (float)(1.0 / dns);
                dmu[0] += (dd[0] - x * inner) * rdn;
                dmu[1] += (dd[1] - y * inner) * rdn;
                dmu[2] += (dd[2] - z * inner) * rdn;
            }
#pragma unroll
            for (int j = 0; j < 3; j++) gr.d_mu[3 * i + j] = dmu[j];
        }
        __syncwarp();
        for (int r = 0; r < nb; r++) {
            float *dst = gr.d_sh + (size_t)(p0 + q[b0 + r]) * ROW;
            for (int c = lane; c < ROW; c += 32) dst[c] = t[r * ROW + c];
        }
        __syncwarp();
    }
}

}  // namespace ssg

extern "C" int ssg_zero_prim_grads(int64_t n, int32_t sh_coeffs, const ssg_grad_buffers *grads, void *stream) {
    using namespace ssg;
    if (!grads || n < 0 || sh_coeffs < 1 || sh_coeffs > 16) return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    float *const f[8] = {grads->d_mu, grads->d_log_scale, grads->d_rot, grads->d_sh,
                         grads->d_opacity_logits, grads->d_eta, grads->g_uv, grads->g_z};
    const int w[8] = {3, 3, 4, 3 * sh_coeffs, 2, 3, 1, 1};
    for (int k = 0; k < 8; k++) {
        if (!f[k]) return SSG_ERR_INVALID_ARGUMENT;
        const cudaError_t e = cudaMemsetAsync(f[k], 0, sizeof(float) * (size_t)w[k] * (size_t)n, st);
        if (e != cudaSuccess) { set_error("memset prim grads", e); return SSG_ERR_CUDA; }
    }
    return SSG_OK;
}

extern "C" int ssg_zero_screen_grads(int64_t n, const ssg_grad_buffers *grads, void *stream) {
    using namespace ssg;
    if (!grads || !grads->screen || n < 0) return SSG_ERR_INVALID_ARGUMENT;
    const cudaError_t e = cudaMemsetAsync(grads->screen, 0, sizeof(float) * 12 * (size_t)n, (cudaStream_t)stream);
    if (e != cudaSuccess) { set_error("memset screen grads", e); return SSG_ERR_CUDA; }
    return SSG_OK;
}

extern "C" int ssg_preprocess_backward_ex(const ssg_scene *scene, const ssg_camera *cam,
                                          const ssg_grad_buffers *grads, int32_t flags, void *stream) {
    using namespace ssg;
    if (!scene || !cam || !grads) return SSG_ERR_INVALID_ARGUMENT;
    if (scene->sh_degree < 0 || scene->sh_degree > 3) return SSG_ERR_INVALID_ARGUMENT;
    if ((flags & ~SSG_PREP_BWD_ACTIVE_ONLY) != 0) return SSG_ERR_INVALID_ARGUMENT;
    if (scene->n == 0) return SSG_OK;
    const int zero = (flags & SSG_PREP_BWD_ACTIVE_ONLY) ? 0 : 1;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t per_block = 4 * (int64_t)kPbSpan;  // 4 warps of kPbSpan primitives
    unsigned blocks = (unsigned)((scene->n + per_block - 1) / per_block);
    switch (scene->sh_degree) {
        case 0: k_preprocess_backward<0><<<blocks, 128, 0, st>>>(*scene, *cam, *grads, zero); break;
        case 1: k_preprocess_backward<1><<<blocks, 128, 0, st>>>(*scene, *cam, *grads, zero); break;
        case 2: k_preprocess_backward<2><<<blocks, 128, 0, st>>>(*scene, *cam, *grads, zero); break;
        default: k_preprocess_backward<3><<<blocks, 128, 0, st>>>(*scene, *cam, *grads, zero); break;
    }
    return check_launch("k_preprocess_backward");
}

extern "C" int ssg_preprocess_backward(const ssg_scene *scene, const ssg_camera *cam,
                                       const ssg_grad_buffers *grads, void *stream) {
    return ssg_preprocess_backward_ex(scene, cam, grads, 0, stream);
}
