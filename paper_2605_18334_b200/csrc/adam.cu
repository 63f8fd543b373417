// adam.cu -- the training-step optimizer of config 5 on the device.
//
// Reference: optimize/adam.py:53-97 (Adam.step): bias-corrected moments with
// BETA1 0.9, BETA2 0.999, EPS 1e-15; primitives with any non-finite
// gradient are skipped (moments untouched, counted); per-field learning
// rates (config.py:19-25, lr_beta shared by beta and dir); quaternions
// renormalised afterwards where they drifted (|norm - 1| > 1e-12), set to
// the identity where degenerate (norm <= 1e-12).
// beta and dir keep separate moments: their rendered gradients are equal
// (projection.py:365-366) but the training step adds the beta regularizer to
// d_beta only (fit2d.py:75, losses.py:127).
// Three passes, all HBM-bound and coalesced: a row check over the gradient
// rows, one element-wise update per field (fp32 arithmetic on the fp32
// moments; the fp64 parameters are updated in fp64), the quaternion fix-up.
#include "ssg_common.cuh"

namespace ssg {

constexpr float kBeta1 = 0.9f, kBeta2 = 0.999f, kEps = 1e-15f;

// One thread per primitive: is every gradient of the row finite
// (adam.py:75-79)?  The (K,3) SH row is read as float4s when 16-byte aligned.
__global__ void k_adam_rowcheck(int64_t n, int K, ssg_grad_buffers g, uint8_t *row_ok, int32_t *n_skipped,
                                const int32_t *skip) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (skip && *skip) {  // the whole step is skipped (hp->skip): no row updates, nothing counted
        if (i < n) row_ok[i] = 0;
        return;
    }
    bool ok = true;
    if (i < n) {
#pragma unroll
        for (int j = 0; j < 3; j++) ok &= isfinite(g.d_mu[3 * i + j]) && isfinite(g.d_log_scale[3 * i + j]) &&
                                          isfinite(g.d_eta[3 * i + j]) &&
                                          (!g.d_beta || isfinite(g.d_beta[3 * i + j]));
#pragma unroll
        for (int j = 0; j < 4; j++) ok &= isfinite(g.d_rot[4 * i + j]);
        ok &= isfinite(g.d_opacity_logits[2 * i]) && isfinite(g.d_opacity_logits[2 * i + 1]);
        const float *sh = g.d_sh + (size_t)i * 3 * K;
        if (((3 * K) & 3) == 0 && (((uintptr_t)g.d_sh) & 15) == 0) {
            const float4 *s4 = reinterpret_cast<const float4 *>(sh);
            for (int q = 0; q < 3 * K / 4; q++) {
                const float4 v = s4[q];
                ok &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
            }
        } else {
            for (int j = 0; j < 3 * K; j++) ok &= isfinite(sh[j]);
        }
        row_ok[i] = ok;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, i < n && !ok);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(n_skipped, __popc(bad));
}

// adam.py:84-90 for one (n, W) field: m += (1-b1)(g-m) form of
// m = b1 m + (1-b1) g, v likewise, p -= lr (m/c1) / (sqrt(v/c2) + eps) on the
// finite rows.  fp32 arithmetic on fp32 moments (memory-bound: 28-36 B per
// element); W is a compile-time constant so the row index is a multiply.
template <typename P, int W>
__global__ void __launch_bounds__(256) k_adam_field(int64_t n, P *__restrict__ p, const float *__restrict__ g,
                                                    float *__restrict__ m, float *__restrict__ v,
                                                    const uint8_t *__restrict__ row_ok, float lr, float rc1,
                                                    float rc2) {
    const uint32_t total = (uint32_t)(n * W);
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        if (!row_ok[e / W]) continue;
        const float gg = g[e];
        const float mm = kBeta1 * m[e] + (1.0f - kBeta1) * gg;
        const float vv = kBeta2 * v[e] + (1.0f - kBeta2) * gg * gg;
        m[e] = mm;
        v[e] = vv;
        const float upd = lr * (mm * rc1) / (sqrtf(vv * rc2) + kEps);
        p[e] = (P)((double)p[e] - (double)upd);
    }
}

// fp32 parameters, 4 elements per thread with 16-byte accesses (each
// element keeps its own row check: a float4 may straddle two rows when W is
// not a multiple of 4).  Same arithmetic as k_adam_field.
template <int W>
__global__ void __launch_bounds__(256) k_adam_field_v4(int64_t n, float4 *__restrict__ p,
                                                       const float4 *__restrict__ g, float4 *__restrict__ m,
                                                       float4 *__restrict__ v, const uint8_t *__restrict__ row_ok,
                                                       float lr, float rc1, float rc2) {
    const uint32_t total4 = (uint32_t)(n * W / 4);
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < total4; q += gridDim.x * blockDim.x) {
        const float4 g4 = g[q];
        float4 m4 = m[q], v4 = v[q], p4 = p[q];
        float *gg = reinterpret_cast<float *>(const_cast<float4 *>(&g4)), *mm = reinterpret_cast<float *>(&m4);
        float *vv = reinterpret_cast<float *>(&v4), *pp = reinterpret_cast<float *>(&p4);
        bool any = false;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            if (!row_ok[(4 * q + c) / W]) continue;
            any = true;
            const float mn = kBeta1 * mm[c] + (1.0f - kBeta1) * gg[c];
            const float vn = kBeta2 * vv[c] + (1.0f - kBeta2) * gg[c] * gg[c];
            mm[c] = mn;
            vv[c] = vn;
            const float upd = lr * (mn * rc1) / (sqrtf(vn * rc2) + kEps);
            pp[c] = (float)((double)pp[c] - (double)upd);
        }
        if (any) {
            m[q] = m4;
            v[q] = v4;
            p[q] = p4;
        }
    }
}

template <typename P, int W>
static void launch_field(int64_t n, P *p, const float *g, float *m, float *v, const uint8_t *row_ok, double lr,
                         double c1, double c2, cudaStream_t st) {
    if constexpr (sizeof(P) == 4) {
        const auto al = [](const void *x) { return (((uintptr_t)x) & 15) == 0; };
        if ((n * W) % 4 == 0 && al(p) && al(g) && al(m) && al(v)) {
            const int64_t b64 = (n * W / 4 + 255) / 256;
            const unsigned blocks = (unsigned)(b64 < 148 * 16 ? b64 : 148 * 16);
            k_adam_field_v4<W><<<blocks, 256, 0, st>>>(n, reinterpret_cast<float4 *>(p),
                                                       reinterpret_cast<const float4 *>(g),
                                                       reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v),
                                                       row_ok, (float)lr, (float)(1.0 / c1), (float)(1.0 / c2));
            return;
        }
    }
    const int64_t blocks64 = (n * W + 255) / 256;
    const unsigned blocks = (unsigned)(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
    k_adam_field<P, W><<<blocks, 256, 0, st>>>(n, p, g, m, v, row_ok, (float)lr, (float)(1.0 / c1),
                                               (float)(1.0 / c2));
}

template <int W>
static void launch_sh(int64_t n, float *p, const float *g, float *m, float *v, const uint8_t *row_ok, double lr,
                      double c1, double c2, cudaStream_t st) {
    launch_field<float, W>(n, p, g, m, v, row_ok, lr, c1, c2, st);
}

__global__ void k_quat_renorm(int64_t n, double *rot, const int32_t *skip) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (skip && *skip)) return;
    double q[4];
#pragma unroll
    for (int j = 0; j < 4; j++) q[j] = rot[4 * i + j];
    const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (nrm <= 1e-12) {
        rot[4 * i] = 1.0; rot[4 * i + 1] = 0.0; rot[4 * i + 2] = 0.0; rot[4 * i + 3] = 0.0;
    } else if (fabs(nrm - 1.0) > 1e-12) {
#pragma unroll
        for (int j = 0; j < 4; j++) rot[4 * i + j] = q[j] / nrm;
    }
}

}  // namespace ssg

extern "C" int ssg_adam_step(const ssg_params *p, const ssg_grad_buffers *g, const ssg_adam_state *s,
                             const ssg_adam_hparams *hp, void *stream) {
    using namespace ssg;
    if (!p || !g || !s || !hp || hp->t < 1 || p->n < 0) return SSG_ERR_INVALID_ARGUMENT;
    if (p->n == 0) return SSG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = p->n;
    const int K = p->sh_coeffs;
    if (K != 1 && K != 4 && K != 9 && K != 16) return SSG_ERR_INVALID_ARGUMENT;
    if (p->n * 3 * K >= (int64_t)UINT32_MAX) return SSG_ERR_CAPACITY;
    k_adam_rowcheck<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, K, *g, s->row_ok, s->n_skipped, hp->skip);
    const double c1 = 1.0 - pow(0.9, (double)hp->t), c2 = 1.0 - pow(0.999, (double)hp->t);
    launch_field<double, 3>(n, p->mu, g->d_mu, s->m_mu, s->v_mu, s->row_ok, hp->lr_mu, c1, c2, st);
    launch_field<double, 3>(n, p->log_scale, g->d_log_scale, s->m_log_scale, s->v_log_scale, s->row_ok,
                            hp->lr_scale, c1, c2, st);
    launch_field<double, 4>(n, p->rot, g->d_rot, s->m_rot, s->v_rot, s->row_ok, hp->lr_rot, c1, c2, st);
    switch (K) {  // (K,3) SH rows: 3, 12, 27 or 48 floats
        case 1: launch_sh<3>(n, p->sh, g->d_sh, s->m_sh, s->v_sh, s->row_ok, hp->lr_sh, c1, c2, st); break;
        case 4: launch_sh<12>(n, p->sh, g->d_sh, s->m_sh, s->v_sh, s->row_ok, hp->lr_sh, c1, c2, st); break;
        case 9: launch_sh<27>(n, p->sh, g->d_sh, s->m_sh, s->v_sh, s->row_ok, hp->lr_sh, c1, c2, st); break;
        default: launch_sh<48>(n, p->sh, g->d_sh, s->m_sh, s->v_sh, s->row_ok, hp->lr_sh, c1, c2, st); break;
    }
    launch_field<float, 2>(n, p->opacity_logits, g->d_opacity_logits, s->m_logits, s->v_logits, s->row_ok,
                           hp->lr_opacity, c1, c2, st);
    if (hp->lr_beta != 0.0) {  // adam.py:63-69: lr_beta drives beta and dir
        launch_field<float, 3>(n, p->beta, g->d_beta ? g->d_beta : g->d_eta, s->m_beta, s->v_beta, s->row_ok,
                               hp->lr_beta, c1, c2, st);
        launch_field<float, 3>(n, p->dir, g->d_eta, s->m_dir, s->v_dir, s->row_ok, hp->lr_beta, c1, c2, st);
    }
    k_quat_renorm<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, p->rot, hp->skip);
    return check_launch("ssg_adam_step");
}
