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
// Three passes, all HBM-bound and coalesced: a row check over the packed
// gradient buffer, one element-wise update per field, the quaternion fix-up.
#include "ssg_common.cuh"

namespace ssg {

constexpr double kBeta1 = 0.9, kBeta2 = 0.999, kEps = 1e-15;

__global__ void k_adam_rowcheck(int64_t n, int K, ssg_grad_buffers g, uint8_t *row_ok, int32_t *n_skipped) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (i < n) {
#pragma unroll
        for (int j = 0; j < 3; j++) ok &= isfinite(g.d_mu[3 * i + j]) && isfinite(g.d_log_scale[3 * i + j]) &&
                                          isfinite(g.d_eta[3 * i + j]) &&
                                          (!g.d_beta || isfinite(g.d_beta[3 * i + j]));
#pragma unroll
        for (int j = 0; j < 4; j++) ok &= isfinite(g.d_rot[4 * i + j]);
        ok &= isfinite(g.d_opacity_logits[2 * i]) && isfinite(g.d_opacity_logits[2 * i + 1]);
        for (int j = 0; j < 3 * K; j++) ok &= isfinite(g.d_sh[(size_t)i * 3 * K + j]);
        row_ok[i] = ok;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, i < n && !ok);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(n_skipped, __popc(bad));
}

// param[e] -= lr * (m/c1) / (sqrt(v/c2) + eps) for every element e of a
// (n, width) field whose row is finite.
template <typename P>
__global__ void k_adam_field(int64_t n, int width, P *__restrict__ p,
                             const float *__restrict__ g, float *__restrict__ m, float *__restrict__ v,
                             const uint8_t *__restrict__ row_ok, double lr, double c1, double c2) {
    const int64_t total = n * width;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (!row_ok[e / width]) continue;
        const double gg = g[e];
        const double mm = kBeta1 * (double)m[e] + (1.0 - kBeta1) * gg;
        const double vv = kBeta2 * (double)v[e] + (1.0 - kBeta2) * gg * gg;
        m[e] = (float)mm;
        v[e] = (float)vv;
        const double upd = lr * (mm / c1) / (sqrt(vv / c2) + kEps);
        p[e] = (P)((double)p[e] - upd);
    }
}

__global__ void k_quat_renorm(int64_t n, double *rot) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
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
    k_adam_rowcheck<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, K, *g, s->row_ok, s->n_skipped);
    const double c1 = 1.0 - pow(kBeta1, (double)hp->t), c2 = 1.0 - pow(kBeta2, (double)hp->t);
    const unsigned grid = 148 * 8;
    k_adam_field<double><<<grid, 256, 0, st>>>(n, 3, p->mu, g->d_mu, s->m_mu, s->v_mu, s->row_ok, hp->lr_mu, c1,
                                               c2);
    k_adam_field<double><<<grid, 256, 0, st>>>(n, 3, p->log_scale, g->d_log_scale, s->m_log_scale, s->v_log_scale,
                                               s->row_ok, hp->lr_scale, c1, c2);
    k_adam_field<double><<<grid, 256, 0, st>>>(n, 4, p->rot, g->d_rot, s->m_rot, s->v_rot, s->row_ok, hp->lr_rot,
                                               c1, c2);
    k_adam_field<float><<<grid, 256, 0, st>>>(n, 3 * K, p->sh, g->d_sh, s->m_sh, s->v_sh, s->row_ok, hp->lr_sh, c1,
                                              c2);
    k_adam_field<float><<<grid, 256, 0, st>>>(n, 2, p->opacity_logits, g->d_opacity_logits, s->m_logits,
                                              s->v_logits, s->row_ok, hp->lr_opacity, c1, c2);
    if (hp->lr_beta != 0.0) {  // adam.py:63-69: lr_beta drives beta and dir
        k_adam_field<float><<<grid, 256, 0, st>>>(n, 3, p->beta, g->d_beta ? g->d_beta : g->d_eta, s->m_beta,
                                                  s->v_beta, s->row_ok, hp->lr_beta, c1, c2);
        k_adam_field<float><<<grid, 256, 0, st>>>(n, 3, p->dir, g->d_eta, s->m_dir, s->v_dir, s->row_ok,
                                                  hp->lr_beta, c1, c2);
    }
    k_quat_renorm<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, p->rot);
    return check_launch("ssg_adam_step");
}
