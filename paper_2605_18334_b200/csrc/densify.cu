// densify.cu -- adaptive density control on the device (SURVEY.md §8(f)
// row 2): clone, split and prune as order-preserving stream compaction.
//
// Reference: optimize/densify.py:24-116 (densify_and_prune), Adam state
// remap optimize/adam.py:99-110 (prune + extend), quat_to_rotmat
// scene.py:66-83, sigmoid kernel_math.py:158-165.
//
//   plan   tau_z calibration when NaN: the 90th percentile of g_z with
//          numpy's linear interpolation (densify.py:39-40), over the device
//          depth sort of the fp32 bit patterns; per-primitive flags
//          (densify.py:42-62) and per-block counts; one-block scan of the
//          block counts -> block offsets and totals (n_keep, n_clone,
//          n_split, n_pruned)
//   apply  every output row written once, in the reference's order:
//          [kept rows in index order | clones in index order | for each
//          split primitive its + then - child] (densify.py:64-105); Adam
//          moments follow the kept rows, new rows start at zero
//          (adam.py:99-110); a device flag records non-finite outputs
//          (densify.py:112-114)
// Compiled with --fmad=false: the fp64 expressions round like numpy's.
#include <math.h>

#include "depth_sort.cuh"
#include "ssg_common.cuh"

namespace ssg {

constexpr int kDThreads = 256;
enum : uint8_t { kKeep = 1, kClone = 2, kSplit = 4, kPrune = 8 };

struct DensifyTemp {
    size_t block_counts, totals, keys, order, sort, total;
};

static DensifyTemp densify_temp(int64_t n) {
    DensifyTemp t;
    const int64_t nb = (n + kDThreads - 1) / kDThreads;
    size_t o = 0;
    auto take = [&](size_t b) { const size_t at = o; o += radix::align256(b); return at; };
    t.block_counts = take(sizeof(uint32_t) * 4 * (size_t)(nb > 0 ? nb : 1));
    t.totals = take(sizeof(int64_t) * 4 + sizeof(double));
    t.keys = take(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    t.order = take(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    t.sort = take(dsort::temp_bytes(n > 0 ? n : 1));
    t.total = o;
    return t;
}

__device__ __forceinline__ double sigmoid_ref(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    const double ex = exp(x);
    return ex / (1.0 + ex);
}

__global__ void k_gz_keys(int64_t n, const float *__restrict__ g_z, uint64_t *__restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint64_t)__float_as_uint(g_z[i]);  // g_z >= 0: bits are monotone
}

// np.percentile(g_z, 90) (method 'linear', numpy's _lerp)
__global__ void k_percentile90(int64_t n, const float *__restrict__ g_z, const uint32_t *__restrict__ order,
                               double *__restrict__ tau) {
    const double virt = 0.9 * (double)(n - 1);
    const double prev = floor(virt);
    const int64_t lo = (int64_t)prev, hi = lo + 1 < n ? lo + 1 : n - 1;
    const double gamma = virt - prev;
    const double a = (double)g_z[order[lo]], b = (double)g_z[order[hi]];
    const double diff = b - a;
    *tau = gamma >= 0.5 ? b - diff * (1.0 - gamma) : a + diff * gamma;
}

// densify.py:42-62: flags and per-block category counts
__global__ void __launch_bounds__(kDThreads) k_densify_flags(int64_t n, ssg_scene sc, ssg_densify_stats st,
                                                             ssg_densify_cfg cfg, const double *__restrict__ tau_dev,
                                                             uint8_t *__restrict__ flags,
                                                             uint32_t *__restrict__ block_counts) {
    __shared__ uint32_t s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint8_t f = 0;
    if (i < n) {
        const double tau_z = tau_dev ? *tau_dev : cfg.tau_z;
        const bool flagged = st.g_uv[i] > cfg.tau_uv || (double)st.g_z[i] > tau_z;
        double ms = exp(sc.log_scale[3 * i]);
        ms = fmax(ms, exp(sc.log_scale[3 * i + 1]));
        ms = fmax(ms, exp(sc.log_scale[3 * i + 2]));
        const bool split = flagged && ms > cfg.split_scale_threshold;
        const double o0 = -cfg.clone_lr * st.d_mu[3 * i], o1 = -cfg.clone_lr * st.d_mu[3 * i + 1],
                     o2 = -cfg.clone_lr * st.d_mu[3 * i + 2];
        const bool clone = flagged && !split && sqrt(o0 * o0 + o1 * o1 + o2 * o2) > 0.0;
        const double s0 = sigmoid_ref((double)sc.opacity_logits[2 * i]);
        const double s1 = sigmoid_ref((double)sc.opacity_logits[2 * i + 1]);
        bool prune = fmax(s0, s1) < cfg.prune_alpha;
        if (cfg.max_radii && cfg.max_screen_radius >= 0.0) prune |= cfg.max_radii[i] > cfg.max_screen_radius;
        if (prune) f |= kPrune;
        if (!prune && !split) f |= kKeep;
        if (clone && !prune) f |= kClone;
        if (split && !prune) f |= kSplit;
        flags[i] = f;
    }
    const unsigned bk = __ballot_sync(0xffffffffu, f & kKeep), bc = __ballot_sync(0xffffffffu, f & kClone);
    const unsigned bs = __ballot_sync(0xffffffffu, f & kSplit), bp = __ballot_sync(0xffffffffu, f & kPrune);
    if ((threadIdx.x & 31) == 0) {
        if (bk) atomicAdd(&s_cnt[0], __popc(bk));
        if (bc) atomicAdd(&s_cnt[1], __popc(bc));
        if (bs) atomicAdd(&s_cnt[2], __popc(bs));
        if (bp) atomicAdd(&s_cnt[3], __popc(bp));
    }
    __syncthreads();
    if (threadIdx.x < 4) block_counts[4 * (size_t)blockIdx.x + threadIdx.x] = s_cnt[threadIdx.x];
}

// one block: exclusive scan of the block counts per category, totals
__global__ void __launch_bounds__(1024) k_densify_scan(int64_t nb, uint32_t *__restrict__ block_counts,
                                                       int64_t *__restrict__ totals) {
    __shared__ uint32_t s_warp[32][4];
    __shared__ uint32_t s_carry[4];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t < 4) s_carry[t] = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nb; c0 += 1024) {
        const int64_t b = c0 + t;
        uint32_t v[4], x[4];
        for (int k = 0; k < 4; k++) {
            v[k] = b < nb ? block_counts[4 * b + k] : 0u;
            x[k] = v[k];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x[k], off);
                if (lane >= off) x[k] += y;
            }
            if (lane == 31) s_warp[w][k] = x[k];
        }
        __syncthreads();
        for (int k = 0; k < 4; k++) {
            uint32_t pre = s_carry[k];
            for (int ww = 0; ww < w; ww++) pre += s_warp[ww][k];
            if (b < nb) block_counts[4 * b + k] = pre + x[k] - v[k];
        }
        __syncthreads();
        if (t < 4) {
            uint32_t tot = 0;
            for (int ww = 0; ww < 32; ww++) tot += s_warp[ww][t];
            s_carry[t] += tot;
        }
        __syncthreads();
    }
    if (t < 4) totals[t] = s_carry[t];
}

__device__ __forceinline__ void copy_row(const ssg_scene &in, const ssg_params &out, int64_t i, int64_t o, int K) {
    for (int j = 0; j < 3; j++) {
        out.mu[3 * o + j] = in.mu[3 * i + j];
        out.log_scale[3 * o + j] = in.log_scale[3 * i + j];
        out.beta[3 * o + j] = in.beta[3 * i + j];
        out.dir[3 * o + j] = in.dir[3 * i + j];
    }
    for (int j = 0; j < 4; j++) out.rot[4 * o + j] = in.rot[4 * i + j];
    for (int j = 0; j < 2; j++) out.opacity_logits[2 * o + j] = in.opacity_logits[2 * i + j];
    for (int j = 0; j < 3 * K; j++) out.sh[(size_t)o * 3 * K + j] = in.sh[(size_t)i * 3 * K + j];
}

__device__ __forceinline__ void moment_row(const ssg_adam_state &a, const ssg_adam_state &b, int64_t i, int64_t o,
                                           int K, bool zero) {
    const float *const src[14] = {a.m_mu, a.v_mu, a.m_log_scale, a.v_log_scale, a.m_rot, a.v_rot, a.m_sh,
                                  a.v_sh, a.m_logits, a.v_logits, a.m_beta, a.v_beta, a.m_dir, a.v_dir};
    float *const dst[14] = {b.m_mu, b.v_mu, b.m_log_scale, b.v_log_scale, b.m_rot, b.v_rot, b.m_sh,
                            b.v_sh, b.m_logits, b.v_logits, b.m_beta, b.v_beta, b.m_dir, b.v_dir};
    const int width[7] = {3, 3, 4, 3 * K, 2, 3, 3};
    for (int f = 0; f < 14; f++) {
        const int wd = width[f / 2];
        if (!dst[f]) continue;
        for (int j = 0; j < wd; j++) dst[f][(size_t)o * wd + j] = zero ? 0.0f : src[f][(size_t)i * wd + j];
    }
}

__device__ __forceinline__ bool row_finite(const ssg_params &p, int64_t o, int K) {
    bool ok = true;
    for (int j = 0; j < 3; j++)
        ok &= isfinite(p.mu[3 * o + j]) && isfinite(p.log_scale[3 * o + j]) && isfinite(p.beta[3 * o + j]) &&
              isfinite(p.dir[3 * o + j]);
    for (int j = 0; j < 4; j++) ok &= isfinite(p.rot[4 * o + j]);
    for (int j = 0; j < 2; j++) ok &= isfinite(p.opacity_logits[2 * o + j]);
    for (int j = 0; j < 3 * K; j++) ok &= isfinite(p.sh[(size_t)o * 3 * K + j]);
    return ok;
}

__global__ void __launch_bounds__(kDThreads) k_densify_apply(int64_t n, ssg_scene in, ssg_params out,
                                                             ssg_adam_state ain, ssg_adam_state aout,
                                                             ssg_densify_stats st, ssg_densify_cfg cfg,
                                                             const uint8_t *__restrict__ flags,
                                                             const uint32_t *__restrict__ block_counts,
                                                             const int64_t *__restrict__ totals,
                                                             int32_t *__restrict__ bad) {
    __shared__ uint32_t s_warp[kDThreads / 32][3];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + t;
    const uint8_t f = i < n ? flags[i] : 0;
    const bool k_ = f & kKeep, c_ = f & kClone, s_ = f & kSplit;
    const uint32_t lt = (1u << lane) - 1u;
    const unsigned bk = __ballot_sync(0xffffffffu, k_), bc = __ballot_sync(0xffffffffu, c_),
                   bs = __ballot_sync(0xffffffffu, s_);
    if (lane == 0) {
        s_warp[w][0] = __popc(bk);
        s_warp[w][1] = __popc(bc);
        s_warp[w][2] = __popc(bs);
    }
    __syncthreads();
    uint32_t pk = block_counts[4 * (size_t)blockIdx.x], pc = block_counts[4 * (size_t)blockIdx.x + 1],
             ps = block_counts[4 * (size_t)blockIdx.x + 2];
    for (int ww = 0; ww < w; ww++) {
        pk += s_warp[ww][0];
        pc += s_warp[ww][1];
        ps += s_warp[ww][2];
    }
    pk += __popc(bk & lt);
    pc += __popc(bc & lt);
    ps += __popc(bs & lt);
    if (i >= n) return;
    const int K = out.sh_coeffs;
    const int64_t n_keep = totals[0], n_clone = totals[1];
    bool ok = true;
    if (k_) {  // densify.py:100-105 (kept rows), adam.py:99-102
        copy_row(in, out, i, pk, K);
        moment_row(ain, aout, i, pk, K, false);
        ok &= row_finite(out, pk, K);
    }
    if (c_) {  // densify.py:67-74
        const int64_t o = n_keep + pc;
        copy_row(in, out, i, o, K);
        for (int j = 0; j < 3; j++) out.mu[3 * o + j] = in.mu[3 * i + j] + (-cfg.clone_lr * st.d_mu[3 * i + j]);
        moment_row(ain, aout, i, o, K, true);
        ok &= row_finite(out, o, K);
    }
    if (s_) {  // densify.py:76-97
        const double *q = in.rot + 4 * i;
        const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        const double qw = q[0] / nrm, qx = q[1] / nrm, qy = q[2] / nrm, qz = q[3] / nrm;
        const double *ls = in.log_scale + 3 * i;
        const int k = (ls[1] > ls[0]) ? ((ls[2] > ls[1]) ? 2 : 1) : ((ls[2] > ls[0]) ? 2 : 0);  // np.argmax
        double axis[3];  // column k of quat_to_rotmat (scene.py:74-82)
        if (k == 0) {
            axis[0] = 1 - 2 * (qy * qy + qz * qz);
            axis[1] = 2 * (qx * qy + qw * qz);
            axis[2] = 2 * (qx * qz - qw * qy);
        } else if (k == 1) {
            axis[0] = 2 * (qx * qy - qw * qz);
            axis[1] = 1 - 2 * (qx * qx + qz * qz);
            axis[2] = 2 * (qy * qz + qw * qx);
        } else {
            axis[0] = 2 * (qx * qz + qw * qy);
            axis[1] = 2 * (qy * qz - qw * qx);
            axis[2] = 1 - 2 * (qx * qx + qy * qy);
        }
        const double half = 0.5 * exp(ls[k]);
        const double eta0 = (double)in.beta[3 * i] + (double)in.dir[3 * i];
        const double eta1 = (double)in.beta[3 * i + 1] + (double)in.dir[3 * i + 1];
        const double eta2 = (double)in.beta[3 * i + 2] + (double)in.dir[3 * i + 2];
        const float l0 = in.opacity_logits[2 * i], l1 = in.opacity_logits[2 * i + 1];
        const float l_hi = fmaxf(l0, l1), l_lo = fminf(l0, l1);
        const bool plus_near = eta0 * axis[0] + eta1 * axis[1] + eta2 * axis[2] >= 0.0;
        for (int c = 0; c < 2; c++) {
            const double sign = c == 0 ? 1.0 : -1.0;
            const bool near = (sign > 0) == plus_near;
            const float lv = near ? l_hi : l_lo;
            const int64_t o = n_keep + n_clone + 2 * (int64_t)ps + c;
            copy_row(in, out, i, o, K);
            for (int j = 0; j < 3; j++) {
                out.mu[3 * o + j] = in.mu[3 * i + j] + sign * half * axis[j];
                out.log_scale[3 * o + j] = ls[j] - 0.47000362924573563;  // math.log(1.6), densify.py:21
            }
            out.opacity_logits[2 * o] = lv;
            out.opacity_logits[2 * o + 1] = lv;
            moment_row(ain, aout, i, o, K, true);
            ok &= row_finite(out, o, K);
        }
    }
    if (!ok) atomicOr(bad, 1);
}

}  // namespace ssg

extern "C" size_t ssg_densify_temp_bytes(int64_t n) { return ssg::densify_temp(n).total; }

extern "C" int ssg_densify_plan(const ssg_scene *scene, const ssg_densify_stats *stats, const ssg_densify_cfg *cfg,
                                uint8_t *flags, void *temp, size_t temp_bytes, int64_t *counts_host,
                                double *tau_z_host, void *stream) {
    using namespace ssg;
    if (!scene || !stats || !cfg || scene->n < 0 || !counts_host || !tau_z_host) return SSG_ERR_INVALID_ARGUMENT;
    const int64_t n = scene->n;
    const DensifyTemp T = densify_temp(n);
    if (temp_bytes < T.total || (n > 0 && (!flags || !temp))) return SSG_ERR_CAPACITY;
    cudaStream_t st = (cudaStream_t)stream;
    char *tp = (char *)temp;
    int64_t *totals = (int64_t *)(tp + T.totals);
    double *tau_dev = (double *)(totals + 4);
    if (n == 0) {
        for (int k = 0; k < 4; k++) counts_host[k] = 0;
        *tau_z_host = cfg->tau_z;
        return SSG_OK;
    }
    const unsigned nb = (unsigned)((n + kDThreads - 1) / kDThreads);
    const bool calibrate = isnan(cfg->tau_z);
    if (calibrate) {  // densify.py:39-40
        uint64_t *keys = (uint64_t *)(tp + T.keys);
        uint32_t *order = (uint32_t *)(tp + T.order);
        k_gz_keys<<<nb, kDThreads, 0, st>>>(n, stats->g_z, keys);
        cudaError_t e = dsort::sort_and_scan(keys, order, nullptr, nullptr, nullptr, n, tp + T.sort, st);
        if (e != cudaSuccess) { set_error("densify percentile sort", e); return SSG_ERR_CUDA; }
        k_percentile90<<<1, 1, 0, st>>>(n, stats->g_z, order, tau_dev);
    }
    uint32_t *bc = (uint32_t *)(tp + T.block_counts);
    k_densify_flags<<<nb, kDThreads, 0, st>>>(n, *scene, *stats, *cfg, calibrate ? tau_dev : nullptr, flags, bc);
    k_densify_scan<<<1, 1024, 0, st>>>(nb, bc, totals);
    int rc = check_launch("ssg_densify_plan");
    if (rc != SSG_OK) return rc;
    int64_t host[4];
    cudaError_t e = cudaMemcpyAsync(host, totals, sizeof(host), cudaMemcpyDeviceToHost, st);
    double tau = cfg->tau_z;
    if (e == cudaSuccess && calibrate) e = cudaMemcpyAsync(&tau, tau_dev, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("densify counts", e); return SSG_ERR_CUDA; }
    for (int k = 0; k < 4; k++) counts_host[k] = host[k];
    *tau_z_host = tau;
    return SSG_OK;
}

extern "C" int ssg_densify_apply(const ssg_scene *scene, const ssg_params *out, const ssg_adam_state *adam_in,
                                 const ssg_adam_state *adam_out, const ssg_densify_stats *stats,
                                 const ssg_densify_cfg *cfg, const uint8_t *flags, void *temp, int32_t *bad,
                                 void *stream) {
    using namespace ssg;
    if (!scene || !out || !stats || !cfg || !bad || scene->n < 0) return SSG_ERR_INVALID_ARGUMENT;
    if (out->sh_coeffs != scene->sh_coeffs) return SSG_ERR_INVALID_ARGUMENT;
    const int64_t n = scene->n;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) { set_error("memset bad", e); return SSG_ERR_CUDA; }
    if (n == 0) return SSG_OK;
    const DensifyTemp T = densify_temp(n);
    char *tp = (char *)temp;
    ssg_adam_state none;
    memset(&none, 0, sizeof(none));
    const unsigned nb = (unsigned)((n + kDThreads - 1) / kDThreads);
    k_densify_apply<<<nb, kDThreads, 0, st>>>(n, *scene, *out, adam_in ? *adam_in : none,
                                              adam_out ? *adam_out : none, *stats, *cfg, flags,
                                              (const uint32_t *)(tp + T.block_counts),
                                              (const int64_t *)(tp + T.totals), bad);
    return check_launch("ssg_densify_apply");
}
