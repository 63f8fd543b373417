// train.cu -- the training-step glue around the rasterizer, on the device
// (SURVEY.md §8(f) row 1): the photometric loss with its analytic pixel
// gradient, the scene regularizers, and the densification interval
// statistics.
//
// Reference:
//   optimize/losses.py:38-41    l1_loss: mean |x - y|, grad sign(x - y) / size
//   optimize/losses.py:44-100   ssim: mean SSIM over 'valid' 11x11 Gaussian
//                               windows (sigma 1.5, C1 = 0.01^2, C2 = 0.03^2),
//                               channels averaged, and its adjoint through
//                               'full' convolutions
//   optimize/losses.py:103-113  image_loss: (1 - l) L1 + l (1 - SSIM)
//   optimize/losses.py:116-136  scene_regularizers: lambda_beta * sum |beta|^2,
//                               lambda_opacity * sum |sig(l1) - sig(l2)|
//   trainer.py:40-58            _IntervalStats: sum g_uv, max g_z, sum d_mu
//
// The 11x11 window is the outer product of one normalised 1-D Gaussian, so
// every windowed mean is two 11-tap passes over a shared-memory tile.  One
// CTA produces a 32x32 block of outputs, channel by channel; the loss
// values are accumulated in fp64 with one atomic per CTA.
#include "ssg_common.cuh"

namespace ssg {

constexpr int kWin = 11, kHalo = kWin - 1;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

__constant__ float c_gauss[kWin];

__device__ __forceinline__ double block_sum(double v, double *s_red) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) tot += s_red[i];
    __syncthreads();
    return tot;
}

// The two passes below work on 32x32 output blocks (256 threads) one
// channel at a time.  Both separable 11-tap passes are register-blocked: a
// horizontal task produces 4 adjacent outputs of one row from 14 staged
// inputs, a vertical task 4 adjacent outputs of one column from 14 rows, so
// each shared-memory load feeds ~4 FMAs instead of 1.  The adjoint maps are
// planar in `gm` ([3c + k][Hv][Wv]): coalesced stores and loads.
constexpr int kBT = 32, kBR = kBT + kHalo, kBS = kBR + 1;  // block, block + halo, padded row stride
constexpr int kGrp = kBT / 4;                               // 4-wide groups per block row

// 11-tap weighted sums of 4 consecutive outputs from 14 inputs
__device__ __forceinline__ void taps4(const float (&v)[14], float (&o)[4]) {
#pragma unroll
    for (int q = 0; q < 4; q++) o[q] = 0.f;
#pragma unroll
    for (int u = 0; u < kWin; u++) {
        const float w = c_gauss[u];
#pragma unroll
        for (int q = 0; q < 4; q++) o[q] = fmaf(w, v[q + u], o[q]);
    }
}

// Pass 1: per valid window (output (i, j) covers input rows i..i+10, columns
// j..j+10) and channel: SSIM s and the three adjoint maps of losses.py:86-93
// (g_mu_x, g_wxx, g_wxy), plus the L1 and SSIM sums.
__global__ void __launch_bounds__(256) k_loss_stats(const float *__restrict__ img, const float *__restrict__ tgt,
                                                    int H, int W, int with_ssim, float inv_n,
                                                    float *__restrict__ gm, double *__restrict__ sums) {
    __shared__ float sx[kBR * kBS], sy[kBR * kBS];
    __shared__ float hs[5][kBR][kBT + 1];  // +1: conflict-free 4-wide row writes
    __shared__ double s_red[8];
    const int t = threadIdx.x;
    const int i0 = blockIdx.y * kBT, j0 = blockIdx.x * kBT;
    double l1 = 0.0, ss = 0.0;
    // L1 over the block's own pixels (every pixel counted once)
    for (int q = t; q < kBT * kBT; q += 256) {
        const int i = i0 + q / kBT, j = j0 + q % kBT;
        if (i < H && j < W)
            for (int c = 0; c < 3; c++) {
                const size_t p = ((size_t)i * W + j) * 3 + c;
                l1 += fabsf(img[p] - tgt[p]);
            }
    }
    if (with_ssim) {
        const int Hv = H - kHalo, Wv = W - kHalo;
        const size_t plane = (size_t)Hv * Wv;
        const int vx = t % kBT, vg = t / kBT;  // vertical task: column vx, rows 4vg..4vg+3
        for (int c = 0; c < 3; c++) {
            for (int q = t; q < kBR * kBR; q += 256) {
                const int r = q / kBR, cc = q % kBR;
                const int i = i0 + r, j = j0 + cc;
                const bool in = i < H && j < W;
                const size_t p = ((size_t)i * W + j) * 3 + c;
                sx[r * kBS + cc] = in ? img[p] : 0.0f;
                sy[r * kBS + cc] = in ? tgt[p] : 0.0f;
            }
            __syncthreads();
            // horizontal: row r, columns 4g..4g+3 of the block
            for (int q = t; q < kBR * kGrp; q += 256) {
                const int r = q / kGrp, g = q % kGrp;
                float x[14], y[14], o[4];
#pragma unroll
                for (int u = 0; u < 14; u++) {
                    x[u] = sx[r * kBS + 4 * g + u];
                    y[u] = sy[r * kBS + 4 * g + u];
                }
                taps4(x, o);
#pragma unroll
                for (int k = 0; k < 4; k++) hs[0][r][4 * g + k] = o[k];
                taps4(y, o);
#pragma unroll
                for (int k = 0; k < 4; k++) hs[1][r][4 * g + k] = o[k];
                float pr[14];
#pragma unroll
                for (int u = 0; u < 14; u++) pr[u] = x[u] * x[u];
                taps4(pr, o);
#pragma unroll
                for (int k = 0; k < 4; k++) hs[2][r][4 * g + k] = o[k];
#pragma unroll
                for (int u = 0; u < 14; u++) pr[u] = y[u] * y[u];
                taps4(pr, o);
#pragma unroll
                for (int k = 0; k < 4; k++) hs[3][r][4 * g + k] = o[k];
#pragma unroll
                for (int u = 0; u < 14; u++) pr[u] = x[u] * y[u];
                taps4(pr, o);
#pragma unroll
                for (int k = 0; k < 4; k++) hs[4][r][4 * g + k] = o[k];
            }
            __syncthreads();
            // vertical: column vx, rows 4vg..4vg+3 -> SSIM terms
            float st[5][4];
#pragma unroll
            for (int m = 0; m < 5; m++) {
                float v[14];
#pragma unroll
                for (int u = 0; u < 14; u++) v[u] = hs[m][4 * vg + u][vx];
                taps4(v, st[m]);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int i = i0 + 4 * vg + q, j = j0 + vx;
                if (i >= Hv || j >= Wv) continue;
                const float mx = st[0][q], my = st[1][q];
                const float vxx = st[2][q] - mx * mx, vyy = st[3][q] - my * my, cov = st[4][q] - mx * my;
                const float a1 = 2.f * mx * my + kC1, a2 = 2.f * cov + kC2;
                const float b1 = mx * mx + my * my + kC1, b2 = vxx + vyy + kC2;
                const float sv = (a1 * a2) / (b1 * b2);
                ss += sv;
                // losses.py:86-93, divided by n = Hv * Wv * 3
                const float g_a1 = a2 / (b1 * b2) * inv_n, g_a2 = a1 / (b1 * b2) * inv_n;
                const float g_b1 = -sv / b1 * inv_n, g_b2 = -sv / b2 * inv_n;
                const float g_mu = 2.f * my * g_a1 + 2.f * mx * g_b1 - 2.f * mx * g_b2 - my * 2.f * g_a2;
                const size_t o = (size_t)i * Wv + j;
                gm[(3 * c) * plane + o] = g_mu;
                gm[(3 * c + 1) * plane + o] = g_b2;
                gm[(3 * c + 2) * plane + o] = 2.f * g_a2;
            }
            __syncthreads();  // sx / sy / hs reused by the next channel
        }
    }
    const double t1 = block_sum(l1, s_red);
    const double t2 = block_sum(ss, s_red);
    if (t == 0) {
        atomicAdd(&sums[0], t1);
        if (with_ssim) atomicAdd(&sums[1], t2);
    }
}

// Pass 2: dL/dpixel = (1 - l) sign(x - y) / size - l * dSSIM/dx, with
// dSSIM/dx = full(g_mu) + 2 x full(g_wxx) + y full(g_wxy) (losses.py:94-96,
// 112).  Full convolution: output (i, j) gathers windows i-10..i, j-10..j.
__global__ void __launch_bounds__(256) k_loss_grad(const float *__restrict__ img, const float *__restrict__ tgt,
                                                   const float *__restrict__ gm, int H, int W, int with_ssim,
                                                   float w_l1, float w_ssim, float *__restrict__ dL) {
    __shared__ float sg[3][kBR * kBS];
    __shared__ float hs[3][kBR][kBT + 1];
    const int t = threadIdx.x;
    const int i0 = blockIdx.y * kBT, j0 = blockIdx.x * kBT;
    const int Hv = H - kHalo, Wv = W - kHalo;
    const size_t plane = (size_t)(with_ssim ? Hv : 0) * (with_ssim ? Wv : 0);
    const int vx = t % kBT, vg = t / kBT;
    for (int c = 0; c < 3; c++) {
        float f[3][4];
        if (with_ssim) {
            // gm rows i0-10 .. i0+31, columns j0-10 .. j0+31 of channel c's three maps
            for (int q = t; q < kBR * kBR; q += 256) {
                const int r = q / kBR, cc = q % kBR;
                const int i = i0 - kHalo + r, j = j0 - kHalo + cc;
                const bool in = i >= 0 && j >= 0 && i < Hv && j < Wv;
                const size_t o = in ? (size_t)i * Wv + j : 0;
#pragma unroll
                for (int k = 0; k < 3; k++) sg[k][r * kBS + cc] = in ? gm[(3 * c + k) * plane + o] : 0.0f;
            }
            __syncthreads();
            for (int q = t; q < 3 * kBR * kGrp; q += 256) {
                const int k = q / (kBR * kGrp), rem = q % (kBR * kGrp);
                const int r = rem / kGrp, g = rem % kGrp;
                float v[14], o[4];
#pragma unroll
                for (int u = 0; u < 14; u++) v[u] = sg[k][r * kBS + 4 * g + u];
                taps4(v, o);
#pragma unroll
                for (int e = 0; e < 4; e++) hs[k][r][4 * g + e] = o[e];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 3; k++) {
                float v[14];
#pragma unroll
                for (int u = 0; u < 14; u++) v[u] = hs[k][4 * vg + u][vx];
                taps4(v, f[k]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = i0 + 4 * vg + q, j = j0 + vx;
            if (i >= H || j >= W) continue;
            const size_t p = ((size_t)i * W + j) * 3 + c;
            const float x = img[p], y = tgt[p], d = x - y;
            float g = w_l1 * (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f));
            if (with_ssim) g -= w_ssim * (f[0][q] + 2.f * x * f[1][q] + y * f[2][q]);
            dL[p] = g;
        }
        if (with_ssim) __syncthreads();  // sg / hs reused by the next channel
    }
}

// losses.py:116-136 on the device: d_beta = d_eta + 2 lb beta (the rendered
// part of d_beta equals d_eta, projection.py:365-366), d_logits += the
// opacity-gap term; sums[2] += lb sum beta^2 + lo sum |gap|.
__global__ void k_regularize(int64_t n, const float *__restrict__ beta, const float *__restrict__ logits,
                             const float *__restrict__ d_eta, float lb, float lo, float *__restrict__ d_beta,
                             float *__restrict__ d_logits, double *__restrict__ sums) {
    __shared__ double s_red[8];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double val = 0.0;
    if (i < n) {
        for (int j = 0; j < 3; j++) {
            const float b = beta[3 * i + j];
            if (d_beta) d_beta[3 * i + j] = d_eta[3 * i + j] + (lb > 0.f ? 2.f * lb * b : 0.f);
            if (lb > 0.f) val += (double)lb * (double)b * (double)b;
        }
        if (lo > 0.f) {
            // kernel_math.py:158-165 branch-stable sigmoid, in fp64 like the reference
            double sg[2];
            for (int j = 0; j < 2; j++) {
                const double l = logits[2 * i + j];
                sg[j] = l >= 0 ? 1.0 / (1.0 + exp(-l)) : exp(l) / (1.0 + exp(l));
            }
            const double gap = sg[0] - sg[1];
            val += (double)lo * fabs(gap);
            const double sgn = gap > 0 ? 1.0 : (gap < 0 ? -1.0 : 0.0);
            if (d_logits) {
                d_logits[2 * i] += (float)(lo * sgn * sg[0] * (1.0 - sg[0]));
                d_logits[2 * i + 1] += (float)(-lo * sgn * sg[1] * (1.0 - sg[1]));
            }
        }
    }
    const double t = block_sum(val, s_red);
    if (threadIdx.x == 0 && t != 0.0) atomicAdd(&sums[2], t);
}

// trainer.py:49-53: uv_sum += g_uv; z_max = max(z_max, g_z); mu_sum += d_mu
__global__ void k_stats_add(int64_t n, const float *__restrict__ g_uv, const float *__restrict__ g_z,
                            const float *__restrict__ d_mu, double *__restrict__ uv_sum, float *__restrict__ z_max,
                            double *__restrict__ mu_sum, const int32_t *__restrict__ skip) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (skip && *skip)) return;
    uv_sum[i] += (double)g_uv[i];
    z_max[i] = fmaxf(z_max[i], g_z[i]);
    for (int j = 0; j < 3; j++) mu_sum[3 * i + j] += (double)d_mu[3 * i + j];
}

}  // namespace ssg

extern "C" int64_t ssg_loss_scratch_floats(int32_t width, int32_t height) {
    if (width < ssg::kWin || height < ssg::kWin) return 9;
    return 9 * (int64_t)(width - ssg::kHalo) * (height - ssg::kHalo);
}

extern "C" int ssg_image_loss(const float *rendered, const float *target, int32_t width, int32_t height,
                              float lambda_ssim, float *scratch, float *dL_dpixels, double *sums, void *stream) {
    using namespace ssg;
    if (!rendered || !target || !dL_dpixels || !sums || width < 1 || height < 1 || lambda_ssim < 0.f)
        return SSG_ERR_INVALID_ARGUMENT;
    const int with_ssim = lambda_ssim != 0.0f;
    if (with_ssim && (width < kWin || height < kWin)) return SSG_ERR_INVALID_ARGUMENT;  // losses.py:58-59
    if (with_ssim && !scratch) return SSG_ERR_INVALID_ARGUMENT;
    // __constant__ memory belongs to each device: upload once per device ordinal
    static DeviceOnce gauss_once;
    {
        const cudaError_t e = gauss_once.run([](int) {  // losses.py:28-32, normalised in fp64
            double g[kWin], sum = 0.0;
            for (int u = 0; u < kWin; u++) {
                const double x = u - (kWin - 1) / 2.0;
                g[u] = exp(-x * x / (2.0 * 1.5 * 1.5));
                sum += g[u];
            }
            float gf[kWin];
            for (int u = 0; u < kWin; u++) gf[u] = (float)(g[u] / sum);
            return cudaMemcpyToSymbol(c_gauss, gf, sizeof(gf));
        });
        if (e != cudaSuccess) { set_error("gauss constant", e); return SSG_ERR_CUDA; }
    }
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(sums, 0, 2 * sizeof(double), st);
    if (e != cudaSuccess) { set_error("memset sums", e); return SSG_ERR_CUDA; }
    const dim3 grid((width + kBT - 1) / kBT, (height + kBT - 1) / kBT);
    const float inv_n = with_ssim ? 1.0f / (3.0f * (float)(width - kHalo) * (float)(height - kHalo)) : 0.0f;
    k_loss_stats<<<grid, 256, 0, st>>>(rendered, target, height, width, with_ssim, inv_n, scratch, sums);
    const float w_l1 = (1.0f - lambda_ssim) / (3.0f * (float)width * (float)height);
    k_loss_grad<<<grid, 256, 0, st>>>(rendered, target, scratch, height, width, with_ssim, w_l1, lambda_ssim,
                                      dL_dpixels);
    return check_launch("ssg_image_loss");
}

extern "C" int ssg_regularize(int64_t n, const float *beta, const float *opacity_logits, const float *d_eta,
                              float lambda_beta, float lambda_opacity, float *d_beta, float *d_logits,
                              double *sums, void *stream) {
    using namespace ssg;
    // d_eta, d_beta and d_logits all NULL = the penalty value only (the
    // finite-loss test of a step runs before its backward)
    const bool value_only = !d_eta && !d_beta && !d_logits;
    if (n < 0 || (n > 0 && (!beta || !opacity_logits || (!value_only && (!d_eta || !d_beta || !d_logits)))) ||
        !sums)
        return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(sums + 2, 0, sizeof(double), st);
    if (e != cudaSuccess) { set_error("memset reg", e); return SSG_ERR_CUDA; }
    if (n == 0) return SSG_OK;
    k_regularize<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, beta, opacity_logits, d_eta, lambda_beta,
                                                               lambda_opacity, d_beta, d_logits, sums);
    return check_launch("ssg_regularize");
}

extern "C" int ssg_interval_stats_add_ex(int64_t n, const float *g_uv, const float *g_z, const float *d_mu,
                                         double *uv_sum, float *z_max, double *mu_sum, const int32_t *skip,
                                         void *stream) {
    using namespace ssg;
    if (n < 0 || (n > 0 && (!g_uv || !g_z || !d_mu || !uv_sum || !z_max || !mu_sum))) return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    k_stats_add<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, g_uv, g_z, d_mu, uv_sum, z_max,
                                                                               mu_sum, skip);
    return check_launch("ssg_interval_stats_add");
}

extern "C" int ssg_interval_stats_add(int64_t n, const float *g_uv, const float *g_z, const float *d_mu,
                                      double *uv_sum, float *z_max, double *mu_sum, void *stream) {
    return ssg_interval_stats_add_ex(n, g_uv, g_z, d_mu, uv_sum, z_max, mu_sum, nullptr, stream);
}

namespace ssg {
__global__ void k_step_value(const double *sums, int32_t W, int32_t H, double lam, const int64_t *n_inst,
                             int64_t capacity, double *loss, int32_t *flag) {
    // explicit roundings: the operations of ImageLoss.value_tensor (torch fp64)
    const double l1 = __ddiv_rn(sums[0], __dmul_rn(__dmul_rn(3.0, (double)W), (double)H));
    double img = l1;
    if (lam != 0.0) {
        const double n = __dmul_rn(__dmul_rn(3.0, (double)(W - 10)), (double)(H - 10));
        img = __dadd_rn(__dmul_rn(__dsub_rn(1.0, lam), l1), __dmul_rn(lam, __dsub_rn(1.0, __ddiv_rn(sums[1], n))));
    }
    const double v = __dadd_rn(img, sums[2]);
    *loss = v;
    if (flag) *flag = (n_inst && n_inst[1] > capacity) ? 2 : (isfinite(v) ? 0 : 1);
}
}  // namespace ssg

extern "C" int ssg_step_value(const double *sums, int32_t width, int32_t height, double lambda_ssim,
                              const int64_t *n_instances, int64_t capacity, double *loss, int32_t *flag,
                              void *stream) {
    using namespace ssg;
    if (!sums || !loss || width < 1 || height < 1 || lambda_ssim < 0.0) return SSG_ERR_INVALID_ARGUMENT;
    k_step_value<<<1, 1, 0, (cudaStream_t)stream>>>(sums, width, height, lambda_ssim, n_instances, capacity, loss,
                                                    flag);
    return check_launch("k_step_value");
}
