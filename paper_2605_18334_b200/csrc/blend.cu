// blend.cu -- K5/K6: per-tile front-to-back skew-kernel blending and its
// back-to-front backward replay.
//
// Reference: raster/_core.pyx:77-166 (_forward_tile) and :203-312
// (_backward_tile), twin raster/_cpu.py:31-158; per-primitive reduction of
// the (M,12) slots raster/backward.py:70-73.
//
// Layout: one CTA per 16x16 tile, one thread per pixel (thread t -> local
// pixel (t & 15, t >> 4)).  Instance batches of 256 are staged in shared
// memory as three float4 rows per splat with the mean made tile-local in
// fp64 before rounding to fp32 (|offset| stays small, so dx/dy keep ~1e-6 px
// precision even at x ~ 2000).  The block leaves the instance loop when
// every pixel has stopped (__syncthreads_count vote, _core.pyx:155-156).
// Backward: the 12 per-instance sums are reduced with a transposed butterfly
// (16 shuffles per warp instead of 60), accumulated per instance in shared
// memory, and flushed once per instance with float4 global atomics.
#include "ssg_common.cuh"

namespace ssg {

struct __align__(16) StagedSplat {
    float4 a;  // mx_local, my_local, conic_a, conic_b
    float4 b;  // conic_c, skew_x, skew_y, o1
    float4 c;  // o2, r, g, b
};

__device__ __forceinline__ void stage_splat(const ssg_splat *splat, uint32_t p, double ox, double oy,
                                            float4 &A, float4 &B, float4 &C) {
    const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
    const float4 q1 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 1);
    const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
    const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
    // q1 = (a, b, c, sx)  q2 = (sy, o1, o2, r)  q3 = (g, b, pad, pad)
    A = make_float4((float)(m.x - ox), (float)(m.y - oy), q1.x, q1.y);
    B = make_float4(q1.z, q1.w, q2.x, q2.y);
    C = make_float4(q2.z, q2.w, q3.x, q3.y);
}

__global__ void __launch_bounds__(256)
k_blend_forward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                const int32_t *__restrict__ ranges, float *__restrict__ color,
                float *__restrict__ final_T, int32_t *__restrict__ n_contrib,
                int32_t *__restrict__ last_idx) {
    __shared__ float4 sA[256], sB[256], sC[256];
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool inside = px < W && py < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);

    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int nc = 0, li = -1;
    bool done = !inside;

    for (int base = start; base < end; base += 256) {
        if (__syncthreads_count(done) == 256) break;
        const int k = base + threadIdx.x;
        if (k < end) {
            float4 A, B, C;
            stage_splat(splat, inst_prim[k], ox, oy, A, B, C);
            sA[threadIdx.x] = A;
            sB[threadIdx.x] = B;
            sC[threadIdx.x] = C;
        }
        __syncthreads();
        const int cnt = min(256, end - base);
        if (!done) {
            for (int j = 0; j < cnt; j++) {
                const float4 A = sA[j];
                const float4 B = sB[j];
                const float dx = fx - A.x, dy = fy - A.y;
                // _core.pyx:133-135
                const float power = -0.5f * (A.z * dx * dx + B.x * dy * dy) - A.w * dx * dy;
                if (power > 0.0f) continue;
                const float4 C = sC[j];
                float E = 1.0f, o = 0.5f * (B.w + C.x);
                if (B.y != 0.0f || B.z != 0.0f) {  // warp-uniform: skew-free splats skip erf
                    const float z = (B.y * dx + B.z * dy) * SSG_SQRT1_2;   // :136
                    E = skew_E(z);                                          // :137
                    o = 0.5f * ((B.w + C.x) + (B.w - C.x) * (E - 1.0f));    // :138
                }
                const float Aval = o * fast_exp2(power * SSG_LOG2E) * E;   // :139
                const float alpha = fminf(Aval, SSG_ALPHA_MAX);             // :140
                if (alpha < SSG_ALPHA_SKIP) continue;                       // :141-142
                const float test_T = T * (1.0f - alpha);                    // :143
                if (test_T < SSG_T_STOP) { done = true; break; }            // :144-147
                const float w = alpha * T;                                  // :148-154
                C0 = fmaf(w, C.y, C0);
                C1 = fmaf(w, C.z, C1);
                C2 = fmaf(w, C.w, C2);
                T = test_T;
                nc++;
                li = base + j;
            }
        }
    }
    if (inside) {  // :158-166
        const int64_t pix = (int64_t)py * W + px;
        color[3 * pix] = C0 + T * bg0;
        color[3 * pix + 1] = C1 + T * bg1;
        color[3 * pix + 2] = C2 + T * bg2;
        final_T[pix] = T;
        n_contrib[pix] = nc;
        last_idx[pix] = li;
    }
}

// Transposed butterfly: v[0..15] per lane -> lane holds the warp sum of
// component (lane >> 1) & 15 in v[0] (lanes 2i and 2i+1 both).
__device__ __forceinline__ float warp_reduce_transposed16(float (&v)[16], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        float send = b4 ? v[i] : v[i + 8];
        float keep = b4 ? v[i + 8] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        float send = b3 ? v[i] : v[i + 4];
        float keep = b3 ? v[i + 4] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int i = 0; i < 2; i++) {
        float send = b2 ? v[i] : v[i + 2];
        float keep = b2 ? v[i + 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {
        float send = b1 ? v[0] : v[1];
        float keep = b1 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__global__ void __launch_bounds__(256)
k_blend_backward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                 const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                 const int32_t *__restrict__ ranges, const float *__restrict__ final_T,
                 const int32_t *__restrict__ last_idx, const float *__restrict__ dL,
                 float *__restrict__ grad_screen) {
    __shared__ float4 sA[256], sB[256], sC[256];
    __shared__ uint32_t sP[256];
    __shared__ float sAcc[256 * 12];
    __shared__ int sMax[8];
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool inside = px < W && py < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    if (end <= start) return;
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);
    const int64_t pix = (int64_t)py * W + px;

    // _core.pyx:232-246
    float T = 1.0f, d0 = 0.0f, d1 = 0.0f, d2 = 0.0f;
    int li = -1;
    if (inside) {
        T = final_T[pix];
        li = last_idx[pix];
        d0 = dL[3 * pix];
        d1 = dL[3 * pix + 1];
        d2 = dL[3 * pix + 2];
    }
    float R0 = bg0, R1 = bg1, R2 = bg2;
    int wmax = __reduce_max_sync(0xffffffffu, li);
    if (lane == 0) sMax[warp] = wmax;
    __syncthreads();
    int maxli = sMax[0];
#pragma unroll
    for (int w = 1; w < 8; w++) maxli = max(maxli, sMax[w]);
    if (maxli < start) return;  // any_hit == 0 (:245-246); uniform
    const int hi = min(maxli + 1, end);

    for (int top = hi; top > start; top -= 256) {
        const int lo = max(start, top - 256);
        const int cnt = top - lo;
        __syncthreads();  // previous batch fully flushed
        if (threadIdx.x < cnt) {
            const uint32_t p = inst_prim[lo + threadIdx.x];
            float4 A, B, C;
            stage_splat(splat, p, ox, oy, A, B, C);
            sA[threadIdx.x] = A;
            sB[threadIdx.x] = B;
            sC[threadIdx.x] = C;
            sP[threadIdx.x] = p;
        }
#pragma unroll
        for (int q = 0; q < 12; q++) sAcc[q * 256 + threadIdx.x] = 0.0f;
        __syncthreads();

        for (int j = cnt - 1; j >= 0; j--) {
            const int k = lo + j;
            float g[16];
#pragma unroll
            for (int q = 0; q < 16; q++) g[q] = 0.0f;
            bool contrib = false;
            if (k <= li) {  // :263-264
                const float4 A = sA[j];
                const float4 B = sB[j];
                const float dx = fx - A.x, dy = fy - A.y;
                const float power = -0.5f * (A.z * dx * dx + B.x * dy * dy) - A.w * dx * dy;
                if (power <= 0.0f) {
                    const float4 C = sC[j];
                    const bool skewed = (B.y != 0.0f || B.z != 0.0f);
                    float E = 1.0f, z = 0.0f;
                    if (skewed) {
                        z = (B.y * dx + B.z * dy) * SSG_SQRT1_2;
                        E = skew_E(z);
                    }
                    const float o1 = B.w, o2 = C.x;
                    const float o = 0.5f * ((o1 + o2) + (o1 - o2) * (E - 1.0f));
                    const float G = fast_exp2(power * SSG_LOG2E);
                    const float Aval = o * G * E;
                    const float alpha = fminf(Aval, SSG_ALPHA_MAX);
                    if (alpha >= SSG_ALPHA_SKIP) {
                        contrib = true;
                        T = __fdividef(T, 1.0f - alpha);                                  // :280
                        const float d_alpha = T * ((C.y - R0) * d0 + (C.z - R1) * d1 + (C.w - R2) * d2);
                        const float aT = alpha * T;
                        g[9] = aT * d0;
                        g[10] = aT * d1;
                        g[11] = aT * d2;
                        const float DA = Aval <= SSG_ALPHA_MAX ? d_alpha : 0.0f;          // :290
                        const float d_power = DA * Aval;
                        const float Gez2 = skewed ? fast_exp2((power - z * z) * SSG_LOG2E) : G;
                        const float d_z = DA * SSG_TWO_OVER_SQRT_PI * Gez2 * (o + 0.5f * (o1 - o2) * E);
                        const float d_dx = d_power * (-(A.z * dx + A.w * dy)) + d_z * B.y * SSG_SQRT1_2;
                        const float d_dy = d_power * (-(B.x * dy + A.w * dx)) + d_z * B.z * SSG_SQRT1_2;
                        const float GE = G * E;
                        g[0] = -d_dx;
                        g[1] = -d_dy;
                        g[2] = d_power * (-0.5f * dx * dx);
                        g[3] = d_power * (-dx * dy);
                        g[4] = d_power * (-0.5f * dy * dy);
                        g[5] = d_z * dx * SSG_SQRT1_2;
                        g[6] = d_z * dy * SSG_SQRT1_2;
                        g[7] = DA * 0.5f * GE * E;
                        g[8] = DA * 0.5f * (2.0f - E) * GE;
                        R0 = alpha * C.y + (1.0f - alpha) * R0;                           // :306-308
                        R1 = alpha * C.z + (1.0f - alpha) * R1;
                        R2 = alpha * C.w + (1.0f - alpha) * R2;
                    }
                }
            }
            if (__any_sync(0xffffffffu, contrib)) {
                const float v = warp_reduce_transposed16(g, lane);
                const int idx = (lane >> 1) & 15;
                if (!(lane & 1) && idx < 12) atomicAdd(&sAcc[j * 12 + idx], v);
            }
        }
        __syncthreads();
        if (threadIdx.x < cnt) {  // raster/backward.py:70-73, one flush per instance
            float s[12];
            bool any = false;
#pragma unroll
            for (int q = 0; q < 12; q++) {
                s[q] = sAcc[threadIdx.x * 12 + q];
                any |= s[q] != 0.0f;
            }
            if (any) {
                float4 *dst = reinterpret_cast<float4 *>(grad_screen + (size_t)sP[threadIdx.x] * 12);
                atomicAdd(dst, make_float4(s[0], s[1], s[2], s[3]));
                atomicAdd(dst + 1, make_float4(s[4], s[5], s[6], s[7]));
                atomicAdd(dst + 2, make_float4(s[8], s[9], s[10], s[11]));
            }
        }
    }
}

}  // namespace ssg

extern "C" int ssg_blend_forward(int64_t m, int32_t width, int32_t height, const float background[3],
                                 const ssg_splat *splat, const ssg_bin_buffers *bins,
                                 const ssg_frame_buffers *frame, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !background || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    (void)m;
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    cudaStream_t st = (cudaStream_t)stream;
    k_blend_forward<<<ntx * nty, 256, 0, st>>>(ntx, width, height, background[0], background[1],
                                               background[2], splat, bins->inst_prim, bins->ranges,
                                               frame->color, frame->final_T, frame->n_contrib,
                                               frame->last_idx);
    return check_launch("k_blend_forward");
}

extern "C" int ssg_blend_backward(int64_t n, int64_t m, int32_t width, int32_t height,
                                  const float background[3], const ssg_splat *splat,
                                  const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                  const float *dL_dpixels, const ssg_grad_buffers *grads, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !grads || !background || !dL_dpixels || width < 1 || height < 1)
        return SSG_ERR_INVALID_ARGUMENT;
    (void)m;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(grads->screen, 0, sizeof(float) * 12 * (size_t)n, st);
    if (e != cudaSuccess) { set_error("memset screen grads", e); return SSG_ERR_CUDA; }
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_backward<<<ntx * nty, 256, 0, st>>>(ntx, width, height, background[0], background[1],
                                                background[2], splat, bins->inst_prim, bins->ranges,
                                                frame->final_T, frame->last_idx, dL_dpixels,
                                                grads->screen);
    return check_launch("k_blend_backward");
}
