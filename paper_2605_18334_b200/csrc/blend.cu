// blend.cu -- K5/K6: per-tile front-to-back skew-kernel blending and its
// back-to-front backward replay.
//
// Reference: raster/_core.pyx:77-166 (_forward_tile) and :203-312
// (_backward_tile), twin raster/_cpu.py:31-158; per-primitive reduction of
// the (M,12) slots raster/backward.py:70-73.
//
// Layout: one CTA of 256 threads per 16x16 tile, one thread per pixel; warp
// w owns the 8x4 pixel block at (8*(w&1), 4*(w>>1)).  Instance batches of 256
// are staged in shared memory with the mean made tile-local in fp64 before
// rounding to fp32 (offsets stay small, so dx/dy keep ~1e-6 px precision at
// x ~ 2000).  Every staged instance also carries the bounding box of the
// ellipse outside of which its alpha is certainly below 1/255 (see
// stage_splat).  Each warp then walks the batch 32 instances at a time: one
// lane per instance tests the box against the warp's 8x4 block, a ballot
// gives the hit mask, and the warp evaluates only the hits, in order.  The
// culling is conservative, so the per-pixel decisions (skip / blend / stop)
// are exactly those of the unculled loop; it removes the pixel-instance pairs
// that cannot contribute before any arithmetic is spent on them.
// Backward: the 12 per-instance sums of a warp are reduced with a transposed
// butterfly (13 shuffles instead of 60) and added to the primitive's
// gradient row by the 12 lanes holding them, one scalar global reduction
// each (one RED instruction; measured 2.4 % faster than gathering them into
// three float4 vector REDs; the shared-memory fp32 atomic on sm_100 is a CAS
// loop, so no smem staging).
#include "ssg_common.cuh"

#ifdef SSG_BLEND_STATS
// diagnostic build only (tools/blend_stats.py): warp-level event counters
__device__ unsigned long long g_blend_stats[32];
#define SSG_STAT(i, v) atomicAdd(&g_blend_stats[i], (unsigned long long)(v))
#endif

namespace ssg {

constexpr int kThreads = 256;
constexpr int kBatch = 256;

// Shared-memory image of one instance:
//   A = (mx_local, my_local, conic_a, conic_b)
//   B = (conic_c, far_thr, skew_x, skew_y)
//   C = (o_sum, o_diff, r, g),  D = b
//   X = (k, h, m, r2m): the ellipse {d : a dx^2 + 2b dx dy + c dy^2 <= r2m}
//       in completed-square form, k = b/a, h = det/a, m = b/c
// far_thr is a per-instance lower bound on the Gaussian exponent below which
// alpha < 1/255 is certain: A = o*G*E <= omax*G*Emax with Emax = 2 (1 for
// skew-free splats), so power < ln(1/(255*omax*Emax)) implies the reference's
// ALPHA_SKIP test (_core.pyx:141) fires.  A 1e-4 margin keeps the shortcut
// strictly inside the region where the full fp32 evaluation also skips.  The
// ellipse {power >= far_thr} (r2 = -2 far_thr, widened by 1e-3 relative +
// 1e-4 absolute) is what the per-warp culling tests against the warp's 8x4
// block of pixel centres, exactly (not via its bounding box).
struct SmemBatch {
    float4 A[kBatch];
    float4 B[kBatch];
    float4 C[kBatch];
    float4 X[kBatch];
    float D[kBatch];
};

template <typename S>
__device__ __forceinline__ void stage_splat(const ssg_splat *splat, uint32_t p, double ox, double oy,
                                            S &s, int slot) {
    const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
    const float4 q1 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 1);
    const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
    const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
    // q1 = (a, b, c, sx)  q2 = (sy, o1, o2, r)  q3 = (g, b, pad, pad)
    const bool skewed = (q1.w != 0.0f || q2.x != 0.0f);
    const float omax = fmaxf(q2.y, q2.z) * (skewed ? 2.0f : 1.0f);
    const float thr = omax > 0.0f ? -logf(255.0f * omax) - 1e-4f : INFINITY;
    const float mx = (float)(m.x - ox), my = (float)(m.y - oy);
    const float a = q1.x, b = q1.y, c = q1.z;
    const float r2 = -2.0f * thr;
    float4 ell;
    if (!(r2 > 0.0f)) {
        ell = make_float4(0.0f, 0.0f, 0.0f, -1.0f);                 // never blends: never hits
    } else {
        const double det = (double)a * (double)c - (double)b * (double)b;   // exact products
        if (a > 0.0f && c > 0.0f && det > 0.0)
            ell = make_float4(b / a, (float)(det / (double)a), b / c, fmaf(r2, 1.001f, 1e-4f));
        else
            ell = make_float4(0.0f, 0.0f, 0.0f, INFINITY);          // degenerate: always evaluate
    }
    s.A[slot] = make_float4(mx, my, a, b);
    s.B[slot] = make_float4(c, thr, q1.w, q2.x);
    s.C[slot] = make_float4(0.5f * (q2.y + q2.z), 0.5f * (q2.y - q2.z), q2.w, q3.x);
    s.D[slot] = q3.y;
    s.X[slot] = ell;
}

// Does the instance's ellipse meet the rectangle spanned by the warp's pixel
// centres [wx0+0.5, wx0+7.5] x [wy0+0.5, wy0+3.5]?  Minimum of the quadratic
// form over the rectangle: 0 if the mean is inside, else the least of the
// four clamped edge minima, each a sum of non-negative terms
// a (dx + k dy)^2 + h dy^2 (no cancellation).
//
// Skewed splats: far_thr assumes the largest skew factor, E <= 2.  Where the
// whole block lies on the negative side of the skew direction (z <= zmax <
// 0 at every pixel centre, z = (sx dx + sy dy)/sqrt2), E = erfc(-z) <=
// exp(-zmax^2) < 1 there, so alpha < 1/255 already for power < far_thr +
// ln 2 + zmax^2: the ellipse shrinks by 2 (ln 2 + zmax^2) in r2 for this
// block (the 1e-4 margin of far_thr and the 1.001 widening carry over).
// Skew-free splats have zmax = 0 and keep their (E = 1) ellipse.  The
// positive side (E <= 1 + 2 zmax / sqrt(pi)) was measured to cull ~1 % more
// hits for no time gain and is not used.
__device__ __forceinline__ bool ellipse_meets_block(const float4 A, const float4 B, const float4 X, float wx0,
                                                    float wy0) {
    const float X0 = wx0 + 0.5f - A.x, X1 = X0 + 7.0f;
    const float Y0 = wy0 + 0.5f - A.y, Y1 = Y0 + 3.0f;
    float r2 = X.w;
    {
        const float zmax = (fmaxf(B.z * X0, B.z * X1) + fmaxf(B.w * Y0, B.w * Y1)) * SSG_SQRT1_2;
        if (zmax < 0.0f) r2 = fmaf(-2.002f, fmaf(zmax, zmax, 0.69314718f), r2);  // 2 (ln 2 + zmax^2) x 1.001
    }
    const float a = A.z, k = X.x, h = X.y, mm = X.z;
    const float ya = fminf(fmaxf(-mm * X0, Y0), Y1), yb = fminf(fmaxf(-mm * X1, Y0), Y1);
    const float ua = fmaf(k, ya, X0), ub = fmaf(k, yb, X1);
    const float xa = fminf(fmaxf(-k * Y0, X0), X1), xb = fminf(fmaxf(-k * Y1, X0), X1);
    const float va = fmaf(k, Y0, xa), vb = fmaf(k, Y1, xb);
    const float q = fminf(fminf(fmaf(a * ua, ua, h * ya * ya), fmaf(a * ub, ub, h * yb * yb)),
                          fminf(fmaf(a * va, va, h * Y0 * Y0), fmaf(a * vb, vb, h * Y1 * Y1)));
    const bool inside = X0 <= 0.0f && X1 >= 0.0f && Y0 <= 0.0f && Y1 >= 0.0f;
    return inside ? r2 >= 0.0f : !(q > r2);
}

// Word of the per-(tile, warp, 32-instance chunk) blend mask: bit b of word
// (start/32 + tile + chunk) * 8 + warp is set when some pixel of the warp
// blended instance start + 32*chunk + b in the forward.  The bases never
// overlap: consecutive tiles' bases differ by >= ceil(len/32).
__device__ __forceinline__ size_t mask_word(int start, int tile, int chunk, int warp) {
    return ((size_t)(start >> 5) + (size_t)tile + (size_t)chunk) * 8 + (size_t)warp;
}

// -------------------------------------------------------------- forward
// kVanilla = true compiles the plain 3DGS blend (no skew term, alpha =
// o * G): the config-3 regression reference for skew-free splats, which
// must come out bit-identical from the skew kernel (E = 1, o_sum = o).
// With blend_mask != nullptr the kernel records, per warp and 32-instance
// chunk, which instances any of the warp's pixels blended; the backward
// then visits exactly those (same arithmetic, same decisions).
#ifndef SSG_FWD_MINB
#define SSG_FWD_MINB 5
#endif
#ifndef SSG_BWD_MINB
#define SSG_BWD_MINB 5
#endif

template <bool kVanilla>
__global__ void __launch_bounds__(kThreads, SSG_FWD_MINB)
k_blend_forward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                const int32_t *__restrict__ ranges, float *__restrict__ color,
                float *__restrict__ final_T, int32_t *__restrict__ n_contrib,
                int32_t *__restrict__ last_idx, uint32_t *__restrict__ blend_mask) {
    __shared__ SmemBatch s;
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool inside = px < W && py < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
    const float fwx0 = (float)wx0, fwy0 = (float)wy0;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);

    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int nc = 0, li = -1;
    int done = !inside;
#ifdef SSG_BLEND_STATS
    __shared__ int sTileH[kThreads / 32];
    if (lane == 0) sTileH[warp] = 0;
#endif
    const uint32_t aA = smem_addr(s.A), aB = smem_addr(s.B), aC = smem_addr(s.C);
    const uint32_t aX = smem_addr(s.X), aD = smem_addr(s.D);

    for (int base = start; base < end; base += kBatch) {
        if (__syncthreads_count(done) == kThreads) break;
        if (base + (int)threadIdx.x < end)
            stage_splat(splat, inst_prim[base + threadIdx.x], ox, oy, s, threadIdx.x);
        __syncthreads();
        const int cnt = min(kBatch, end - base);
#ifdef SSG_BLEND_STATS
        int bh = 0;  // this warp's hits in the batch (imbalance diagnostics)
#endif
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            if (__all_sync(0xffffffffu, done)) break;
            const int i = c0 + lane;
            bool hit = false;
            if (i < cnt)
                hit = ellipse_meets_block(lds128(aA + 16 * i), lds128(aB + 16 * i), lds128(aX + 16 * i), fwx0, fwy0);
            unsigned mask = __ballot_sync(0xffffffffu, hit);
            uint32_t lbits = 0;  // instances of this chunk the lane's pixel blended
#ifdef SSG_BLEND_STATS
            if (lane == 0) SSG_STAT(0, __popc(mask));
            bh += __popc(mask);
#endif
            while (mask) {
                const int bit = __ffs(mask) - 1;
                mask &= mask - 1;
                const int j = c0 + bit;
                // branch-free per lane (the warp skips an instance no live
                // pixel can blend); blending lanes run exactly the
                // reference's operations, the others carry zero weight
                const float4 A = lds128(aA + 16 * j);
                const float4 B = lds128(aB + 16 * j);
                const float dx = fx - A.x, dy = fy - A.y;
                const float power = -0.5f * (A.z * dx * dx + B.x * dy * dy) - A.w * dx * dy;   // :133-135
                const bool live = !done && power >= B.y && power <= 0.0f;
                if (!__any_sync(0xffffffffu, live)) continue;
                const float4 C = lds128(aC + 16 * j);
                const float cb = lds32(aD + 4 * j);
                float E = 1.0f, o = C.x;
                if (!kVanilla && (B.z != 0.0f || B.w != 0.0f)) {     // warp-uniform
                    const float z = (B.z * dx + B.w * dy) * SSG_SQRT1_2;   // :136
                    E = skew_E(z);                                          // :137
                    o = fmaf(C.y, E - 1.0f, C.x);                           // :138
                }
                const float pw = fminf(power, 0.0f);
                const float Aval = kVanilla ? o * fast_exp2(pw * SSG_LOG2E)
                                            : o * fast_exp2(pw * SSG_LOG2E) * E;      // :139
                const float alpha = fminf(Aval, SSG_ALPHA_MAX);                         // :140
                const bool pass = live && alpha >= SSG_ALPHA_SKIP;                     // :141-142
                const float test_T = T * (1.0f - alpha);                                // :143
                const bool stop = pass && test_T < SSG_T_STOP;                          // :144-147
                const bool blend = pass && !stop;                                       // :148-154
                done |= stop;
                const float w = blend ? alpha * T : 0.0f;
                C0 = fmaf(w, C.z, C0);
                C1 = fmaf(w, C.w, C1);
                C2 = fmaf(w, cb, C2);
                T = blend ? test_T : T;
                lbits |= (uint32_t)blend << bit;
            }
            // n_contrib and last_idx from the chunk's blend bits (ascending k)
            if (lbits) {
                nc += __popc(lbits);
                li = base + c0 + 31 - __clz(lbits);
            }
            if (blend_mask) {
                const uint32_t bmask = __reduce_or_sync(0xffffffffu, lbits);
#ifdef SSG_BLEND_STATS
                if (lane == 0) SSG_STAT(1, __popc(bmask));
#endif
                if (lane == 0) blend_mask[mask_word(start, tile, (base - start + c0) >> 5, warp)] = bmask;
            }
        }
#ifdef SSG_BLEND_STATS
        {   // per batch: the slowest warp's hits vs the warps' total (barrier imbalance)
            __shared__ int sH[kThreads / 32];
            if (lane == 0) sH[warp] = bh;
            __syncthreads();
            if (threadIdx.x == 0) {
                int mx = 0, sm = 0;
                for (int w = 0; w < kThreads / 32; w++) { mx = max(mx, sH[w]); sm += sH[w]; }
                SSG_STAT(2, mx);
                SSG_STAT(3, sm);
            }
            if (lane == 0) sTileH[warp] += bh;
            __syncthreads();
        }
#endif
    }
#ifdef SSG_BLEND_STATS
    __syncthreads();
    if (threadIdx.x == 0) {  // per tile: the slowest warp's hits vs the total
        int mx = 0, sm = 0;
        for (int w = 0; w < kThreads / 32; w++) { mx = max(mx, sTileH[w]); sm += sTileH[w]; }
        SSG_STAT(4, mx);
        SSG_STAT(5, sm);
    }
#endif
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

// ------------------------------------------------------------- backward
// Transposed butterfly over 12 components: after it, lane L holds the warp
// sum of component 6*b4 + 3*b3 + c(b2, b1), c = 0 / 1 / 2 for (b2, b1) =
// (0,0) / (0,1) / (1,0) (bit bk = lane bit k; (1,1) is padding): 13 shuffles
// instead of 5 x 12.
__device__ __forceinline__ float warp_reduce_transposed12(float (&v)[12], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
    for (int i = 0; i < 6; i++) {
        const float send = b4 ? v[i] : v[i + 6];
        const float keep = b4 ? v[i + 6] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
        const float send = b3 ? v[i] : v[i + 3];
        const float keep = b3 ? v[i + 3] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        const float send0 = b2 ? v[0] : v[2], keep0 = b2 ? v[2] : v[0];
        const float send1 = b2 ? v[1] : 0.0f, keep1 = b2 ? 0.0f : v[1];
        v[0] = keep0 + __shfl_xor_sync(0xffffffffu, send0, 4);
        v[1] = keep1 + __shfl_xor_sync(0xffffffffu, send1, 4);
    }
    {
        const float send = b1 ? v[0] : v[1], keep = b1 ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// d_z * SQRT1_2 of _core.pyx:293-302 (d_z = DA G (2/sqrt(pi)) e^-z^2 (o + (o1-o2)E/2))
constexpr float kDzScale = SSG_TWO_OVER_SQRT_PI * SSG_SQRT1_2;

__global__ void __launch_bounds__(kThreads, SSG_BWD_MINB)
k_blend_backward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                 const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                 const int32_t *__restrict__ ranges, const float *__restrict__ final_T,
                 const int32_t *__restrict__ last_idx, const uint32_t *__restrict__ blend_mask,
                 const float *__restrict__ dL, float *__restrict__ grad_screen, float *__restrict__ slots) {
    __shared__ SmemBatch s;
    __shared__ float *sRow[kBatch];  // destination gradient row of each staged instance
    __shared__ int sMax[kThreads / 32];
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool inside = px < W && py < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    if (end <= start) return;
    const float fx = (float)lx + 0.5f, fy = (float)ly + 0.5f;
    const float fwx0 = (float)wx0, fwy0 = (float)wy0;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);

    // _core.pyx:232-246
    float T = 1.0f, d0 = 0.0f, d1 = 0.0f, d2 = 0.0f;
    int li = -1;
    if (inside) {
        const int64_t pix = (int64_t)py * W + px;
        T = final_T[pix];
        li = last_idx[pix];
        d0 = dL[3 * pix];
        d1 = dL[3 * pix + 1];
        d2 = dL[3 * pix + 2];
    }
    float R0 = bg0, R1 = bg1, R2 = bg2;
    const int wmax = __reduce_max_sync(0xffffffffu, li);
    if (lane == 0) sMax[warp] = wmax;
    __syncthreads();
    int maxli = sMax[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; w++) maxli = max(maxli, sMax[w]);
    if (maxli < start) return;  // any_hit == 0 (:245-246); block-uniform
    const int hi = min(maxli + 1, end);
    const uint32_t aA = smem_addr(s.A), aB = smem_addr(s.B), aC = smem_addr(s.C);
    const uint32_t aX = smem_addr(s.X), aD = smem_addr(s.D);
    // lane 8g + 2c (c < 3) holds component 3g + c after the reduction
    const bool holder = (lane & 1) == 0 && ((lane >> 1) & 3) < 3;
    const int my_comp = 3 * (lane >> 3) + ((lane >> 1) & 3);

    // batches aligned to the forward's chunk grid (start + 256 b), top down
    for (int b = (hi - start - 1) / kBatch; b >= 0; b--) {
        const int lo = start + b * kBatch;
        const int cnt = min(kBatch, hi - lo);
        // this warp's mask words of the batch (lane q < 8 holds chunk q)
        uint32_t words = 0;
        if (blend_mask && lane < 8 && 32 * lane < cnt)
            words = blend_mask[mask_word(start, tile, b * (kBatch / 32) + lane, warp)];
        __syncthreads();  // previous batch fully consumed
        if ((int)threadIdx.x < cnt) {
            const uint32_t p = inst_prim[lo + threadIdx.x];
            stage_splat(splat, p, ox, oy, s, threadIdx.x);
            // per-primitive accumulator, or (plugin slot mode) the per-instance
            // (M,12) slot row of _core.pyx:309-312 (raster/backward.py:70-73)
            sRow[threadIdx.x] = slots ? slots + (size_t)(lo + threadIdx.x) * 12 : grad_screen + (size_t)p * 12;
        }
        __syncthreads();

        const int cwarp = min(cnt, wmax - lo + 1);  // instances past the warp's last_idx never blend
        for (int c0 = ((cwarp - 1) >> 5) << 5; c0 >= 0 && cwarp > 0; c0 -= 32) {
            unsigned mask;
            if (blend_mask) {
                mask = __shfl_sync(0xffffffffu, words, c0 >> 5);
                if (cwarp - c0 < 32) mask &= (1u << (cwarp - c0)) - 1u;
            } else {
                const int i = c0 + lane;
                bool hit = false;
                if (i < cwarp)
                    hit = ellipse_meets_block(lds128(aA + 16 * i), lds128(aB + 16 * i), lds128(aX + 16 * i), fwx0,
                                              fwy0);
                mask = __ballot_sync(0xffffffffu, hit);
            }
#ifdef SSG_BLEND_STATS
            if (lane == 0) SSG_STAT(16, __popc(mask));
#endif
            // per-lane replay of instance j (global index k): updates T, R
            // and writes the 12 slot values g (zero off-contribution)
            auto replay = [&](int j, int k, float (&g)[12], bool &live, bool &contrib) {
                // Branch-free per lane (every visited instance has a
                // contributing pixel, so no warp-wide skip is lost): lanes that
                // do not contribute compute with a zero weight and keep T, R;
                // contributing lanes run exactly the reference's operations.
                const float4 A = lds128(aA + 16 * j);
                const float4 B = lds128(aB + 16 * j);
                const float4 C = lds128(aC + 16 * j);
                const float cb = lds32(aD + 4 * j);
                const float dx = fx - A.x, dy = fy - A.y;
                const float power = -0.5f * (A.z * dx * dx + B.x * dy * dy) - A.w * dx * dy;
                live = k <= li && power >= B.y && power <= 0.0f;                           // :263-264, :265-269
                const float pw = fminf(power, 0.0f);   // == power on live lanes; finite exps elsewhere
                const bool skewed = (B.z != 0.0f || B.w != 0.0f);                          // warp-uniform
                float E = 1.0f, z = 0.0f, o = C.x;
                if (skewed) {
                    z = (B.z * dx + B.w * dy) * SSG_SQRT1_2;
                    E = skew_E(z);
                    o = fmaf(C.y, E - 1.0f, C.x);
                }
                const float G = fast_exp2(pw * SSG_LOG2E);
                const float Aval = o * G * E;
                const float alpha = fminf(Aval, SSG_ALPHA_MAX);
                contrib = live && alpha >= SSG_ALPHA_SKIP;
                const float Tn = T * fast_rcp(1.0f - alpha);                                   // :280
                T = contrib ? Tn : T;
                const float e0 = C.z - R0, e1 = C.w - R1, e2 = cb - R2;
                const float d_alpha = T * (e0 * d0 + e1 * d1 + e2 * d2);
                const float aT = contrib ? alpha * T : 0.0f;
                g[9] = aT * d0;
                g[10] = aT * d1;
                g[11] = aT * d2;
                const float DA = contrib && Aval <= SSG_ALPHA_MAX ? d_alpha : 0.0f;            // :290
                const float d_power = DA * Aval;
                const float Gez2 = skewed ? fast_exp2((pw - z * z) * SSG_LOG2E) : G;
                const float dzs = (DA * kDzScale) * Gez2 * fmaf(C.y, E, o);
                const float px_ = d_power * dx, py_ = d_power * dy;
                g[0] = fmaf(A.z, px_, fmaf(A.w, py_, -dzs * B.z));                           // -d_dx
                g[1] = fmaf(B.x, py_, fmaf(A.w, px_, -dzs * B.w));                           // -d_dy
                g[2] = -0.5f * px_ * dx;
                g[3] = -px_ * dy;
                g[4] = -0.5f * py_ * dy;
                g[5] = dzs * dx;
                g[6] = dzs * dy;
                const float hGE = 0.5f * DA * G * E;
                g[7] = hGE * E;
                g[8] = hGE * (2.0f - E);
                const float ae = contrib ? alpha : 0.0f;                                       // :306-308
                R0 = fmaf(ae, e0, R0);
                R1 = fmaf(ae, e1, R1);
                R2 = fmaf(ae, e2, R2);
#ifdef SSG_BLEND_STATS
                const unsigned cbal = __ballot_sync(0xffffffffu, contrib);
                if (lane == 0) {
                    SSG_STAT(17, cbal != 0);
                    SSG_STAT(18, __popc(cbal));
                }
#endif
            };
            // the 12 holder lanes add their component straight into the
            // primitive's accumulator row, or (plugin slot mode) the
            // per-instance (M,12) slot row of _core.pyx:309-312
            // (raster/backward.py:70-73).  Two loops, so the visit itself
            // carries no mask-mode test.
            if (blend_mask) {
                // the forward's mask: every visited instance has a contributing pixel
                while (mask) {
                    const int bit = 31 - __clz(mask);
                    mask &= ~(1u << bit);
                    const int j = c0 + bit;
                    float g[12];
                    bool live, contrib;
                    replay(j, lo + j, g, live, contrib);
                    const float v = warp_reduce_transposed12(g, lane);
                    if (holder) atomicAdd(sRow[j] + my_comp, v);
                }
            } else {
                // test-driven walk: skip empty hits
                while (mask) {
                    const int bit = 31 - __clz(mask);
                    mask &= ~(1u << bit);
                    const int j = c0 + bit;
                    float g[12];
                    bool live, contrib;
                    replay(j, lo + j, g, live, contrib);
                    if (!__any_sync(0xffffffffu, live) || !__any_sync(0xffffffffu, contrib)) continue;
                    const float v = warp_reduce_transposed12(g, lane);
                    if (holder) atomicAdd(sRow[j] + my_comp, v);
                }
            }
        }
    }
}

}  // namespace ssg

extern "C" int64_t ssg_blend_mask_words(int64_t m, int32_t n_tiles) {
    // mask_word(): bases start/32 + tile + chunk, 8 warps each
    return m < 0 || n_tiles < 0 ? -1 : 8 * (m / 32 + (int64_t)n_tiles + 1);
}

extern "C" int ssg_blend_forward(int64_t m, int32_t width, int32_t height, const float background[3],
                                 const ssg_splat *splat, const ssg_bin_buffers *bins,
                                 const ssg_frame_buffers *frame, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !background || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    (void)m;
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    cudaStream_t st = (cudaStream_t)stream;
    k_blend_forward<false><<<ntx * nty, kThreads, 0, st>>>(ntx, width, height, background[0], background[1],
                                                           background[2], splat, bins->inst_prim, bins->ranges,
                                                           frame->color, frame->final_T, frame->n_contrib,
                                                           frame->last_idx, frame->blend_mask);
    return check_launch("k_blend_forward");
}

extern "C" int ssg_test_blend_forward_vanilla(int32_t width, int32_t height, const float background[3],
                                              const ssg_splat *splat, const ssg_bin_buffers *bins,
                                              const ssg_frame_buffers *frame, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !background || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_forward<true><<<ntx * nty, kThreads, 0, (cudaStream_t)stream>>>(
        ntx, width, height, background[0], background[1], background[2], splat, bins->inst_prim, bins->ranges,
        frame->color, frame->final_T, frame->n_contrib, frame->last_idx, nullptr);
    return check_launch("k_blend_forward<vanilla>");
}

extern "C" int ssg_blend_backward(int64_t n, int64_t m, int32_t width, int32_t height,
                                  const float background[3], const ssg_splat *splat,
                                  const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                  const float *dL_dpixels, const ssg_grad_buffers *grads, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !grads || !background || !dL_dpixels || width < 1 || height < 1 || n < 0)
        return SSG_ERR_INVALID_ARGUMENT;
    (void)m;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(grads->screen, 0, sizeof(float) * 12 * (size_t)n, st);
    if (e != cudaSuccess) { set_error("memset screen grads", e); return SSG_ERR_CUDA; }
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_backward<<<ntx * nty, kThreads, 0, st>>>(ntx, width, height, background[0], background[1],
                                                     background[2], splat, bins->inst_prim, bins->ranges,
                                                     frame->final_T, frame->last_idx, frame->blend_mask,
                                                     dL_dpixels, grads->screen, nullptr);
    return check_launch("k_blend_backward");
}

extern "C" int ssg_blend_backward_slots(int64_t m, int32_t width, int32_t height, const float background[3],
                                        const ssg_splat *splat, const ssg_bin_buffers *bins,
                                        const ssg_frame_buffers *frame, const float *dL_dpixels, float *slots,
                                        void *stream) {
    using namespace ssg;
    if (!bins || !frame || !background || !dL_dpixels || !slots || width < 1 || height < 1 || m < 0)
        return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(slots, 0, sizeof(float) * 12 * (size_t)m, st);
    if (e != cudaSuccess) { set_error("memset slots", e); return SSG_ERR_CUDA; }
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_backward<<<ntx * nty, kThreads, 0, st>>>(ntx, width, height, background[0], background[1],
                                                     background[2], splat, bins->inst_prim, bins->ranges,
                                                     frame->final_T, frame->last_idx, frame->blend_mask,
                                                     dL_dpixels, nullptr, slots);
    return check_launch("k_blend_backward(slots)");
}

#ifdef SSG_BLEND_STATS
extern "C" int ssg_test_blend_stats(unsigned long long *out, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out, g_blend_stats, sizeof(unsigned long long) * 32);
    if (e == cudaSuccess && reset) {
        static const unsigned long long zero[32] = {0};
        e = cudaMemcpyToSymbol(g_blend_stats, zero, sizeof(zero));
    }
    return e == cudaSuccess ? SSG_OK : SSG_ERR_CUDA;
}
#endif
