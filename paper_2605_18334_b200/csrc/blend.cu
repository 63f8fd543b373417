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
// rounding to fp32.  Every staged instance also carries the ellipse outside
// of which its alpha is certainly below 1/255 (see stage_values).  Each warp
// walks the batch 32 instances at a time: one lane per instance tests the
// ellipse against the warp's 8x4 block, a ballot gives the hit mask, and the
// warp evaluates only the hits, in order.  The culling is conservative.
//
// Decisions equal the fp64 reference's.  The blend arithmetic is fp32, and
// every skip (alpha >= 1/255), clamp (A <= 0.99) and stop (T (1 - alpha) <
// 1e-4) decision it takes is certified: each primitive carries a bound
// `band` on the relative error of its fp32 alpha (ssg_common.cuh
// alpha_band), each pixel a running bound `dT` on the absolute error of its
// fp32 transmittance.  A pixel that meets a decision its bounds cannot
// certify stops there and is flagged (redo_mask / redo_list); the redo
// kernels then recompute exactly those pixels on the exact path: candidate
// instances from an fp32 scan (a superset of the reference's passing
// instances), their alphas in fp64 (ref_pair), transmittance as an fp64
// prefix product, colour / gradients in fp64.  No fp64 and no calls on the
// hot loop.
//
// Backward: the 12 per-instance sums of a warp are reduced with a transposed
// butterfly (13 shuffles instead of 60).  Default: the 12 lanes holding them
// add them to the primitive's gradient row, one scalar global reduction each.
// Deterministic modes: each warp stores its sums in shared memory, the tile's
// eight warps are combined in a fixed order and one thread per instance
// stores the row (no atomics): per instance (the reference's (M,12) slots) or
// primitive-major (each primitive's rows in ascending instance order, summed
// in that order by k_reduce_rank_rows); their redo runs one warp per tile in
// pixel order.
#include "ssg_common.cuh"

namespace ssg {

constexpr int kThreads = 128;       // blend kernels: 4 warps per 16x16 tile
constexpr int kBatch = 256;          // instances staged per batch (2 per thread)
constexpr int kWarps = kThreads / 32;
constexpr int kBlocks = 8;           // 8x4-pixel blocks per tile (the redo mask's words)
constexpr float kNearT = 1.05e-4f;   // candidate transmittance below which the stop test needs its bound
constexpr int kCand = 256;           // redo: candidate instances per segment (per warp)
constexpr int kRedoWarps = 4;        // redo: warps per CTA
constexpr int kDoneNaN = 0x7fc00001;   // row coordinate of a pixel that is outside / stopped
constexpr int kUnsureNaN = 0x7fc00002; // ... of a pixel on the exact path

// Shared-memory image of one instance:
//   A = (mx_local, my_local, conic_a, conic_b)
//   B = (conic_c, hw, skew_x, skew_y), hw = -far_thr / 2: a pair is live when
//       its exponent lies in [far_thr, 0], i.e. |power + hw| <= hw (one compare)
//   C = (o_sum, o_diff, r, g)
//   D = (b, sband, g0, g1): the pair's relative alpha error is <= g0 + g1 |power|
//       (alpha_band); sband = (1/255) (g0 + 6.3 g1): fp32 alpha - 1/255 >= sband
//       certainly passes the reference's 1/255 test, < -sband certainly fails
//   X = (k, h, m, r2m): the ellipse {d : a dx^2 + 2b dx dy + c dy^2 <= r2m}
//       in completed-square form, k = b/a, h = det/a, m = b/c
// far_thr is a per-instance lower bound on the Gaussian exponent below which
// alpha < 1/255 is certain: A = o*G*E <= omax*G*Emax with Emax = 2 (1 for
// skew-free splats), so power < ln(1/(255*omax*Emax)) implies the reference's
// ALPHA_SKIP test (_core.pyx:141) fires; the margin max(1e-4, 2 band) keeps
// the shortcut strictly inside the region where the true alpha also skips.
// The ellipse {power >= far_thr} (r2 = -2 far_thr, widened by max(1e-3,
// 4 band) relative + 1e-4 absolute) is what the per-warp culling tests
// against the warp's 8x4 block of pixel centres, exactly.
template <int NB>
struct SmemBatchT {
    float4 A[NB];
    float4 B[NB];
    float4 C[NB];
    float4 D[NB];
    float4 X[NB];
};
using SmemBatch = SmemBatchT<kBatch>;
// the deterministic backward stages half batches: its per-warp partial sums
// ([warp][instance][12] floats) then take 24 KB instead of 48 KB, and twice
// as many CTAs fit an SM
#ifndef SSG_DET_BATCH
#define SSG_DET_BATCH 128
#endif
constexpr int kDetBatch = SSG_DET_BATCH;
#ifndef SSG_DET_MINB
#define SSG_DET_MINB 8
#endif
struct Staged {
    float4 A, B, C, D, X;
};

__device__ __forceinline__ Staged stage_values(const ssg_splat *splat, uint32_t p, double ox, double oy) {
    const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
    const float4 q1 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 1);
    const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
    const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
    // q1 = (a, b, c, sx)  q2 = (sy, o1, o2, r)  q3 = (g, b, band0, band1)
    const bool skewed = (q1.w != 0.0f || q2.x != 0.0f);
    const float band = fmaf(6.3f, q3.w, q3.z);      // the band anywhere a decision can fall
    const float omax = fmaxf(q2.y, q2.z) * (skewed ? 2.0f : 1.0f);
    const float thr = omax > 0.0f ? -logf(255.0f * omax) - fmaxf(1e-4f, 2.0f * band) : INFINITY;
    const float mx = (float)(m.x - ox), my = (float)(m.y - oy);
    const float a = q1.x, b = q1.y, c = q1.z;
    const float r2 = -2.0f * thr;
    Staged v;
    if (!(r2 > 0.0f)) {
        v.X = make_float4(0.0f, 0.0f, 0.0f, -1.0f);                 // never blends: never hits
    } else {
        const double det = (double)a * (double)c - (double)b * (double)b;   // exact products
        if (a > 0.0f && c > 0.0f && det > 0.0)
            v.X = make_float4(b / a, (float)(det / (double)a), b / c, fmaf(r2, 1.0f + fmaxf(1e-3f, 4.0f * band), 1e-4f));
        else
            v.X = make_float4(0.0f, 0.0f, 0.0f, INFINITY);          // degenerate: always evaluate
    }
    v.A = make_float4(mx, my, a, b);
    v.B = make_float4(c, -0.5f * thr, q1.w, q2.x);
    v.C = make_float4(0.5f * (q2.y + q2.z), 0.5f * (q2.y - q2.z), q2.w, q3.x);
    v.D = make_float4(q3.y, SSG_ALPHA_SKIP * band, q3.z, q3.w);
    return v;
}

template <int NB>
__device__ __forceinline__ void stage_splat(const ssg_splat *splat, uint32_t p, double ox, double oy,
                                            SmemBatchT<NB> &s, int slot) {
    const Staged v = stage_values(splat, p, ox, oy);
    s.A[slot] = v.A;
    s.B[slot] = v.B;
    s.C[slot] = v.C;
    s.D[slot] = v.D;
    s.X[slot] = v.X;
}

// Does the instance's ellipse meet the rectangle spanned by the warp's pixel
// centres [wx0+0.5, wx0+7.5] x [wy0+0.5, wy0+7.5]?  Minimum of the quadratic
// form over the rectangle: 0 if the mean is inside, else the least of the
// four clamped edge minima, each a sum of non-negative terms
// a (dx + k dy)^2 + h dy^2 (no cancellation).
//
// Skewed splats: far_thr assumes the largest skew factor, E <= 2.  Where the
// whole block lies on the negative side of the skew direction (z <= zmax <
// 0 at every pixel centre, z = (sx dx + sy dy)/sqrt2), E = erfc(-z) <=
// exp(-zmax^2) < 1 there, so alpha < 1/255 already for power < far_thr +
// ln 2 + zmax^2: the ellipse shrinks by 2 (ln 2 + zmax^2) in r2 for this
// block (far_thr's margin and the widening carry over).  Skew-free splats
// have zmax = 0 and keep their (E = 1) ellipse.
__device__ __forceinline__ bool ellipse_meets_block(const float4 A, const float4 B, const float4 X, float wx0,
                                                    float wy0) {
    const float X0 = wx0 + 0.5f - A.x, X1 = X0 + 7.0f;
    const float Y0 = wy0 + 0.5f - A.y, Y1 = Y0 + 7.0f;
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
// (start/32 + tile + chunk) * 4 + warp is set when some pixel of the warp's
// 8x8 block blended instance start + 32*chunk + b in the forward.  The bases
// never overlap: consecutive tiles' bases differ by >= ceil(len/32).
__device__ __forceinline__ size_t mask_word(int start, int tile, int chunk, int warp) {
    return ((size_t)(start >> 5) + (size_t)tile + (size_t)chunk) * kWarps + (size_t)warp;
}

// fp32 pre-clamp alpha of one pixel-instance pair: the same operation
// sequence in every kernel (explicit fmaf, no contraction choices left to
// the compiler), so all of them see bit-identical values.
struct Pair {
    float dx, dy, power, E, z, o, G, A;
};
__device__ __forceinline__ void pair_power(float fx, float fy, const float4 &A, const float4 &B, Pair &q) {
    q.dx = fx - A.x;
    q.dy = fy - A.y;
    const float t = fmaf(B.x * q.dy, q.dy, A.z * q.dx * q.dx);
    q.power = fmaf(-0.5f, t, -(A.w * q.dx) * q.dy);                                      // :133
}
template <bool kVanilla>
__device__ __forceinline__ void pair_alpha(const float4 &B, const float4 &C, Pair &q) {
    q.E = 1.0f;
    q.z = 0.0f;
    q.o = C.x;
    if (!kVanilla && (B.z != 0.0f || B.w != 0.0f)) {     // warp-uniform on the hot loop
        q.z = fmaf(B.z, q.dx, B.w * q.dy) * SSG_SQRT1_2;     // :136
        q.E = skew_E(q.z);                                  // :137
        q.o = fmaf(C.y, q.E - 1.0f, C.x);                   // :138
    }
    q.G = fast_exp2(fminf(q.power, 0.0f) * SSG_LOG2E);
    q.A = kVanilla ? q.o * q.G : (q.o * q.G) * q.E;         // :139
}

// ---- two pixels per thread (rows y and y + 4 of one column) ------------
// The blend kernels give each thread the pixel pair (x, y), (x, y + 4): the
// dx terms are shared, the per-row terms run as packed fp32x2 operations
// (FFMA2 / FMUL2 / FADD2, one issue slot for two lanes' worth of FP32 work:
// profiles/r2_ffma2.txt), and every per-instance cost -- shared-memory
// loads, the culling ballot, loop control, the backward's 12-value warp
// reduction -- is paid once per 64 pixels instead of 32.  Every packed op
// is the same IEEE operation per component as the scalar sequence above.
__device__ __forceinline__ uint64_t pk(float2 a) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk(uint64_t r) {
    float2 a;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return upk(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 sel2(bool px, bool py, float2 a, float2 b) {
    return make_float2(px ? a.x : b.x, py ? a.y : b.y);
}

// erfc_pos / skew_E (ssg_common.cuh) on a pair: the same operations per
// component, the polynomial packed
__device__ __forceinline__ float2 skew_E2(float2 z) {
    const float2 x = make_float2(fabsf(z.x), fabsf(z.y));
    const float2 u = fma2(f2(0.5f), x, f2(1.0f));
    const float2 t = make_float2(fast_rcp(u.x), fast_rcp(u.y));
    float2 p = fma2(t, f2(0.17087277f), f2(-0.82215223f));
    p = fma2(t, p, f2(1.48851587f));
    p = fma2(t, p, f2(-1.13520398f));
    p = fma2(t, p, f2(0.27886807f));
    p = fma2(t, p, f2(-0.18628806f));
    p = fma2(t, p, f2(0.09678418f));
    p = fma2(t, p, f2(0.37409196f));
    p = fma2(t, p, f2(1.00002368f));
    p = fma2(t, p, f2(-1.26551223f));
    const float2 a = mul2(fma2(make_float2(-x.x, -x.y), x, p), f2(SSG_LOG2E));
    const float2 y = mul2(t, make_float2(fast_exp2(a.x), fast_exp2(a.y)));
    const float2 ny = sub2(f2(2.0f), y);
    return make_float2(z.x > 0.0f ? ny.x : y.x, z.y > 0.0f ? ny.y : y.y);
}

struct Pair2 {
    float dx;
    float2 dy, power, E, z, o, G, A;
};
__device__ __forceinline__ void pair_power2(float fx, float2 fy, const float4 &A, const float4 &B, Pair2 &q) {
    q.dx = fx - A.x;
    q.dy = sub2(fy, f2(A.y));
    const float adx2 = A.z * q.dx * q.dx;
    const float2 t = fma2(mul2(f2(B.x), q.dy), q.dy, f2(adx2));
    q.power = fma2(f2(-0.5f), t, mul2(f2(-(A.w * q.dx)), q.dy));                        // :133
}
template <bool kVanilla>
__device__ __forceinline__ void pair_alpha2(const float4 &B, const float4 &C, Pair2 &q) {
    q.E = f2(1.0f);
    q.z = f2(0.0f);
    q.o = f2(C.x);
    if (!kVanilla && (B.z != 0.0f || B.w != 0.0f)) {     // warp-uniform
        q.z = mul2(fma2(f2(B.z), f2(q.dx), mul2(f2(B.w), q.dy)), f2(SSG_SQRT1_2));        // :136
        q.E = skew_E2(q.z);                                                                 // :137
        q.o = fma2(f2(C.y), sub2(q.E, f2(1.0f)), f2(C.x));                                 // :138
    }
    const float2 pl = mul2(make_float2(fminf(q.power.x, 0.0f), fminf(q.power.y, 0.0f)), f2(SSG_LOG2E));
    q.G = make_float2(fast_exp2(pl.x), fast_exp2(pl.y));
    q.A = kVanilla ? mul2(q.o, q.G) : mul2(mul2(q.o, q.G), q.E);                           // :139
}

// -------------------------------------------------------------- forward
// kVanilla = true compiles the plain 3DGS blend (no skew term, alpha =
// o * G): the config-3 regression reference for skew-free splats, which
// must come out bit-identical from the skew kernel (E = 1, o_sum = o).
// With blend_mask != nullptr the kernel records, per warp and 32-instance
// chunk, which instances any of the warp's pixels blended; the backward
// then visits exactly those (same arithmetic, same decisions).
#ifndef SSG_FWD_MINB
#define SSG_FWD_MINB 8
#endif
#ifndef SSG_BWD_MINB
#define SSG_BWD_MINB 8
#endif

template <bool kVanilla>
__global__ void __launch_bounds__(kThreads, SSG_FWD_MINB)
k_blend_forward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                const int32_t *__restrict__ ranges, float *__restrict__ color, float *__restrict__ final_T,
                int32_t *__restrict__ n_contrib, int32_t *__restrict__ last_idx, uint32_t *__restrict__ blend_mask,
                uint32_t *__restrict__ redo_mask, uint32_t *__restrict__ redo_list,
                uint32_t *__restrict__ redo_count, int all_exact) {
    __shared__ SmemBatch s;
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 8;     // the warp's 8x8 block
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);   // pixels (lx, ly), (lx, ly + 4)
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool in0 = px < W && py < H, in1 = px < W && py + 4 < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const float fx = (float)lx + 0.5f;
    const float fwx0 = (float)wx0, fwy0 = (float)wy0;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);

    float2 T = f2(1.0f), dT = f2(0.0f);          // dT: bound on |T - T_reference|
    float2 C0 = f2(0.0f), C1 = f2(0.0f), C2 = f2(0.0f);
    int nc0 = 0, nc1 = 0, li0 = -1, li1 = -1;
    // A pixel that is done (outside, stopped, or on the exact path) gets a NaN
    // row coordinate: its exponent is NaN and every later test fails, so the
    // hot loop carries no per-pixel done state.  un*: met a decision its
    // bounds cannot certify (all_exact: every pixel does -- a test mode).
    float2 fy = make_float2((float)ly + 0.5f, (float)ly + 4.5f);
    if (!in0) fy.x = __int_as_float(kDoneNaN);
    else if (all_exact) fy.x = __int_as_float(kUnsureNaN);
    if (!in1) fy.y = __int_as_float(kDoneNaN);
    else if (all_exact) fy.y = __int_as_float(kUnsureNaN);
    const uint32_t aA = smem_addr(s.A), aB = smem_addr(s.B), aC = smem_addr(s.C);
    const uint32_t aX = smem_addr(s.X), aD = smem_addr(s.D);
    int kdone = start;    // instances [start, kdone) walked by this warp (mask words written)

    for (int base = start; base < end; base += kBatch) {
        if (__syncthreads_count(isnan(fy.x) && isnan(fy.y)) == kThreads) break;
        for (int t = threadIdx.x; t < kBatch && base + t < end; t += kThreads)
            stage_splat(splat, inst_prim[base + t], ox, oy, s, t);
        __syncthreads();
        const int cnt = min(kBatch, end - base);
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            if (__all_sync(0xffffffffu, isnan(fy.x) && isnan(fy.y))) break;
            kdone = base + c0 + 32;
            const int i = c0 + lane;
            bool hit = false;
            if (i < cnt)
                hit = ellipse_meets_block(lds128(aA + 16 * i), lds128(aB + 16 * i), lds128(aX + 16 * i), fwx0, fwy0);
            unsigned mask = __ballot_sync(0xffffffffu, hit);
            uint32_t lb0 = 0, lb1 = 0;  // instances of this chunk each pixel blended
            while (mask) {
                const uint32_t lowb = mask & (0u - mask);
                const int bit = __ffs(mask) - 1;
                mask ^= lowb;
                const int j = c0 + bit;
                // branch-free per lane (the warp skips an instance no live
                // pixel can blend); blending lanes run exactly the
                // reference's operations, the others carry zero weight
                const float4 A = lds128(aA + 16 * j);
                const float4 B = lds128(aB + 16 * j);
                Pair2 q;
                pair_power2(fx, fy, A, B, q);
                const float2 pc = add2(q.power, f2(B.y));
                const bool live0 = fabsf(pc.x) <= B.y, live1 = fabsf(pc.y) <= B.y;
                if (!__any_sync(0xffffffffu, live0 | live1)) continue;
                const float4 C = lds128(aC + 16 * j);
                const float4 D = lds128(aD + 16 * j);
                pair_alpha2<kVanilla>(B, C, q);
                const float2 alpha = make_float2(fminf(q.A.x, SSG_ALPHA_MAX), fminf(q.A.y, SSG_ALPHA_MAX));   // :140
                const float2 dA = sub2(q.A, f2(SSG_ALPHA_SKIP));
                const bool pass0 = live0 & (dA.x >= D.y), pass1 = live1 & (dA.y >= D.y);   // certainly >= 1/255
                const float2 gp = fma2(f2(D.w), make_float2(-q.power.x, -q.power.y), f2(D.z));  // alpha error bounds
                const float2 dc = sub2(q.A, f2(SSG_ALPHA_MAX)), cb = mul2(f2(SSG_ALPHA_MAX), gp);
                // uncertain: the 1/255 skip, or the backward's clamp cut (A <= 0.99, :290)
                bool bad0 = live0 & ((fabsf(dA.x) < D.y) | (fabsf(dc.x) <= cb.x));
                bool bad1 = live1 & ((fabsf(dA.y) < D.y) | (fabsf(dc.y) <= cb.y));
                const float2 oma = sub2(f2(1.0f), alpha);
                const float2 test_T = mul2(T, oma);                                                // :143
                const float2 nthr = add2(f2(kNearT), dT);
                const bool near0 = pass0 & (test_T.x < nthr.x), near1 = pass1 & (test_T.y < nthr.y);
                bool bl0 = pass0, bl1 = pass1;
                if (__any_sync(0xffffffffu, near0 | near1 | bad0 | bad1)) {
                    // rare: a candidate stop, or an uncertain decision
                    // |T (1 - alpha) - T_ref (1 - alpha_ref)| <= dT (1 - alpha) + T alpha gp
                    //   + 2 roundings per blend so far (eps / 2 each, relative)
                    const float e0 = fmaf(dT.x, oma.x, T.x * alpha.x * gp.x) +
                                     (float)(nc0 + __popc(lb0) + 2) * 6e-8f * test_T.x;
                    const float e1 = fmaf(dT.y, oma.y, T.y * alpha.y * gp.y) +
                                     (float)(nc1 + __popc(lb1) + 2) * 6e-8f * test_T.y;
                    bad0 |= near0 & (fabsf(test_T.x - SSG_T_STOP) <= e0);
                    bad1 |= near1 & (fabsf(test_T.y - SSG_T_STOP) <= e1);
                    const bool stop0 = near0 & (test_T.x < SSG_T_STOP);                          // :144-147
                    const bool stop1 = near1 & (test_T.y < SSG_T_STOP);
                    if (stop0 | bad0) {                                                            // :148-154
                        bl0 = false;
                        fy.x = __int_as_float(bad0 ? kUnsureNaN : kDoneNaN);
                    }
                    if (stop1 | bad1) {
                        bl1 = false;
                        fy.y = __int_as_float(bad1 ? kUnsureNaN : kDoneNaN);
                    }
                }
                const float2 bm = make_float2(bl0 ? 1.0f : 0.0f, bl1 ? 1.0f : 0.0f);
                const float2 w = mul2(mul2(alpha, T), bm);
                C0 = fma2(w, f2(C.z), C0);
                C1 = fma2(w, f2(C.w), C1);
                C2 = fma2(w, f2(D.x), C2);
                const float2 omb = fma2(make_float2(-alpha.x, -alpha.y), bm, f2(1.0f));   // 1 - alpha or 1
                dT = fma2(w, gp, mul2(dT, omb));
                T = mul2(T, omb);
                lb0 |= bl0 ? lowb : 0u;
                lb1 |= bl1 ? lowb : 0u;
            }
            // n_contrib and last_idx from the chunk's blend bits (ascending k)
            if (lb0) {
                nc0 += __popc(lb0);
                li0 = base + c0 + 31 - __clz(lb0);
            }
            if (lb1) {
                nc1 += __popc(lb1);
                li1 = base + c0 + 31 - __clz(lb1);
            }
            if (blend_mask) {
                const uint32_t bmask = __reduce_or_sync(0xffffffffu, lb0 | lb1);
                if (lane == 0) blend_mask[mask_word(start, tile, (base - start + c0) >> 5, warp)] = bmask;
            }
        }
    }
    // the mask words past this warp's walk are zeroed, so every word of the
    // tile is valid for the exact path (which reads a pixel's candidates there)
    if (blend_mask)
        for (int c = (kdone - start) / 32 + lane; c < (end - start + 31) / 32; c += 32)
            blend_mask[mask_word(start, tile, c, warp)] = 0u;
    // the redo mask is kept per 8x4 block: rows ly (block 4 (warp >> 1) +
    // (warp & 1)) and ly + 4 (two blocks further)
    const bool un0 = in0 && __float_as_int(fy.x) == kUnsureNaN, un1 = in1 && __float_as_int(fy.y) == kUnsureNaN;
    const uint32_t r0 = __ballot_sync(0xffffffffu, un0), r1 = __ballot_sync(0xffffffffu, un1);
    if (lane == 0) {
        const int b0 = (warp >> 1) * 4 + (warp & 1);
        redo_mask[(size_t)tile * kBlocks + b0] = r0;
        redo_mask[(size_t)tile * kBlocks + b0 + 2] = r1;
    }
    // :158-166; pixels on the exact path: every blend so far is <= li and set
    // in the warp's mask words, the exact path resumes the scan at li + 1
    if (in0) {
        const int64_t pix = (int64_t)py * W + px;
        if (un0) {
            redo_list[atomicAdd(redo_count, 1u)] = (uint32_t)pix;
            last_idx[pix] = li0;
        } else {
            color[3 * pix] = C0.x + T.x * bg0;
            color[3 * pix + 1] = C1.x + T.x * bg1;
            color[3 * pix + 2] = C2.x + T.x * bg2;
            final_T[pix] = T.x;
            n_contrib[pix] = nc0;
            last_idx[pix] = li0;
        }
    }
    if (in1) {
        const int64_t pix = (int64_t)(py + 4) * W + px;
        if (un1) {
            redo_list[atomicAdd(redo_count, 1u)] = (uint32_t)pix;
            last_idx[pix] = li1;
        } else {
            color[3 * pix] = C0.y + T.y * bg0;
            color[3 * pix + 1] = C1.y + T.y * bg1;
            color[3 * pix + 2] = C2.y + T.y * bg2;
            final_T[pix] = T.y;
            n_contrib[pix] = nc1;
            last_idx[pix] = li1;
        }
    }
}

// ------------------------------------------------------------ exact path
// One flagged pixel, evaluated by one warp.
struct RedoPixel {
    int px, py, tile, tx, ty, start, end, warp_in_tile;
    double pxc, pyc, ox, oy;
    float fx, fy;
};
__device__ __forceinline__ RedoPixel redo_pixel(uint32_t pix, int32_t W, int32_t ntx, const int32_t *ranges) {
    RedoPixel r;
    r.py = (int)(pix / (uint32_t)W);
    r.px = (int)(pix - (uint32_t)r.py * (uint32_t)W);
    r.tx = r.px >> 4;
    r.ty = r.py >> 4;
    r.tile = r.ty * ntx + r.tx;
    r.start = ranges[2 * r.tile];
    r.end = ranges[2 * r.tile + 1];
    const int lx = r.px & 15, ly = r.py & 15;
    r.warp_in_tile = (ly >> 3) * 2 + (lx >> 3);
    r.fx = (float)lx + 0.5f;
    r.fy = (float)ly + 0.5f;
    r.ox = (double)(r.tx * 16);
    r.oy = (double)(r.ty * 16);
    r.pxc = (double)r.px + 0.5;   // _core.pyx:131-132
    r.pyc = (double)r.py + 0.5;
    return r;
}

// Could instance p's alpha at this pixel reach 1/255?  fp32 alpha >=
// (1/255) (1 - band): a superset of the reference's passing instances (the
// band bounds the fp32 error).  Lean: no culling data, just the pair.
template <bool kVanilla>
__device__ __forceinline__ bool redo_maybe(const RedoPixel &P, const ssg_splat *splat, uint32_t p) {
    const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
    const float4 q1 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 1);
    const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
    const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
    const float4 A = make_float4((float)(m.x - P.ox), (float)(m.y - P.oy), q1.x, q1.y);
    const float4 B = make_float4(q1.z, 0.0f, q1.w, q2.x);
    const float4 C = make_float4(0.5f * (q2.y + q2.z), 0.5f * (q2.y - q2.z), 0.0f, 0.0f);
    Pair q;
    pair_power(P.fx, P.fy, A, B, q);
    pair_alpha<kVanilla>(B, C, q);
    return q.A >= SSG_ALPHA_SKIP * (1.0f - fmaf(6.3f, q3.w, q3.z));
}

// Collect, in order, the instances k in [kb, kend) that redo_maybe admits.
// Instances k <= kmask are taken from the pixel's warp-block blend mask (a
// superset of the pixel's blends there: 32 mask words per load, only set
// bits evaluated); later ones by a full scan (four chunks in flight per step
// to cover load latency).  Fills list[0, n) and returns n; kb advances past
// the examined instances (stops early when the segment is full).
template <bool kVanilla>
__device__ __forceinline__ int redo_candidates(const RedoPixel &P, int &kb, int kend, int kmask,
                                               const uint32_t *blend_mask, const ssg_splat *splat,
                                               const uint32_t *inst_prim, uint32_t *list) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int n = 0;
    // mask-driven part: chunks are aligned to start + 32 c
    while (kb < kend && kb <= kmask && n <= kCand - 32) {
        const int c0 = (kb - P.start) >> 5;
        const int kstop = min(kend, kmask + 1);
        const int nch = min(32, ((kstop - P.start + 31) >> 5) - c0);
        uint32_t word = 0;
        if (lane < nch) word = blend_mask[mask_word(P.start, P.tile, c0 + lane, P.warp_in_tile)];
        int c = 0;
        for (; c < nch && n <= kCand - 32; c++) {
            const int kc = P.start + 32 * (c0 + c);
            uint32_t bits = __shfl_sync(0xffffffffu, word, c);
            const int lo = max(kb, kc), hi = min(kstop, kc + 32);     // [lo, hi) of this chunk
            if (lo >= hi) continue;
            bits &= (hi - kc >= 32 ? 0xffffffffu : ((1u << (hi - kc)) - 1u)) & ~((1u << (lo - kc)) - 1u);
            const int k = kc + lane;
            const bool maybe = ((bits >> lane) & 1u) && redo_maybe<kVanilla>(P, splat, inst_prim[k]);
            const uint32_t b = __ballot_sync(0xffffffffu, maybe);
            if (maybe) list[n + __popc(b & lt)] = (uint32_t)k;
            n += __popc(b);
        }
        kb = min(kstop, P.start + 32 * (c0 + c));
        if (kb == kmask + 1) break;
    }
    while (kb < kend && n <= kCand - 128) {
        uint32_t p[4];
        bool v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int k = kb + 32 * u + lane;
            v[u] = k < kend;
            p[u] = v[u] ? inst_prim[k] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const bool maybe = v[u] && redo_maybe<kVanilla>(P, splat, p[u]);
            const uint32_t b = __ballot_sync(0xffffffffu, maybe);
            if (maybe) list[n + __popc(b & lt)] = (uint32_t)(kb + 32 * u + lane);
            n += __popc(b);
        }
        kb = min(kend, kb + 128);
    }
    __syncwarp();
    return n;
}

// inclusive prefix product / sum over the warp's lanes, and the warp sum (fp64)
__device__ __forceinline__ double warp_prefix_prod(double f) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, f, off);
        if (lane >= off) f *= y;
    }
    return f;
}
__device__ __forceinline__ double warp_prefix_sum(double f) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, f, off);
        if (lane >= off) f += y;
    }
    return f;
}
__device__ __forceinline__ double warp_sum(double f) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
    return f;
}

// The exact front-to-back blend of one pixel (raster/_core.pyx:125-166) over
// the tile's instances [start, kend), in fp64 with the reference's
// decisions: the pass test on fp64 alphas, transmittance as a prefix
// product, the first passing instance whose test_T < 1e-4 stops the pixel
// unblended (with_stop).  Calls visit(k, p, pair, alpha, T_before, blended)
// on every lane for every round (lanes in instance order).  Returns the
// final transmittance; nc / li as the reference counts them.
template <bool kVanilla, typename Visit>
__device__ __forceinline__ double redo_blend(const RedoPixel &P, int kend, int kmask, const uint32_t *blend_mask,
                                             bool with_stop, const ssg_splat *splat, const ssg_splat64 *splat64,
                                             const uint32_t *inst_prim, uint32_t *list, int &nc, int &li,
                                             Visit &&visit) {
    const int lane = threadIdx.x & 31;
    double T = 1.0;
    nc = 0;
    li = -1;
    int kb = P.start;
    bool stopped = false;
    while (kb < kend && !stopped) {
        const int n = redo_candidates<kVanilla>(P, kb, kend, kmask, blend_mask, splat, inst_prim, list);
        for (int r = 0; r < n && !stopped; r += 32) {
            const int idx = r + lane;
            const bool valid = idx < n;
            const int k = valid ? (int)list[idx] : 0;
            uint32_t p = 0;
            bool pass = false;
            double al = 0.0;
            RefPair rp = {};
            if (valid) {
                p = inst_prim[k];
                const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
                rp = ref_pair(P.pxc, P.pyc, m.x, m.y, splat64[p], kVanilla);
                al = rp.A < 0.99 ? rp.A : 0.99;                        // :140
                pass = !rp.skip && al >= 1.0 / 255.0;                  // :133-135, :141-142
            }
            const double f = pass ? 1.0 - al : 1.0;
            const double incl = warp_prefix_prod(f);
            double excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0;
            const double Tb = T * excl;
            const bool stop_l = with_stop && pass && T * incl < 1e-4;  // :143-147
            const uint32_t sb = __ballot_sync(0xffffffffu, stop_l);
            const int first = sb ? __ffs(sb) - 1 : 32;
            const bool blended = pass && lane < first;
            visit(k, p, rp, al, Tb, blended);
            const uint32_t bb = __ballot_sync(0xffffffffu, blended);
            nc += __popc(bb);
            if (bb) li = __shfl_sync(0xffffffffu, k, 31 - __clz(bb));
            if (sb) {
                T = __shfl_sync(0xffffffffu, Tb, first);
                stopped = true;
            } else {
                T = T * __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncwarp();
    }
    return T;
}

template <bool kVanilla>
__global__ void __launch_bounds__(32 * kRedoWarps)
k_blend_forward_redo(int32_t ntx, int32_t W, float bg0, float bg1, float bg2, const ssg_splat *__restrict__ splat,
                     const ssg_splat64 *__restrict__ splat64, const uint32_t *__restrict__ inst_prim,
                     const int32_t *__restrict__ ranges, float *__restrict__ color, float *__restrict__ final_T,
                     int32_t *__restrict__ n_contrib, int32_t *__restrict__ last_idx,
                     uint32_t *__restrict__ blend_mask, const uint32_t *__restrict__ redo_list,
                     const uint32_t *__restrict__ redo_count) {
    __shared__ uint32_t s_list[kRedoWarps][kCand];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t count = *redo_count;
    for (uint32_t i = blockIdx.x * kRedoWarps + wid; i < count; i += gridDim.x * kRedoWarps) {
        const uint32_t pix = redo_list[i];
        const RedoPixel P = redo_pixel(pix, W, ntx, ranges);
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;  // per-lane partial colour
        int nc, li;
        // the main kernel left the pixel's last certified blend in last_idx
        const int kmask = blend_mask ? last_idx[pix] : -1;
        const double T = redo_blend<kVanilla>(
            P, P.end, kmask, blend_mask, true, splat, splat64, inst_prim, s_list[wid], nc, li,
            [&](int k, uint32_t p, const RefPair &, double al, double Tb, bool blended) {
                if (!blended) return;
                const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
                const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
                const double w = al * Tb;                               // :148-152
                c0 += w * (double)q2.w;
                c1 += w * (double)q3.x;
                c2 += w * (double)q3.y;
                if (blend_mask)
                    atomicOr(&blend_mask[mask_word(P.start, P.tile, (k - P.start) >> 5, P.warp_in_tile)],
                             1u << ((k - P.start) & 31));
            });
        c0 = warp_sum(c0);
        c1 = warp_sum(c1);
        c2 = warp_sum(c2);
        if (lane == 0) {  // :158-166
            color[3 * (size_t)pix] = (float)(c0 + T * bg0);
            color[3 * (size_t)pix + 1] = (float)(c1 + T * bg1);
            color[3 * (size_t)pix + 2] = (float)(c2 + T * bg2);
            final_T[pix] = (float)T;
            n_contrib[pix] = nc;
            last_idx[pix] = li;
        }
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

// one fp32 reduction into global memory (RED, no return value): the
// destination rows are global, so no generic-address dispatch
__device__ __forceinline__ void red_add_global(float *p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ float *lds_ptr(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return reinterpret_cast<float *>(v);
}

// d_z * SQRT1_2 of _core.pyx:293-302 (d_z = DA G (2/sqrt(pi)) e^-z^2 (o + (o1-o2)E/2))
constexpr float kDzScale = SSG_TWO_OVER_SQRT_PI * SSG_SQRT1_2;

// destination row of instance (k, p) of tile (tx, ty) in the three modes:
// 0 = per-primitive accumulator, 1 = per-instance (M,12) slots
// (_core.pyx:309-312), 2 = primitive-major row prim_row[p] + rank of the tile
// in p's rectangle (ascending instance order per primitive)
template <int kMode>
__device__ __forceinline__ float *dest_row(float *out, int k, uint32_t p, int tx, int ty, const uint64_t *prim_row,
                                           const uint64_t *tile_rect) {
    if (kMode == 0) return out + (size_t)p * 12;
    if (kMode == 1) return out + (size_t)k * 12;
    const uint64_t rc = tile_rect[p];
    const int x0 = (int)(rc & 0xffff), x1 = (int)((rc >> 16) & 0xffff), y0 = (int)((rc >> 32) & 0xffff);
    const uint64_t rank = (uint64_t)(ty - y0) * (uint64_t)(x1 - x0) + (uint64_t)(tx - x0);
    return out + (size_t)(prim_row[p] + rank) * 12;
}

template <int kMode>
__global__ void __launch_bounds__(kThreads, kMode == 0 ? SSG_BWD_MINB : SSG_DET_MINB)
k_blend_backward(int32_t ntx, int32_t W, int32_t H, float bg0, float bg1, float bg2,
                 const ssg_splat *__restrict__ splat, const uint32_t *__restrict__ inst_prim,
                 const int32_t *__restrict__ ranges, const float *__restrict__ final_T,
                 const int32_t *__restrict__ last_idx, const uint32_t *__restrict__ blend_mask,
                 const uint32_t *__restrict__ redo_mask, const float *__restrict__ dL, float *__restrict__ out,
                 const uint64_t *__restrict__ prim_row, const uint64_t *__restrict__ tile_rect) {
    constexpr int kB = kMode == 0 ? kBatch : kDetBatch;  // instances staged per batch
    __shared__ SmemBatchT<kB> s;
    __shared__ float *sRow[kB];  // destination gradient row of each staged instance
    __shared__ int sMax[kWarps];
    extern __shared__ __align__(16) float s_part[];  // deterministic modes: [warp][instance][12]
    const int tile = blockIdx.x;
    const int tyi = tile / ntx, txi = tile - tyi * ntx;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 8;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
    const int px = txi * 16 + lx, py = tyi * 16 + ly;
    const bool in0 = px < W && py < H, in1 = px < W && py + 4 < H;
    const int start = ranges[2 * tile], end = ranges[2 * tile + 1];
    if (end <= start) return;
    const float fx = (float)lx + 0.5f;
    const float2 fy = make_float2((float)ly + 0.5f, (float)ly + 4.5f);
    const float fwx0 = (float)wx0, fwy0 = (float)wy0;
    const double ox = (double)(txi * 16), oy = (double)(tyi * 16);

    // _core.pyx:232-246; pixels on the exact path are done by the redo kernel
    float2 T = f2(1.0f), d0 = f2(0.0f), d1 = f2(0.0f), d2 = f2(0.0f);
    int li0 = -1, li1 = -1;
    {
        const int b0 = (warp >> 1) * 4 + (warp & 1);
        const bool redo0 = (redo_mask[(size_t)tile * kBlocks + b0] >> lane) & 1u;
        const bool redo1 = (redo_mask[(size_t)tile * kBlocks + b0 + 2] >> lane) & 1u;
        if (in0 && !redo0) {
            const int64_t pix = (int64_t)py * W + px;
            T.x = final_T[pix];
            li0 = last_idx[pix];
            d0.x = dL[3 * pix];
            d1.x = dL[3 * pix + 1];
            d2.x = dL[3 * pix + 2];
        }
        if (in1 && !redo1) {
            const int64_t pix = (int64_t)(py + 4) * W + px;
            T.y = final_T[pix];
            li1 = last_idx[pix];
            d0.y = dL[3 * pix];
            d1.y = dL[3 * pix + 1];
            d2.y = dL[3 * pix + 2];
        }
    }
    float2 R0 = f2(bg0), R1 = f2(bg1), R2 = f2(bg2);
    const int wmax = __reduce_max_sync(0xffffffffu, max(li0, li1));
    if (lane == 0) sMax[warp] = wmax;
    __syncthreads();
    int maxli = sMax[0];
#pragma unroll
    for (int w = 1; w < kWarps; w++) maxli = max(maxli, sMax[w]);
    if (maxli < start) return;  // any_hit == 0 (:245-246); block-uniform
    const int hi = min(maxli + 1, end);
    const uint32_t aA = smem_addr(s.A), aB = smem_addr(s.B), aC = smem_addr(s.C);
    const uint32_t aX = smem_addr(s.X), aD = smem_addr(s.D);
    // lane 8g + 2c (c < 3) holds component 3g + c after the reduction
    const bool holder = (lane & 1) == 0 && ((lane >> 1) & 3) < 3;
    const int my_comp = 3 * (lane >> 3) + ((lane >> 1) & 3);
    // this lane's destination pointer slot: sRow[j] + my_comp, read as one
    // 64-bit shared load per visit (the pointer array's shared-window address)
    const uint32_t aRow = smem_addr(sRow);
    float *part = kMode != 0 ? s_part + (size_t)warp * kB * 12 : nullptr;

    // batches aligned to the forward's chunk grid (start + 256 b), top down
    for (int b = (hi - start - 1) / kB; b >= 0; b--) {
        const int lo = start + b * kB;
        const int cnt = min(kB, hi - lo);
        // this warp's mask words of the batch (lane q < 8 holds chunk q)
        uint32_t words = 0;
        if (blend_mask && lane < 8 && 32 * lane < cnt)
            words = blend_mask[mask_word(start, tile, b * (kB / 32) + lane, warp)];
        __syncthreads();  // previous batch fully consumed
        for (int t = threadIdx.x; t < cnt; t += kThreads) {
            const uint32_t p = inst_prim[lo + t];
            stage_splat(splat, p, ox, oy, s, t);
            sRow[t] = dest_row<kMode>(out, lo + t, p, txi, tyi, prim_row, tile_rect);
        }
        if (kMode != 0) {  // this warp's partial sums of the batch start at zero
            for (int i = lane; i < cnt * 3; i += 32)
                reinterpret_cast<float4 *>(part)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
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
            while (mask) {
                const int bit = 31 - __clz(mask);
                mask &= ~(1u << bit);
                const int j = c0 + bit;
                const int k = lo + j;
                // Branch-free per lane: pixels that do not contribute compute
                // with a zero weight and keep T, R; contributing ones run
                // exactly the reference's operations (every decision here
                // was certified by the forward for non-redo pixels).
                const float4 A = lds128(aA + 16 * j);
                const float4 B = lds128(aB + 16 * j);
                Pair2 q;
                pair_power2(fx, fy, A, B, q);
                const float2 pc = add2(q.power, f2(B.y));                                      // :263-269
                const bool live0 = (k <= li0) & (fabsf(pc.x) <= B.y), live1 = (k <= li1) & (fabsf(pc.y) <= B.y);
                if (!blend_mask && !__any_sync(0xffffffffu, live0 | live1)) continue;
                const float4 C = lds128(aC + 16 * j);
                const float4 D = lds128(aD + 16 * j);
                pair_alpha2<false>(B, C, q);
                const float2 alpha = make_float2(fminf(q.A.x, SSG_ALPHA_MAX), fminf(q.A.y, SSG_ALPHA_MAX));
                const bool ct0 = live0 & (q.A.x >= SSG_ALPHA_SKIP), ct1 = live1 & (q.A.y >= SSG_ALPHA_SKIP);  // :276
                if (!blend_mask && !__any_sync(0xffffffffu, ct0 | ct1)) continue;
                const float2 oma = sub2(f2(1.0f), alpha);
                const float2 Tn = mul2(T, make_float2(fast_rcp(oma.x), fast_rcp(oma.y)));    // :280
                T = sel2(ct0, ct1, Tn, T);
                const float2 e0 = sub2(f2(C.z), R0), e1 = sub2(f2(C.w), R1), e2 = sub2(f2(D.x), R2);
                const float2 d_alpha = mul2(T, fma2(e2, d2, fma2(e1, d1, mul2(e0, d0))));
                const float2 aT = sel2(ct0, ct1, mul2(alpha, T), f2(0.0f));
                // DA = 0 past the clamp (:290)
                const float2 DA = sel2(ct0 & (q.A.x <= SSG_ALPHA_MAX), ct1 & (q.A.y <= SSG_ALPHA_MAX), d_alpha,
                                       f2(0.0f));
                const float2 d_power = mul2(DA, q.A);
                // d_z (:293) exists for skew-free splats too (z = 0, E = 1: e^-z^2 G = G)
                const bool skewed = (B.z != 0.0f || B.w != 0.0f);                            // warp-uniform
                float2 Gez2 = q.G;
                if (skewed) {
                    const float2 pw = make_float2(fminf(q.power.x, 0.0f), fminf(q.power.y, 0.0f));
                    const float2 a2 = mul2(fma2(make_float2(-q.z.x, -q.z.y), q.z, pw), f2(SSG_LOG2E));
                    Gez2 = make_float2(fast_exp2(a2.x), fast_exp2(a2.y));
                }
                const float2 dzs = mul2(mul2(mul2(DA, f2(kDzScale)), Gez2), fma2(f2(C.y), q.E, q.o));
                const float2 px_ = mul2(d_power, f2(q.dx)), py_ = mul2(d_power, q.dy);
                // per-pixel terms, then the pair's sum per component
                float g[12];
                {
                    const float2 g0 = fma2(f2(A.z), px_, fma2(f2(A.w), py_, mul2(dzs, f2(-B.z))));   // -d_dx
                    const float2 g1 = fma2(f2(B.x), py_, fma2(f2(A.w), px_, mul2(dzs, f2(-B.w))));   // -d_dy
                    const float2 g2 = mul2(mul2(f2(-0.5f), px_), f2(q.dx));
                    const float2 g3 = mul2(make_float2(-px_.x, -px_.y), q.dy);
                    const float2 g4 = mul2(mul2(f2(-0.5f), py_), q.dy);
                    const float2 g5 = mul2(dzs, f2(q.dx));
                    const float2 g6 = mul2(dzs, q.dy);
                    const float2 hGE = mul2(mul2(mul2(f2(0.5f), DA), q.G), q.E);
                    const float2 g7 = mul2(hGE, q.E);
                    const float2 g8 = mul2(hGE, sub2(f2(2.0f), q.E));
                    const float2 g9 = mul2(aT, d0), g10 = mul2(aT, d1), g11 = mul2(aT, d2);
                    g[0] = g0.x + g0.y;
                    g[1] = g1.x + g1.y;
                    g[2] = g2.x + g2.y;
                    g[3] = g3.x + g3.y;
                    g[4] = g4.x + g4.y;
                    g[5] = g5.x + g5.y;
                    g[6] = g6.x + g6.y;
                    g[7] = g7.x + g7.y;
                    g[8] = g8.x + g8.y;
                    g[9] = g9.x + g9.y;
                    g[10] = g10.x + g10.y;
                    g[11] = g11.x + g11.y;
                }
                const float2 ae = sel2(ct0, ct1, alpha, f2(0.0f));                               // :306-308
                R0 = fma2(ae, e0, R0);
                R1 = fma2(ae, e1, R1);
                R2 = fma2(ae, e2, R2);
                const float v = warp_reduce_transposed12(g, lane);
                if (holder) {
                    if (kMode == 0) red_add_global(lds_ptr(aRow + 8 * j) + my_comp, v);
                    else part[j * 12 + my_comp] = v;
                }
            }
        }
        if (kMode != 0) {
            // fixed-order combination of the warps' sums, one row per thread
            __syncthreads();
            for (int j = threadIdx.x; j < cnt; j += kThreads) {
                float4 acc[3];
#pragma unroll
                for (int c = 0; c < 3; c++) acc[c] = reinterpret_cast<const float4 *>(s_part + j * 12)[c];
#pragma unroll
                for (int w = 1; w < kWarps; w++) {
                    const float4 *src = reinterpret_cast<const float4 *>(s_part + ((size_t)w * kB + j) * 12);
#pragma unroll
                    for (int c = 0; c < 3; c++) {
                        const float4 v = src[c];
                        acc[c].x += v.x;
                        acc[c].y += v.y;
                        acc[c].z += v.z;
                        acc[c].w += v.w;
                    }
                }
                float4 *dst = reinterpret_cast<float4 *>(sRow[j]);
#pragma unroll
                for (int c = 0; c < 3; c++) dst[c] = acc[c];
            }
        }
    }
}

// Per-warp scratch of the backward redo: the candidate list and, per
// candidate, its alpha (< 0: not passing), transmittance before it and the
// running colour . dL up to and including it.
struct RedoBwdSmem {
    uint32_t list[kCand];
    double al[kCand], tb[kCand], fdl[kCand];
};

// The 12 per-instance sums of one blended pair (raster/_core.pyx:280-305) in
// fp64, added to the destination row (atomics in mode 0; plain adds in the
// deterministic modes, where one warp owns all rows of its tile).
template <int kMode>
__device__ __forceinline__ void redo_emit(const RedoPixel &P, int k, uint32_t p, const RefPair &rp, double al,
                                          double Tb, double d_alpha, double dl0, double dl1, double dl2,
                                          const ssg_splat64 *splat64, float *out, const uint64_t *prim_row,
                                          const uint64_t *tile_rect) {
    const ssg_splat64 e = splat64[p];
    const double DA = rp.A <= 0.99 ? d_alpha : 0.0;                                          // :290
    const double d_power = DA * rp.A;
    const double ez2 = exp(-rp.z * rp.z);
    const double d_z = DA * rp.G * SSG_REF_TWO_OVER_SQRT_PI * ez2 * (rp.o + 0.5 * (e.o1 - e.o2) * rp.E);  // :293
    const double d_dx = d_power * (-(e.conic_a * rp.dx + e.conic_b * rp.dy)) + d_z * e.skew_x * SSG_REF_SQRT1_2;
    const double d_dy = d_power * (-(e.conic_c * rp.dy + e.conic_b * rp.dx)) + d_z * e.skew_y * SSG_REF_SQRT1_2;
    const double aT = al * Tb;
    float g[12];
    g[0] = (float)(-d_dx);
    g[1] = (float)(-d_dy);
    g[2] = (float)(d_power * (-0.5 * rp.dx * rp.dx));
    g[3] = (float)(d_power * (-rp.dx * rp.dy));
    g[4] = (float)(d_power * (-0.5 * rp.dy * rp.dy));
    g[5] = (float)(d_z * rp.dx * SSG_REF_SQRT1_2);
    g[6] = (float)(d_z * rp.dy * SSG_REF_SQRT1_2);
    g[7] = (float)(DA * 0.5 * rp.G * rp.E * rp.E);
    g[8] = (float)(DA * 0.5 * (2.0 - rp.E) * rp.G * rp.E);
    g[9] = (float)(aT * dl0);
    g[10] = (float)(aT * dl1);
    g[11] = (float)(aT * dl2);
    float *row = dest_row<kMode>(out, k, p, P.tx, P.ty, prim_row, tile_rect);
#pragma unroll
    for (int c = 0; c < 12; c++) {
        if (kMode == 0) atomicAdd(row + c, g[c]);
        else row[c] += g[c];
    }
}

// Exact backward of one flagged pixel (raster/_core.pyx:232-312 for it) in
// fp64.  The reference's R behind instance k satisfies
// T_before(k) R_k = (C - F_k) / (1 - alpha_k), C the pixel colour and F_k the
// colour blended up to and including k, so one front-to-back pass gives F_k
// (stored per candidate) and C, and a second sweep over the stored
// candidates emits d_alpha = T_k c.dL - (C.dL - F_k.dL) / (1 - alpha_k).
// Candidate lists longer than one segment take a two-pass fallback.
template <int kMode>
__device__ __forceinline__ void redo_backward_pixel(const RedoPixel &P, int li, const float *dLp, float bg0,
                                                    float bg1, float bg2, const ssg_splat *splat,
                                                    const ssg_splat64 *splat64, const uint32_t *inst_prim,
                                                    const uint32_t *blend_mask, RedoBwdSmem &sm, float *out,
                                                    const uint64_t *prim_row, const uint64_t *tile_rect) {
    if (li < P.start) return;
    const int lane = threadIdx.x & 31;
    const int kend = li + 1;
    const double dl0 = dLp[0], dl1 = dLp[1], dl2 = dLp[2];
    int kb = P.start;
    const int kmask = blend_mask ? li : -1;
    const int n = redo_candidates<false>(P, kb, kend, kmask, blend_mask, splat, inst_prim, sm.list);
    if (kb >= kend) {
        // front to back over the candidates: alpha, T_before, F.dL
        double T = 1.0, Fdl = 0.0;
        for (int r = 0; r < n; r += 32) {
            const int idx = r + lane;
            const bool valid = idx < n;
            double al = 0.0, cdl = 0.0;
            bool pass = false;
            if (valid) {
                const int k = (int)sm.list[idx];
                const uint32_t p = inst_prim[k];
                const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
                const RefPair rp = ref_pair(P.pxc, P.pyc, m.x, m.y, splat64[p], false);
                al = rp.A < 0.99 ? rp.A : 0.99;
                pass = !rp.skip && al >= 1.0 / 255.0;
                const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
                const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
                cdl = (double)q2.w * dl0 + (double)q3.x * dl1 + (double)q3.y * dl2;
            }
            const double f = pass ? 1.0 - al : 1.0;
            const double incl = warp_prefix_prod(f);
            double excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0;
            const double Tb = T * excl;
            const double fdl = warp_prefix_sum(pass ? al * Tb * cdl : 0.0) + Fdl;
            if (valid) {
                sm.al[idx] = pass ? al : -1.0;
                sm.tb[idx] = Tb;
                sm.fdl[idx] = fdl;
            }
            T *= __shfl_sync(0xffffffffu, incl, 31);
            Fdl = __shfl_sync(0xffffffffu, fdl, 31);
        }
        const double Cdl = Fdl + T * ((double)bg0 * dl0 + (double)bg1 * dl1 + (double)bg2 * dl2);
        __syncwarp();
        for (int idx = lane; idx < n; idx += 32) {
            const double al = sm.al[idx];
            if (al < 0.0) continue;
            const int k = (int)sm.list[idx];
            const uint32_t p = inst_prim[k];
            const double2 m = __ldg(reinterpret_cast<const double2 *>(splat + p));
            const RefPair rp = ref_pair(P.pxc, P.pyc, m.x, m.y, splat64[p], false);
            const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
            const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
            const double Tb = sm.tb[idx];
            const double cdl = (double)q2.w * dl0 + (double)q3.x * dl1 + (double)q3.y * dl2;
            const double d_alpha = Tb * cdl - (Cdl - sm.fdl[idx]) / (1.0 - al);              // :282-285
            redo_emit<kMode>(P, k, p, rp, al, Tb, d_alpha, dl0, dl1, dl2, splat64, out, prim_row, tile_rect);
        }
        __syncwarp();
        return;
    }
    // long candidate lists: pass 1 gives C.dL, pass 2 the gradients
    int nc, li2;
    double f0 = 0.0;
    const double Tf = redo_blend<false>(P, kend, kmask, blend_mask, false, splat, splat64, inst_prim, sm.list, nc, li2,
                                        [&](int, uint32_t p, const RefPair &, double al, double Tb, bool blended) {
                                            if (!blended) return;
                                            const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
                                            const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
                                            f0 += al * Tb * ((double)q2.w * dl0 + (double)q3.x * dl1 +
                                                             (double)q3.y * dl2);
                                        });
    const double Cdl = warp_sum(f0) + Tf * ((double)bg0 * dl0 + (double)bg1 * dl1 + (double)bg2 * dl2);
    double Fdl = 0.0;
    redo_blend<false>(P, kend, kmask, blend_mask, false, splat, splat64, inst_prim, sm.list, nc, li2,
                      [&](int k, uint32_t p, const RefPair &rp, double al, double Tb, bool blended) {
                          double cdl = 0.0;
                          if (blended) {
                              const float4 q2 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 2);
                              const float4 q3 = __ldg(reinterpret_cast<const float4 *>(splat + p) + 3);
                              cdl = (double)q2.w * dl0 + (double)q3.x * dl1 + (double)q3.y * dl2;
                          }
                          const double fdl = warp_prefix_sum(blended ? al * Tb * cdl : 0.0) + Fdl;
                          Fdl = __shfl_sync(0xffffffffu, fdl, 31);
                          if (!blended) return;
                          const double d_alpha = Tb * cdl - (Cdl - fdl) / (1.0 - al);
                          redo_emit<kMode>(P, k, p, rp, al, Tb, d_alpha, dl0, dl1, dl2, splat64, out, prim_row,
                                           tile_rect);
                      });
}

// mode 0: one warp per listed pixel (any order: the rows take atomics)
__global__ void __launch_bounds__(32 * kRedoWarps)
k_blend_backward_redo_list(int32_t ntx, int32_t W, float bg0, float bg1, float bg2, const ssg_splat *__restrict__ splat,
                           const ssg_splat64 *__restrict__ splat64, const uint32_t *__restrict__ inst_prim,
                           const int32_t *__restrict__ ranges, const int32_t *__restrict__ last_idx,
                           const float *__restrict__ dL, const uint32_t *__restrict__ blend_mask,
                           const uint32_t *__restrict__ redo_list, const uint32_t *__restrict__ redo_count,
                           float *__restrict__ out) {
    __shared__ RedoBwdSmem s_redo[kRedoWarps];
    const int wid = threadIdx.x >> 5;
    const uint32_t count = *redo_count;
    for (uint32_t i = blockIdx.x * kRedoWarps + wid; i < count; i += gridDim.x * kRedoWarps) {
        const uint32_t pix = redo_list[i];
        const RedoPixel P = redo_pixel(pix, W, ntx, ranges);
        redo_backward_pixel<0>(P, last_idx[pix], dL + 3 * (size_t)pix, bg0, bg1, bg2, splat, splat64, inst_prim,
                               blend_mask, s_redo[wid], out, nullptr, nullptr);
    }
}

// deterministic modes: one warp per tile, its flagged pixels in a fixed order
template <int kMode>
__global__ void __launch_bounds__(32 * kRedoWarps)
k_blend_backward_redo_tiles(int32_t ntx, int32_t n_tiles, int32_t W, float bg0, float bg1, float bg2,
                            const ssg_splat *__restrict__ splat, const ssg_splat64 *__restrict__ splat64,
                            const uint32_t *__restrict__ inst_prim, const int32_t *__restrict__ ranges,
                            const int32_t *__restrict__ last_idx, const float *__restrict__ dL,
                            const uint32_t *__restrict__ blend_mask, const uint32_t *__restrict__ redo_mask,
                            float *__restrict__ out,
                            const uint64_t *__restrict__ prim_row, const uint64_t *__restrict__ tile_rect) {
    __shared__ RedoBwdSmem s_redo[kRedoWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tile = blockIdx.x * kRedoWarps + wid;
    if (tile >= n_tiles) return;
    const uint32_t word = lane < kBlocks ? redo_mask[(size_t)tile * kBlocks + lane] : 0u;
    if (!__any_sync(0xffffffffu, word != 0u)) return;
    const int ty = tile / ntx, tx = tile - ty * ntx;
    for (int w = 0; w < kBlocks; w++) {
        uint32_t bits = __shfl_sync(0xffffffffu, word, w);
        while (bits) {
            const int l = __ffs(bits) - 1;
            bits &= bits - 1;
            const int px = tx * 16 + (w & 1) * 8 + (l & 7), py = ty * 16 + (w >> 1) * 4 + (l >> 3);
            const uint32_t pix = (uint32_t)py * (uint32_t)W + (uint32_t)px;
            const RedoPixel P = redo_pixel(pix, W, ntx, ranges);
            redo_backward_pixel<kMode>(P, last_idx[pix], dL + 3 * (size_t)pix, bg0, bg1, bg2, splat, splat64,
                                       inst_prim, blend_mask, s_redo[wid], out, prim_row, tile_rect);
            __syncwarp();
        }
    }
}

// deterministic mode: depth rank of each primitive (inverse of the depth order)
__global__ void k_depth_rank(int64_t n, const uint32_t *__restrict__ order, uint32_t *__restrict__ rank) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) rank[order[r]] = (uint32_t)r;
}

// deterministic mode: first primitive-major row of each primitive
// (rank_offset is the exclusive scan of the counts in depth order)
__global__ void k_prim_rows(int64_t n, const uint32_t *__restrict__ rank, const uint64_t *__restrict__ rank_offset,
                            uint64_t *__restrict__ prim_row) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) prim_row[p] = rank_offset[rank[p]];
}

// deterministic mode: each primitive's rows summed in ascending instance
// order (raster/backward.py:70-73: np.add.at visits k in order), walked in
// depth-rank order: thread r reads the rows of primitive order[r], which sit
// right after rank r - 1's (rank_offset), so a warp reads one contiguous range
__global__ void k_reduce_rank_rows(int64_t n, const uint32_t *__restrict__ order,
                                   const uint64_t *__restrict__ rank_offset, const float *__restrict__ rows,
                                   float *__restrict__ screen) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    float4 acc[3] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f),
                     make_float4(0.f, 0.f, 0.f, 0.f)};
    const uint64_t r0 = rank_offset[r], r1 = rank_offset[r + 1];
    for (uint64_t i = r0; i < r1; i++) {
        const float4 *src = reinterpret_cast<const float4 *>(rows + (size_t)i * 12);
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const float4 v = src[q];
            acc[q].x += v.x;
            acc[q].y += v.y;
            acc[q].z += v.z;
            acc[q].w += v.w;
        }
    }
    float4 *dst = reinterpret_cast<float4 *>(screen + (size_t)order[r] * 12);
#pragma unroll
    for (int q = 0; q < 3; q++) dst[q] = acc[q];
}

__global__ void k_erf_probe(const double *x, int64_t n, float *e32, double *e64) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (e32) e32[i] = skew_E2(f2((float)x[i])).x;   // the blend kernels' packed evaluation
    if (e64) e64[i] = ref_erf(x[i]);
}

constexpr size_t kDetSmem = sizeof(float) * kWarps * kDetBatch * 12;

// per-device one-time launch setup (function attributes are per device)
struct DevSetup {
    int redo_grid;
};
static int dev_setup(DevSetup &out) {
    static DevSetup cache[64];
    static DeviceOnce once;
    cudaError_t e = once.run([](int dev) {
        cudaError_t r = cudaFuncSetAttribute(k_blend_backward<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kDetSmem);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k_blend_backward<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDetSmem);
        int sms = 148;
        if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess) cache[dev].redo_grid = sms * 12;  // 48 redo warps per SM
        return r;
    });
    int dev = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { set_error("blend setup", e); return SSG_ERR_CUDA; }
    out = cache[dev];
    return SSG_OK;
}

static int launch_forward(bool vanilla, int32_t width, int32_t height, const float bg[3], const ssg_splat *splat,
                          const ssg_splat64 *splat64, const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                          int32_t flags, cudaStream_t st) {
    DevSetup ds;
    int rc = dev_setup(ds);
    if (rc != SSG_OK) return rc;
    const int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    if (!(flags & SSG_BLEND_EXACT_ONLY)) {
        cudaError_t e = cudaMemsetAsync(frame->redo_count, 0, sizeof(uint32_t), st);
        if (e != cudaSuccess) { set_error("memset redo count", e); return SSG_ERR_CUDA; }
        if (vanilla)
            k_blend_forward<true><<<ntx * nty, kThreads, 0, st>>>(
                ntx, width, height, bg[0], bg[1], bg[2], splat, bins->inst_prim, bins->ranges, frame->color,
                frame->final_T, frame->n_contrib, frame->last_idx, frame->blend_mask, frame->redo_mask,
                frame->redo_list, frame->redo_count, (flags & SSG_BLEND_ALL_EXACT) != 0);
        else
            k_blend_forward<false><<<ntx * nty, kThreads, 0, st>>>(
                ntx, width, height, bg[0], bg[1], bg[2], splat, bins->inst_prim, bins->ranges, frame->color,
                frame->final_T, frame->n_contrib, frame->last_idx, frame->blend_mask, frame->redo_mask,
                frame->redo_list, frame->redo_count, (flags & SSG_BLEND_ALL_EXACT) != 0);
        rc = check_launch("k_blend_forward");
        if (rc != SSG_OK) return rc;
    }
    if (flags & SSG_BLEND_MAIN_ONLY) return SSG_OK;
    if (vanilla)
        k_blend_forward_redo<true><<<ds.redo_grid, 32 * kRedoWarps, 0, st>>>(
            ntx, width, bg[0], bg[1], bg[2], splat, splat64, bins->inst_prim, bins->ranges, frame->color,
            frame->final_T, frame->n_contrib, frame->last_idx, frame->blend_mask, frame->redo_list, frame->redo_count);
    else
        k_blend_forward_redo<false><<<ds.redo_grid, 32 * kRedoWarps, 0, st>>>(
            ntx, width, bg[0], bg[1], bg[2], splat, splat64, bins->inst_prim, bins->ranges, frame->color,
            frame->final_T, frame->n_contrib, frame->last_idx, frame->blend_mask, frame->redo_list, frame->redo_count);
    return check_launch("k_blend_forward_redo");
}

static bool frame_ok(const ssg_frame_buffers *f) {
    return f && f->color && f->final_T && f->n_contrib && f->last_idx && f->redo_mask && f->redo_list &&
           f->redo_count;
}

}  // namespace ssg

extern "C" int64_t ssg_blend_mask_words(int64_t m, int32_t n_tiles) {
    // mask_word(): bases start/32 + tile + chunk, kWarps (4) warps each
    return m < 0 || n_tiles < 0 ? -1 : (int64_t)ssg::kWarps * (m / 32 + (int64_t)n_tiles + 1);
}

extern "C" int ssg_blend_forward(int64_t m, int32_t width, int32_t height, const float background[3],
                                 const ssg_splat *splat, const ssg_splat64 *splat64, const ssg_bin_buffers *bins,
                                 const ssg_frame_buffers *frame, void *stream) {
    using namespace ssg;
    if (!bins || !frame_ok(frame) || !background || !splat64 || width < 1 || height < 1)
        return SSG_ERR_INVALID_ARGUMENT;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    (void)m;
    return launch_forward(false, width, height, background, splat, splat64, bins, frame, 0, (cudaStream_t)stream);
}

extern "C" int ssg_blend_forward_ex(int64_t m, int32_t width, int32_t height, const float background[3],
                                    const ssg_splat *splat, const ssg_splat64 *splat64, const ssg_bin_buffers *bins,
                                    const ssg_frame_buffers *frame, int32_t flags, void *stream) {
    using namespace ssg;
    if (!bins || !frame_ok(frame) || !background || !splat64 || width < 1 || height < 1 ||
        (flags & ~(SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY | SSG_BLEND_ALL_EXACT)) ||
        (flags & (SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY)) == (SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY))
        return SSG_ERR_INVALID_ARGUMENT;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    (void)m;
    return launch_forward(false, width, height, background, splat, splat64, bins, frame, flags,
                          (cudaStream_t)stream);
}

extern "C" int ssg_test_blend_forward_vanilla(int32_t width, int32_t height, const float background[3],
                                              const ssg_splat *splat, const ssg_splat64 *splat64,
                                              const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                              void *stream) {
    using namespace ssg;
    if (!bins || !frame_ok(frame) || !background || !splat64 || width < 1 || height < 1)
        return SSG_ERR_INVALID_ARGUMENT;
    return launch_forward(true, width, height, background, splat, splat64, bins, frame, 0, (cudaStream_t)stream);
}

extern "C" int ssg_blend_backward_ex(int64_t n, int64_t m, int32_t width, int32_t height,
                                     const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                                     const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                     const float *dL_dpixels, const ssg_grad_buffers *grads, int32_t flags,
                                     void *stream) {
    using namespace ssg;
    if (!bins || !frame || !frame->final_T || !frame->last_idx || !frame->redo_mask || !frame->redo_list ||
        !frame->redo_count || !grads || !background || !dL_dpixels || !splat64 || width < 1 || height < 1 || n < 0 ||
        (flags & ~(SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY | SSG_BLEND_NO_ZERO)) ||
        (flags & (SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY)) == (SSG_BLEND_MAIN_ONLY | SSG_BLEND_EXACT_ONLY))
        return SSG_ERR_INVALID_ARGUMENT;
    (void)m;
    DevSetup ds;
    int rc = dev_setup(ds);
    if (rc != SSG_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (!(flags & SSG_BLEND_NO_ZERO)) {
        cudaError_t e = cudaMemsetAsync(grads->screen, 0, sizeof(float) * 12 * (size_t)n, st);
        if (e != cudaSuccess) { set_error("memset screen grads", e); return SSG_ERR_CUDA; }
    }
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    if (!(flags & SSG_BLEND_EXACT_ONLY)) {
        k_blend_backward<0><<<ntx * nty, kThreads, 0, st>>>(ntx, width, height, background[0], background[1],
                                                            background[2], splat, bins->inst_prim, bins->ranges,
                                                            frame->final_T, frame->last_idx, frame->blend_mask,
                                                            frame->redo_mask, dL_dpixels, grads->screen, nullptr,
                                                            nullptr);
        rc = check_launch("k_blend_backward");
        if (rc != SSG_OK) return rc;
    }
    if (flags & SSG_BLEND_MAIN_ONLY) return SSG_OK;
    k_blend_backward_redo_list<<<ds.redo_grid, 32 * kRedoWarps, 0, st>>>(
        ntx, width, background[0], background[1], background[2], splat, splat64, bins->inst_prim, bins->ranges,
        frame->last_idx, dL_dpixels, frame->blend_mask, frame->redo_list, frame->redo_count, grads->screen);
    return check_launch("k_blend_backward_redo");
}

extern "C" int ssg_blend_backward(int64_t n, int64_t m, int32_t width, int32_t height,
                                  const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                                  const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                  const float *dL_dpixels, const ssg_grad_buffers *grads, void *stream) {
    return ssg_blend_backward_ex(n, m, width, height, background, splat, splat64, bins, frame, dL_dpixels, grads, 0,
                                 stream);
}

extern "C" size_t ssg_blend_det_temp_bytes(int64_t n, int64_t m) {
    if (n < 0 || m < 0) return 0;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    return al(sizeof(uint32_t) * (size_t)(n + 1)) + al(sizeof(uint64_t) * (size_t)(n + 1)) +
           al(sizeof(float) * 12 * (size_t)(m + 1));
}

extern "C" int ssg_blend_backward_det(int64_t n, int64_t m, int32_t width, int32_t height,
                                      const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                                      const ssg_prim_buffers *prim, const ssg_bin_buffers *bins,
                                      const ssg_frame_buffers *frame, const float *dL_dpixels,
                                      const ssg_grad_buffers *grads, void *temp, size_t temp_bytes, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !frame->final_T || !frame->last_idx || !frame->redo_mask || !grads || !prim ||
        !background || !dL_dpixels || !splat64 || width < 1 || height < 1 || n < 0 || m < 0 || !temp)
        return SSG_ERR_INVALID_ARGUMENT;
    if (temp_bytes < ssg_blend_det_temp_bytes(n, m)) return SSG_ERR_CAPACITY;
    DevSetup ds;
    int rc = dev_setup(ds);
    if (rc != SSG_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    char *t = (char *)temp;
    uint32_t *rank = (uint32_t *)t;
    uint64_t *prim_row = (uint64_t *)(t + al(sizeof(uint32_t) * (size_t)(n + 1)));
    float *rows = (float *)(t + al(sizeof(uint32_t) * (size_t)(n + 1)) + al(sizeof(uint64_t) * (size_t)(n + 1)));
    cudaError_t e = cudaMemsetAsync(rows, 0, sizeof(float) * 12 * (size_t)m, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(grads->screen, 0, sizeof(float) * 12 * (size_t)n, st);
    if (e != cudaSuccess) { set_error("memset det rows", e); return SSG_ERR_CUDA; }
    if (n == 0) return SSG_OK;
    const unsigned gb = (unsigned)((n + 255) / 256);
    k_depth_rank<<<gb, 256, 0, st>>>(n, bins->depth_order, rank);
    k_prim_rows<<<gb, 256, 0, st>>>(n, rank, bins->rank_offset, prim_row);
    const int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_backward<2><<<ntx * nty, kThreads, kDetSmem, st>>>(
        ntx, width, height, background[0], background[1], background[2], splat, bins->inst_prim, bins->ranges,
        frame->final_T, frame->last_idx, frame->blend_mask, frame->redo_mask, dL_dpixels, rows, prim_row,
        prim->tile_rect);
    k_blend_backward_redo_tiles<2><<<(ntx * nty + kRedoWarps - 1) / kRedoWarps, 32 * kRedoWarps, 0, st>>>(
        ntx, ntx * nty, width, background[0], background[1], background[2], splat, splat64, bins->inst_prim,
        bins->ranges, frame->last_idx, dL_dpixels, frame->blend_mask, frame->redo_mask, rows, prim_row,
        prim->tile_rect);
    k_reduce_rank_rows<<<gb, 256, 0, st>>>(n, bins->depth_order, bins->rank_offset, rows, grads->screen);
    return check_launch("k_blend_backward(det)");
}

extern "C" int ssg_blend_backward_slots(int64_t m, int32_t width, int32_t height, const float background[3],
                                        const ssg_splat *splat, const ssg_splat64 *splat64,
                                        const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                        const float *dL_dpixels, float *slots, void *stream) {
    using namespace ssg;
    if (!bins || !frame || !frame->final_T || !frame->last_idx || !frame->redo_mask || !background ||
        !dL_dpixels || !slots || !splat64 || width < 1 || height < 1 || m < 0)
        return SSG_ERR_INVALID_ARGUMENT;
    DevSetup ds;
    int rc = dev_setup(ds);
    if (rc != SSG_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(slots, 0, sizeof(float) * 12 * (size_t)m, st);
    if (e != cudaSuccess) { set_error("memset slots", e); return SSG_ERR_CUDA; }
    const int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_blend_backward<1><<<ntx * nty, kThreads, kDetSmem, st>>>(
        ntx, width, height, background[0], background[1], background[2], splat, bins->inst_prim, bins->ranges,
        frame->final_T, frame->last_idx, frame->blend_mask, frame->redo_mask, dL_dpixels, slots, nullptr, nullptr);
    k_blend_backward_redo_tiles<1><<<(ntx * nty + kRedoWarps - 1) / kRedoWarps, 32 * kRedoWarps, 0, st>>>(
        ntx, ntx * nty, width, background[0], background[1], background[2], splat, splat64, bins->inst_prim,
        bins->ranges, frame->last_idx, dL_dpixels, frame->blend_mask, frame->redo_mask, slots, nullptr, nullptr);
    return check_launch("k_blend_backward(slots)");
}

extern "C" int ssg_erf_probe(const double *x, int64_t n, float *e32, double *e64, void *stream) {
    using namespace ssg;
    if (n < 0 || (n > 0 && !x)) return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    k_erf_probe<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, e32, e64);
    return check_launch("k_erf_probe");
}
