// depth_sort.cuh -- binning steps 1+2 in ONE cooperative launch: stable LSD
// radix sort of the primitives by their 64-bit fp64 depth key, then the
// instance counts in depth order and their scan (M).
//
// Reference: raster/tiles.py:72 (np.lexsort((prim, depth[prim], tile))): the
// per-tile order is depth ascending, primitive id ascending on ties, which is
// exactly a stable sort of the ids by the full depth bits.
//
// Every CTA is resident (cooperative launch, one per SM), so the passes are
// separated by grid-wide barriers instead of kernel launches:
//   phase 0   min / max of the valid keys; keys are rebased, k' = k - min
//             (no-instance keys map to ~0), nbits = significant bits of the
//             largest k'
//   passes    LSD over the top kWindow (24) significant bits only (3 byte
//             digits), one grid barrier per pass:
//             counts  per-(tile, digit) counts of the pass, tile_counts
//                     [pass][tile][digit]: pass 0 from a shared-memory
//                     histogram of each tile; pass k+1 accumulated by pass k's
//                     scatter (one global reduction per key, into the tile the
//                     key lands in)
//             prefix  every CTA sums the count table itself: digit totals
//                     (-> bucket bases) and the counts of the tiles before
//                     its own (-> the tile's run starts); no scan phase
//             scatter stable in-tile ranking (warp-striped, match_any per
//                     step), tile reordered by digit in shared memory,
//                     written out in digit runs (coalesced)
//   fix-up    runs of keys equal in those 24 bits but out of order in the low
//             bits (1 part in 2^24 of the depth range: rare, short) are
//             insertion-sorted by the full key, stably; runs without an inversion (exact ties,
//             no-instance keys) are already right; an inverted run longer
//             than 32 triggers the exact fallback, a full LSD over every
//             significant byte
//   final     counts in depth order, exclusive scan over ranks -> rank_offset,
//             n_instances
// Tiles are 8192 keys (1024 threads x 8), one CTA per SM; a CTA loops over
// several tiles when N > tiles x CTAs.
#pragma once

#include <cooperative_groups.h>

#include "radix_sort.cuh"
#include "ssg_common.cuh"

namespace ssg {
namespace dsort {

namespace cg = cooperative_groups;

#ifndef SSG_DS_THREADS
#define SSG_DS_THREADS 1024
#endif
#ifndef SSG_DS_WINDOW
#define SSG_DS_WINDOW 24
#endif
constexpr int kThreads = SSG_DS_THREADS;      // one CTA per SM
constexpr int kWarps = kThreads / 32;
constexpr int kWindow = SSG_DS_WINDOW;        // significant key bits sorted by the passes
constexpr int kIPT = 8;                       // keys per lane per tile
constexpr int kTile = kThreads * kIPT;        // 8192 keys
constexpr uint64_t kInvalid = ~0ull;          // primitives without instances

struct Ctl {
    unsigned long long kmin, kmax;            // range of the valid keys
    uint32_t long_run;                        // fix-up found a run > kFixMax
    uint32_t pad;
};

constexpr int kFixMax = 32;
constexpr unsigned long long kReady = 1ull << 63;  // tile_sums flag (final phase)
constexpr int kMaxPasses = 8;                 // 64-bit keys, byte digits
constexpr int kSub = kThreads / 256;          // threads per digit in the prefix sums
constexpr int kPre = 4;                       // tiles per multi-tile prefix sweep
static_assert(kThreads == 1024, "prefix_sweep maps 64 digit quads x 16 lanes: exactly 1024 threads");

__host__ __device__ inline int64_t num_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

// temp = [Ctl | tile_counts passes x tiles x 256 | tile_sums tiles | keys x2 | vals x1]
inline size_t temp_bytes(int64_t n) {
    const int64_t nt = num_tiles(n > 0 ? n : 1);
    return radix::align256(sizeof(Ctl)) + radix::align256(sizeof(uint32_t) * kMaxPasses * 256 * nt) +
           radix::align256(sizeof(uint64_t) * nt) + 2 * radix::align256(sizeof(uint64_t) * n) +
           radix::align256(sizeof(uint32_t) * n);
}

struct Args {
    const uint64_t *keys_in;      // (n), not modified
    uint32_t *order_out;          // (n) depth order (final permutation)
    const uint32_t *count;        // (n) instances per primitive (nullptr: sort only)
    uint64_t *rank_offset;        // (n+1)
    int64_t *n_instances;         // (2): [0] M, [1] running max of M (caller-reset)
    int64_t n;
    Ctl *ctl;
    uint32_t *tile_counts;        // [kMaxPasses][ntiles][256]
    uint64_t *tile_sums;          // [ntiles]
    uint64_t *keys_a, *keys_b;    // ping-pong keys
    uint32_t *vals_a;             // ping-pong values (the other buffer is order_out)
    const uint32_t *gate;         // optional: run only when *gate != 0 (the onesweep's fallback)
};

struct Smem {
    uint64_t keys[kTile];
    uint32_t vals[kTile];
    uint32_t wcnt[kWarps][256];
    uint32_t base[256];           // bucket base of the current pass
    uint32_t tstart[256];         // tile-local start of each digit run
    uint32_t excl[256];           // global start of this tile's digit run
    uint32_t red[2][kSub][256];   // prefix sums: partial (before tile, total) per sub-thread
    uint32_t pre[4][256];         // multi-tile prefix sweep: counts before each of 4 tiles
    uint32_t swarp[kWarps];
    uint64_t sum64[kWarps];
    unsigned long long kmin, kmax;
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    return x;
}

// 256-entry exclusive scan by the first 8 warps: out[t] = sum in[< t]
__device__ __forceinline__ void scan256(const uint32_t *in, uint32_t *out, uint32_t *swarp) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v = 0, x = 0;
    if (t < 256) {
        v = in[t];
        x = warp_incl_scan(v, lane);
        if (lane == 31) swarp[w] = x;
    }
    __syncthreads();
    if (t < 256) {
        uint32_t pre = 0;
        for (int ww = 0; ww < w; ww++) pre += swarp[ww];
        out[t] = pre + x - v;
    }
    __syncthreads();
}

// Multi-tile CTAs (ntiles > grid): prefix sums over a pass's count table for
// up to kPre of this CTA's tiles (tile, tile + grid, ...) in ONE sweep:
// digit totals (first sweep of the pass -> s.base) and, per tile g, the
// counts of the tiles before it (s.pre[g]).  16 B loads (4 digits), 16 lanes
// per digit quad, reduced by shuffles.  (With one tile per CTA the plain
// 4-byte sweep in the kernel is cheaper.)
__device__ __forceinline__ void prefix_sweep(const uint32_t *cnt, int64_t ntiles, int64_t tile, bool first, Smem &s) {
    const int t = threadIdx.x;
    const int d4 = t >> 4, j = t & 15;  // digits 4*d4 .. 4*d4+3, sweep lane j
    int64_t tl[kPre];
#pragma unroll
    for (int g = 0; g < kPre; g++) tl[g] = tile + (int64_t)g * gridDim.x;  // may be >= ntiles
    const int64_t qend = first ? ntiles : (tl[kPre - 1] < ntiles ? tl[kPre - 1] : ntiles);
    uint4 tot = make_uint4(0, 0, 0, 0), pre[kPre];
#pragma unroll
    for (int g = 0; g < kPre; g++) pre[g] = make_uint4(0, 0, 0, 0);
#pragma unroll 4
    for (int64_t q = j; q < qend; q += 16) {
        const uint4 c = __ldcg(reinterpret_cast<const uint4 *>(cnt + (size_t)q * 256) + d4);
        tot.x += c.x; tot.y += c.y; tot.z += c.z; tot.w += c.w;
#pragma unroll
        for (int g = 0; g < kPre; g++)
            if (q < tl[g]) {
                pre[g].x += c.x; pre[g].y += c.y; pre[g].z += c.z; pre[g].w += c.w;
            }
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        tot.x += __shfl_xor_sync(0xffffffffu, tot.x, off);
        tot.y += __shfl_xor_sync(0xffffffffu, tot.y, off);
        tot.z += __shfl_xor_sync(0xffffffffu, tot.z, off);
        tot.w += __shfl_xor_sync(0xffffffffu, tot.w, off);
#pragma unroll
        for (int g = 0; g < kPre; g++) {
            pre[g].x += __shfl_xor_sync(0xffffffffu, pre[g].x, off);
            pre[g].y += __shfl_xor_sync(0xffffffffu, pre[g].y, off);
            pre[g].z += __shfl_xor_sync(0xffffffffu, pre[g].z, off);
            pre[g].w += __shfl_xor_sync(0xffffffffu, pre[g].w, off);
        }
    }
    if (j == 0) {
        if (first) reinterpret_cast<uint4 *>(s.wcnt[0])[d4] = tot;
#pragma unroll
        for (int g = 0; g < kPre; g++) reinterpret_cast<uint4 *>(s.pre[g])[d4] = pre[g];
    }
    __syncthreads();
    if (first) scan256(s.wcnt[0], s.base, s.swarp);  // bucket bases of this pass
}

static __global__ void __launch_bounds__(kThreads, 1024 / kThreads) k_depth_sort(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    cg::grid_group grid = cg::this_grid();
    if (a.gate && *((volatile const uint32_t *)a.gate) == 0) return;   // every CTA sees the same flag
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t n = a.n, ntiles = num_tiles(n);
    const uint32_t lt = radix::lanemask_lt();

    // ---------------------------------------------------------- phase 0
    if (t == 0) {
        s.kmin = ~0ull;
        s.kmax = 0ull;
    }
    __syncthreads();
    {
        unsigned long long mn = ~0ull, mx = 0ull;
        for (int64_t i = (int64_t)blockIdx.x * kThreads + t; i < n; i += (int64_t)gridDim.x * kThreads) {
            const uint64_t k = a.keys_in[i];
            if (k == kInvalid) continue;
            mn = min(mn, (unsigned long long)k);
            mx = max(mx, (unsigned long long)k);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        }
        if (lane == 0) {
            atomicMin(&s.kmin, mn);
            atomicMax(&s.kmax, mx);
        }
    }
    __syncthreads();
    if (t == 0) {
        atomicMin(&a.ctl->kmin, s.kmin);
        atomicMax(&a.ctl->kmax, s.kmax);
    }
    const size_t slot = (size_t)ntiles * 256;       // one pass's count table
    // zero the count tables of passes 1.. (pass 0's is stored, not accumulated)
    auto zero_counts = [&]() {
        for (size_t q = (size_t)blockIdx.x * kThreads + t + slot; q < kMaxPasses * slot;
             q += (size_t)gridDim.x * kThreads)
            a.tile_counts[q] = 0u;
    };
    zero_counts();
    for (int64_t q = (int64_t)blockIdx.x * kThreads + t; q < ntiles; q += (int64_t)gridDim.x * kThreads)
        a.tile_sums[q] = 0ull;
    grid.sync();
    const uint64_t kmin = *((volatile unsigned long long *)&a.ctl->kmin);
    const uint64_t kmax = *((volatile unsigned long long *)&a.ctl->kmax);
    const int nbits = kmax >= kmin && kmax != kmin ? 64 - __clzll((long long)(kmax - kmin)) : 0;
    const int sh = nbits > kWindow ? nbits - kWindow : 0;  // window [sh, nbits)
    const int npw = (nbits - sh + 7) / 8;                    // window passes

    // ---------------------------------------------------------- passes
    auto run_passes = [&](int np, int shift0) {
        // pass 0 counts: shared-memory histogram per tile
        if (np > 0) {
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                if (t < 256) s.base[t] = 0u;
                __syncthreads();
                const int64_t base = tile * kTile;
#pragma unroll
                for (int i = 0; i < kIPT; i++) {
                    const int64_t idx = base + (int64_t)i * kThreads + t;
                    if (idx < n) {
                        const uint64_t kk = a.keys_in[idx];
                        const uint64_t kr = kk == kInvalid ? ~0ull : kk - kmin;
                        atomicAdd(&s.base[(uint32_t)(kr >> shift0) & 255u], 1u);
                    }
                }
                __syncthreads();
                if (t < 256) a.tile_counts[(size_t)tile * 256 + t] = s.base[t];
                __syncthreads();
            }
            grid.sync();
        }
        for (int k = 0; k < np; k++) {
            const int shift = shift0 + 8 * k;
            const uint64_t *kin = (k & 1) ? a.keys_a : a.keys_b;  // k == 0 reads keys_in (rebased)
            uint64_t *kout = (k & 1) ? a.keys_b : a.keys_a;
            // value ping-pong ends in order_out: pass k writes order_out iff
            // (np - 1 - k) is even; pass 0 generates the ids
            uint32_t *vout = ((np - 1 - k) & 1) ? a.vals_a : a.order_out;
            const uint32_t *vin = k == 0 ? nullptr : (((np - k) & 1) ? a.vals_a : a.order_out);
            const uint32_t *cnt = a.tile_counts + (size_t)k * slot;
            uint32_t *cnext = k + 1 < np ? a.tile_counts + (size_t)(k + 1) * slot : nullptr;
            auto load_key = [&](int64_t idx) -> uint64_t {
                if (k > 0) return kin[idx];
                const uint64_t kk = a.keys_in[idx];
                return kk == kInvalid ? ~0ull : kk - kmin;
            };

            const bool multi = ntiles > (int64_t)gridDim.x;  // some CTA owns several tiles
            int ti = 0;                                       // index of `tile` among this CTA's
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ti++) {
                if (multi) {
                    // one sweep of the count table per group of kPre tiles
                    if (ti % kPre == 0) prefix_sweep(cnt, ntiles, tile, ti == 0, s);
                    if (t < 256) s.excl[t] = s.pre[ti % kPre][t];
                    __syncthreads();
                } else {
                    // prefix sums over the count table: digit totals (-> bucket
                    // bases) and counts of the tiles before this one
                    const int d = t & 255, j = t >> 8;
                    const bool first = tile == blockIdx.x;
                    const int64_t qend = first ? ntiles : tile;
                    uint32_t pre = 0, tot = 0;
#pragma unroll 4
                    for (int64_t q = j; q < qend; q += kSub) {
                        const uint32_t c = __ldcg(cnt + (size_t)q * 256 + d);
                        tot += c;
                        pre += q < tile ? c : 0u;
                    }
                    s.red[0][j][d] = pre;
                    s.red[1][j][d] = tot;
                    __syncthreads();
                    if (t < 256) {
                        uint32_t p = 0, tt = 0;
#pragma unroll
                        for (int q = 0; q < kSub; q++) {
                            p += s.red[0][q][t];
                            tt += s.red[1][q][t];
                        }
                        s.excl[t] = p;
                        if (first) s.wcnt[0][t] = tt;
                    }
                    __syncthreads();
                    if (first) scan256(s.wcnt[0], s.base, s.swarp);  // bucket bases of this pass
                }
                for (int q = t; q < kWarps * 256; q += kThreads) (&s.wcnt[0][0])[q] = 0;
                __syncthreads();
                const int64_t base = tile * kTile;
                const int tile_n = (int)(n - base < kTile ? n - base : kTile);
                uint64_t key[kIPT];
                uint32_t val[kIPT], dig[kIPT], rnk[kIPT];
#pragma unroll
                for (int i = 0; i < kIPT; i++) {
                    const int local = w * (32 * kIPT) + i * 32 + lane;
                    const bool ok = local < tile_n;
                    const int64_t idx = base + local;
                    key[i] = ok ? load_key(idx) : 0ull;
                    val[i] = ok ? (vin ? vin[idx] : (uint32_t)idx) : 0u;
                    dig[i] = ok ? ((uint32_t)(key[i] >> shift) & 255u) : 256u;
                }
#pragma unroll
                for (int i = 0; i < kIPT; i++) {
                    const uint32_t peers = __match_any_sync(0xffffffffu, dig[i]);
                    const uint32_t before = dig[i] < 256u ? s.wcnt[w][dig[i]] : 0u;
                    rnk[i] = before + __popc(peers & lt);
                    __syncwarp();
                    if (dig[i] < 256u && (peers & lt) == 0) s.wcnt[w][dig[i]] = before + __popc(peers);
                    __syncwarp();
                }
                __syncthreads();
                if (t < 256) {  // per digit: warp prefixes, tile count, global run start
                    uint32_t run = 0;
#pragma unroll 8
                    for (int ww = 0; ww < kWarps; ww++) {
                        const uint32_t c = s.wcnt[ww][t];
                        s.wcnt[ww][t] = run;
                        run += c;
                    }
                    s.excl[t] += s.base[t];
                    s.tstart[t] = run;  // tile count, scanned below
                }
                __syncthreads();
                scan256(s.tstart, s.tstart, s.swarp);
#pragma unroll
                for (int i = 0; i < kIPT; i++) {
                    if (dig[i] < 256u) {
                        const uint32_t pos = s.tstart[dig[i]] + s.wcnt[w][dig[i]] + rnk[i];
                        s.keys[pos] = key[i];
                        s.vals[pos] = val[i];
                    }
                }
                __syncthreads();
                for (int p = t; p < tile_n; p += kThreads) {
                    const uint64_t kk = s.keys[p];
                    const uint32_t d = (uint32_t)(kk >> shift) & 255u;
                    const uint32_t dest = s.excl[d] + (uint32_t)p - s.tstart[d];
                    kout[dest] = kk;
                    vout[dest] = s.vals[p];
                    // next pass's count of (destination tile, next digit)
                    if (cnext) atomicAdd(cnext + (size_t)(dest / kTile) * 256 + ((uint32_t)(kk >> (shift + 8)) & 255u), 1u);
                }
                __syncthreads();
            }
            grid.sync();
        }
        if (np == 0) {  // every valid key equal: the identity is the stable order
            for (int64_t i = (int64_t)blockIdx.x * kThreads + t; i < n; i += (int64_t)gridDim.x * kThreads)
                a.order_out[i] = (uint32_t)i;
            grid.sync();
        }
    };
    run_passes(npw, sh);

    // ---------------------------------------------------------- fix-up
    if (sh > 0 && npw > 0) {
        const uint64_t *K = ((npw - 1) & 1) ? a.keys_b : a.keys_a;   // last pass output
        // A run (keys equal in the window) needs work only where it holds an
        // inversion in the full key; the run's first inversion sorts it.
        for (int64_t i = 1 + (int64_t)blockIdx.x * kThreads + t; i < n; i += (int64_t)gridDim.x * kThreads) {
            const uint64_t ki = K[i], kp = K[i - 1];
            const uint64_t hi = ki >> sh;
            if ((kp >> sh) != hi || kp <= ki) continue;           // no inversion at i
            int64_t st = i - 1;                                   // run start
            while (st > 0 && i - st <= kFixMax && (K[st - 1] >> sh) == hi) st--;
            int64_t e = i + 1;                                    // run end
            while (e < n && e - st <= kFixMax && (K[e] >> sh) == hi) e++;
            const int len = (int)(e - st);
            if (len > kFixMax || (st > 0 && (K[st - 1] >> sh) == hi)) {
                atomicOr(&a.ctl->long_run, 1u);
                continue;
            }
            bool first = true;                                    // no earlier inversion in the run
            for (int64_t q = st + 1; q < i && first; q++) first = K[q - 1] <= K[q];
            if (!first) continue;
            uint64_t rk[kFixMax];
            uint32_t rv[kFixMax];
            for (int q = 0; q < len; q++) {
                rk[q] = K[st + q];
                rv[q] = a.order_out[st + q];
            }
            for (int q = 1; q < len; q++) {       // stable insertion sort by the full key
                const uint64_t kq = rk[q];
                const uint32_t vq = rv[q];
                int j = q - 1;
                while (j >= 0 && rk[j] > kq) {
                    rk[j + 1] = rk[j];
                    rv[j + 1] = rv[j];
                    j--;
                }
                rk[j + 1] = kq;
                rv[j + 1] = vq;
            }
            for (int q = 0; q < len; q++) a.order_out[st + q] = rv[q];
        }
        grid.sync();
        if (*((volatile uint32_t *)&a.ctl->long_run)) {
            // exact fallback: full LSD over every significant byte
            zero_counts();
            grid.sync();
            run_passes((nbits + 7) / 8, 0);
        }
    }
    if (!a.count) return;

    // ---------------------------------------------------------- final
    // counts in depth order; rank_offset[r+1] = sum of counts of ranks <= r.
    // One pass: each tile publishes its sum with a ready flag (bit 63) and
    // adds the sums of the tiles before it as they appear.  Every CTA is
    // resident and walks its tiles in increasing order, so the lowest
    // unfinished tile never waits.
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * kTile;
        uint64_t v[kIPT], sum = 0;
#pragma unroll
        for (int i = 0; i < kIPT; i++) {
            const int64_t r = base + (int64_t)t * kIPT + i;
            v[i] = r < n ? a.count[a.order_out[r]] : 0u;
            sum += v[i];
        }
        uint64_t x = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) s.sum64[w] = x;
        __syncthreads();
        uint64_t wpre = 0, tot = 0;
        for (int ww = 0; ww < kWarps; ww++) {
            const uint64_t c = s.sum64[ww];
            wpre += ww < w ? c : 0u;
            tot += c;
        }
        if (t == 0) {
            __threadfence();
            *((volatile unsigned long long *)&a.tile_sums[tile]) = (unsigned long long)(tot | kReady);
        }
        // prefix of the earlier tiles
        uint64_t pre = 0;
        for (int64_t q = t; q < tile; q += kThreads) {
            unsigned long long f;
            do {
                f = *((volatile unsigned long long *)&a.tile_sums[q]);
            } while (!(f & kReady));
            pre += f & ~kReady;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, off);
        __syncthreads();  // sum64 reads done
        if (lane == 0) s.sum64[w] = pre;
        __syncthreads();
        uint64_t tile_pre = 0;
        for (int ww = 0; ww < kWarps; ww++) tile_pre += s.sum64[ww];
        uint64_t run = tile_pre + wpre + x - sum;
#pragma unroll
        for (int i = 0; i < kIPT; i++) {
            const int64_t r = base + (int64_t)t * kIPT + i;
            run += v[i];
            if (r < n) a.rank_offset[r + 1] = run;
        }
        if (tile == 0 && t == 0) a.rank_offset[0] = 0;
        if (tile == ntiles - 1 && t == kThreads - 1) {
            a.n_instances[0] = (int64_t)run;
            atomicMax(reinterpret_cast<unsigned long long *>(a.n_instances + 1), (unsigned long long)run);
        }
        __syncthreads();
    }
}

// Host side: sort (and, with count != nullptr, scan the counts in depth
// order).  keys are not modified.  With a gate, the launch returns at once
// unless *gate != 0 (the exact fallback of onesweep.cuh).
static inline cudaError_t sort_and_scan(const uint64_t *keys, uint32_t *order, const uint32_t *count, uint64_t *rank_offset,
                                 int64_t *n_instances, int64_t n, void *temp, cudaStream_t st,
                                 const uint32_t *gate = nullptr) {
    if (n <= 0) return cudaSuccess;
    char *tp = (char *)temp;
    const int64_t nt = num_tiles(n);
    Args a;
    a.keys_in = keys;
    a.order_out = order;
    a.count = count;
    a.rank_offset = rank_offset;
    a.n_instances = n_instances;
    a.n = n;
    a.gate = gate;
    a.ctl = (Ctl *)tp;
    tp += radix::align256(sizeof(Ctl));
    a.tile_counts = (uint32_t *)tp;
    tp += radix::align256(sizeof(uint32_t) * kMaxPasses * 256 * nt);
    a.tile_sums = (uint64_t *)tp;
    tp += radix::align256(sizeof(uint64_t) * nt);
    a.keys_a = (uint64_t *)tp;
    tp += radix::align256(sizeof(uint64_t) * n);
    a.keys_b = (uint64_t *)tp;
    tp += radix::align256(sizeof(uint64_t) * n);
    a.vals_a = (uint32_t *)tp;
    cudaError_t e = cudaMemsetAsync(&a.ctl->kmin, 0xff, sizeof(unsigned long long), st);  // min identity
    if (e == cudaSuccess) e = cudaMemsetAsync(&a.ctl->kmax, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    // the smem attribute and the co-resident grid size belong to the device:
    // cached per device ordinal (function attributes are per device)
    static int grid_max_dev[64] = {0};
    static DeviceOnce setup_once;
    const int smem = (int)sizeof(Smem);
    e = setup_once.run([smem](int dev) {
        cudaError_t r = cudaFuncSetAttribute(k_depth_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (r != cudaSuccess) return r;
        int sms = 0, per = 0;
        r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_depth_sort, kThreads, smem);
        if (r != cudaSuccess) return r;
        if (per < 1) return cudaErrorInvalidConfiguration;
        grid_max_dev[dev] = sms * per;
        return cudaSuccess;
    });
    if (e != cudaSuccess) return e;
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int grid_max = grid_max_dev[dev];
    const int grid = (int)(nt < grid_max ? nt : grid_max);
    void *params[] = {&a};
    return cudaLaunchCooperativeKernel((const void *)k_depth_sort, dim3(grid), dim3(kThreads), params, smem, st);
}

}  // namespace dsort
}  // namespace ssg
