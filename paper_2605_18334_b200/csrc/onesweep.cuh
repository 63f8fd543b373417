// onesweep.cuh -- binning steps 1+2: stable radix sort of the primitives by
// their 64-bit fp64 depth key (one kernel per pass, decoupled look-back),
// then the instance counts in depth order and their scan (M).
//
// Reference: raster/tiles.py:72 (np.lexsort((prim, depth[prim], tile))): the
// per-tile order is depth ascending, primitive id ascending on ties -- a
// stable sort of the ids by the full depth bits.
//
//   minmax   range of the valid keys; keys are rebased, w(k) = (k - min) >>
//            sh with sh = max(0, bits(max - min) - 31), so every valid key's
//            window value is < 2^32 - 1 and no-instance keys (~0) take
//            2^32 - 1: they sort last
//   hist     the four 8-bit digit histograms of the window in one read
//   pass x4  LSD over the window digits: each CTA takes the next 8192-key
//            tile (dynamic tile index), ranks its keys stably (warp-striped,
//            match_any per step), and finds its digit offsets by decoupled
//            look-back over the earlier tiles' published counts, 16 tiles per
//            round trip (no grid barrier, no count table); keys and ids are
//            scattered directly
//   fix-up   runs of keys equal in the window but out of order in the low
//            bits (rare and short) are insertion-sorted by the full key,
//            stably; a run longer than 32 with an inversion flags the exact
//            fallback (the full-width cooperative sort of depth_sort.cuh,
//            launched always and returning at once unless flagged)
//   scan     counts in depth order, exclusive scan (decoupled look-back over
//            tiles) -> rank_offset, n_instances
// Per key and pass: ~30 instructions and 24 bytes of traffic, against the
// cooperative sort's grid barriers (K2-K4 are HBM-bound).
#pragma once

#include "depth_sort.cuh"
#include "radix_sort.cuh"
#include "ssg_common.cuh"

namespace ssg {
namespace osort {

constexpr int kT = 512;                   // threads per CTA
constexpr int kW = kT / 32;
constexpr int kIPT = 16;                  // keys per thread
constexpr int kTile = kT * kIPT;          // 8192 keys per tile
constexpr int kPasses = 4;                // 32-bit window
constexpr int kWinBits = 8 * kPasses - 1; // significant bits a valid key keeps
constexpr int kLook = 16;                 // look-back loads in flight per digit
constexpr int64_t kOnesweepMin = 2000000;    // smaller sorts use the cooperative kernel
constexpr size_t kPassSmem = (sizeof(uint64_t) + sizeof(uint32_t)) * kTile;   // the reordered tile
constexpr int kFix = 32;                  // longest run the fix-up sorts in place
constexpr uint32_t kAgg = 1u << 30, kInc = 2u << 30, kCntMask = kAgg - 1;
constexpr unsigned long long kReady = 1ull << 63;

struct Ctl {
    unsigned long long kmin, kmax;
    uint32_t tile_ctr[kPasses + 1];       // dynamic tile indices (passes, scan)
    uint32_t long_run;                    // fix-up found a long inverted run
    uint32_t pad;
};

__host__ __device__ inline int64_t num_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

struct Layout {
    size_t ctl, hist, status, tsum, keys_a, keys_b, vals_a, old, total;
};
inline Layout layout(int64_t n) {
    const int64_t nt = num_tiles(n > 0 ? n : 1);
    Layout L;
    size_t o = 0;
    auto take = [&](size_t b) { const size_t at = o; o += radix::align256(b); return at; };
    L.ctl = take(sizeof(Ctl));
    L.hist = take(sizeof(uint32_t) * kPasses * 256);
    L.status = take(sizeof(uint32_t) * kPasses * 256 * (size_t)nt);
    L.tsum = take(sizeof(unsigned long long) * (size_t)nt);
    L.keys_a = take(sizeof(uint64_t) * (size_t)n);
    L.keys_b = take(sizeof(uint64_t) * (size_t)n);
    L.vals_a = take(sizeof(uint32_t) * (size_t)n);
    L.old = o;                            // the fallback's own work area
    L.total = o + dsort::temp_bytes(n);
    return L;
}
inline size_t temp_bytes(int64_t n) { return layout(n).total; }

__device__ __forceinline__ int window_shift(unsigned long long kmin, unsigned long long kmax) {
    if (kmax < kmin) return 0;            // no valid key
    const unsigned long long span = kmax - kmin;
    const int bits = span ? 64 - __clzll((long long)span) : 0;
    return bits > kWinBits ? bits - kWinBits : 0;
}
__device__ __forceinline__ uint32_t window(uint64_t k, unsigned long long kmin, int sh) {
    return k == ~0ull ? 0xFFFFFFFFu : (uint32_t)((k - kmin) >> sh);
}

__global__ void __launch_bounds__(kT) k_minmax(const uint64_t *__restrict__ keys, int64_t n, Ctl *ctl) {
    __shared__ unsigned long long smin[kW], smax[kW];
    unsigned long long mn = ~0ull, mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
        const uint64_t k = keys[i];
        if (k != ~0ull) {
            mn = min(mn, (unsigned long long)k);
            mx = max(mx, (unsigned long long)k);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        smin[w] = mn;
        smax[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kW; q++) {
            mn = min(mn, smin[q]);
            mx = max(mx, smax[q]);
        }
        if (mn != ~0ull) atomicMin(&ctl->kmin, mn);
        if (mx != 0) atomicMax(&ctl->kmax, mx);
    }
}

__global__ void __launch_bounds__(kT) k_hist(const uint64_t *__restrict__ keys, int64_t n, const Ctl *ctl,
                                             uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[kPasses][256];
    for (int i = threadIdx.x; i < kPasses * 256; i += kT) (&h[0][0])[i] = 0;
    __syncthreads();
    const unsigned long long kmin = ctl->kmin;
    const int sh = window_shift(kmin, ctl->kmax);
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
        const uint32_t wv = window(keys[i], kmin, sh);
#pragma unroll
        for (int p = 0; p < kPasses; p++) atomicAdd(&h[p][(wv >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPasses * 256; i += kT) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

// One LSD pass over window digit p.  in_vals == nullptr: the ids 0..n-1.
__global__ void __launch_bounds__(kT) k_pass(int p, const uint64_t *__restrict__ in_keys,
                                             const uint32_t *__restrict__ in_vals, uint64_t *__restrict__ out_keys,
                                             uint32_t *__restrict__ out_vals, int64_t n, Ctl *ctl,
                                             const uint32_t *__restrict__ hist, uint32_t *status) {
    __shared__ uint32_t wc[kW][256];      // per-warp digit counts, then per-warp prefixes
    __shared__ uint32_t goff[256];        // global bucket start + look-back prefix of this tile
    __shared__ uint32_t tstart[256];      // tile-local start of each digit run
    __shared__ uint32_t s_tile;
    extern __shared__ __align__(16) unsigned char s_dyn[];   // the tile reordered by digit
    uint64_t *s_keys = reinterpret_cast<uint64_t *>(s_dyn);
    uint32_t *s_vals = reinterpret_cast<uint32_t *>(s_dyn + sizeof(uint64_t) * kTile);
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_tile = atomicAdd(&ctl->tile_ctr[p], 1u);
    for (int i = t; i < kW * 256; i += kT) (&wc[0][0])[i] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kTile + (int64_t)w * (kIPT * 32);
    const unsigned long long kmin = ctl->kmin;
    const int sh = window_shift(kmin, ctl->kmax);
    uint64_t k[kIPT];
    uint32_t v[kIPT], rank[kIPT];
    uint32_t dig[kIPT];
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const int64_t idx = base + 32 * i + lane;
        const bool ok = idx < n;
        k[i] = ok ? in_keys[idx] : ~0ull;
        v[i] = ok ? (in_vals ? in_vals[idx] : (uint32_t)idx) : 0u;
        dig[i] = ok ? (window(k[i], kmin, sh) >> (8 * p)) & 0xFF : 256u;   // 256: padding
    }
    // stable rank inside the warp: keys in order i-major, lane-minor
    const uint32_t lt = radix::lanemask_lt();
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const uint32_t d = dig[i];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t c = d < 256 ? wc[w][d] : 0u;
        __syncwarp();
        rank[i] = c + (uint32_t)__popc(peers & lt);
        if (d < 256 && (peers & lt) == 0) wc[w][d] = c + (uint32_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // threads 0..255 (digit d = t): warp prefixes, tile count, look-back;
    // threads 256..511 (d = t - 256): the digit's global bucket start, the
    // exclusive scan of the pass histogram
    __shared__ uint32_t hbase[256], wsum[8], tsum[8];
    if (t < 256) {
        const int d = t;
        uint32_t run = 0;
#pragma unroll
        for (int q = 0; q < kW; q++) {
            const uint32_t c = wc[q][d];
            wc[q][d] = run;
            run += c;
        }
        {   // tile-local run starts: exclusive scan of the tile's digit counts
            uint32_t x = run;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            if (lane == 31) tsum[w] = x;
            asm volatile("bar.sync 2, 256;");   // the digit warps only
            uint32_t pre = 0;
            for (int q = 0; q < w; q++) pre += tsum[q];
            tstart[d] = pre + x - run;
        }
        uint32_t *st = status + (size_t)p * 256 * num_tiles(n);
        if (tile == 0) {
            atomicExch(st + d, kInc | run);
            goff[d] = 0;
        } else {
            atomicExch(st + (size_t)tile * 256 + d, kAgg | run);
            uint32_t excl = 0;
            // kLook predecessors per round trip: sum back to the nearest
            // inclusive value (a round that meets a not-yet-published tile
            // resumes there)
            for (int64_t q0 = tile - 1; q0 >= 0;) {
                uint32_t f[kLook];
#pragma unroll
                for (int u = 0; u < kLook; u++)
                    f[u] = q0 - u >= 0 ? *((volatile uint32_t *)(st + (size_t)(q0 - u) * 256 + d)) : (uint32_t)(2u << 30);
                int u = 0;
                uint32_t part = 0;
                bool inc = false, gap = false;
#pragma unroll
                for (int uu = 0; uu < kLook; uu++) {
                    if (inc || gap) continue;
                    if (!(f[uu] & (kAgg | kInc))) { gap = true; continue; }
                    part += f[uu] & kCntMask;
                    u = uu + 1;
                    inc = (f[uu] & kInc) != 0;
                }
                excl += part;
                if (inc) break;
                q0 -= u;
            }
            atomicExch(st + (size_t)tile * 256 + d, kInc | (excl + run));
            goff[d] = excl;
        }
    } else {
        const int d = t - 256;
        const uint32_t hv = hist[p * 256 + d];
        uint32_t x = hv;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) wsum[w - 8] = x;
        asm volatile("bar.sync 1, 256;");   // the histogram warps only
        uint32_t pre = 0;
        for (int q = 0; q < w - 8; q++) pre += wsum[q];
        hbase[d] = pre + x - hv;
    }
    __syncthreads();
    if (t < 256) goff[t] += hbase[t];
    // reorder the tile by digit in shared memory ...
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const uint32_t d = dig[i];
        if (d < 256) {
            const uint32_t lp = tstart[d] + wc[w][d] + rank[i];
            s_keys[lp] = k[i];
            s_vals[lp] = v[i];
        }
    }
    __syncthreads();
    // ... and write each digit run contiguously (coalesced)
    const int64_t nvalid = n - tile * kTile < kTile ? n - tile * kTile : (int64_t)kTile;
    for (int j = t; j < nvalid; j += kT) {
        const uint64_t kk = s_keys[j];
        const uint32_t d = (window(kk, kmin, sh) >> (8 * p)) & 0xFF;
        const uint32_t pos = goff[d] + (uint32_t)j - tstart[d];
        out_keys[pos] = kk;
        out_vals[pos] = s_vals[j];
    }
}

// Window-equal runs with an inversion in the full key: stable insertion sort.
__global__ void __launch_bounds__(kT) k_fixup(const uint64_t *__restrict__ K, uint32_t *__restrict__ V, int64_t n,
                                              Ctl *ctl) {
    const unsigned long long kmin = ctl->kmin;
    const int sh = window_shift(kmin, ctl->kmax);
    if (sh == 0) return;                  // the window holds every significant bit
    for (int64_t i = 1 + (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
        const uint64_t ki = K[i], kp = K[i - 1];
        const uint32_t hi = window(ki, kmin, sh);
        if (window(kp, kmin, sh) != hi || kp <= ki) continue;   // no inversion at i
        int64_t st = i - 1;                                     // run start
        while (st > 0 && i - st <= kFix && window(K[st - 1], kmin, sh) == hi) st--;
        int64_t e = i + 1;                                      // run end
        while (e < n && e - st <= kFix && window(K[e], kmin, sh) == hi) e++;
        const int len = (int)(e - st);
        if (len > kFix || (st > 0 && window(K[st - 1], kmin, sh) == hi)) {
            atomicOr(&ctl->long_run, 1u);
            continue;
        }
        // keys stay as they are: other threads read them to find their runs
        bool first = true;                                      // the run's first inversion sorts it
        for (int64_t q = st + 1; q < i && first; q++) first = K[q - 1] <= K[q];
        if (!first) continue;
        uint64_t rk[kFix];
        uint32_t rv[kFix];
        for (int q = 0; q < len; q++) {
            rk[q] = K[st + q];
            rv[q] = V[st + q];
        }
        for (int q = 1; q < len; q++) {
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
        for (int q = 0; q < len; q++) V[st + q] = rv[q];
    }
}

// counts in depth order; rank_offset[r + 1] = sum of the counts of ranks <= r
__global__ void __launch_bounds__(kT) k_count_scan(const uint32_t *__restrict__ order, const uint32_t *__restrict__ count,
                                                   int64_t n, Ctl *ctl, unsigned long long *tsum,
                                                   uint64_t *__restrict__ rank_offset, int64_t *n_instances) {
    __shared__ unsigned long long wsum[kW];
    __shared__ unsigned long long s_pre;
    __shared__ uint32_t s_tile;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_tile = atomicAdd(&ctl->tile_ctr[kPasses], 1u);
    __syncthreads();
    const int64_t tile = s_tile, base = tile * kTile + (int64_t)t * kIPT;
    unsigned long long c[kIPT], sum = 0;
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        c[i] = base + i < n ? count[order[base + i]] : 0u;
        sum += c[i];
    }
    unsigned long long x = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (t == 0) {
        unsigned long long tot = 0;
        for (int q = 0; q < kW; q++) tot += wsum[q];
        unsigned long long pre = 0;
        if (tile > 0) {
            atomicExch(tsum + tile, tot | (1ull << 62));     // aggregate
            for (int64_t q = tile - 1; q >= 0; q--) {
                unsigned long long f;
                do {
                    f = *((volatile unsigned long long *)(tsum + q));
                } while (!(f & (kReady | (1ull << 62))));
                pre += f & ((1ull << 62) - 1);
                if (f & kReady) break;
            }
        }
        atomicExch(tsum + tile, (pre + tot) | kReady);
        s_pre = pre;
        if (tile == num_tiles(n) - 1) {
            n_instances[0] = (int64_t)(pre + tot);
            atomicMax(reinterpret_cast<unsigned long long *>(n_instances + 1), pre + tot);
        }
    }
    __syncthreads();
    unsigned long long run = s_pre + x - sum;
    for (int q = 0; q < w; q++) run += wsum[q];
    if (tile == 0 && t == 0) rank_offset[0] = 0;
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        run += c[i];
        if (base + i < n) rank_offset[base + i + 1] = run;
    }
}

// Host side: sort (and, with count != nullptr, scan the counts in depth
// order).  keys are not modified.
static inline cudaError_t sort_and_scan(const uint64_t *keys, uint32_t *order, const uint32_t *count,
                                        uint64_t *rank_offset, int64_t *n_instances, int64_t n, void *temp,
                                        cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const Layout L = layout(n);
    char *tp = (char *)temp;
    // Below ~2M keys the cooperative sort (one launch, every CTA resident)
    // is faster: 131 vs 155 us at config 2's 1M keys; above it the onesweep
    // wins (config 4's 3M keys), profiles/r2_binning.md.
    if (n < kOnesweepMin)
        return dsort::sort_and_scan(keys, order, count, rank_offset, n_instances, n, tp + L.old, st);
    Ctl *ctl = (Ctl *)(tp + L.ctl);
    uint32_t *hist = (uint32_t *)(tp + L.hist), *status = (uint32_t *)(tp + L.status);
    unsigned long long *tsum = (unsigned long long *)(tp + L.tsum);
    uint64_t *ka = (uint64_t *)(tp + L.keys_a), *kb = (uint64_t *)(tp + L.keys_b);
    uint32_t *va = (uint32_t *)(tp + L.vals_a);
    const int64_t nt = num_tiles(n);
    // ctl (kmin = ~0, the rest 0), histograms and the look-back flags
    cudaError_t e = cudaMemsetAsync(ctl, 0, L.keys_a - L.ctl, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(&ctl->kmin, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static DeviceOnce attr_once;   // function attributes are per device
    e = attr_once.run([](int) {
        return cudaFuncSetAttribute(k_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem);
    });
    if (e != cudaSuccess) return e;
    const unsigned g = (unsigned)(nt < (int64_t)sms * 4 ? nt : (int64_t)sms * 4);
    k_minmax<<<g, kT, 0, st>>>(keys, n, ctl);
    k_hist<<<g, kT, 0, st>>>(keys, n, ctl, hist);
    // passes: keys -> ka -> kb -> ka -> kb ; ids iota -> va -> order -> va -> order
    k_pass<<<(unsigned)nt, kT, kPassSmem, st>>>(0, keys, nullptr, ka, va, n, ctl, hist, status);
    k_pass<<<(unsigned)nt, kT, kPassSmem, st>>>(1, ka, va, kb, order, n, ctl, hist, status);
    k_pass<<<(unsigned)nt, kT, kPassSmem, st>>>(2, kb, order, ka, va, n, ctl, hist, status);
    k_pass<<<(unsigned)nt, kT, kPassSmem, st>>>(3, ka, va, kb, order, n, ctl, hist, status);
    k_fixup<<<g, kT, 0, st>>>(kb, order, n, ctl);
    if (count) k_count_scan<<<(unsigned)nt, kT, 0, st>>>(order, count, n, ctl, tsum, rank_offset, n_instances);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // exact fallback: the cooperative full-width sort, gated on the fix-up flag
    return dsort::sort_and_scan(keys, order, count, rank_offset, n_instances, n, tp + L.old, st, &ctl->long_run);
}

}  // namespace osort
}  // namespace ssg
