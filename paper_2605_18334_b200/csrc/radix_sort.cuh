// radix_sort.cuh -- hand-written stable LSD onesweep radix sort (key, u32
// value) for the binning stage.
//
// One histogram kernel counts the 8-bit digits of every pass in a single read
// of the keys; a one-block scan turns them into bucket bases and drops passes
// whose digit is the same for every (valid) key (the fp64 depth keys of a
// scene share their sign/exponent prefix, the 13-bit tile keys need only two
// passes).  Each pass is reduce-then-scan: a CTA per key tile counts, ranks
// its keys stably inside shared memory (warp-striped order, __match_any_sync
// per step), takes its per-digit global offsets from an upsweep (per-tile
// digit counts) + per-digit row scan -- no inter-CTA spin waits -- reorders
// the tile by digit in shared memory and writes it out in digit runs
// (coalesced).
#pragma once

#include "ssg_common.cuh"

namespace ssg {
namespace radix {

constexpr int kThreads = 256;
constexpr int kMaxPasses = 8;
constexpr uint64_t kFlagAgg = 1ull << 62;     // tile aggregate published
constexpr uint64_t kFlagPre = 2ull << 62;     // inclusive prefix published
constexpr uint64_t kValMask = (1ull << 62) - 1;

template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<uint16_t> {
    static constexpr bool has_invalid = false;
    static constexpr int ipt = 8;              // 2048-key tiles: M ~ 1e7 instances
    static __device__ __forceinline__ bool valid(uint16_t) { return true; }
};
template <>
struct KeyTraits<uint64_t> {
    static constexpr bool has_invalid = true;
    static constexpr int ipt = 8;              // 2048-key tiles
    // the depth key of a primitive that emits no instances is ~0: its
    // position is irrelevant, so it does not veto skipping a constant digit
    static __device__ __forceinline__ bool valid(uint64_t k) { return k != ~0ull; }
};

struct Control {                       // device-side pass schedule
    uint32_t hist_all[kMaxPasses][256];
    uint32_t hist_valid[kMaxPasses][256];
    uint32_t base[kMaxPasses][256];
    int32_t active[kMaxPasses];        // digit index of the k-th executed pass
    int32_t n_active;
    uint32_t n_valid;
    uint32_t tile_counter[kMaxPasses];
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
template <typename K>
__host__ __device__ constexpr int tile_keys() { return kThreads * KeyTraits<K>::ipt; }
template <typename K>
__host__ __device__ inline int64_t num_tiles(int64_t n) { return (n + tile_keys<K>() - 1) / tile_keys<K>(); }

// temp = [Control | tile_counts 256 x tiles u32 | keys_alt | vals_alt]
template <typename K>
inline size_t temp_bytes(int64_t n) {
    return align256(sizeof(Control)) + align256(sizeof(uint32_t) * 256 * num_tiles<K>(n)) +
           align256(sizeof(K) * n) + align256(sizeof(uint32_t) * n);
}

template <typename K>
__global__ void __launch_bounds__(256) k_hist(const K *__restrict__ keys, int64_t n, int npass,
                                              Control *ctl) {
    __shared__ uint32_t h_all[kMaxPasses][256], h_val[kMaxPasses][256];
    __shared__ uint32_t s_nvalid;
    for (int q = threadIdx.x; q < kMaxPasses * 256; q += 256) {
        (&h_all[0][0])[q] = 0;
        (&h_val[0][0])[q] = 0;
    }
    if (threadIdx.x == 0) s_nvalid = 0;
    __syncthreads();
    uint32_t nv = 0;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
        const K k = keys[i];
        const bool v = KeyTraits<K>::valid(k);
        nv += v;
        for (int p = 0; p < npass; p++) {
            const uint32_t d = (uint32_t)(k >> (8 * p)) & 255u;
            atomicAdd(&h_all[p][d], 1u);
            if (KeyTraits<K>::has_invalid && v) atomicAdd(&h_val[p][d], 1u);
        }
    }
    // (the grid-stride loop above is not warp-uniform at the tail, so the
    // per-key atomics are not warp-aggregated; contention is low because the
    // keys of neighbouring threads differ in their low digits)
    nv = __reduce_add_sync(0xffffffffu, nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicAdd(&s_nvalid, nv);
    __syncthreads();
    for (int q = threadIdx.x; q < npass * 256; q += 256) {
        const uint32_t a = (&h_all[0][0])[q];
        const uint32_t b = KeyTraits<K>::has_invalid ? (&h_val[0][0])[q] : a;
        if (a) atomicAdd(&ctl->hist_all[0][0] + q, a);
        if (b) atomicAdd(&ctl->hist_valid[0][0] + q, b);
    }
    if (threadIdx.x == 0 && s_nvalid) atomicAdd(&ctl->n_valid, s_nvalid);
}

// One block of 256 threads: bucket bases and the active-pass schedule.
__global__ void __launch_bounds__(256) k_schedule(Control *ctl, int npass, int64_t n) {
    __shared__ uint32_t s[256];
    __shared__ int s_skip[kMaxPasses];
    const int t = threadIdx.x;
    for (int p = 0; p < npass; p++) {
        const uint32_t c = ctl->hist_all[p][t];
        const uint32_t cv = ctl->hist_valid[p][t];
        // inclusive scan (Hillis-Steele; 256 entries)
        s[t] = c;
        __syncthreads();
        for (int off = 1; off < 256; off <<= 1) {
            const uint32_t add = t >= off ? s[t - off] : 0u;
            __syncthreads();
            s[t] += add;
            __syncthreads();
        }
        ctl->base[p][t] = s[t] - c;
        if (t == 0) s_skip[p] = 0;
        __syncthreads();
        if (cv == ctl->n_valid) s_skip[p] = 1;  // every valid key has digit t: constant digit
        __syncthreads();
    }
    if (t == 0) {
        int na = 0;
        for (int p = 0; p < npass; p++)
            if (!s_skip[p]) ctl->active[na++] = p;
        ctl->n_active = na;
    }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Per-tile digit counts of pass k -> tile_counts[digit][tile] (digit-major).
template <typename K>
__global__ void __launch_bounds__(kThreads) k_upsweep(const K *__restrict__ key0, const K *__restrict__ key1,
                                                      int64_t n, int k_pass, const Control *ctl,
                                                      uint32_t *__restrict__ tile_counts) {
    if (k_pass >= ctl->n_active) return;
    constexpr int kIPT = KeyTraits<K>::ipt, kTile = tile_keys<K>();
    __shared__ uint32_t s_cnt[kThreads / 32][256];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int q = t; q < (kThreads / 32) * 256; q += kThreads) (&s_cnt[0][0])[q] = 0;
    __syncthreads();
    const int shift = 8 * ctl->active[k_pass];
    const K *kin = (k_pass & 1) ? key1 : key0;
    const int64_t tile = blockIdx.x, base = tile * kTile;
    const uint32_t lt = lanemask_lt();
    uint32_t dg[kIPT];
#pragma unroll
    for (int i = 0; i < kIPT; i++) {  // all loads in flight before the ranking chain
        const int64_t idx = base + w * (32 * kIPT) + i * 32 + lane;
        dg[i] = idx < n ? ((uint32_t)(kin[idx] >> shift) & 255u) : 256u;
    }
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const uint32_t d = dg[i];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (d < 256u && (peers & lt) == 0) s_cnt[w][d] += __popc(peers);  // one writer per digit per warp
        __syncwarp();
    }
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int ww = 0; ww < kThreads / 32; ww++) c += s_cnt[ww][t];
    tile_counts[(size_t)t * num_tiles<K>(n) + tile] = c;
}

// Exclusive scan of each digit row of tile_counts (one block per digit).
__global__ void __launch_bounds__(1024) k_rowscan(uint32_t *tile_counts, int64_t ntiles, int k_pass,
                                                  const Control *ctl) {
    if (k_pass >= ctl->n_active) return;
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    uint32_t *row = tile_counts + (size_t)blockIdx.x * ntiles;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < ntiles; c0 += 1024) {
        const int64_t i = c0 + t;
        const uint32_t v = i < ntiles ? row[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (lane == 31) s_warp[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t z = s_warp[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, z, off);
                if (lane >= off) z += y;
            }
            s_warp[lane] = z;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        const uint32_t excl = carry + (w > 0 ? s_warp[w - 1] : 0u) + x - v;
        if (i < ntiles) row[i] = excl;
        __syncthreads();
        if (t == 1023) s_carry = excl + v;
        __syncthreads();
    }
}

// Scatter of pass `k` of the schedule (no-op when k >= n_active).
// Ping-pong: even k reads buffer 0, writes buffer 1.  With iota_vals the
// first executed pass generates the values (input positions).
template <typename K>
__global__ void __launch_bounds__(kThreads) k_downsweep(K *__restrict__ key0, K *__restrict__ key1,
                                                        uint32_t *__restrict__ val0, uint32_t *__restrict__ val1,
                                                        bool iota_vals, int64_t n, int k_pass, const Control *ctl,
                                                        const uint32_t *__restrict__ tile_counts) {
    if (k_pass >= ctl->n_active) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K *s_keys = reinterpret_cast<K *>(smem_raw);
    constexpr int kIPT = KeyTraits<K>::ipt, kTile = tile_keys<K>();
    uint32_t *s_vals = reinterpret_cast<uint32_t *>(smem_raw + sizeof(K) * kTile);
    __shared__ uint32_t s_wcnt[kThreads / 32][256];
    __shared__ uint32_t s_excl[256], s_tstart[256], s_warp[8];

    const int digit_idx = ctl->active[k_pass];
    const int shift = 8 * digit_idx;
    const K *kin = (k_pass & 1) ? key1 : key0;
    K *kout = (k_pass & 1) ? key0 : key1;
    const uint32_t *vin = (k_pass & 1) ? val1 : val0;
    uint32_t *vout = (k_pass & 1) ? val0 : val1;
    const bool gen_vals = iota_vals && k_pass == 0;
    const int64_t ntiles = num_tiles<K>(n);

    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int q = t; q < (kThreads / 32) * 256; q += kThreads) (&s_wcnt[0][0])[q] = 0;
    __syncthreads();
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * kTile;
    const int tile_n = (int)(n - base < kTile ? n - base : kTile);

    // load (warp-striped within the warp's 512-key segment) and rank stably
    K key[kIPT];
    uint32_t val[kIPT], dig[kIPT], rnk[kIPT];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const int local = w * (32 * kIPT) + i * 32 + lane;
        const bool ok = local < tile_n;
        const int64_t idx = base + local;
        key[i] = ok ? kin[idx] : (K)0;
        val[i] = ok ? (gen_vals ? (uint32_t)idx : vin[idx]) : 0u;
        dig[i] = ok ? ((uint32_t)(key[i] >> shift) & 255u) : 256u;
    }
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const uint32_t peers = __match_any_sync(0xffffffffu, dig[i]);
        const uint32_t before = dig[i] < 256u ? s_wcnt[w][dig[i]] : 0u;
        rnk[i] = before + __popc(peers & lt);
        __syncwarp();
        if (dig[i] < 256u && (peers & lt) == 0) s_wcnt[w][dig[i]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // per digit (thread t == digit t): warp prefixes and the tile count
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kThreads / 32; ww++) {
        const uint32_t c = s_wcnt[ww][t];
        s_wcnt[ww][t] = run;
        run += c;
    }
    const uint32_t total = run;
    // offset of this tile's digit-t run among all keys with digit t
    // (exclusive scan over tiles produced by k_upsweep + k_rowscan)
    const uint32_t excl = tile_counts[(size_t)t * ntiles + tile];
    s_excl[t] = ctl->base[digit_idx][t] + excl;
    // exclusive scan of the tile's digit counts -> start of each digit run
    uint32_t x = total;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int ww = 0; ww < kThreads / 32; ww++) wpre += ww < w ? s_warp[ww] : 0u;
    s_tstart[t] = wpre + x - total;
    __syncthreads();

    // reorder the tile by digit in shared memory
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        if (dig[i] < 256u) {
            const uint32_t pos = s_tstart[dig[i]] + s_wcnt[w][dig[i]] + rnk[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    // write out in digit runs: consecutive positions of a digit are contiguous
    for (int p = t; p < tile_n; p += kThreads) {
        const K kk = s_keys[p];
        const uint32_t d = (uint32_t)(kk >> shift) & 255u;
        const uint32_t dest = s_excl[d] + (uint32_t)p - s_tstart[d];
        kout[dest] = kk;
        vout[dest] = s_vals[p];
    }
}

// after the schedule: move keys/values to buffer 0 when an odd number of
// passes left them in buffer 1, and materialise the iota values when no pass
// ran at all (so callers always find the result in key0 / val0)
template <typename K>
__global__ void k_settle(const Control *ctl, const K *__restrict__ key1, K *__restrict__ key0,
                         const uint32_t *__restrict__ val1, uint32_t *__restrict__ val0, bool iota_vals,
                         int64_t n) {
    const int na = ctl->n_active;
    if ((na & 1) == 0 && !(na == 0 && iota_vals)) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (na & 1) {
            key0[i] = key1[i];
            val0[i] = val1[i];
        } else {
            val0[i] = (uint32_t)i;
        }
    }
}

// Stable sort of (key, value) pairs by bits [0, 8*npass) of the key, in
// place: keys0/vals0 hold the input and, on return, the sorted pairs.  With
// iota_vals the input values are the positions 0..n-1 (vals0 is output only).
template <typename K>
inline cudaError_t sort_pairs(K *keys0, uint32_t *vals0, bool iota_vals, int64_t n, int npass, void *temp,
                              cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    char *tp = (char *)temp;
    Control *ctl = (Control *)tp;
    tp += align256(sizeof(Control));
    uint32_t *tile_counts = (uint32_t *)tp;
    const int64_t ntiles = num_tiles<K>(n);
    tp += align256(sizeof(uint32_t) * 256 * ntiles);
    K *keys1 = (K *)tp;
    tp += align256(sizeof(K) * n);
    uint32_t *vals1 = (uint32_t *)tp;
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(Control), st);
    if (e != cudaSuccess) return e;
    const int hist_blocks = (int)((n + 255) / 256 < 4 * 148 ? (n + 255) / 256 : 4 * 148);
    k_hist<K><<<hist_blocks, 256, 0, st>>>(keys0, n, npass, ctl);
    k_schedule<<<1, 256, 0, st>>>(ctl, npass, n);
    const size_t smem = (sizeof(K) + sizeof(uint32_t)) * tile_keys<K>();
    static bool attr_set = false;
    if (!attr_set) {
        e = cudaFuncSetAttribute(k_downsweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    for (int k = 0; k < npass; k++) {
        k_upsweep<K><<<(unsigned)ntiles, kThreads, 0, st>>>(keys0, keys1, n, k, ctl, tile_counts);
        k_rowscan<<<256, 1024, 0, st>>>(tile_counts, ntiles, k, ctl);
        k_downsweep<K><<<(unsigned)ntiles, kThreads, smem, st>>>(keys0, keys1, vals0, vals1, iota_vals, n, k,
                                                                ctl, tile_counts);
    }
    k_settle<K><<<(unsigned)hist_blocks, 256, 0, st>>>(ctl, keys1, keys0, vals1, vals0, iota_vals, n);
    return cudaGetLastError();
}

}  // namespace radix
}  // namespace ssg
