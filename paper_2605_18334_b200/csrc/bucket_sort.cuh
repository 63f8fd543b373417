// bucket_sort.cuh -- binning steps 1+2 without radix passes: the stable
// depth order of the primitives by an MSD bucket scatter and small exact
// sorts, then the instance counts in depth order and their scan (M).
//
// Reference: raster/tiles.py:72 (np.lexsort((prim, depth[prim], tile))): the
// per-tile order is depth ascending, primitive id ascending on ties -- a
// stable sort of the ids by the full 64-bit depth key, i.e. a sort by the
// pair (key, id), which is a total order.
//
//   minmax   range of the valid keys (osort::k_minmax)
//   count    bucket b(k) = (k - kmin) >> sh over 2^nbits buckets (about
//            kPerBucket keys each); one atomic per key, whose return value is
//            the key's slot in its bucket; no-instance keys (~0) are counted
//            per chunk instead (they keep id order, last)
//   scan     bucket starts (decoupled look-back, a warp reading 32
//            predecessors per round trip); buckets of kSmall+1 .. kBig keys
//            are listed for the big sorter, a larger one flags the fallback
//   scatter  (key, id, count) records, 16 B, to bucket start + slot (no
//            atomics); no-instance ids by a stable block compaction behind
//            the valid ones
//   rank     every key of a bucket of <= kSmall keys: its final position is
//            the bucket start plus the number of the bucket's (key, id)
//            pairs before it, counted over the bucket in shared memory (a CTA
//            stages its 256 positions plus 32 on each side)
//   big      one warp per listed bucket: bitonic sort in shared memory
//   scan     counts in depth order (written beside the ids by rank / big, so
//            read contiguously) -> rank_offset, n_instances (look-back as above)
//   fallback a bucket above kBig (keys crowded into a sliver of the range):
//            the full-width cooperative sort of depth_sort.cuh, launched
//            always and returning at once unless flagged
// Exact whatever the distribution; no per-digit passes.
#pragma once

#include "onesweep.cuh"

namespace ssg {
namespace bsort {

constexpr int kT = 256;                       // threads per CTA
constexpr int kIPT = 16;                      // keys per thread (count, scatter, scans)
constexpr int kChunk = kT * kIPT;             // 4096 keys per CTA (blocked: id order)
constexpr int kPerBucket = 4;                 // mean keys per bucket
constexpr int kSmall = 32;                    // buckets ranked in place
constexpr int kBig = 2048;                    // largest bucket the warp sorter takes
constexpr int kBigWarps = 4;                  // warps per CTA of the big-bucket sorter
constexpr size_t kBigSmem = (size_t)kBigWarps * kBig * (sizeof(uint64_t) + sizeof(uint32_t));
constexpr int kHalo = kSmall;                 // rank kernel: staged positions either side
constexpr unsigned long long kAggF = 1ull << 62, kIncF = 1ull << 63, kValM = kAggF - 1;

__host__ __device__ inline int bucket_bits(int64_t n) {
    int b = 12;                               // >= one scan tile (kChunk buckets)
    while (b < 22 && ((int64_t)1 << b) * kPerBucket < n) b++;
    return b;
}
__host__ __device__ inline int64_t num_chunks(int64_t n) { return (n + kChunk - 1) / kChunk; }

struct Ctl {
    unsigned long long kmin, kmax;            // osort::k_minmax writes these two
    uint32_t tile_ctr[2];                     // dynamic tile indices: bucket scan, count scan
    uint32_t long_run;                        // a bucket above kBig: run the fallback
    uint32_t nbig;                            // listed big buckets
};

struct Layout {
    size_t ctl, cnt, status, csum, zero_end, bstart, slot, inv, big, rec, rcount, old, total;
};
inline Layout layout(int64_t n) {
    const int64_t nb = (int64_t)1 << bucket_bits(n);
    Layout L;
    size_t o = 0;
    auto take = [&](size_t b) { const size_t at = o; o += radix::align256(b); return at; };
    L.ctl = take(sizeof(Ctl));
    L.cnt = take(sizeof(uint32_t) * (size_t)nb);
    L.status = take(sizeof(unsigned long long) * (size_t)(nb / kChunk));
    L.csum = take(sizeof(unsigned long long) * (size_t)num_chunks(n));
    L.zero_end = o;                           // everything above is zeroed per sort
    L.bstart = take(sizeof(uint32_t) * (size_t)(nb + 1));
    L.slot = take(sizeof(uint32_t) * (size_t)n);
    L.inv = take(sizeof(uint32_t) * (size_t)num_chunks(n));
    L.big = take(sizeof(uint32_t) * (size_t)nb);
    L.rec = take(sizeof(uint4) * (size_t)n);
    L.rcount = take(sizeof(uint32_t) * (size_t)n);
    L.old = o;                                // the fallback's own work area
    L.total = o + dsort::temp_bytes(n);
    return L;
}
inline size_t temp_bytes(int64_t n) { return layout(n).total; }

__device__ __forceinline__ int key_shift(const Ctl *ctl, int nbits) {
    const unsigned long long kmin = ctl->kmin, kmax = ctl->kmax;
    if (kmax < kmin) return 0;                // no valid key
    const unsigned long long span = kmax - kmin;
    const int bits = span ? 64 - __clzll((long long)span) : 0;
    return bits > nbits ? bits - nbits : 0;
}

// (key, id) lexicographic: true when (ka, va) sorts before (kb, vb)
__device__ __forceinline__ bool before(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka < kb || (ka == kb && va < vb);
}

// Decoupled look-back by one warp: the sum of the tiles before `tile`.
// status: 0 = unpublished, kAggF | v = the tile's own sum, kIncF | v = the
// sum through that tile.  Lane i reads tile - 1 - i; a round stops at the
// nearest inclusive entry.
__device__ __forceinline__ unsigned long long lookback(unsigned long long *status, int64_t tile, int lane) {
    unsigned long long pre = 0;
    for (int64_t q0 = tile - 1; q0 >= 0; q0 -= 32) {
        const int64_t q = q0 - lane;
        unsigned long long f = kIncF;         // before tile 0: an inclusive zero
        if (q >= 0) {
            do {
                f = *((volatile unsigned long long *)(status + q));
            } while (!(f & (kAggF | kIncF)));
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (f & kIncF) != 0);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long v = lane <= stop ? (f & kValM) : 0ull;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        pre += v;
        if (inc) break;
    }
    return pre;
}

// Tile scan in a warp-striped layout: warp w owns the tile's elements
// [w * 32 kIPT, (w + 1) * 32 kIPT), element j * 32 + lane of that run in
// c[j] (coalesced loads and stores).  The tile's prefix comes from the
// look-back (warp 0 publishes the aggregate, looks back, publishes the
// inclusive sum).  On return c[j] holds the EXCLUSIVE prefix of its element;
// *tile_total = the sum through this tile.
template <typename T>
__device__ __forceinline__ void tile_scan(T (&c)[kIPT], unsigned long long *status, int64_t tile, T *s_w,
                                          T *s_pre, T *tile_total) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    T sum = 0;
#pragma unroll
    for (int j = 0; j < kIPT; j++) sum += c[j];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) s_w[w] = sum;
    __syncthreads();
    if (w == 0) {
        T tot = 0;
        for (int q = 0; q < kT / 32; q++) tot += s_w[q];
        if (lane == 0 && tile > 0) atomicExch(status + tile, (unsigned long long)tot | kAggF);
        const unsigned long long pre = tile > 0 ? lookback(status, tile, lane) : 0ull;
        if (lane == 0) {
            atomicExch(status + tile, (pre + (unsigned long long)tot) | kIncF);
            *s_pre = (T)pre;
            *tile_total = (T)(pre + tot);
        }
    }
    __syncthreads();
    T carry = *s_pre;
    for (int q = 0; q < w; q++) carry += s_w[q];
#pragma unroll
    for (int j = 0; j < kIPT; j++) {
        const T v = c[j];
        T x = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        c[j] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

// bucket counts; each key's slot in its bucket; no-instance count per chunk
__global__ void __launch_bounds__(kT) k_count(const uint64_t *__restrict__ keys, int64_t n, int nbits,
                                              const Ctl *ctl, uint32_t *__restrict__ cnt,
                                              uint32_t *__restrict__ slot, uint32_t *__restrict__ inv) {
    __shared__ uint32_t s_inv[kT / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned long long kmin = ctl->kmin;
    const int sh = key_shift(ctl, nbits);
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    uint32_t ninv = 0;
#pragma unroll 4
    for (int i = 0; i < kIPT; i++) {
        const int64_t idx = base + i * kT + t;
        const uint64_t k = idx < n ? keys[idx] : 0ull;
        const bool bad = idx < n && k == ~0ull;
        ninv += __popc(__ballot_sync(0xffffffffu, bad));
        if (idx < n && !bad) slot[idx] = atomicAdd(cnt + ((k - kmin) >> sh), 1u);
    }
    if (lane == 0) s_inv[w] = ninv;
    __syncthreads();
    if (t == 0) {
        uint32_t s = 0;
        for (int q = 0; q < kT / 32; q++) s += s_inv[q];
        inv[blockIdx.x] = s;
    }
}

// bucket starts; bstart[nb] = the number of valid keys
__global__ void __launch_bounds__(kT) k_scan(const uint32_t *__restrict__ cnt, int64_t nb, Ctl *ctl,
                                             unsigned long long *status, uint32_t *__restrict__ bstart,
                                             uint32_t *__restrict__ big) {
    __shared__ uint32_t s_w[kT / 32], s_pre, s_tot, s_tile;
    const int t = threadIdx.x;
    if (t == 0) s_tile = atomicAdd(&ctl->tile_ctr[0], 1u);
    __syncthreads();
    const int64_t tile = s_tile, b0 = tile * kChunk + (int64_t)(t >> 5) * 32 * kIPT + (t & 31);
    uint32_t c[kIPT];
#pragma unroll
    for (int j = 0; j < kIPT; j++) {          // nb is a power of two >= kChunk: no tail
        c[j] = cnt[b0 + 32 * j];
        if (c[j] > (uint32_t)kSmall) {
            if (c[j] > (uint32_t)kBig) atomicOr(&ctl->long_run, 1u);
            else big[atomicAdd(&ctl->nbig, 1u)] = (uint32_t)(b0 + 32 * j);
        }
    }
    tile_scan<uint32_t>(c, status, tile, s_w, &s_pre, &s_tot);
#pragma unroll
    for (int j = 0; j < kIPT; j++) bstart[b0 + 32 * j] = c[j];
    if (tile == nb / kChunk - 1 && t == 0) bstart[nb] = s_tot;
}

// keys and ids to bucket start + slot; no-instance ids, stably, behind them
__global__ void __launch_bounds__(kT) k_scatter(const uint64_t *__restrict__ keys, int64_t n, int nbits, int64_t nb,
                                                const Ctl *ctl, const uint32_t *__restrict__ inv,
                                                const uint32_t *__restrict__ bstart,
                                                const uint32_t *__restrict__ slot, const uint32_t *__restrict__ count,
                                                uint4 *__restrict__ rec, uint32_t *__restrict__ order,
                                                uint32_t *__restrict__ rcount) {
    __shared__ uint32_t s_cnt[kIPT][kT / 32];
    __shared__ uint32_t s_red[kT / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned long long kmin = ctl->kmin;
    const int sh = key_shift(ctl, nbits);
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    uint32_t before_inv = 0;                   // no-instance keys of the earlier chunks
    for (int64_t q = t; q < (int64_t)blockIdx.x; q += kT) before_inv += inv[q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) before_inv += __shfl_xor_sync(0xffffffffu, before_inv, off);
    if (lane == 0) s_red[w] = before_inv;
    uint64_t k[kIPT];
    uint32_t badm = 0, ballots[kIPT];
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const int64_t idx = base + i * kT + t;
        k[i] = idx < n ? keys[idx] : 0ull;
        const bool bad = idx < n && k[i] == ~0ull;
        badm |= (uint32_t)bad << i;
        ballots[i] = __ballot_sync(0xffffffffu, bad);
        if (lane == 0) s_cnt[i][w] = __popc(ballots[i]);
    }
    __syncthreads();
    if (badm == 0) {                           // the common case: no marker in this thread's keys
#pragma unroll
        for (int i = 0; i < kIPT; i++) {
            const int64_t idx = base + i * kT + t;
            if (idx < n) {
                const uint32_t pos = bstart[(k[i] - kmin) >> sh] + slot[idx];
                rec[pos] = make_uint4((uint32_t)k[i], (uint32_t)(k[i] >> 32), (uint32_t)idx, count ? count[idx] : 0u);
            }
        }
        return;
    }
    uint32_t inv_base = bstart[nb];
    for (int q = 0; q < kT / 32; q++) inv_base += s_red[q];
    const uint32_t lt = radix::lanemask_lt();
    uint32_t run = 0;                          // no-instance keys earlier in this chunk
#pragma unroll
    for (int i = 0; i < kIPT; i++) {
        const int64_t idx = base + i * kT + t;
        uint32_t before_w = 0, round = 0;
#pragma unroll
        for (int q = 0; q < kT / 32; q++) {
            const uint32_t c = s_cnt[i][q];
            before_w += q < w ? c : 0u;
            round += c;
        }
        if (idx < n) {
            if ((badm >> i) & 1u) {               // no instances: count 0
                const uint32_t pos = inv_base + run + before_w + __popc(ballots[i] & lt);
                order[pos] = (uint32_t)idx;
                rcount[pos] = 0u;
            } else {
                const uint32_t pos = bstart[(k[i] - kmin) >> sh] + slot[idx];
                rec[pos] = make_uint4((uint32_t)k[i], (uint32_t)(k[i] >> 32), (uint32_t)idx, count ? count[idx] : 0u);
            }
        }
        run += round;
    }
}

// final position of every key of a bucket of <= kSmall keys: bucket start +
// the number of the bucket's pairs before it
__global__ void __launch_bounds__(kT) k_rank(const uint4 *__restrict__ rec, int nbits, const Ctl *ctl,
                                             const uint32_t *__restrict__ bstart, int64_t nb,
                                             uint32_t *__restrict__ order, uint32_t *__restrict__ rcount) {
    __shared__ uint64_t s_k[kT + 2 * kHalo];
    __shared__ uint32_t s_v[kT + 2 * kHalo], s_c[kT + 2 * kHalo];
    const int t = threadIdx.x;
    const int64_t nv = bstart[nb];
    const int64_t p0 = (int64_t)blockIdx.x * kT;
    if (p0 >= nv) return;
    const int64_t s0 = p0 - kHalo;            // s_k[i] holds position s0 + i
    for (int i = t; i < kT + 2 * kHalo; i += kT) {
        const int64_t p = s0 + i;
        uint4 r = make_uint4(0u, 0u, 0u, 0u);
        if (p >= 0 && p < nv) r = rec[p];
        s_k[i] = ((uint64_t)r.y << 32) | r.x;
        s_v[i] = r.z;
        s_c[i] = r.w;
    }
    __syncthreads();
    const int64_t p = p0 + t;
    if (p >= nv) return;
    const uint64_t k = s_k[kHalo + t];
    const uint32_t v = s_v[kHalo + t];
    const uint64_t b = (k - ctl->kmin) >> key_shift(ctl, nbits);
    const uint32_t st = bstart[b], sz = bstart[b + 1] - st;
    if (sz > (uint32_t)kSmall) return;        // the big sorter's
    uint32_t r = 0;
    const int i0 = (int)((int64_t)st - s0);
    for (int i = i0; i < i0 + (int)sz; i++) r += before(s_k[i], s_v[i], k, v) ? 1u : 0u;
    order[st + r] = v;
    rcount[st + r] = s_c[kHalo + t];
}

// one warp per listed bucket (kSmall < size <= kBig): bitonic in shared memory
__global__ void __launch_bounds__(32 * kBigWarps) k_big(const uint4 *__restrict__ rec,
                                                        const uint32_t *__restrict__ bstart,
                                                        const uint32_t *__restrict__ big, const Ctl *ctl,
                                                        const uint32_t *__restrict__ count,
                                                        uint32_t *__restrict__ order, uint32_t *__restrict__ rcount) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t *sk = reinterpret_cast<uint64_t *>(s_raw) + (size_t)w * kBig;
    uint32_t *sv = reinterpret_cast<uint32_t *>(s_raw + sizeof(uint64_t) * kBig * kBigWarps) + (size_t)w * kBig;
    const uint32_t nl = ctl->nbig;
    for (uint32_t q = blockIdx.x * kBigWarps + w; q < nl; q += gridDim.x * kBigWarps) {
        const uint32_t b = big[q], s0 = bstart[b], sz = bstart[b + 1] - s0;
        int P = 64;
        while (P < (int)sz) P <<= 1;
        for (int i = lane; i < P; i += 32) {
            uint4 r = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0u);
            if (i < (int)sz) r = rec[s0 + i];
            sk[i] = ((uint64_t)r.y << 32) | r.x;
            sv[i] = r.z;
        }
        __syncwarp();
        for (int kk = 2; kk <= P; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int p = lane; p < P / 2; p += 32) {
                    const int i = 2 * p - (p & (j - 1));   // lower element of the pair
                    const int l = i + j;
                    const bool up = (i & kk) == 0;
                    const uint64_t ki = sk[i], kl = sk[l];
                    const uint32_t vi = sv[i], vl = sv[l];
                    if (before(kl, vl, ki, vi) == up) {
                        sk[i] = kl; sk[l] = ki;
                        sv[i] = vl; sv[l] = vi;
                    }
                }
                __syncwarp();
            }
        }
        for (int i = lane; i < (int)sz; i += 32) {
            order[s0 + i] = sv[i];
            rcount[s0 + i] = count ? count[sv[i]] : 0u;
        }
        __syncwarp();
    }
}

// counts in depth order; rank_offset[r + 1] = sum of the counts of ranks <= r
__global__ void __launch_bounds__(kT) k_count_scan(const uint32_t *__restrict__ rcount, int64_t n, Ctl *ctl,
                                                   unsigned long long *status, uint64_t *__restrict__ rank_offset,
                                                   int64_t *n_instances) {
    __shared__ unsigned long long s_w[kT / 32], s_pre, s_tot;
    __shared__ uint32_t s_tile;
    const int t = threadIdx.x;
    if (t == 0) s_tile = atomicAdd(&ctl->tile_ctr[1], 1u);
    __syncthreads();
    const int64_t tile = s_tile, r0 = tile * kChunk + (int64_t)(t >> 5) * 32 * kIPT + (t & 31);
    unsigned long long c[kIPT];
#pragma unroll
    for (int j = 0; j < kIPT; j++) c[j] = r0 + 32 * j < n ? rcount[r0 + 32 * j] : 0u;
    tile_scan<unsigned long long>(c, status, tile, s_w, &s_pre, &s_tot);
    // rank_offset[r] = exclusive prefix of rank r; [n] = the total
#pragma unroll
    for (int j = 0; j < kIPT; j++)
        if (r0 + 32 * j < n) rank_offset[r0 + 32 * j] = c[j];
    if (tile == num_chunks(n) - 1 && t == 0) {
        rank_offset[n] = s_tot;
        n_instances[0] = (int64_t)s_tot;
        atomicMax(reinterpret_cast<unsigned long long *>(n_instances + 1), s_tot);
    }
}

// Host side: sort (and, with count != nullptr, scan the counts in depth
// order).  keys are not modified.
static inline cudaError_t sort_and_scan(const uint64_t *keys, uint32_t *order, const uint32_t *count,
                                        uint64_t *rank_offset, int64_t *n_instances, int64_t n, void *temp,
                                        cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const Layout L = layout(n);
    const int nbits = bucket_bits(n);
    const int64_t nb = (int64_t)1 << nbits;
    char *tp = (char *)temp;
    Ctl *ctl = (Ctl *)(tp + L.ctl);
    uint32_t *cnt = (uint32_t *)(tp + L.cnt), *bstart = (uint32_t *)(tp + L.bstart);
    unsigned long long *status = (unsigned long long *)(tp + L.status), *csum = (unsigned long long *)(tp + L.csum);
    uint32_t *slot = (uint32_t *)(tp + L.slot), *inv = (uint32_t *)(tp + L.inv), *big = (uint32_t *)(tp + L.big);
    uint4 *rec = (uint4 *)(tp + L.rec);
    uint32_t *rcount = (uint32_t *)(tp + L.rcount);
    cudaError_t e = cudaMemsetAsync(tp, 0, L.zero_end, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(&ctl->kmin, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static DeviceOnce attr_once;       // function attributes are per device
    e = attr_once.run([](int) {
        return cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBigSmem);
    });
    if (e != cudaSuccess) return e;
    const int64_t nc = num_chunks(n);
    const unsigned gm = (unsigned)(nc < (int64_t)sms * 4 ? nc : (int64_t)sms * 4);
    // k_minmax reads only kmin / kmax, the first two fields of both Ctl types
    osort::k_minmax<<<gm, osort::kT, 0, st>>>(keys, n, reinterpret_cast<osort::Ctl *>(ctl));
    k_count<<<(unsigned)nc, kT, 0, st>>>(keys, n, nbits, ctl, cnt, slot, inv);
    k_scan<<<(unsigned)(nb / kChunk), kT, 0, st>>>(cnt, nb, ctl, status, bstart, big);
    k_scatter<<<(unsigned)nc, kT, 0, st>>>(keys, n, nbits, nb, ctl, inv, bstart, slot, count, rec, order, rcount);
    k_rank<<<(unsigned)((n + kT - 1) / kT), kT, 0, st>>>(rec, nbits, ctl, bstart, nb, order, rcount);
    k_big<<<(unsigned)(sms * 2), 32 * kBigWarps, kBigSmem, st>>>(rec, bstart, big, ctl, count, order, rcount);
    if (count) k_count_scan<<<(unsigned)nc, kT, 0, st>>>(rcount, n, ctl, csum, rank_offset, n_instances);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // exact fallback: the cooperative full-width sort, gated on the flag
    return dsort::sort_and_scan(keys, order, count, rank_offset, n_instances, n, tp + L.old, st, &ctl->long_run);
}

}  // namespace bsort
}  // namespace ssg
