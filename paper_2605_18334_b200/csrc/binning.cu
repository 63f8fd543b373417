// binning.cu -- K2-K4: tile binning with bit-exact reference ordering.
//
// Reference: raster/tiles.py:43-79 (bin_arrays).  The reference emits one
// instance per covered tile and lexsorts by (tile, depth, primitive id).
// Here the same order is produced without ever sorting the instances:
//   1. stable radix sort of primitives by their full 64-bit fp64 depth key
//      (equal depths keep primitive-id order)                 -> depth rank
//   2. counts in depth-rank order, single-pass look-back scan -> M
//   3. two-level stable counting scatter of the depth-ordered primitives:
//      tile rows, then the tiles of each row (see below)  -> (tile, depth, id)
// The ranges fall out of step 3 as the exclusive scan of the per-tile counts:
// [start, start + count), empty tiles at the insertion point, i.e. exactly
// np.searchsorted(..., "left"/"right") (tiles.py:76-78).
#include "bucket_sort.cuh"
#include "ssg_common.cuh"

namespace ssg {

// temp = one work area: the depth sort (bin_prepare), then the counting-
// scatter tables (bin_finish).  width < 1 sizes the bin_prepare part only.
struct BinTemp {
    size_t sort_depth, sort_tile, total;
};

static size_t cs_temp_bytes(int64_t n, int64_t capacity, int32_t width, int32_t height);

// steps 1+2: the bucket sort (bucket_sort.cuh); SSG_DEPTH_SORT=1 selects the
// onesweep radix sort instead (A/B builds)
#ifndef SSG_DEPTH_SORT
#define SSG_DEPTH_SORT 0
#endif
static inline size_t depth_sort_temp(int64_t n) {
    return SSG_DEPTH_SORT == 1 ? osort::temp_bytes(n) : bsort::temp_bytes(n);
}
static inline cudaError_t depth_sort(const uint64_t *keys, uint32_t *order, const uint32_t *count,
                                     uint64_t *rank_offset, int64_t *n_instances, int64_t n, void *temp,
                                     cudaStream_t st) {
    if (SSG_DEPTH_SORT == 1) return osort::sort_and_scan(keys, order, count, rank_offset, n_instances, n, temp, st);
    return bsort::sort_and_scan(keys, order, count, rank_offset, n_instances, n, temp, st);
}

static BinTemp bin_temp(int64_t n, int64_t capacity, int32_t width, int32_t height) {
    BinTemp b;
    b.sort_depth = depth_sort_temp(n > 0 ? n : 1);
    b.sort_tile = width < 1 ? 0 : cs_temp_bytes(n, capacity, width, height);
    b.total = b.sort_depth > b.sort_tile ? b.sort_depth : b.sort_tile;
    return b;
}

// ------------------------------------------------------------------------
// Two-level counting scatter (default path for step 3).
//
// Level 1 splits every primitive's tile rectangle into row segments and
// scatters them, stably, into per-row lists (buckets = tile rows); level 2
// scatters each row list, stably, into per-tile lists (buckets = the row's
// tiles).  Both levels are the same stable counting scatter over an ordered
// item stream where each item covers a contiguous bucket range [b0, b1):
//   count    per (chunk of items, bucket) counts            (smem atomics)
//   scan     per bucket over chunks, then over buckets      (-> bases, ranges)
//   scatter  one warp per chunk walks its items in order, 32 per step; the
//            lanes of a step rank themselves inside each bucket by an
//            atomicOr lane mask (rank = popcount of lower lanes), the lowest
//            lane advances the warp's per-bucket cursor.
// Bucket counts per level are <= 4096 (rows or tiles of one row), so each
// warp's cursors and masks live in shared memory and every item costs a few
// instructions per covered bucket -- no instance sort.
#ifndef SSG_CS_C1
#define SSG_CS_C1 256
#endif
#ifndef SSG_CS_C2
#define SSG_CS_C2 256
#endif
#ifndef SSG_CS_STAGE
#define SSG_CS_STAGE 1024
#endif
constexpr int kCsWarps = 4;                  // chunk workers per CTA
constexpr int kCsC1 = SSG_CS_C1;             // primitives per level-1 chunk
constexpr int kCsC2 = SSG_CS_C2;             // row segments per level-2 chunk
constexpr int kCsStage = SSG_CS_STAGE;       // staged outputs per warp (coalesced flush)

struct CsLayout {
    int64_t nch1;                            // level-1 chunks
    int64_t max_ch2;                         // bound on level-2 chunks
    size_t cnt1, row_total, row_start, chunk_base, ctl, cnt2, tile_total, tile_start, rowlist, total;
};

static CsLayout cs_layout(int64_t n, int64_t capacity, int32_t ntx, int32_t nty) {
    CsLayout L;
    L.nch1 = (n + kCsC1 - 1) / kCsC1;
    if (L.nch1 < 1) L.nch1 = 1;
    const int64_t cap = capacity > 0 ? capacity : 1;
    L.max_ch2 = cap / kCsC2 + nty + 1;
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o += radix::align256(bytes); return at; };
    L.cnt1 = take(sizeof(uint32_t) * (size_t)nty * L.nch1);
    L.row_total = take(sizeof(uint32_t) * (size_t)(nty + 1));
    L.row_start = take(sizeof(uint32_t) * (size_t)(nty + 1));
    L.chunk_base = take(sizeof(uint32_t) * (size_t)(nty + 1));
    L.ctl = take(sizeof(uint32_t) * 4);
    L.cnt2 = take(sizeof(uint32_t) * (size_t)ntx * L.max_ch2);
    L.tile_total = take(sizeof(uint32_t) * (size_t)ntx * nty);
    L.tile_start = take(sizeof(uint32_t) * (size_t)ntx * nty);
    L.rowlist = take(sizeof(uint64_t) * (size_t)cap);
    L.total = o;
    return L;
}

static size_t cs_temp_bytes(int64_t n, int64_t capacity, int32_t width, int32_t height) {
    const int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    return cs_layout(n, capacity, ntx, nty).total;
}

// shared memory per scatter warp: staging (u64 / u32 payload + u16 bucket)
// then two u32 arrays over the buckets (cursor, flush delta)
template <typename P>
__host__ __device__ constexpr size_t cs_stage_bytes() { return (sizeof(P) + sizeof(uint16_t)) * kCsStage; }
template <typename P>
__host__ __device__ inline size_t cs_warp_smem(int nb) { return cs_stage_bytes<P>() + 8 * (size_t)nb; }

__device__ __forceinline__ void rect_unpack(uint64_t rc, int &x0, int &x1, int &y0, int &y1) {
    x0 = (int)(rc & 0xffff);
    x1 = (int)((rc >> 16) & 0xffff);
    y0 = (int)((rc >> 32) & 0xffff);
    y1 = (int)(rc >> 48);
}

// Warp-wide exclusive scan, in place, of a[0, len) (sequential 32-wide blocks).
__device__ __forceinline__ uint32_t warp_exclusive_scan(uint32_t *a, int len, int lane) {
    uint32_t carry = 0;
    for (int b = 0; b < len; b += 32) {
        const int i = b + lane;
        const uint32_t v = i < len ? a[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        if (i < len) a[i] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    return carry;
}

// Lanes holding the same bucket b (NB low bits), from NB ballots.  Not
// __match_any_sync: MATCH.ANY issues on the ADU pipe, which saturates at a
// small fraction of the issue rate on sm_100 (ncu: adu 59 % of cycles in
// this kernel with it, profiles/r2_binning.md).  Lanes with v == false
// belong to no set.
template <int NB>
__device__ __forceinline__ uint32_t lane_peers(uint32_t b, bool v) {
    uint32_t m = __ballot_sync(0xffffffffu, v);
#pragma unroll
    for (int k = 0; k < NB; k++) {
        const uint32_t bb = __ballot_sync(0xffffffffu, (b >> k) & 1u);
        m &= ((b >> k) & 1u) ? bb : ~bb;
    }
    return m;
}

// bits of the largest bucket index (buckets < 4096 per level)
static inline int bucket_bits(int nb) {
    int k = 1;
    while ((1 << k) < nb) k++;
    return k;
}

// Ordered walk of one warp's items [i0, i1): each item covers buckets
// [b0, b1) and carries a payload.  Items are expanded 32 instances per step
// (item-major, bucket-minor: the output order); equal buckets inside a step
// are ranked by lane (lane_peers), across steps by the warp's cursors scur[].
template <int NB, typename P, typename Load, typename Emit>
__device__ __forceinline__ void cs_walk(int64_t i0, int64_t i1, int lane, uint32_t *scur, Load &&load, Emit &&emit) {
    const uint32_t lt = radix::lanemask_lt();
    for (int64_t a = i0; a < i1; a += 32) {
        const int64_t i = a + lane;
        int b0 = 0, b1 = 0;
        P pay = 0;
        if (i < i1) load(i, b0, b1, pay);
        const uint32_t len = (uint32_t)(b1 - b0);
        uint32_t inc = len;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += y;
        }
        const uint32_t pre = inc - len, tot = __shfl_sync(0xffffffffu, inc, 31);
        for (uint32_t g0 = 0; g0 < tot; g0 += 32) {
            const uint32_t g = g0 + lane;
            int j = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
                if (__shfl_sync(0xffffffffu, pre, j + step) <= g) j += step;
            const uint32_t pj = __shfl_sync(0xffffffffu, pre, j);
            const int bj = __shfl_sync(0xffffffffu, b0, j);
            P payj;
            if constexpr (sizeof(P) == 8) {
                const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)pay, j);
                const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)((uint64_t)pay >> 32), j);
                payj = (P)(((uint64_t)hi << 32) | lo);
            } else {
                payj = __shfl_sync(0xffffffffu, pay, j);
            }
            const bool v = g < tot;
            const int b = bj + (int)(g - pj);
            const uint32_t peers = lane_peers<NB>((uint32_t)b, v);
            const uint32_t base = v ? scur[b] : 0u;
            __syncwarp();
            if (v && (peers & lt) == 0) scur[b] = base + (uint32_t)__popc(peers);
            __syncwarp();
            if (v) emit(b, base + (uint32_t)__popc(peers & lt), payj);
        }
    }
}

// Per-chunk cursor setup shared by both scatters.  count_of(b) = the chunk's
// items in bucket b, gbase_of(b) = its first global output position.  The
// chunk's outputs are staged in shared memory (bucket-major) when they fit
// and flushed in coalesced runs; otherwise written in place.
// Returns the chunk's output count; staged iff it is <= kCsStage.
template <typename CountOf, typename GbaseOf>
__device__ __forceinline__ uint32_t cs_setup(uint32_t *scur, uint32_t *delta, int nb, int lane, CountOf &&count_of,
                                             GbaseOf &&gbase_of) {
    for (int b = lane; b < nb; b += 32) scur[b] = count_of(b);
    __syncwarp();
    const uint32_t total = warp_exclusive_scan(scur, nb, lane);  // local starts
    const bool staged = total <= (uint32_t)kCsStage;
    for (int b = lane; b < nb; b += 32) {
        const uint32_t g = gbase_of(b), l = scur[b];
        delta[b] = g - l;
        if (!staged) scur[b] = g;
    }
    __syncwarp();
    return total;
}

// level 1, count (difference array over rows): cnt1[row][chunk]
__global__ void __launch_bounds__(32 * kCsWarps) k_cs1_count(const uint32_t *__restrict__ order,
                                                             const uint32_t *__restrict__ count,
                                                             const uint64_t *__restrict__ rect, int64_t n,
                                                             int64_t nch1, int32_t nty, uint32_t *__restrict__ cnt1) {
    extern __shared__ uint32_t s_cs[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t *h = s_cs + (size_t)w * (nty + 1);
    const int64_t c = (int64_t)blockIdx.x * kCsWarps + w;
    if (c >= nch1) return;
    for (int y = lane; y <= nty; y += 32) h[y] = 0;
    __syncwarp();
    const int64_t r1 = min(n, (c + 1) * kCsC1);
    for (int64_t r = c * kCsC1 + lane; r < r1; r += 32) {
        const uint32_t p = order[r];
        if (count[p] == 0) continue;
        int x0, x1, y0, y1;
        rect_unpack(rect[p], x0, x1, y0, y1);
        atomicAdd(&h[y0], 1u);
        atomicAdd(&h[y1], 0xffffffffu);
    }
    __syncwarp();
    uint32_t carry = 0;
    for (int b = 0; b < nty; b += 32) {
        const int y = b + lane;
        uint32_t x = y < nty ? h[y] : 0u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += u;
        }
        if (y < nty) cnt1[(size_t)y * nch1 + c] = carry + x;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

// Exclusive scan with one CTA of 1024 threads, each owning a contiguous run
// (read twice): src -> dst (may alias); returns the total.
__device__ __forceinline__ uint32_t cta_scan_runs(const uint32_t *src, uint32_t *dst, int len, uint32_t *s_warp) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int per = (len + 1023) / 1024;
    const int lo = min(len, t * per), hi = min(len, lo + per);
    uint32_t sum = 0;
    for (int q = lo; q < hi; q++) sum += src[q];
    uint32_t x = sum;
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
    uint32_t run = (w > 0 ? s_warp[w - 1] : 0u) + x - sum;
    const uint32_t total = s_warp[31];
    for (int q = lo; q < hi; q++) {
        const uint32_t v = src[q];
        dst[q] = run;
        run += v;
    }
    return total;
}

// level 1, per-row scan over chunks (one CTA of 1024 threads per row, each
// thread a contiguous run: one pass, no per-256 loop of barriers)
__global__ void __launch_bounds__(1024) k_cs1_rowscan(uint32_t *__restrict__ cnt1, int64_t nch1,
                                                      uint32_t *__restrict__ row_total) {
    __shared__ uint32_t s_warp[32];
    uint32_t *row = cnt1 + (size_t)blockIdx.x * nch1;
    const uint32_t tot = cta_scan_runs(row, row, (int)nch1, s_warp);
    if (threadIdx.x == 0) row_total[blockIdx.x] = tot;
}

// one CTA: row starts (exclusive scan of row totals) and level-2 chunk bases
// (exclusive scan of ceil(total / C2)); ctl[0] = number of level-2 chunks
// A sync-free frame (ssg_bin_finish with m < 0) may find more instances than
// the buffers hold: chunk bases are clamped to max_ch2 so no table is
// overrun (the caller detects the overflow as n_instances > capacity).
__global__ void __launch_bounds__(1024) k_cs1_rowstart(const uint32_t *__restrict__ row_total, int32_t nty,
                                                       uint32_t max_ch2, uint32_t *__restrict__ row_start,
                                                       uint32_t *__restrict__ chunk_base, uint32_t *__restrict__ ctl) {
    __shared__ uint32_t s_warp[32];
    for (int y = threadIdx.x; y < nty; y += blockDim.x) chunk_base[y] = (row_total[y] + kCsC2 - 1) / kCsC2;
    __syncthreads();
    const uint32_t rt = cta_scan_runs(row_total, row_start, nty, s_warp);
    __syncthreads();
    const uint32_t ct = cta_scan_runs(chunk_base, chunk_base, nty, s_warp);
    __syncthreads();
    for (int y = threadIdx.x; y < nty; y += blockDim.x) chunk_base[y] = min(chunk_base[y], max_ch2);
    if (threadIdx.x == 0) {
        row_start[nty] = rt;
        chunk_base[nty] = min(ct, max_ch2);
        ctl[0] = min(ct, max_ch2);
    }
}

// level 1, scatter: row segments (prim | x0 << 32 | x1 << 48) into per-row lists
template <int NB>
__global__ void __launch_bounds__(32 * kCsWarps) k_cs1_scatter(const uint32_t *__restrict__ order,
                                                               const uint32_t *__restrict__ count,
                                                               const uint64_t *__restrict__ rect, int64_t n,
                                                               int64_t nch1, int32_t nty,
                                                               const uint32_t *__restrict__ cnt1,
                                                               const uint32_t *__restrict__ row_total,
                                                               const uint32_t *__restrict__ row_start,
                                                               uint64_t *__restrict__ rowlist, uint32_t cap) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char *base = s_raw + (size_t)w * cs_warp_smem<uint64_t>(nty);
    uint64_t *st_pay = reinterpret_cast<uint64_t *>(base);
    uint16_t *st_b = reinterpret_cast<uint16_t *>(base + sizeof(uint64_t) * kCsStage);
    uint32_t *scur = reinterpret_cast<uint32_t *>(base + cs_stage_bytes<uint64_t>()), *delta = scur + nty;
    const int64_t c = (int64_t)blockIdx.x * kCsWarps + w;
    if (c >= nch1) return;
    const uint32_t total = cs_setup(
        scur, delta, nty, lane,
        [&](int y) {
            const uint32_t e = c + 1 < nch1 ? cnt1[(size_t)y * nch1 + c + 1] : row_total[y];
            return e - cnt1[(size_t)y * nch1 + c];
        },
        [&](int y) { return row_start[y] + cnt1[(size_t)y * nch1 + c]; });
    const bool staged = total <= (uint32_t)kCsStage;
    const int64_t r1 = min(n, (c + 1) * kCsC1);
    cs_walk<NB, uint64_t>(
        c * kCsC1, r1, lane, scur,
        [&](int64_t r, int &b0, int &b1, uint64_t &pay) {
            const uint32_t p = order[r];
            if (count[p] == 0) return;
            int x0, x1;
            rect_unpack(rect[p], x0, x1, b0, b1);
            pay = (uint64_t)p | ((uint64_t)x0 << 32) | ((uint64_t)x1 << 48);
        },
        [&](int y, uint32_t pos, uint64_t pay) {
            if (staged) {
                st_pay[pos] = pay;
                st_b[pos] = (uint16_t)y;
            } else if (pos < cap) {
                rowlist[pos] = pay;
            }
        });
    if (staged) {  // bucket-major local order: runs of one row are contiguous in rowlist
        __syncwarp();
        for (uint32_t i = lane; i < total; i += 32) {
            const uint32_t pos = delta[st_b[i]] + i;
            if (pos < cap) rowlist[pos] = st_pay[i];
        }
    }
}

// level-2 chunk id -> row by binary search of chunk_base
__device__ __forceinline__ int cs2_row_of(const uint32_t *__restrict__ chunk_base, int32_t nty, uint32_t c) {
    int lo = 0, hi = nty;  // chunk_base[lo] <= c < chunk_base[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (chunk_base[mid] <= c) lo = mid; else hi = mid;
    }
    return lo;
}

// level 2, count (difference array over the row's tiles): cnt2 block of row y
// laid out [x][k] (tile-major, chunk-minor)
__global__ void __launch_bounds__(32 * kCsWarps) k_cs2_count(const uint64_t *__restrict__ rowlist,
                                                             const uint32_t *__restrict__ row_start,
                                                             const uint32_t *__restrict__ chunk_base,
                                                             const uint32_t *__restrict__ ctl, int32_t ntx,
                                                             int32_t nty, uint32_t *__restrict__ cnt2, uint32_t cap) {
    extern __shared__ uint32_t s_cs[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t *h = s_cs + (size_t)w * (ntx + 1);
    const uint32_t nch2 = ctl[0];
    for (uint32_t c = blockIdx.x * kCsWarps + w; c < nch2; c += gridDim.x * kCsWarps) {
        const int y = cs2_row_of(chunk_base, nty, c);
        const uint32_t k = c - chunk_base[y], nk = chunk_base[y + 1] - chunk_base[y];
        for (int x = lane; x <= ntx; x += 32) h[x] = 0;
        __syncwarp();
        const uint32_t i0 = row_start[y] + k * kCsC2, i1 = min(min(row_start[y + 1], i0 + kCsC2), cap);
        for (uint32_t i = i0 + lane; i < i1; i += 32) {
            const uint64_t seg = rowlist[i];
            atomicAdd(&h[(int)((seg >> 32) & 0xffff)], 1u);
            atomicAdd(&h[(int)(seg >> 48)], 0xffffffffu);
        }
        __syncwarp();
        uint32_t *blk = cnt2 + (size_t)chunk_base[y] * ntx;
        uint32_t carry = 0;
        for (int b = 0; b < ntx; b += 32) {
            const int x = b + lane;
            uint32_t v = x < ntx ? h[x] : 0u;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += u;
            }
            if (x < ntx) blk[(size_t)x * nk + k] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
        __syncwarp();
    }
}

// level 2, per-tile exclusive scan over the row's chunks (one warp per tile)
__global__ void __launch_bounds__(256) k_cs2_tilescan(uint32_t *__restrict__ cnt2,
                                                      const uint32_t *__restrict__ chunk_base, int32_t ntx,
                                                      int32_t nty, uint32_t *__restrict__ tile_total) {
    const int lane = threadIdx.x & 31;
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= (int64_t)ntx * nty) return;
    const int y = (int)(t / ntx), x = (int)(t - (int64_t)y * ntx);
    const uint32_t nk = chunk_base[y + 1] - chunk_base[y];
    uint32_t *a = cnt2 + (size_t)chunk_base[y] * ntx + (size_t)x * nk;
    uint32_t carry = 0;
    for (uint32_t k0 = 0; k0 < nk; k0 += 32) {
        const uint32_t k = k0 + lane;
        const uint32_t v = k < nk ? a[k] : 0u;
        uint32_t s = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += u;
        }
        if (k < nk) a[k] = carry + s - v;
        carry += __shfl_sync(0xffffffffu, s, 31);
    }
    if (lane == 0) tile_total[t] = carry;
}

// one CTA: tile starts (exclusive scan of the totals) and ranges
// [start, start + total): empty tiles sit at the insertion point, exactly
// np.searchsorted left/right (tiles.py:76-78)
__global__ void __launch_bounds__(1024) k_cs2_tilestart(const uint32_t *__restrict__ tile_total, int32_t n_tiles,
                                                        uint32_t cap, uint32_t *__restrict__ tile_start,
                                                        int32_t *__restrict__ ranges) {
    __shared__ uint32_t s_warp[32];
    cta_scan_runs(tile_total, tile_start, n_tiles, s_warp);
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint32_t st = tile_start[t];
        // clamped to the capacity: an overflowing sync-free frame never reads past it
        ranges[2 * t] = (int32_t)min(st, cap);
        ranges[2 * t + 1] = (int32_t)min(st + tile_total[t], cap);
    }
}

// level 2, scatter: per-tile instance lists (inst_prim, inst_tile)
template <int NB>
__global__ void __launch_bounds__(32 * kCsWarps) k_cs2_scatter(const uint64_t *__restrict__ rowlist,
                                                               const uint32_t *__restrict__ row_start,
                                                               const uint32_t *__restrict__ chunk_base,
                                                               const uint32_t *__restrict__ ctl,
                                                               const uint32_t *__restrict__ cnt2,
                                                               const uint32_t *__restrict__ tile_total,
                                                               const uint32_t *__restrict__ tile_start,
                                                               int32_t ntx, int32_t nty,
                                                               uint32_t *__restrict__ inst_prim,
                                                               uint32_t *__restrict__ inst_tile, uint32_t cap) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char *base = s_raw + (size_t)w * cs_warp_smem<uint32_t>(ntx);
    uint32_t *st_pay = reinterpret_cast<uint32_t *>(base);
    uint16_t *st_b = reinterpret_cast<uint16_t *>(base + sizeof(uint32_t) * kCsStage);
    uint32_t *scur = reinterpret_cast<uint32_t *>(base + cs_stage_bytes<uint32_t>()), *delta = scur + ntx;
    const uint32_t nch2 = ctl[0];
    for (uint32_t c = blockIdx.x * kCsWarps + w; c < nch2; c += gridDim.x * kCsWarps) {
        const int y = cs2_row_of(chunk_base, nty, c);
        const uint32_t k = c - chunk_base[y], nk = chunk_base[y + 1] - chunk_base[y];
        const uint32_t *blk = cnt2 + (size_t)chunk_base[y] * ntx;
        const uint32_t trow = (uint32_t)y * (uint32_t)ntx;
        const uint32_t total = cs_setup(
            scur, delta, ntx, lane,
            [&](int x) {
                const uint32_t e = k + 1 < nk ? blk[(size_t)x * nk + k + 1] : tile_total[trow + x];
                return e - blk[(size_t)x * nk + k];
            },
            [&](int x) { return tile_start[trow + x] + blk[(size_t)x * nk + k]; });
        const bool staged = total <= (uint32_t)kCsStage;
        const uint32_t i0 = row_start[y] + k * kCsC2, i1 = min(min(row_start[y + 1], i0 + kCsC2), cap);
        cs_walk<NB, uint32_t>(
            i0, i1, lane, scur,
            [&](int64_t i, int &b0, int &b1, uint32_t &pay) {
                const uint64_t seg = rowlist[i];
                pay = (uint32_t)seg;
                b0 = (int)((seg >> 32) & 0xffff);
                b1 = (int)(seg >> 48);
            },
            [&](int x, uint32_t pos, uint32_t p) {
                if (staged) {
                    st_pay[pos] = p;
                    st_b[pos] = (uint16_t)x;
                } else if (pos < cap) {
                    inst_prim[pos] = p;
                    if (inst_tile) inst_tile[pos] = trow + (uint32_t)x;
                }
            });
        if (staged) {
            __syncwarp();
            for (uint32_t i = lane; i < total; i += 32) {
                const int x = st_b[i];
                const uint32_t pos = delta[x] + i;
                if (pos >= cap) continue;
                inst_prim[pos] = st_pay[i];
                if (inst_tile) inst_tile[pos] = trow + (uint32_t)x;
            }
        }
        __syncwarp();
    }
}

// Binning from caller-provided screen arrays (tiles.py:43-57 inputs), used by
// the bin_arrays mirror: rect, count and depth key per primitive.
__global__ void k_rects_from_arrays(int64_t n, const double *mean2d, const double *radius,
                                    const double *depth, const uint8_t *valid, int ntx, int nty,
                                    uint32_t *count, uint64_t *rect, uint64_t *key) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t rc;
    bool v = valid[i] != 0;
    count[i] = tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], v, ntx, nty, rc);
    rect[i] = rc;
    // order-preserving bits for any finite double (sign flip for negatives);
    // the all-ones pattern is reserved for primitives without instances
    uint64_t b = (uint64_t)__double_as_longlong(depth[i] == 0.0 ? 0.0 : depth[i]);
    uint64_t kk = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    key[i] = count[i] ? (kk == ~0ull ? kk - 1 : kk) : ~0ull;
}

}  // namespace ssg

extern "C" int ssg_bin_rects(int64_t n, const double *mean2d, const double *radius,
                             const double *depth, const uint8_t *valid, int32_t width,
                             int32_t height, const ssg_prim_buffers *out, void *stream) {
    using namespace ssg;
    if (!out || n < 0 || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    if (n == 0) return SSG_OK;
    int ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    k_rects_from_arrays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n, mean2d, radius, depth, valid, ntx, nty, out->tile_count, out->tile_rect, out->depth_key);
    return check_launch("k_rects_from_arrays");
}

extern "C" int ssg_bin_temp_bytes(int64_t n, int64_t capacity, int32_t width, int32_t height, size_t *bytes) {
    using namespace ssg;
    if (!bytes || n < 0 || capacity < 0 || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    *bytes = bin_temp(n, capacity, width, height).total;
    return SSG_OK;
}

extern "C" int ssg_bin_prepare(int64_t n, const ssg_prim_buffers *prim, const ssg_bin_buffers *bins,
                               void *stream) {
    using namespace ssg;
    if (!prim || !bins || n < 0 || n >= (int64_t)UINT32_MAX) return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(bins->n_instances, 0, sizeof(int64_t), st);  // [1] (max) unchanged
        if (e == cudaSuccess) e = cudaMemsetAsync(bins->rank_offset, 0, sizeof(uint64_t), st);
        if (e != cudaSuccess) { set_error("memset", e); return SSG_ERR_CUDA; }
        return SSG_OK;
    }
    const BinTemp L = bin_temp(n, bins->capacity, 0, 0);
    if (bins->temp_bytes < L.total) return SSG_ERR_CAPACITY;
    // 1+2. stable sort of the ids by depth key, counts in depth order, scan
    cudaError_t e = depth_sort(prim->depth_key, bins->depth_order, prim->tile_count, bins->rank_offset,
                               bins->n_instances, n, bins->temp, (cudaStream_t)stream);
    if (e != cudaSuccess) { set_error("depth sort", e); return SSG_ERR_CUDA; }
    return check_launch("ssg_bin_prepare");
}

#define CS_KERNELS(K)                                                                                       \
    (const void *)K<1>, (const void *)K<2>, (const void *)K<3>, (const void *)K<4>, (const void *)K<5>,         \
        (const void *)K<6>, (const void *)K<7>, (const void *)K<8>, (const void *)K<9>, (const void *)K<10>,    \
        (const void *)K<11>, (const void *)K<12>

extern "C" int ssg_bin_finish(int64_t n, int64_t m, int32_t width, int32_t height,
                              const ssg_prim_buffers *prim, const ssg_bin_buffers *bins, void *stream) {
    using namespace ssg;
    if (!prim || !bins || n < 0 || width < 1 || height < 1) return SSG_ERR_INVALID_ARGUMENT;
    // m < 0: sync-free frame, M not read back; the kernels stay inside the
    // capacity and the caller checks n_instances <= capacity afterwards
    if (m > bins->capacity || m >= (int64_t)INT32_MAX || bins->capacity >= (int64_t)UINT32_MAX)
        return SSG_ERR_CAPACITY;
    if (width > SSG_MAX_IMAGE_DIM || height > SSG_MAX_IMAGE_DIM) return SSG_ERR_DIM_OVERFLOW;
    const int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    const int32_t n_tiles = ntx * nty;
    cudaStream_t st = (cudaStream_t)stream;
    const BinTemp T = bin_temp(n, bins->capacity, width, height);
    if (bins->temp_bytes < T.total) return SSG_ERR_CAPACITY;
    char *work = (char *)bins->temp;
    const CsLayout L = cs_layout(n, bins->capacity, ntx, nty);
    uint32_t *cnt1 = (uint32_t *)(work + L.cnt1), *row_total = (uint32_t *)(work + L.row_total);
    uint32_t *row_start = (uint32_t *)(work + L.row_start), *chunk_base = (uint32_t *)(work + L.chunk_base);
    uint32_t *ctl = (uint32_t *)(work + L.ctl), *cnt2 = (uint32_t *)(work + L.cnt2);
    uint32_t *tile_total = (uint32_t *)(work + L.tile_total);
    uint64_t *rowlist = (uint64_t *)(work + L.rowlist);
    uint32_t *tile_start = (uint32_t *)(work + L.tile_start);
    const size_t sm1 = kCsWarps * cs_warp_smem<uint64_t>(nty), sm2 = kCsWarps * cs_warp_smem<uint32_t>(ntx);
    const size_t smc1 = sizeof(uint32_t) * kCsWarps * (nty + 1), smc2 = sizeof(uint32_t) * kCsWarps * (ntx + 1);
    // the largest grids (4096 tiles per side) need > 48 KB; function
    // attributes are per device, so the one-time setup is per device ordinal
    static DeviceOnce attr_once;
    int sms = 148, dev = 0;
    {
        cudaError_t e = attr_once.run([](int) {
            const int mx = (int)(kCsWarps * cs_warp_smem<uint64_t>(4096));
            const void *fs[] = {CS_KERNELS(k_cs1_scatter), CS_KERNELS(k_cs2_scatter), (const void *)k_cs1_count,
                                (const void *)k_cs2_count};
            cudaError_t r = cudaSuccess;
            for (const void *f : fs)
                if (r == cudaSuccess) r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            return r;
        });
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e != cudaSuccess) { set_error("cudaFuncSetAttribute(binning)", e); return SSG_ERR_CUDA; }
    }
    const unsigned g1 = (unsigned)((L.nch1 + kCsWarps - 1) / kCsWarps);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g2 = (unsigned)(sms * 8);
    // level 1: row segments in per-row lists
    k_cs1_count<<<g1, 32 * kCsWarps, smc1, st>>>(bins->depth_order, prim->tile_count, prim->tile_rect, n, L.nch1,
                                                 nty, cnt1);
    k_cs1_rowscan<<<nty, 1024, 0, st>>>(cnt1, L.nch1, row_total);
    const uint32_t cap = (uint32_t)(bins->capacity > 0 ? bins->capacity : 0);
    k_cs1_rowstart<<<1, 1024, 0, st>>>(row_total, nty, (uint32_t)L.max_ch2, row_start, chunk_base, ctl);
    if (n > 0)
        switch (bucket_bits(nty)) {
#define SSG_CS1(B)                                                                                              \
    case B:                                                                                                     \
        k_cs1_scatter<B><<<g1, 32 * kCsWarps, sm1, st>>>(bins->depth_order, prim->tile_count, prim->tile_rect, \
                                                         n, L.nch1, nty, cnt1, row_total, row_start, rowlist, cap); \
        break;
            SSG_CS1(1) SSG_CS1(2) SSG_CS1(3) SSG_CS1(4) SSG_CS1(5) SSG_CS1(6) SSG_CS1(7) SSG_CS1(8) SSG_CS1(9)
            SSG_CS1(10) SSG_CS1(11) SSG_CS1(12)
#undef SSG_CS1
            default: return SSG_ERR_INVALID_ARGUMENT;
        }
    // level 2: per-tile lists of each row
    k_cs2_count<<<g2, 32 * kCsWarps, smc2, st>>>(rowlist, row_start, chunk_base, ctl, ntx, nty, cnt2, cap);
    k_cs2_tilescan<<<(unsigned)(((int64_t)n_tiles * 32 + 255) / 256), 256, 0, st>>>(cnt2, chunk_base, ntx, nty,
                                                                                    tile_total);
    k_cs2_tilestart<<<1, 1024, 0, st>>>(tile_total, n_tiles, cap, tile_start, bins->ranges);
    switch (bucket_bits(ntx)) {
#define SSG_CS2(B)                                                                                              \
    case B:                                                                                                     \
        k_cs2_scatter<B><<<g2, 32 * kCsWarps, sm2, st>>>(rowlist, row_start, chunk_base, ctl, cnt2, tile_total, \
                                                         tile_start, ntx, nty, bins->inst_prim, bins->inst_tile,  \
                                                         cap);                                                   \
        break;
        SSG_CS2(1) SSG_CS2(2) SSG_CS2(3) SSG_CS2(4) SSG_CS2(5) SSG_CS2(6) SSG_CS2(7) SSG_CS2(8) SSG_CS2(9)
        SSG_CS2(10) SSG_CS2(11) SSG_CS2(12)
#undef SSG_CS2
        default: return SSG_ERR_INVALID_ARGUMENT;
    }
    return check_launch("ssg_bin_finish");
}

// ---- test hooks (tests/ only): the depth sort in isolation ---------------
extern "C" size_t ssg_test_sort_temp_bytes(int64_t n, int key_bytes) {
    using namespace ssg;
    return key_bytes == 8 ? depth_sort_temp(n) : 0;
}

// stable sort of u64 keys (not modified): vals <- ids in sorted order
extern "C" int ssg_test_sort(void *keys, uint32_t *vals, int key_bytes, int iota, int64_t n, int npass,
                             void *temp, void *stream) {
    using namespace ssg;
    if (key_bytes != 8 || !iota || npass != 8) return SSG_ERR_INVALID_ARGUMENT;
    cudaError_t e = depth_sort((const uint64_t *)keys, vals, nullptr, nullptr, nullptr, n, temp, (cudaStream_t)stream);
    if (e != cudaSuccess) { set_error("test sort", e); return SSG_ERR_CUDA; }
    return SSG_OK;
}
