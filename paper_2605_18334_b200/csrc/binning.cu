// binning.cu -- K2-K4: tile binning with bit-exact reference ordering.
//
// Reference: raster/tiles.py:43-79 (bin_arrays).  The reference emits one
// instance per covered tile and lexsorts by (tile, depth, primitive id).
// Here the same order is produced in two stable stages, all hand-written:
//   1. stable radix sort of primitives by their full 64-bit fp64 depth key
//      (equal depths keep primitive-id order)            -> depth rank
//   2. counts in depth-rank order, single-pass look-back scan -> offsets
//   3. warp-cooperative duplication (coalesced writes) of each primitive's
//      tiles in depth-rank order, then a stable radix sort of the instances
//      by tile id (13-16 bit key, two passes)          -> (tile, depth, id)
// Ranges are the per-tile [first, last+1) of the sorted tile ids with empty
// tiles set to the insertion point, i.e. exactly np.searchsorted(...,
// "left"/"right") (tiles.py:76-78).
#include "radix_sort.cuh"
#include "ssg_common.cuh"

namespace ssg {

static int tile_passes(int32_t n_tiles) {
    int b = 1;
    while ((1 << b) < n_tiles) b++;
    return (b + 7) / 8;
}

constexpr int kScanThreads = 256, kScanIPT = 16, kScanTile = kScanThreads * kScanIPT;

struct BinTemp {
    size_t sort_depth, sort_tile, scan_lookback, total;
};

static BinTemp bin_temp(int64_t n, int64_t capacity) {
    BinTemp b;
    b.sort_depth = radix::temp_bytes<uint64_t>(n > 0 ? n : 1);
    b.sort_tile = radix::temp_bytes<uint16_t>(capacity > 0 ? capacity : 1);
    b.scan_lookback = radix::align256(sizeof(uint64_t) * (size_t)((n + kScanTile - 1) / kScanTile + 1) + 256);
    size_t m = b.sort_depth > b.sort_tile ? b.sort_depth : b.sort_tile;
    b.total = m + b.scan_lookback;
    return b;
}

// Counts in depth order + inclusive scan in one pass (decoupled look-back).
// rank_offset[r+1] = sum of counts of ranks <= r; rank_offset[0] = 0.
__global__ void __launch_bounds__(kScanThreads)
k_scan_counts(const uint32_t *__restrict__ order, const uint32_t *__restrict__ count, int64_t n,
              uint64_t *__restrict__ rank_offset, uint64_t *__restrict__ lookback, int64_t *n_instances) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_warp[kScanThreads / 32];
    __shared__ uint64_t s_prefix;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t *counter = reinterpret_cast<uint32_t *>(lookback + (n + kScanTile - 1) / kScanTile);
    if (t == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)t * kScanIPT;
    uint64_t v[kScanIPT];
    uint64_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; i++) {
        const int64_t r = base + i;
        v[i] = r < n ? count[order[r]] : 0u;
        sum += v[i];
    }
    // block exclusive scan of the per-thread sums
    uint64_t x = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    uint64_t wpre = 0, total = 0;
#pragma unroll
    for (int ww = 0; ww < kScanThreads / 32; ww++) {
        wpre += ww < w ? s_warp[ww] : 0ull;
        total += s_warp[ww];
    }
    if (t == 0) {
        uint64_t excl = 0;
        if (tile == 0) {
            atomicExch(reinterpret_cast<unsigned long long *>(lookback), radix::kFlagPre | total);
        } else {
            atomicExch(reinterpret_cast<unsigned long long *>(lookback + tile), radix::kFlagAgg | total);
            for (int64_t p = tile - 1;; p--) {
                const volatile uint64_t *q = lookback + p;
                uint64_t val = *q;
                while ((val >> 62) == 0) val = *q;
                excl += val & radix::kValMask;
                if ((val >> 62) == 2) break;
            }
            atomicExch(reinterpret_cast<unsigned long long *>(lookback + tile), radix::kFlagPre | (excl + total));
        }
        s_prefix = excl;
        if (base <= n && tile == (n - 1) / kScanTile) *n_instances = (int64_t)(excl + total);
        if (tile == 0) rank_offset[0] = 0;
    }
    __syncthreads();
    uint64_t run = s_prefix + wpre + x - sum;
#pragma unroll
    for (int i = 0; i < kScanIPT; i++) {
        const int64_t r = base + i;
        run += v[i];
        if (r < n) rank_offset[r + 1] = run;
    }
}

// tiles.py:59-70: each primitive's instances in row-major tile order, in
// depth-rank order.  A warp owns 32 consecutive ranks, whose instances are
// contiguous in the output; lanes stride over that span (coalesced stores)
// and find their primitive by a 5-step shuffle binary search.
__global__ void __launch_bounds__(256)
k_duplicate(const uint32_t *__restrict__ order, const uint64_t *__restrict__ rank_offset,
            const uint64_t *__restrict__ rect, int32_t ntx, int64_t n, uint16_t *__restrict__ inst_tile,
            uint32_t *__restrict__ inst_prim) {
    const int lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
    if (r0 >= n) return;
    const int64_t r = r0 + lane;
    const uint64_t off = rank_offset[r < n ? r : n];
    const uint64_t end = __shfl_sync(0xffffffffu, rank_offset[r0 + 32 < n ? r0 + 32 : n], 0);
    uint32_t prim = 0;
    uint64_t rc = 0;
    if (r < n) {
        prim = order[r];
        const uint64_t nxt = rank_offset[r + 1];
        if (nxt > off) rc = rect[prim];
    }
    const uint64_t first = __shfl_sync(0xffffffffu, off, 0);
    const uint32_t rlo = (uint32_t)rc, rhi = (uint32_t)(rc >> 32);
    for (uint64_t g0 = first; g0 < end; g0 += 32) {  // warp-uniform trip count (shuffles below)
        const uint64_t g = g0 + lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint64_t oc = __shfl_sync(0xffffffffu, off, j + step);
            if (oc <= g) j += step;
        }
        const uint64_t oj = __shfl_sync(0xffffffffu, off, j);
        const uint32_t lo = __shfl_sync(0xffffffffu, rlo, j), hi = __shfl_sync(0xffffffffu, rhi, j);
        const uint32_t pj = __shfl_sync(0xffffffffu, prim, j);
        const int x0 = (int)(lo & 0xffff), x1 = (int)(lo >> 16), y0 = (int)(hi & 0xffff);
        const int nx = x1 - x0;
        if (g < end) {
            const int local = (int)(g - oj);
            const int ty = y0 + local / nx, tx = x0 + local % nx;
            inst_tile[g] = (uint16_t)(ty * ntx + tx);
            inst_prim[g] = pj;
        }
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

// Per-tile [first, last+1) of the sorted tile ids; empty tiles marked -1.
__global__ void k_tile_bounds(const uint16_t *__restrict__ tile, int64_t m, int32_t *__restrict__ ranges) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int t = tile[i];
    if (i == 0 || tile[i - 1] != t) ranges[2 * t] = (int32_t)i;
    if (i == m - 1 || tile[i + 1] != t) ranges[2 * t + 1] = (int32_t)(i + 1);
}

// Empty tiles get start == end == first instance of the next non-empty tile
// (M if none): a block-wide suffix-min over the tile starts.
__global__ void __launch_bounds__(1024) k_fill_empty(int32_t *ranges, int32_t n_tiles, int32_t m) {
    __shared__ int32_t s_min[1024];
    const int t = threadIdx.x;
    const int chunk = (n_tiles + 1023) / 1024;
    const int lo = t * chunk, hi = min(lo + chunk, n_tiles);
    int32_t mn = INT32_MAX;
    for (int i = lo; i < hi; i++)
        if (ranges[2 * i] >= 0) { mn = ranges[2 * i]; break; }
    s_min[t] = mn;
    __syncthreads();
    // suffix min over chunks (Hillis-Steele, right to left)
    for (int off = 1; off < 1024; off <<= 1) {
        const int32_t o = t + off < 1024 ? s_min[t + off] : INT32_MAX;
        __syncthreads();
        s_min[t] = min(s_min[t], o);
        __syncthreads();
    }
    int32_t next = t + 1 < 1024 ? s_min[t + 1] : INT32_MAX;
    if (next == INT32_MAX) next = m;
    for (int i = hi - 1; i >= lo; i--) {
        if (ranges[2 * i] >= 0) {
            next = ranges[2 * i];
        } else {
            ranges[2 * i] = next;
            ranges[2 * i + 1] = next;
        }
    }
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

extern "C" int ssg_bin_temp_bytes(int64_t n, int64_t capacity, int32_t n_tiles, size_t *bytes) {
    using namespace ssg;
    if (!bytes || n < 0 || capacity < 0 || n_tiles < 1 || n_tiles > 65536) return SSG_ERR_INVALID_ARGUMENT;
    *bytes = bin_temp(n, capacity).total;
    return SSG_OK;
}

extern "C" int ssg_bin_prepare(int64_t n, const ssg_prim_buffers *prim, const ssg_bin_buffers *bins,
                               void *stream) {
    using namespace ssg;
    if (!prim || !bins || n < 0 || n >= (int64_t)UINT32_MAX) return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(bins->n_instances, 0, sizeof(int64_t), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(bins->rank_offset, 0, sizeof(uint64_t), st);
        if (e != cudaSuccess) { set_error("memset", e); return SSG_ERR_CUDA; }
        return SSG_OK;
    }
    const BinTemp L = bin_temp(n, bins->capacity);
    if (bins->temp_bytes < L.total) return SSG_ERR_CAPACITY;
    char *tmp = (char *)bins->temp;
    // 1. stable sort of primitive ids by depth key (the key buffer is consumed)
    cudaError_t e = radix::sort_pairs<uint64_t>(prim->depth_key, bins->depth_order, true, n, 8, tmp, st);
    if (e != cudaSuccess) { set_error("depth sort", e); return SSG_ERR_CUDA; }
    // 2. counts in depth order, scanned
    uint64_t *lb = (uint64_t *)(tmp + (L.total - L.scan_lookback));
    const int64_t scan_tiles = (n + kScanTile - 1) / kScanTile;
    e = cudaMemsetAsync(lb, 0, sizeof(uint64_t) * (scan_tiles + 1), st);
    if (e != cudaSuccess) { set_error("memset scan", e); return SSG_ERR_CUDA; }
    k_scan_counts<<<(unsigned)scan_tiles, kScanThreads, 0, st>>>(bins->depth_order, prim->tile_count, n,
                                                                bins->rank_offset, lb, bins->n_instances);
    return check_launch("ssg_bin_prepare");
}

extern "C" int ssg_bin_finish(int64_t n, int64_t m, int32_t width, int32_t height,
                              const ssg_prim_buffers *prim, const ssg_bin_buffers *bins, void *stream) {
    using namespace ssg;
    if (!prim || !bins || n < 0 || m < 0) return SSG_ERR_INVALID_ARGUMENT;
    if (m > bins->capacity || m >= (int64_t)INT32_MAX) return SSG_ERR_CAPACITY;
    int32_t ntx = (width + SSG_TILE - 1) / SSG_TILE, nty = (height + SSG_TILE - 1) / SSG_TILE;
    int32_t n_tiles = ntx * nty;
    if (n_tiles > 65536) return SSG_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(bins->ranges, 0xff, sizeof(int32_t) * 2 * (size_t)n_tiles, st);
    if (e != cudaSuccess) { set_error("memset ranges", e); return SSG_ERR_CUDA; }
    if (m > 0) {
        const BinTemp L = bin_temp(n, bins->capacity);
        if (bins->temp_bytes < L.total) return SSG_ERR_CAPACITY;
        k_duplicate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(bins->depth_order, bins->rank_offset,
                                                                 prim->tile_rect, ntx, n, bins->inst_tile,
                                                                 bins->inst_prim);
        e = radix::sort_pairs<uint16_t>(bins->inst_tile, bins->inst_prim, false, m, tile_passes(n_tiles),
                                        bins->temp, st);
        if (e != cudaSuccess) { set_error("tile sort", e); return SSG_ERR_CUDA; }
        k_tile_bounds<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(bins->inst_tile, m, bins->ranges);
    }
    k_fill_empty<<<1, 1024, 0, st>>>(bins->ranges, n_tiles, (int32_t)m);
    return check_launch("ssg_bin_finish");
}

// ---- test hooks (tests/ only): the radix sort in isolation -------------
extern "C" size_t ssg_test_sort_temp_bytes(int64_t n, int key_bytes) {
    using namespace ssg;
    return key_bytes == 2 ? radix::temp_bytes<uint16_t>(n) : radix::temp_bytes<uint64_t>(n);
}

extern "C" int ssg_test_sort(void *keys, uint32_t *vals, int key_bytes, int iota, int64_t n, int npass,
                             void *temp, void *stream) {
    using namespace ssg;
    cudaError_t e = key_bytes == 2
        ? radix::sort_pairs<uint16_t>((uint16_t *)keys, vals, iota != 0, n, npass, temp, (cudaStream_t)stream)
        : radix::sort_pairs<uint64_t>((uint64_t *)keys, vals, iota != 0, n, npass, temp, (cudaStream_t)stream);
    if (e != cudaSuccess) { set_error("test sort", e); return SSG_ERR_CUDA; }
    return SSG_OK;
}
