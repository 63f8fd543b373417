// binning.cu -- K2-K4: tile binning with bit-exact reference ordering.
//
// Reference: raster/tiles.py:43-79 (bin_arrays).  The reference emits one
// instance per covered tile and lexsorts by (tile, depth, primitive id).
// Here the same order is produced in two stable stages:
//   1. sort primitives by their full 64-bit fp64 depth (stable, so equal
//      depths keep primitive-id order)               -> depth rank
//   2. emit each primitive's instances in depth-rank order, then stable-sort
//      the instances by tile id (13-16 bit key)        -> (tile, depth, id)
// Ranges are per-tile lower/upper bounds of the sorted tile ids, i.e.
// exactly np.searchsorted(..., side="left"/"right") (tiles.py:76-78),
// including the start==end position of empty tiles.
#include <cub/cub.cuh>

#include "ssg_common.cuh"

namespace ssg {

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int tile_bits(int32_t n_tiles) {
    int b = 1;
    while ((1 << b) < n_tiles) b++;
    return b;
}

struct TempLayout {
    size_t cub_bytes;
    size_t off_keys, off_iota, off_cnt, total;
};

static cudaError_t temp_layout(int64_t n, int64_t capacity, int32_t n_tiles, TempLayout &L) {
    size_t a = 0, b = 0, c = 0;
    cudaError_t e;
    int nn = (int)(n > 0 ? n : 1);
    int cc = (int)(capacity > 0 ? capacity : 1);
    e = cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                        (const uint32_t *)nullptr, (uint32_t *)nullptr, nn, 0, 64);
    if (e != cudaSuccess) return e;
    e = cub::DeviceScan::InclusiveSum(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr, nn);
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(nullptr, c, (const uint16_t *)nullptr, (uint16_t *)nullptr,
                                        (const uint32_t *)nullptr, (uint32_t *)nullptr, cc, 0,
                                        tile_bits(n_tiles));
    if (e != cudaSuccess) return e;
    size_t m = a > b ? a : b;
    m = m > c ? m : c;
    L.cub_bytes = align256(m);
    L.off_keys = L.cub_bytes;
    L.off_iota = L.off_keys + align256(sizeof(uint64_t) * (size_t)nn);
    L.off_cnt = L.off_iota + align256(sizeof(uint32_t) * (size_t)nn);
    L.total = L.off_cnt + align256(sizeof(uint64_t) * (size_t)nn);
    return cudaSuccess;
}

__global__ void k_iota(uint32_t *v, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__global__ void k_gather_counts(const uint32_t *order, const uint32_t *count, uint64_t *out, int64_t n) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) out[r] = count[order[r]];
}

__global__ void k_finish_scan(uint64_t *rank_offset, int64_t n, int64_t *n_instances) {
    rank_offset[0] = 0;
    *n_instances = (int64_t)rank_offset[n];
}

// tiles.py:59-70: the instances of one primitive in row-major tile order.
__global__ void k_duplicate(const uint32_t *order, const uint64_t *rank_offset,
                            const uint64_t *rect, int32_t ntx, int64_t n, uint16_t *inst_tile,
                            uint32_t *inst_prim) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    uint64_t base = rank_offset[r], end = rank_offset[r + 1];
    if (end == base) return;
    uint32_t prim = order[r];
    uint64_t rc = rect[prim];
    int x0 = (int)(rc & 0xffff), x1 = (int)((rc >> 16) & 0xffff);
    int y0 = (int)((rc >> 32) & 0xffff), y1 = (int)((rc >> 48) & 0xffff);
    uint64_t k = base;
    for (int ty = y0; ty < y1; ty++)
        for (int tx = x0; tx < x1; tx++) {
            inst_tile[k] = (uint16_t)(ty * ntx + tx);
            inst_prim[k] = prim;
            k++;
        }
}

// np.searchsorted(inst_tile, t, 'left') / (t, 'right') for every tile id
__global__ void k_ranges(const uint16_t *inst_tile, int64_t m, int32_t n_tiles, int32_t *ranges) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int)inst_tile[mid] < t) lo = mid + 1; else hi = mid;
    }
    int64_t s = lo;
    hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int)inst_tile[mid] <= t) lo = mid + 1; else hi = mid;
    }
    ranges[2 * t] = (int32_t)s;
    ranges[2 * t + 1] = (int32_t)lo;
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
    // order-preserving bits for any finite double (sign flip for negatives)
    uint64_t b = (uint64_t)__double_as_longlong(depth[i] == 0.0 ? 0.0 : depth[i]);
    key[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
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
    TempLayout L;
    cudaError_t e = temp_layout(n, capacity, n_tiles, L);
    if (e != cudaSuccess) { set_error("cub temp query", e); return SSG_ERR_CUDA; }
    *bytes = L.total;
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
    TempLayout L;
    cudaError_t e = temp_layout(n, bins->capacity, 1, L);
    if (e != cudaSuccess) { set_error("cub temp query", e); return SSG_ERR_CUDA; }
    if (bins->temp_bytes < L.total) return SSG_ERR_CAPACITY;
    char *tmp = (char *)bins->temp;
    uint64_t *keys_sorted = (uint64_t *)(tmp + L.off_keys);
    uint32_t *iota = (uint32_t *)(tmp + L.off_iota);
    uint64_t *cnt = (uint64_t *)(tmp + L.off_cnt);
    unsigned blocks = (unsigned)((n + 255) / 256);
    k_iota<<<blocks, 256, 0, st>>>(iota, n);
    size_t cb = L.cub_bytes;
    e = cub::DeviceRadixSort::SortPairs(tmp, cb, prim->depth_key, keys_sorted, iota, bins->depth_order,
                                        (int)n, 0, 64, st);
    if (e != cudaSuccess) { set_error("depth sort", e); return SSG_ERR_CUDA; }
    k_gather_counts<<<blocks, 256, 0, st>>>(bins->depth_order, prim->tile_count, cnt, n);
    cb = L.cub_bytes;
    e = cub::DeviceScan::InclusiveSum(tmp, cb, cnt, bins->rank_offset + 1, (int)n, st);
    if (e != cudaSuccess) { set_error("count scan", e); return SSG_ERR_CUDA; }
    k_finish_scan<<<1, 1, 0, st>>>(bins->rank_offset, n, bins->n_instances);
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
    if (m > 0) {
        TempLayout L;
        cudaError_t e = temp_layout(n, bins->capacity, n_tiles, L);
        if (e != cudaSuccess) { set_error("cub temp query", e); return SSG_ERR_CUDA; }
        if (bins->temp_bytes < L.total) return SSG_ERR_CAPACITY;
        k_duplicate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            bins->depth_order, bins->rank_offset, prim->tile_rect, ntx, n, bins->inst_tile_tmp,
            bins->inst_prim_tmp);
        size_t cb = L.cub_bytes;
        e = cub::DeviceRadixSort::SortPairs(bins->temp, cb, bins->inst_tile_tmp, bins->inst_tile,
                                            bins->inst_prim_tmp, bins->inst_prim, (int)m, 0,
                                            tile_bits(n_tiles), st);
        if (e != cudaSuccess) { set_error("tile sort", e); return SSG_ERR_CUDA; }
    }
    k_ranges<<<(n_tiles + 255) / 256, 256, 0, st>>>(bins->inst_tile, m, n_tiles, bins->ranges);
    return check_launch("ssg_bin_finish");
}
