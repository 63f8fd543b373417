/*
 * ssg_b200.h -- C ABI of the B200-native skew-Gaussian rasterizer
 * (libssg_b200.so, sm_100a).
 *
 * Plain C: device pointers, sizes, and an opaque CUDA stream (void*, a
 * cudaStream_t).  No allocation happens inside these calls except where a
 * function says so; the caller owns every buffer (two-phase size queries
 * for the temporary storage).  Every call is asynchronous on `stream` and
 * returns an ssg_status; errors are never thrown across the ABI.
 *
 * The entry points replace the reference's hot path
 * (reference: pkg/src/skewsplat/...):
 *   ssg_preprocess_forward   projection.py:151-235 project_scene (+ tiles.py:43-57
 *                            per-primitive tile rect and count)
 *   ssg_bin_prepare          tiles.py:58-59 counts/offsets, ordering key of tiles.py:72
 *   ssg_bin_finish           tiles.py:59-79 duplicate + lexsort + searchsorted ranges
 *   ssg_blend_forward        raster/_core.pyx:169-200 forward_tiles (plugin slot of
 *                            raster/backend.py:41-43)
 *   ssg_blend_backward       raster/_core.pyx:315-343 backward_tiles fused with the
 *                            per-primitive slot reduction of raster/backward.py:70-73
 *   ssg_preprocess_backward  projection.py:255-379 projection_backward
 *   ssg_blend_backward_slots raster/_core.pyx:315-343 backward_tiles as is (per-instance
 *                            slots), for the reference's kernel plugin slot
 * The Python host layer (paper_2605_18334_b200.raster) keeps the reference's
 * render_forward / render_backward signatures (raster/forward.py:37-38,
 * raster/backward.py:77-79) on top of these.
 */
#ifndef SSG_B200_H
#define SSG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SSG_OK = 0,
    SSG_ERR_INVALID_ARGUMENT = 1, /* -> ValueError */
    SSG_ERR_DIM_OVERFLOW = 2,     /* -> ValueError("image dimension overflow"), forward.py:40-41 */
    SSG_ERR_CAPACITY = 3,         /* caller buffer too small (instances / temp storage) */
    SSG_ERR_CUDA = 4              /* a CUDA launch or runtime error; see ssg_last_error() */
} ssg_status;

#define SSG_TILE 16               /* raster/tiles.py:16 */
#define SSG_MAX_IMAGE_DIM 65535   /* raster/forward.py:21 */
#define SSG_MAX_BATCH_VIEWS 8     /* cameras per ssg_preprocess_forward_views call */

/* Scene on the device (reference Scene, scene.py:99-121).  Geometry that
 * decides tile membership and depth order stays fp64 so the tile lists are
 * bit-exact; appearance is fp32. */
typedef struct ssg_scene {
    int64_t n;
    int32_t sh_degree;          /* 0..3 */
    int32_t sh_coeffs;          /* K = (degree+1)^2; sh row stride is 3*K floats */
    const double *mu;           /* (n,3) */
    const double *log_scale;    /* (n,3) */
    const double *rot;          /* (n,4) quaternion w,x,y,z (normalised in use) */
    const float *sh;            /* (n,K,3) coefficient-major, then RGB */
    const float *opacity_logits;/* (n,2) */
    const float *beta;          /* (n,3) */
    const float *dir;           /* (n,3) */
} ssg_scene;

/* Camera, already in OpenCV convention (camera.py:53-75, projection.py:152-167).
 * R and t are the host's fp64 world_to_cam result; they feed the depth bits. */
typedef struct ssg_camera {
    double R[9];                /* R_w2c, row-major */
    double t[3];                /* -R_w2c @ eye */
    double campos[3];           /* c2w[:3,3] */
    double fx, fy, cx, cy;
    double tan_fovx, tan_fovy;
    double near_plane;
    double s;                   /* screen dilation */
    int32_t width, height;
} ssg_camera;

/* Per-primitive screen record consumed by the blend kernels (64 bytes,
 * 16-byte aligned): mean in fp64 so blend kernels can form tile-local
 * offsets exactly; the rest fp32.  band0 + band1 |power| bounds the relative
 * error of the blend's fp32 alpha against the reference's fp64 alpha for this
 * primitive (ssg_common.cuh alpha_band): a pixel whose fp32 alpha or
 * transmittance lies within its error bound of a threshold (1/255 skip, 0.99
 * clamp, 1e-4 stop) is decided on the exact fp64 path instead (ssg_splat64),
 * so every decision equals the reference's. */
typedef struct ssg_splat {
    double mean_x, mean_y;
    float conic_a, conic_b, conic_c;
    float skew_x, skew_y;
    float o1, o2;
    float r, g, b;
    float band0, band1;         /* alpha error band g0 + g1 |power| */
} ssg_splat;

/* fp64 twin of the splat's blend inputs (projection.py:194-215 values before
 * any rounding), read only on the rare threshold-band path (64 bytes). */
typedef struct ssg_splat64 {
    double conic_a, conic_b, conic_c;
    double skew_x, skew_y;
    double o1, o2;
    double comp;                /* dilation compensation (projection.py:201); 0 from ssg_pack_splats */
} ssg_splat64;

/* Per-primitive buffers written by ssg_preprocess_forward. */
typedef struct ssg_prim_buffers {
    ssg_splat *splat;           /* (n) */
    uint64_t *depth_key;        /* (n) order-preserving bits of the fp64 depth */
    uint32_t *tile_count;       /* (n) tiles covered (0 if invalid) */
    uint64_t *tile_rect;        /* (n) x0 | x1<<16 | y0<<32 | y1<<48 */
    uint8_t *valid;             /* (n) */
    double *depth;              /* (n) camera-space z (projection.py:161) */
    double *radius;             /* (n) */
    int32_t *n_skew_fallback;   /* (1) accumulated with atomics (zeroed by the call) */
    ssg_splat64 *splat64;       /* (n) fp64 blend inputs (threshold-band path) */
} ssg_prim_buffers;

/* Binning buffers.  depth_order/rank_offset are (n); inst_* are (capacity). */
typedef struct ssg_bin_buffers {
    uint32_t *depth_order;      /* (n) primitive ids sorted by (depth, id) */
    uint64_t *rank_offset;      /* (n+1) exclusive scan of counts in depth order */
    int64_t *n_instances;       /* (2) device: [0] M of the last ssg_bin_prepare, [1] running
                                   max of M (never reset by the library; lets a caller that
                                   skips the read-back check a batch of frames at once) */
    int64_t capacity;           /* allocated instances */
    uint32_t *inst_prim;        /* (capacity) sorted primitive id per instance */
    uint32_t *inst_tile;        /* (capacity) sorted tile id per instance; optional (NULL =
                                   not written: the blend kernels never read it) */
    int32_t *ranges;            /* (n_tiles, 2) half-open [start, end) */
    void *temp;                 /* temporary storage for the sorts and scans
                                   (size from ssg_bin_temp_bytes) */
    size_t temp_bytes;
} ssg_bin_buffers;

/* Frame outputs of the forward blend (raster/forward.py:24-34). */
typedef struct ssg_frame_buffers {
    float *color;               /* (H,W,3) */
    float *final_T;             /* (H,W) */
    int32_t *n_contrib;         /* (H,W) */
    int32_t *last_idx;          /* (H,W) global sorted index or -1 */
    uint32_t *blend_mask;       /* optional (NULL = unused), ssg_blend_mask_words(m, tiles)
                                   words: ssg_blend_forward records which instances each
                                   8x4 pixel block blended; ssg_blend_backward /
                                   ssg_blend_backward_slots then visit exactly those.  Only
                                   valid for the binning, splats and final_T/last_idx of
                                   the forward call that wrote it. */
    /* Exact-path bookkeeping, written by ssg_blend_forward and read by the
     * backward (required by both): pixels whose fp32 evaluation met an
     * uncertain decision are recomputed by the exact fp64 path. */
    uint32_t *redo_mask;        /* (n_tiles, 8) words: bit l of word 8 t + w = pixel l of the
                                   8x4 block w of tile t (lane order: 8 per row) */
    uint32_t *redo_list;        /* (W*H) pixel indices (y*W + x), first *redo_count valid */
    uint32_t *redo_count;       /* (1) */
} ssg_frame_buffers;

/* Gradient outputs (raster/backward.py:28-39).  d_beta == d_dir
 * (projection.py:365-366) so one d_eta array serves both. */
typedef struct ssg_grad_buffers {
    float *screen;              /* (n,12) screen-space sums: d_mean2d(2) d_conic(3)
                                   d_skew2d(2) d_opair(2) d_color(3) (raster/_cpu.py:88-93) */
    float *d_mu;                /* (n,3) */
    float *d_log_scale;         /* (n,3) */
    float *d_rot;               /* (n,4) */
    float *d_sh;                /* (n,K,3) */
    float *d_opacity_logits;    /* (n,2) */
    float *d_eta;               /* (n,3) */
    float *g_uv;                /* (n) */
    float *g_z;                 /* (n) */
    float *d_beta;              /* optional (n,3): d_eta plus the beta regularizer
                                   (ssg_regularize); NULL = d_eta (ssg_adam_step only) */
} ssg_grad_buffers;

/* Mutable parameters for the optimizer (same layout as ssg_scene). */
typedef struct ssg_params {
    int64_t n;
    int32_t sh_degree, sh_coeffs;
    double *mu, *log_scale, *rot;
    float *sh, *opacity_logits, *beta, *dir;
} ssg_params;

/* Adam moments (fp32, one array pair per scene field, adam.py:60-61) and
 * per-step scratch. */
typedef struct ssg_adam_state {
    float *m_mu, *v_mu, *m_log_scale, *v_log_scale, *m_rot, *v_rot;
    float *m_sh, *v_sh, *m_logits, *v_logits, *m_beta, *v_beta, *m_dir, *v_dir;
    uint8_t *row_ok;            /* (n) scratch */
    int32_t *n_skipped;         /* (1) skipped primitive-steps (non-finite gradient), accumulated
                                   across steps like adam.py:79; the caller zeroes it once */
} ssg_adam_state;

typedef struct ssg_adam_hparams {
    int64_t t;                  /* step count after this step (>= 1) */
    double lr_mu, lr_scale, lr_rot, lr_sh, lr_opacity, lr_beta;
    const int32_t *skip;        /* optional device flag: nonzero = this whole step is
                                   skipped (no moment, parameter or quaternion update,
                                   nothing counted), the device-side form of
                                   fit2d.py:70-71 for pipelined training steps; NULL = run */
} ssg_adam_hparams;

/* ---- queries ---------------------------------------------------------- */
int ssg_abi_version(void);
const char *ssg_last_error(void);
void ssg_grid_dims(int32_t width, int32_t height, int32_t *tiles_x, int32_t *tiles_y);
/* temporary storage needed by ssg_bin_prepare / ssg_bin_finish */
int ssg_bin_temp_bytes(int64_t n, int64_t capacity, int32_t width, int32_t height, size_t *bytes);

/* ---- forward ------------------------------------------------------------ */
/* screen records (splat + splat64, with the alpha band) from caller fp64 device
 * arrays mean2d (n,2), conic (n,3), skew2d (n,2), opair (n,2), color (n,3): the
 * inputs of the reference's blend plugin slot (raster/_core.pyx:169-177) */
int ssg_pack_splats(int64_t n, const double *mean2d, const double *conic, const double *skew2d,
                    const double *opair, const double *color, ssg_splat *splat, ssg_splat64 *splat64,
                    void *stream);
int ssg_preprocess_forward(const ssg_scene *scene, const ssg_camera *cam,
                           const ssg_prim_buffers *out, void *stream);
/* ssg_preprocess_forward for a batch of n_views (1..SSG_MAX_BATCH_VIEWS) cameras of
 * one scene in one pass over the scene (each primitive read once per batch; the
 * view-independent part of projection.py:151-235 -- scene.py:66-96 Sigma_world,
 * the sigmoids, Sigma eta -- computed once): outs[v] receives exactly what
 * ssg_preprocess_forward(scene, &cams[v], &outs[v]) writes.  outs[v].valid /
 * .depth / .radius may be NULL (not written).  Replaces the per-view project_scene
 * calls of the reference's trajectory loop (trajectory.py:12-31). */
int ssg_preprocess_forward_views(const ssg_scene *scene, const ssg_camera *cams,
                                 const ssg_prim_buffers *outs, int32_t n_views, void *stream);
/* depth sort, counts in depth order, exclusive scan; writes bins->n_instances */
int ssg_bin_prepare(int64_t n, const ssg_prim_buffers *prim, const ssg_bin_buffers *bins,
                    void *stream);
/* bin_arrays from caller screen arrays (tiles.py:43-57): fills tile_count,
 * tile_rect and depth_key of `out` (the other fields are not touched) */
int ssg_bin_rects(int64_t n, const double *mean2d, const double *radius, const double *depth,
                  const uint8_t *valid, int32_t width, int32_t height,
                  const ssg_prim_buffers *out, void *stream);
/* two-level counting scatter, ranges; m = bins->n_instances[0] read back, or m < 0 to
 * skip the read-back (writes stay inside `capacity`; M > capacity means the frame is
 * invalid and must be redone with larger buffers) */
int ssg_bin_finish(int64_t n, int64_t m, int32_t width, int32_t height,
                   const ssg_prim_buffers *prim, const ssg_bin_buffers *bins, void *stream);
/* words of the optional frame blend mask for m instances over n_tiles tiles */
int64_t ssg_blend_mask_words(int64_t m, int32_t n_tiles);
/* Decisions (alpha skip, transmittance stop) equal the fp64 reference's: the
 * fp32 blend carries an error bound and re-decides in fp64 (splat64, and an
 * fp64 replay of the pixel's transmittance) whenever a value falls inside it. */
int ssg_blend_forward(int64_t m, int32_t width, int32_t height, const float background[3],
                      const ssg_splat *splat, const ssg_splat64 *splat64, const ssg_bin_buffers *bins,
                      const ssg_frame_buffers *frame, void *stream);

/* The two halves of ssg_blend_forward / ssg_blend_backward, for callers that
 * overlap the exact path with other work on a second stream:
 * SSG_BLEND_MAIN_ONLY runs the fp32 kernel (it flags the pixels it cannot
 * certify), SSG_BLEND_EXACT_ONLY the exact path over the flagged pixels
 * (after the forward's main half; the backward's exact half needs the
 * forward's exact half but not the backward's main half -- both only add
 * into grads->screen).  SSG_BLEND_NO_ZERO (backward): grads->screen is
 * already zeroed by the caller.  flags = 0: the whole call. */
#define SSG_BLEND_MAIN_ONLY 1
#define SSG_BLEND_EXACT_ONLY 2
#define SSG_BLEND_NO_ZERO 4
/* (forward, test mode) every pixel takes the exact fp64 path */
#define SSG_BLEND_ALL_EXACT 8
int ssg_blend_forward_ex(int64_t m, int32_t width, int32_t height, const float background[3],
                         const ssg_splat *splat, const ssg_splat64 *splat64, const ssg_bin_buffers *bins,
                         const ssg_frame_buffers *frame, int32_t flags, void *stream);

/* ---- backward ----------------------------------------------------------- */
/* accumulates (n,12) screen gradients into grads->screen (zeroed by the call) */
int ssg_blend_backward(int64_t n, int64_t m, int32_t width, int32_t height,
                       const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                       const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                       const float *dL_dpixels, const ssg_grad_buffers *grads, void *stream);
int ssg_blend_backward_ex(int64_t n, int64_t m, int32_t width, int32_t height,
                          const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                          const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                          const float *dL_dpixels, const ssg_grad_buffers *grads, int32_t flags, void *stream);
/* Deterministic variant (bitwise-repeatable gradients).
 * Each (primitive, tile) pair's 12 sums are combined over the tile's pixel
 * blocks in a fixed order and stored (no atomics) into a primitive-major
 * slot array, each primitive's slots in ascending tile (= ascending
 * instance, raster/backward.py:70-73) order, then summed per primitive in
 * that order.  `prim` must be the buffers of the forward's ssg_bin_prepare
 * (tile_count, tile_rect); temp of ssg_blend_det_temp_bytes(n, m) bytes. */
size_t ssg_blend_det_temp_bytes(int64_t n, int64_t m);
int ssg_blend_backward_det(int64_t n, int64_t m, int32_t width, int32_t height,
                           const float background[3], const ssg_splat *splat, const ssg_splat64 *splat64,
                           const ssg_prim_buffers *prim, const ssg_bin_buffers *bins,
                           const ssg_frame_buffers *frame, const float *dL_dpixels,
                           const ssg_grad_buffers *grads, void *temp, size_t temp_bytes, void *stream);
int ssg_preprocess_backward(const ssg_scene *scene, const ssg_camera *cam,
                            const ssg_grad_buffers *grads, void *stream);
/* The projection backward in two parts, so the zero-fill can overlap the
 * blend (what the engine does: ssg_zero_prim_grads on a second stream while
 * ssg_blend_backward runs, then ssg_preprocess_backward_ex with
 * SSG_PREP_BWD_ACTIVE_ONLY).  ssg_zero_prim_grads zeroes grads' per-primitive
 * fields (d_mu, d_log_scale, d_rot, d_sh with sh_coeffs, d_opacity_logits,
 * d_eta, g_uv, g_z); with SSG_PREP_BWD_ACTIVE_ONLY the projection backward
 * writes only the primitives with a non-zero screen gradient (the others must
 * already be zero).  flags = 0 is ssg_preprocess_backward.  Outputs are
 * identical either way. */
#define SSG_PREP_BWD_ACTIVE_ONLY 1
int ssg_zero_prim_grads(int64_t n, int32_t sh_coeffs, const ssg_grad_buffers *grads, void *stream);
/* zeroes grads->screen (n,12): what ssg_blend_backward_ex does unless
 * SSG_BLEND_NO_ZERO, for callers that split the halves across streams */
int ssg_zero_screen_grads(int64_t n, const ssg_grad_buffers *grads, void *stream);
int ssg_preprocess_backward_ex(const ssg_scene *scene, const ssg_camera *cam,
                               const ssg_grad_buffers *grads, int32_t flags, void *stream);
/* the reference's blend-backward plugin contract (raster/_core.pyx:315-343,
 * backward_tiles): per-instance gradient slots (m,12) instead of the fused
 * per-primitive reduction; slots is zeroed by the call */
int ssg_blend_backward_slots(int64_t m, int32_t width, int32_t height, const float background[3],
                             const ssg_splat *splat, const ssg_splat64 *splat64, const ssg_bin_buffers *bins,
                             const ssg_frame_buffers *frame, const float *dL_dpixels, float *slots,
                             void *stream);

/* ---- training step (config 5) ------------------------ */
/* floats of scratch ssg_image_loss needs for a width x height image */
int64_t ssg_loss_scratch_floats(int32_t width, int32_t height);
/* optimize/losses.py:103-113 image_loss: (1-l) L1 + l (1 - SSIM) of rendered
 * vs target ((H,W,3) f32) and its pixel gradient dL_dpixels (H,W,3);
 * sums[0] = sum |x - y|, sums[1] = sum of SSIM over the valid windows x 3
 * channels (value = (1-l) sums[0]/(3HW) + l (1 - sums[1]/(3 (H-10)(W-10)))).
 * l == 0: L1 only (scratch may be NULL); l > 0 needs W, H >= 11 */
int ssg_image_loss(const float *rendered, const float *target, int32_t width, int32_t height,
                   float lambda_ssim, float *scratch, float *dL_dpixels, double *sums, void *stream);
/* optimize/losses.py:116-136 scene_regularizers folded into the gradients:
 * d_beta = d_eta + 2 lambda_beta beta, d_logits += the opacity-gap term,
 * sums[2] = the penalty value.  d_eta, d_beta and d_logits all NULL: the
 * value only (losses.py:146-149 tests loss + penalty for finiteness) */
int ssg_regularize(int64_t n, const float *beta, const float *opacity_logits, const float *d_eta,
                   float lambda_beta, float lambda_opacity, float *d_beta, float *d_logits, double *sums,
                   void *stream);
/* A step's loss value and fate, on the device (no host read-back): loss[0] =
 * (1-l) sums[0]/(3HW) + l (1 - sums[1]/(3 (H-10)(W-10))) + sums[2] (l == 0: the
 * L1 term only), in the reference's fp64 operation order (losses.py:103-113,
 * fit2d.py:69); flag[0] = 2 when n_instances[1] > capacity (the frame's lists
 * were truncated), else 1 when the loss is not finite (fit2d.py:70-71), else 0.
 * n_instances / flag may be NULL (value only). */
int ssg_step_value(const double *sums, int32_t width, int32_t height, double lambda_ssim,
                   const int64_t *n_instances, int64_t capacity, double *loss, int32_t *flag, void *stream);
/* trainer.py:49-53 _IntervalStats.add: uv_sum += g_uv, z_max = max(z_max, g_z),
 * mu_sum += d_mu */
int ssg_interval_stats_add(int64_t n, const float *g_uv, const float *g_z, const float *d_mu,
                           double *uv_sum, float *z_max, double *mu_sum, void *stream);
/* the same, skipped entirely when *skip != 0 (device flag; NULL = always add) */
int ssg_interval_stats_add_ex(int64_t n, const float *g_uv, const float *g_z, const float *d_mu,
                              double *uv_sum, float *z_max, double *mu_sum, const int32_t *skip,
                              void *stream);
/* optimize/adam.py:71-97 Adam.step on the device (skip non-finite rows,
 * bias-corrected moments, per-field learning rates, quaternion renorm) */
int ssg_adam_step(const ssg_params *params, const ssg_grad_buffers *grads,
                  const ssg_adam_state *state, const ssg_adam_hparams *hp, void *stream);

/* ---- adaptive density control --------------------- */
/* optimize/densify.py:24-116 inputs: the interval statistics bundle */
typedef struct ssg_densify_stats {
    const double *g_uv;         /* (n) mean screen-space positional gradient */
    const float *g_z;           /* (n) max depth gradient */
    const double *d_mu;         /* (n,3) mean position gradient */
} ssg_densify_stats;

typedef struct ssg_densify_cfg {
    double tau_uv;
    double tau_z;               /* NaN: calibrate to the 90th percentile of g_z */
    double split_scale_threshold;
    double prune_alpha;
    double max_screen_radius;   /* < 0: no radius cap */
    double clone_lr;            /* position_lr_at(densify_start), densify.py:49 */
    const double *max_radii;    /* optional (n) screen radii, NULL: none */
} ssg_densify_cfg;

size_t ssg_densify_temp_bytes(int64_t n);
/* flags (n bytes: 1 keep, 2 clone, 4 split, 8 prune) and, on the host,
 * counts[4] = {n_keep, n_clone, n_split, n_pruned} and the tau_z used; the new
 * primitive count is n_keep + n_clone + 2 n_split.  Synchronises the stream. */
int ssg_densify_plan(const ssg_scene *scene, const ssg_densify_stats *stats, const ssg_densify_cfg *cfg,
                     uint8_t *flags, void *temp, size_t temp_bytes, int64_t *counts, double *tau_z,
                     void *stream);
/* writes the new scene into `out` (capacity for the new count; same SH
 * degree) in the reference's row order and, when given, the remapped Adam
 * moments (adam.py:99-110); *bad = 1 when an output is non-finite
 * (densify.py:112-114).  `temp` and `flags` as left by ssg_densify_plan. */
int ssg_densify_apply(const ssg_scene *scene, const ssg_params *out, const ssg_adam_state *adam_in,
                      const ssg_adam_state *adam_out, const ssg_densify_stats *stats,
                      const ssg_densify_cfg *cfg, const uint8_t *flags, void *temp, int32_t *bad,
                      void *stream);

/* ---- frame serving --------------------------------- */
/* dataset.py:33-38 quantize_u8 on the device: dst[i] = rint(clip(src[i], 0, 1)
 * * 255) evaluated in fp64 (round half to even); src is f32 (a rendered
 * frame) or, with src_is_f64, f64 */
int ssg_quantize_u8(const void *src, int32_t src_is_f64, int64_t n_values, uint8_t *dst, void *stream);

/* ---- scene PLY -> device SoA ----------------------- */
/* PLY property types (scene.py:210-216) */
enum { SSG_PLY_ABSENT = -1, SSG_PLY_F32 = 0, SSG_PLY_F64 = 1, SSG_PLY_I8 = 2, SSG_PLY_U8 = 3,
       SSG_PLY_I16 = 4, SSG_PLY_U16 = 5, SSG_PLY_I32 = 6, SSG_PLY_U32 = 7 };
/* Unpack n binary little-endian vertex records (`stride` bytes each, device
 * memory) into `out` (capacity n).  offsets/types (host arrays of 18 + 3K
 * entries) give each destination component's byte offset and type in the
 * record, in the order mu 0-2, log_scale 3-5, rot 6-9, opacity_logits 10-11,
 * beta 12-14, dir 15-17, sh (K,3); type SSG_PLY_ABSENT stores 0 (load_ply,
 * scene.py:222-313: the host resolves names, defaults and errors). */
int ssg_ply_unpack(const uint8_t *payload, int64_t n, int32_t stride, const int32_t *offsets,
                   const int32_t *types, int32_t sh_coeffs, const ssg_params *out, void *stream);

/* ---- test hooks (used by tests/ only) ----------------------------------- */
/* the depth sort of ssg_bin_prepare in isolation: stable sort of u64 keys
 * (not modified), vals <- the ids 0..n-1 in sorted order; key_bytes must be 8,
 * iota 1 and npass 8 (any other combination: SSG_ERR_INVALID_ARGUMENT) */
size_t ssg_test_sort_temp_bytes(int64_t n, int key_bytes);
int ssg_test_sort(void *keys, uint32_t *vals, int key_bytes, int iota, int64_t n, int npass,
                  void *temp, void *stream);
/* the blend forward compiled without the skew term (plain 3DGS: alpha =
 * o * G): the config-3 regression reference for skew-free splats */
int ssg_test_blend_forward_vanilla(int32_t width, int32_t height, const float background[3],
                                   const ssg_splat *splat, const ssg_splat64 *splat64,
                                   const ssg_bin_buffers *bins, const ssg_frame_buffers *frame,
                                   void *stream);
/* device evaluation of the blend's two erf paths at n points x (device
 * arrays): e32[i] = the fp32 E = 1 + erf(x) of the blend kernels, e64[i] =
 * the fp64 c_erf restatement (raster/_core.pyx:57-74) the threshold-band
 * path uses; either output may be NULL (erf_probe, raster/_core.pyx:46-54) */
int ssg_erf_probe(const double *x, int64_t n, float *e32, double *e64, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SSG_B200_H */
