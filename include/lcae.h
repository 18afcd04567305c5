/*
 * lcae.h — C ABI of liblcae.so: one training step of a locally-connected (untied-weight)
 * RICA sparse-autoencoder layer on one B200 (sm_100a).
 *
 * The operation (§3.1 eq. "RICA", read as DESIGN.md "Readings" R1-R11):
 * for every receptive field f of the layer (row-major grid) and every
 * sample x^(i) of the batch (patch x_f^(i) flattened in (ry, rx, c) order):
 *
 *     h    = alpha_f W_f x                                   (encode, "alpha W x")
 *     s_G  = sqrt(eps + sum_{j in G} h_j^2)                   (L2 pooling, groups of g filters; g=1: the
 *                                                              paper's lambda sqrt((alpha W x)^2))
 *     r    = W_f^T h + b_f,  e = r - x                         (decode with offset b)
 *     J   += ||e||^2 + lambda sum_G s_G                        (reconstruction + sparsity, summed; R6)
 *     dW_f, dalpha_f, db_f, dX (overlap-added over fields)     (exact gradients of J; R11)
 *     W_f <- rownorm(W_f - lr dW_f) (optional momentum); alpha_f <- max(alpha_f - lr dalpha_f, alpha_min);
 *     b_f <- b_f - lr db_f                                     (projected SGD)
 *
 * Precision: LCAE_FP32 computes every product and sum in fp32 (FFMA, no TF32) with an fp64 loss sum;
 * LCAE_BF16 feeds bf16 operands (x, W, h, delta, D rounded RN-even) to tcgen05 tensor cores with fp32
 * accumulation (TMEM), fp32 epilogues and fp32 master weights. A bf16 layer runs on one fused step kernel
 * when k <= 128, m <= 256 and n <= 4096; larger layers (e.g. the paper's own layer 1, k = 384)
 * run the same step as five batched tcgen05 GEMMs with epilogue kernels (same operand rounding).
 *
 * Conventions
 *  - All functions return lcae_status; on error, lcae_last_error() (thread-local, library-owned
 *    string) says why. Status codes 2/3/4 mirror SPEC.md:531's exit codes (config/data/numeric).
 *  - Data pointers marked "host or device" may be either: the library inspects them with
 *    cudaPointerGetAttributes and copies host data through its own device staging buffers on the
 *    layer's stream. Device pointers must be on the layer's device.
 *  - Everything is ordered on cfg.stream (a cudaStream_t; NULL = legacy default stream). Calls whose
 *    outputs are host memory or that return a host scalar (loss != NULL) synchronise that stream.
 *  - A layer handle is not thread-safe; one handle per host thread.
 *  - The library owns all device memory it allocates; nothing is freed by the caller.
 *
 * Errors of the data ("non-finite ... numeric error"; SPEC.md:531 exit codes 3/4)
 *  - The input staging kernel flags any non-finite x element on the device; a loss reduction that yields a
 *    non-finite J flags that too. Flags are sticky: while one is set, every parameter-updating kernel of
 *    lcae_step returns without writing (the flagged step itself is skipped when the input was bad; with a
 *    non-finite loss the step that produced it has already updated its parameters, later steps are skipped).
 *  - The flag is reported -- LCAE_ERR_DATA for a non-finite input, LCAE_ERR_NUMERIC for a non-finite loss --
 *    and cleared by the next call that synchronises: a step/forward with loss != NULL, a call with host
 *    outputs, or lcae_sync. lcae_set_params also clears it. With loss == NULL (the asynchronous hot path)
 *    nothing is silently written into W after a bad input: the step is skipped on the device.
 *
 * Layouts (canonical, exchanged with callers and the test oracle)
 *  - image x / dx: NHWC float32 [m][img_h][img_w][img_c].
 *  - W: float32 [F][k][n], n = (ry*rf_w + rx)*img_c + c; alpha: float32 [F]; b: float32 [F][n].
 *  - pooled p: float32 [m][grid_r][grid_c][k/g] (p = s_G, the L2-pooled code).
 *  - F = grid_r*grid_c fields in row-major order over THIS layer's image (a rank of a model-parallel
 *    run passes its extended input region — owned pixels plus halo — as its image; global field ids
 *    are field_row0/field_col0/global_grid_c offsets, used only by the degenerate-row generator).
 */
#ifndef LCAE_H_
#define LCAE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lcae_layer lcae_layer; /* opaque; owns all its device memory */

typedef enum {
  LCAE_OK = 0,
  LCAE_ERR_CONFIG = 2,  /* geometry / pooling / precision / size not supported */
  LCAE_ERR_DATA = 3,    /* bad data pointer, shape or non-finite input */
  LCAE_ERR_NUMERIC = 4, /* non-finite loss ("numeric error") */
  LCAE_ERR_CUDA = 5,    /* CUDA runtime / driver failure (message has the CUDA error string) */
  LCAE_ERR_NCCL = 6,    /* NCCL communicator / transfer failure of a model-parallel layer (lcae_mp_*) */
  LCAE_ERR_ARG = 7      /* NULL handle or NULL required pointer */
} lcae_status;

typedef enum { LCAE_FP32 = 0, LCAE_BF16 = 1 } lcae_precision;

typedef struct {
  int32_t img_h, img_w, img_c; /* input image (this rank's extended region) */
  int32_t rf_h, rf_w, stride;  /* receptive field and stride; (img-rf) % stride == 0 */
  int32_t filters;             /* k per field (PAPER.md:95 'output size 4x4x24' = 384 for the paper) */
  int32_t pool_group;          /* g: divides k and 32; g = 1 == the paper (no pooling) */
  int32_t batch;               /* m: samples per step */
  float lambda_;               /* sparsity weight (0.1 for layers 1-2) */
  float eps;                   /* sqrt smoothing, > 0 recommended */
  float lr;                    /* SGD learning rate */
  float momentum;              /* 0 = plain SGD (hot path); > 0 allocates velocity buffers */
  float alpha_init;            /* initial alpha (when params are not set explicitly) */
  float alpha_min;             /* alpha clamp (1e-8) */
  uint64_t seed;               /* degenerate-row re-initialisation generator seed */
  int32_t precision;           /* lcae_precision */
  int32_t keep_grads;          /* 1: also store dW/dalpha/db of the last step for lcae_get_grads (tests) */
  int32_t field_row0, field_col0, global_grid_c; /* global id of local field (r,c) = (row0+r)*ggc + col0+c
                                                   (caller-tiled mode, world_size == 1; set by the library
                                                   itself when world_size > 1) */
  /* Model parallelism over receptive fields inside the library ("model parallel ...
   * communication ... occurs when a layer's input (or output) field spans multiple GPUs").
   * world_size > 1: img_h/img_w are the GLOBAL image; the field grid is cut into tiles_r x tiles_c contiguous
   * rectangles (rank r = tile (r / tiles_c, r % tiles_c); tiles_r = tiles_c = 0 derives the
   * most square split with tiles_r >= tiles_c); this rank owns the weights of its fields and the pixel
   * rectangle own_px (lcae_geometry). x / dx of lcae_step / lcae_forward are then this rank's OWNED pixels,
   * NHWC f32 [m][own_h][own_w][C]; pooled is [m][local grid_r][local grid_c][k/g]; the loss is the global sum.
   * Each step exchanges the input halo (bf16 on the tensor-core path) and returns the halo dX (fp32) with NCCL
   * send/recv on the layer's comm stream, the halo overlapping the interior fields; the loss is all-reduced. */
  int32_t world_size;          /* 1 (default) = one GPU (with nccl_id set: a one-tile model-parallel layer) */
  int32_t rank;                /* 0 .. world_size-1 */
  int32_t tiles_r, tiles_c;    /* tiles_r * tiles_c == world_size, or both 0 */
  const void *nccl_id;         /* 128-byte ncclUniqueId (lcae_nccl_unique_id on one rank, broadcast by the caller);
                                  NULL with world_size > 1 = test mode: no NCCL, the caller moves the exchange
                                  buffers between phases (lcae_mp_buffer / lcae_mp_phase) */
  void *stream;                /* cudaStream_t; NULL = default stream */
} lcae_config;

/* Fill *cfg with the defaults of DESIGN.md (lambda 0.1, eps 1e-6, lr 1e-3, momentum 0, alpha 1, 1e-8). */
void lcae_config_default(lcae_config *cfg);

/* Validate cfg and report the derived geometry without allocating anything (no GPU needed).
 * grid_r/grid_c/n_params: THIS rank's field grid and parameter count F*(k*n + n + 1) (the
 * whole layer when world_size == 1). own_px = {y0, y1, x0, x1}: the global pixel rectangle this rank owns;
 * own_fields = {R0, R1, C0, C1}: its global field rows / columns. Any output may be NULL.
 * Errors: LCAE_ERR_CONFIG with the residue for non-divisible extents, g not dividing k
 * or 32, rf larger than the image, non-positive sizes, unknown precision, a tile without fields,
 * tiles_r * tiles_c != world_size, rank out of range. */
lcae_status lcae_geometry(const lcae_config *cfg, int32_t *grid_r, int32_t *grid_c, int64_t *n_params,
                          int32_t own_px[4], int32_t own_fields[4]);

/* Write a fresh 128-byte ncclUniqueId to out128 (host memory), for lcae_config.nccl_id of every rank.
 * Errors: LCAE_ERR_NCCL when libnccl.so.2 cannot be loaded or fails. */
lcae_status lcae_nccl_unique_id(void *out128);

/* Model-parallel test mode (world_size > 1, nccl_id == NULL): a step is three calls, and between them the
 * caller copies, for every pair of ranks (a, b), a's send buffer for b into b's receive buffer from a:
 *   lcae_mp_phase(L, 0, x, ...)  stage the owned x, pack the halo neighbours need, run the interior fields;
 *   -- move input-halo buffers (which 0 -> which 1) --
 *   lcae_mp_phase(L, 1, ...)     unpack the halo, run the boundary fields, finalize, local loss, pack halo dX;
 *   -- move dX buffers (which 2 -> which 3) --
 *   lcae_mp_phase(L, 2, ..., dx, loss)  add the returned dX into the owned pixels, write dx (owned, NHWC f32),
 *                                       loss = this rank's local J (the caller sums over ranks).
 * update = 1 trains (lcae_step), 0 = forward (pooled nullable, phases 0-1 only, then 2 for the loss).
 * lcae_mp_buffer: device pointer and byte size of buffer `which` (0 halo send to peer, 1 halo receive from
 * peer, 2 dX send to peer, 3 dX receive from peer); NULL / 0 when the pair exchanges nothing. Buffers are
 * owned by the layer. Errors: ARG (not a model-parallel test-mode layer, bad phase order), CUDA. */
lcae_status lcae_mp_phase(lcae_layer *L, int32_t phase, int32_t update, const float *x, float *dx, float *pooled,
                          double *loss);
lcae_status lcae_mp_buffer(lcae_layer *L, int32_t which, int32_t peer, void **ptr, int64_t *bytes);

/* Interior / boundary field counts of a model-parallel rank (interior fields run while the halo travels). */
lcae_status lcae_mp_fields(lcae_layer *L, int32_t *n_interior, int32_t *n_boundary);

/* Create a layer on the current CUDA device: validates cfg (as lcae_geometry), allocates parameters,
 * gradient/optimizer state and scratch, and initialises W to unit rows from a counter-based generator,
 * alpha = alpha_init, b = 0 (callers normally overwrite them with lcae_set_params).
 * *out receives the handle. Errors: CONFIG, CUDA (e.g. out of memory), ARG. */
lcae_status lcae_create(const lcae_config *cfg, lcae_layer **out);

/* Release everything the handle owns. NULL-safe. Synchronises the layer's stream first. */
lcae_status lcae_destroy(lcae_layer *L);

/* Copy parameters in (canonical layouts above; host or device pointers). W rows are used as given
 * (callers pass unit rows). Any pointer may be NULL to leave that tensor unchanged. */
lcae_status lcae_set_params(lcae_layer *L, const float *W, const float *alpha, const float *b);

/* Copy the current parameters out (host or device pointers; NULL skips). */
lcae_status lcae_get_params(lcae_layer *L, float *W, float *alpha, float *b);

/* The parameters of fields [f0, f0 + count) only (canonical layouts restricted to the range; host or device;
 * NULL skips): sampled checks of layers too large to copy out whole (e.g. the 15 B-weight point).
 * Errors: ARG (range outside the layer), CUDA. */
lcae_status lcae_get_field_params(lcae_layer *L, int64_t f0, int64_t count, float *W, float *alpha, float *b);

/* Gradients of the most recent lcae_step, taken at the pre-update parameters (requires keep_grads=1,
 * else LCAE_ERR_CONFIG). dW [F][k][n], dalpha [F], db [F][n]; host or device; NULL skips. */
lcae_status lcae_get_grads(lcae_layer *L, float *dW, float *dalpha, float *db);

/* Forward only: pooled code p (nullable) and loss J at the current parameters (nullable; if non-NULL the
 * call synchronises and returns LCAE_ERR_NUMERIC when J is not finite). x: host or device NHWC f32. */
lcae_status lcae_forward(lcae_layer *L, const float *x, float *pooled, double *loss);

/* Inference (SPEC.md:490 forward_dataset, "forward propagated 2 million
 * images ... to obtain activation values"): the encode + L2-pooling half of the layer only (no decode, no
 * update). pooled (required) receives p [m][grid_r][grid_c][k/g] (host or device); j_sparse (nullable,
 * synchronises) receives lambda * sum p. Parameters are not modified. Errors: ARG, DATA, CUDA. */
lcae_status lcae_encode(lcae_layer *L, const float *x, float *pooled, double *j_sparse);

/* Streaming top-K stimuli per unit (SPEC.md:500-508 top_k_stimuli; "top 5 stimuli").
 * State: vals [units][K] f32 and ids [units][K] int32 (device), each row sorted by value descending, ties
 * by lower image id; lcae_topk_init fills it with (-inf, INT32_MAX). lcae_topk_update merges one batch of
 * activations act [m][units] (device f32, e.g. the pooled output of lcae_encode with units =
 * grid_r*grid_c*(k/g)) whose sample s has image id id0 + s. 1 <= K <= 32 (else LCAE_ERR_ARG). Ordered on
 * `stream` (cudaStream_t; NULL = default stream); no synchronisation. */
lcae_status lcae_topk_init(float *vals, int32_t *ids, int64_t units, int32_t K, void *stream);
lcae_status lcae_topk_update(const float *act, int64_t m, int64_t units, int32_t K, int64_t id0, float *vals,
                             int32_t *ids, void *stream);

/* Local contrast normalisation of a layer output before the next layer (PAPER.md:95
 * "local contrast normalization (LCN) is applied prior to continuing onto the next layer"; formula
 * SPEC.md:215-223): v = x - mean_w(x), y = v / max(floor, sqrt(mean_w(v^2))), uniform window x window per
 * channel, zero padding with count-correct divisors. x, y: device f32 [m][H][W][C] (y may not alias x);
 * scratch: device f32, 2 m H W C elements. window odd and <= H, W; floor > 0 (else LCAE_ERR_CONFIG).
 * Ordered on `stream`; no synchronisation. */
lcae_status lcae_lcn(const float *x, float *y, float *scratch, int32_t m, int32_t H, int32_t W, int32_t C,
                     int32_t window, float floor_, void *stream);

/* Start copying the NEXT batch (a host NHWC f32 pointer; pinned memory for a truly asynchronous copy) into
 * a device buffer on the layer's own copy stream, so that the transfer overlaps the current step; the
 * lcae_step / lcae_forward / lcae_encode call that is given the same pointer then waits for that copy
 * instead of copying. The host buffer must stay unchanged until that call. Device pointers are a no-op.
 * Errors: ARG, CUDA. */
lcae_status lcae_prefetch_input(lcae_layer *L, const float *x_host);

/* One training step on batch x (host or device NHWC f32): loss and gradients at the current parameters,
 * the input gradient dX overlap-added over fields into dx (nullable: the dX contraction still runs,
 * the result stays in the layer's device buffer — see lcae_dx_device), then the fused projected-SGD
 * update. loss (nullable) receives J = J_rec + J_sparse of the pre-update parameters (synchronises).
 * Errors: ARG, DATA, NUMERIC (non-finite loss, parameters already updated), CUDA. */
lcae_status lcae_step(lcae_layer *L, const float *x, float *dx, double *loss);

/* Wait for the layer's stream and report the sticky data errors (see "Errors of the data" above): LCAE_OK,
 * LCAE_ERR_DATA (a non-finite input was seen) or LCAE_ERR_NUMERIC (a non-finite loss); clears the flag. */
lcae_status lcae_sync(lcae_layer *L);

/* Per-field loss of the last step/forward: out[f][0] = J_rec of field f, out[f][1] = J_sparse (lambda sum s_G),
 * f in this layer's row-major field order; out is host or device memory of 2*F doubles. Synchronises.
 * (Sampled parity checks at full size compare single fields against the oracle.) Errors: ARG, CUDA. */
lcae_status lcae_field_losses(lcae_layer *L, double *out);

/* Loss split of the last step/forward: J_rec and J_sparse (host doubles; synchronises). */
lcae_status lcae_last_loss(lcae_layer *L, double *j_rec, double *j_sparse);

/* Device pointer of the layer's dX buffer (NHWC f32, valid after lcae_step until the next call). */
lcae_status lcae_dx_device(lcae_layer *L, float **dx_dev);

/* Number of steps taken and of degenerate rows re-initialised so far. */
lcae_status lcae_counters(lcae_layer *L, int64_t *steps, int64_t *reinit_rows);

/* Overlap-add for model-parallel halos ("when a layer's input (or output) field spans
 * multiple GPUs"): dst[i][y0+y][x0+x][c] += src[i][y][x][c] for i<m, y<rows, x<cols, c<C.
 * dst is NHWC with row width dst_w, src is dense NHWC [m][rows][cols][C]; both device pointers,
 * ordered on `stream` (cudaStream_t). */
lcae_status lcae_region_add(void *stream, float *dst, int32_t dst_h, int32_t dst_w, const float *src,
                            int32_t m, int32_t rows, int32_t cols, int32_t C, int32_t y0, int32_t x0);

/* Kernel launches issued by the last lcae_step / lcae_forward on this handle (bench accounting). */
int32_t lcae_last_launch_count(lcae_layer *L);

/* Kernel timing for roofline accounting: enable = 1 starts recording CUDA events (on the layer's stream)
 * around the dominant fused step kernel of every subsequent lcae_step (on the general bf16 path, layers with
 * k > 128 / m > 256 / n > 4096: around each of its tcgen05 GEMM launches; up to 4096 ranges); enable = 0 stops.
 * lcae_profile_read synchronises and returns the summed duration (ms) and the number of recorded launches,
 * then clears the record. Events add no synchronisation inside the step. */
lcae_status lcae_profile(lcae_layer *L, int32_t enable);
lcae_status lcae_profile_read(lcae_layer *L, double *main_kernel_ms, int32_t *launches);

/* Thread-local description of the last error (never NULL). */
const char *lcae_last_error(void);

/* Library build string: "lcae <version> sm_100a". */
const char *lcae_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LCAE_H_ */
