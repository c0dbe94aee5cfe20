/*
 * cpi.h — C ABI of the B200 (sm_100a) Correlation Plenoptic Imaging hot path.
 *
 * The hot path (BASELINE.json north_star):
 *   binary SwissSPAD2 frames --(cpi_load_frames)--> device
 *     --(cpi_correlate)--> on-device int8 expansion + single-pixel sums S_a, S_b
 *                          + pair sums S_ab = A^T B on tcgen05 kind::i8 tensor cores
 *                          + fused exact normalisation into fp32 Gamma
 *     --(cpi_finalize)-->  Gamma from kept counts when not fused
 *     --(cpi_refocus)-->   stack of refocused planes.
 *
 * Citations: P:NNN = PAPER.md line (arXiv 2407.20692), S:NNN = SPEC.md line.
 *
 * Conventions shared by every entry point
 *   - Every function returns cpi_status (0 = CPI_OK, < 0 = error).  None throws, none
 *     exits, none prints.  On error the context keeps a message (cpi_last_error) and is
 *     left in the state it had before the call, except for CPI_ERR_CUDA (sticky device
 *     errors: destroy the context).
 *   - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Kernel faults surface at a later call or at
 *     stream synchronisation as CPI_ERR_CUDA.
 *   - Ownership: the caller owns every buffer it passes (inputs and outputs, device or
 *     host); the library owns its workspaces (expanded operands, counts, refocus
 *     scratch) until cpi_destroy.  Device pointers must be allocated on cfg.device.
 *   - Pixel indexing inside a RoI: p = m * width + j, j horizontal (fastest), m
 *     vertical, 0-based (P:69 uses 1-based j,k).  Gamma is row-major
 *     [P_a][P_b]: Gamma_jkmn of Eq. (1) is gamma[(m*W_a + j) * P_b + (n*W_b + k)].
 */
#ifndef CPI_H_
#define CPI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t cpi_status;

/* Status codes (names mirror SPEC's errors where one exists). */
#define CPI_OK                      0
#define CPI_ERR_INVALID_ARG        (-1)  /* NULL pointer, negative size, bad enum */
#define CPI_ERR_LAYOUT             (-2)  /* frame width/height not positive multiples of 8 */
#define CPI_ERR_ROI_OUT_OF_BOUNDS  (-3)  /* RoI not fully inside the frame */
#define CPI_ERR_SIZE_MISMATCH      (-4)  /* byte count not a whole number of frames */
#define CPI_ERR_CAPACITY           (-5)  /* more frames than cfg.max_frames in one batch */
#define CPI_ERR_ZERO_FRAMES        (-6)  /* finalize / Gamma requested with N_TOT = 0 */
#define CPI_ERR_DEGENERATE_ALPHA   (-7)  /* alpha = 0 or non-finite under the default map */
#define CPI_ERR_EMPTY_ANGULAR_GRID (-8)  /* n_planes < 1 or empty B lattice */
#define CPI_ERR_STATE              (-9)  /* call out of order (e.g. correlate before load) */
#define CPI_ERR_CUDA               (-10) /* CUDA runtime/driver failure or no sm_100 device */
#define CPI_ERR_OOM                (-11) /* device allocation failure */
#define CPI_ERR_UNSUPPORTED        (-12) /* feature not available for this configuration */
#define CPI_ERR_NCCL               (-13) /* NCCL unavailable (libnccl.so.2 not loadable) or an NCCL call failed */

/* Frame layout.  bit_order: column c of a row is bit (c % 8) of
 * byte c/8 (CPI_LSB_FIRST, declared convention S:110) or bit 7 - c % 8 (CPI_MSB_FIRST). */
#define CPI_LSB_FIRST 0
#define CPI_MSB_FIRST 1

/* Where cpi_load_frames' pointer lives. */
#define CPI_HOST   0   /* host memory (pinned gives async H2D; pageable is staged by CUDA) */
#define CPI_DEVICE 1   /* device memory on cfg.device, used in place (not copied): it must
                          stay valid and unmodified until the next cpi_correlate completes */

/* cpi_config.flags */
#define CPI_VARIANT_TC    0u  /* S_ab on tcgen05 kind::i8 tensor cores (default) */
#define CPI_VARIANT_POPC  1u  /* S_ab as popcount(a AND b) on CUDA cores */
#define CPI_KEEP_COUNTS   2u  /* keep int32 S_ab [P_a][P_b] in a library workspace: needed for
                                 multi-batch accumulation, cpi_get_counts of S_ab,
                                 and cpi_finalize from counts.  Costs 4*P_a*P_b bytes. */
#define CPI_VARIANT_FP4   4u  /* S_ab on tcgen05 kind::mxf4 (block-scaled FP4) tensor cores: bits
                                 expanded to E2M1 0.0 / 1.0 (2 frames per byte), all block scales
                                 2^0, fp32 accumulation -- every partial sum is an integer
                                 < 2^24, so S_ab is exact for batches of < 2^24 frames; twice the
                                 int8 MMA rate.  Exclusive with CPI_VARIANT_POPC. */
#define CPI_VARIANT_TC_BITS 64u /* SURVEY f1 ("bit unpacking and cross-correlation calculation
                                 occur jointly in the same kernel"): the expansion writes pixel-major
                                 bit streams (1 bit per frame, 1/8 of the u8 operand bytes) and the
                                 CTA-pair kind::i8 GEMM TMA-loads them and unpacks each stage into
                                 the swizzled u8 operand tiles in shared memory (expansion warps,
                                 fence.proxy.async, then the MMA).  Same exact int32 S_ab.
                                 Exclusive with CPI_VARIANT_POPC / CPI_VARIANT_FP4; plain epilogue
                                 (no CPI_FUSED_REDUCE, no SYRK). */
#define CPI_GAMMA_UBLOCKED 8u /* B pixels are ordered u-blocked everywhere in this context: B pixel
                                 q = v*W_b + u has index (u/8)*(8*H_b) + 8*v + u%8 in S_b, in the
                                 columns of S_ab and of every Gamma it writes or cpi_refocus reads
                                 (A pixels and rows unchanged).  The GEMM then produces, and
                                 refocusing stages, each 8 u x 8 v block as one contiguous 256-B
                                 segment (faster refocus, same arithmetic).  Needs
                                 roi_b.width % 8 == 0. */
#define CPI_GAMMA_VMAJOR  16u /* B pixels are ordered v-major in blocks of VB = min(H_b, 128) rows
                                 everywhere in this context: B pixel q = v*W_b + u has index
                                 (v / VB)*(W_b*VB) + u*VB + v % VB in S_b, in the columns of S_ab
                                 and of every Gamma it writes or cpi_refocus reads.  For one A
                                 pixel, one v block and one B column u the VB values are
                                 contiguous (and consecutive u adjacent), which is what the window
                                 stage 1 (KB5w) stages: all lanes of a warp share one
                                 (x, u) sample and reuse the two Gamma rows of neighbouring outputs
                                 from registers.  Needs roi_b.height % 4 == 0 and, above 128, a
                                 multiple of 128; exclusive with CPI_GAMMA_UBLOCKED.  Refocusing spans longer than
                                 the kernel's stage (A-axis map slopes above ~2.2) and W_a > 256 run
                                 a plain staged stage 1 (contiguous row shards only). */
#define CPI_FUSED_REDUCE 32u /* multi-GPU only: the pair-sum GEMM epilogue adds each
                                 finished partial tile straight into the shard of the rank that owns
                                 its A rows (red.global.add.s32 into peer memory mapped with CUDA IPC;
                                 NVLink between GPUs), instead of writing a full-size local partial
                                 and reduce-scattering it: no 4 P_a P_b-byte local partial, no
                                 separate reduction pass, the exchange overlaps the GEMM tile by
                                 tile.  Exact: integer adds.  CTA-pair tensor-core variants only.
                                 With nccl_id the library maps the peers itself (handles
                                 all-gathered over its communicator) and cpi_reset / cpi_finalize
                                 order the ranks; without nccl_id (external mode) the caller
                                 exchanges cpi_shard_ipc_handle bytes, calls cpi_open_peer_shards,
                                 and orders the ranks itself (all shards zeroed by cpi_reset before
                                 any rank correlates; all correlates done before the shard,
                                 cpi_counts_dev's s_ab, is read). */
#define CPI_SHARD_HANDLE_BYTES 64

/* Boundary policy of refocusing. */
#define CPI_SKIP_RENORMALIZE 0  /* sample counts only if 0 <= c_A <= W-1 on both axes; mean */
#define CPI_CLAMP            1  /* c_A clamped into [0, W-1]; every sample counts */

typedef struct {
    int32_t x0, y0, width, height;   /* 0-based inclusive top-left, size in px */
} cpi_roi;

typedef struct {
    int32_t width_px, height_px, bit_order;   /* SwissSPAD2: 512, 256, CPI_LSB_FIRST */
} cpi_layout;

typedef struct {
    cpi_layout layout;
    cpi_roi roi_a, roi_b;   /* spatial arm rho_a (image A) and angular arm rho_b (image B),
                               P:68-69: A = left half, B = right half for the paper's data */
    int64_t max_frames;     /* capacity of one cpi_load_frames batch (>= 1) */
    int32_t device;         /* CUDA device ordinal; must be compute capability 10.0 */
    uint32_t flags;         /* CPI_VARIANT_* | CPI_KEEP_COUNTS | CPI_GAMMA_* */
    /* Frame-sharded multi-GPU mode (north_star; one context per GPU, one process per
     * GPU): world >= 2 makes this context rank `rank` of `world`.  cpi_create then joins a library-
     * owned NCCL communicator (collective: every rank must call cpi_create) identified by nccl_id
     * (CPI_NCCL_ID_BYTES bytes from cpi_nccl_unique_id on one rank, shared out of band), and needs
     * CPI_KEEP_COUNTS and H_a % world == 0.  Each rank loads and correlates its own contiguous
     * slice of the frame sequence (Eq. (1)'s sums are additive); cpi_finalize reduces
     * across ranks and finalises the rank's own Gamma rows; cpi_refocus from the current totals
     * (gamma_dev NULL) refocuses them and all-reduces the planes.  world == 1 with a non-NULL
     * nccl_id runs the same multi-GPU code path as a one-rank group.  Otherwise (world <= 1, no id):
     * single GPU (a zero-initialised config is a single-GPU config). */
    int32_t rank, world;
    const uint8_t *nccl_id;
} cpi_config;

#define CPI_NCCL_ID_BYTES 128

typedef struct {
    const double *alphas;   /* HOST array of n_planes refocusing parameters alpha (finite, != 0) */
    int32_t n_planes;       /* >= 1 */
    int32_t boundary;       /* CPI_SKIP_RENORMALIZE | CPI_CLAMP */
    const float *gamma_dev; /* DEVICE Gamma rows [row0, row0 + rows) of [P_a][P_b], row-major,
                               leading dimension P_b (e.g. cpi_correlate's output), or NULL:
                               refocus this context's current totals (SURVEY §8(b)
                               CPI_FROM_COUNTS) -- the Gamma the last cpi_correlate /
                               cpi_finalize wrote, else Gamma finalised from the kept counts
                               into a library workspace (CPI_KEEP_COUNTS, 4 P_a P_b bytes);
                               then row0 = 0, rows = P_a. */
    int64_t row0, rows;     /* multiples of roi_a.width; a single GPU passes 0, P_a.  A row
                               shard yields that shard's additive share of every plane. */
    int32_t row_block;      /* A-row layout of the shard (SURVEY §8(e) load balance): the
                               shard's local A-row l is global A-row
                                 m(l) = row0/W_a + (l / row_block) * row_stride + l % row_block,
                               i.e. blocks of row_block consecutive A-rows every row_stride
                               A-rows (block-cyclic ownership).  row_block <= 0: contiguous
                               (m(l) = row0/W_a + l).  Needs row_stride >= row_block. */
    int32_t row_stride;
    const double *affine;   /* HOST [n_planes][12] general RefocusMap per plane (SURVEY
                               f3(ii)), or NULL for the default map from alphas.  Row
                               {ax, bx, cx, dx, ex, fx, ay, by, cy, dy, ey, fy}, coordinates
                               relative to the arm centres c = (W-1)/2:
                                 c_Ax = ax (x - c_ax) + bx (u - c_bx) + cx + c_ax
                                 c_Bx = dx (x - c_ax) + ex (u - c_bx) + fx + c_bx
                               (y, v likewise; evaluated left to right in fp64).  A sample counts
                               only if all four coordinates lie on their lattices (skip policy).
                               B coordinates independent of the output pixel (dx = dy = 0):
                               integral B (ex = ey = 1, fx = fy = 0) runs the
                               fast separable kernels directly.  Any other (ex, fx, ey, fy):
                               the library resamples Gamma onto the B lattice once per distinct
                               B map (a rows x P_b fp32 workspace, allocated on first use and
                               kept) and runs the same fast kernels, consecutive planes with
                               one B map fused; if that workspace cannot be allocated it falls
                               back to general-B kernels (2 x 2 corners per stage, row-major B
                               order, contiguous row shards only).  dx or dy != 0 (B
                               coordinates depending on the output pixel): per-axis support
                               tables and two image-sampling stages (refocus_gen.cu; row-major
                               B order, A RoIs up to 256 px per side, contiguous row shards;
                               otherwise CPI_ERR_UNSUPPORTED).  The default map is
                               {a, 1 - a, 0, 0, 1, 0} on both axes. */
} cpi_refocus_spec;

typedef struct cpi_ctx cpi_ctx;   /* opaque, owned by the library */

/* Create a context on cfg->device: validates the layout and RoIs, allocates
 * the expanded-operand workspaces for max_frames, the marginals and (CPI_KEEP_COUNTS) the
 * counts, and encodes the TMA descriptors.  *out is set only on success.
 * Errors: INVALID_ARG, LAYOUT, ROI_OUT_OF_BOUNDS, CUDA (no sm_100 device), OOM. */
cpi_status cpi_create(const cpi_config *cfg, cpi_ctx **out);

/* Release every library-owned resource.  NULL is a no-op.  Synchronises the device. */
void cpi_destroy(cpi_ctx *ctx);

/* Message for the last error on ctx (never NULL; "" when none).  ctx may be NULL (then
 * the message of the last failed cpi_create on this thread). */
const char *cpi_last_error(const cpi_ctx *ctx);

/* Static name of a status code. */
const char *cpi_status_string(cpi_status s);

/* Load one batch of n_frames whole packed frames (frame-major, row-major, 1 bpp,
 * layout.width_px/8 bytes per row: "Input Dataset") as the input of the
 * next cpi_correlate.  where = CPI_HOST: asynchronous copy into one of two device staging
 * buffers on an internal copy stream, so it overlaps the compute of the previous batch; the
 * next cpi_correlate makes `stream` wait for it.  The host buffer must stay unchanged until
 * the work of that cpi_correlate has completed on `stream` (pinned memory gives a truly
 * asynchronous copy).  where = CPI_DEVICE uses the pointer in place.  Errors: INVALID_ARG,
 * CAPACITY (n_frames > max_frames), CUDA.  n_frames = 0 is allowed (the next correlate adds
 * nothing). */
cpi_status cpi_load_frames(cpi_ctx *ctx, const void *packed, int64_t n_frames, int32_t where,
                           void *stream);

/* Dataset files ("Input Dataset": sets of headerless .bin files, 8 MiB = 512 frames
 * each; S:57-64 parse_bin_file, S:91-100 scan_dataset).  Host-only: these two need no device
 * and no context.  A file is a whole number of packed frames of `layout`
 * (width_px/8 * height_px bytes each) and nothing else.
 *   cpi_bin_frames: *n_frames = file size / frame bytes.  Errors: INVALID_ARG (NULL, bad
 *     layout -> LAYOUT), SIZE_MISMATCH (size not a multiple of the frame bytes), CUDA is
 *     never returned; an unreadable file is INVALID_ARG with the errno text in
 *     cpi_last_error(NULL).  An empty file has 0 frames.
 *   cpi_read_bin: copies frames [frame0, frame0 + n_frames) of the file, bit for bit, into
 *     the caller's host buffer `dst` (n_frames * frame bytes; pinned memory can then go straight
 *     to cpi_load_frames).  Errors: INVALID_ARG (NULL, negative range, range past the end of
 *     the file, read failure), LAYOUT, SIZE_MISMATCH.
 * Ordering of a dataset's files (SPEC scan_dataset: lexicographic) is the caller's; the Python
 * binding's scan_dataset sorts names and checks that every file has the same frame count. */
cpi_status cpi_bin_frames(const char *path, const cpi_layout *layout, int64_t *n_frames);
cpi_status cpi_read_bin(const char *path, const cpi_layout *layout, int64_t frame0, int64_t n_frames, void *dst);

/* Accumulate the loaded batch into the context's sums (Eq. (1) numerators):
 *   S_a[p] += sum_i A^i_p,  S_b[q] += sum_i B^i_q,  N_TOT += n_frames,
 *   S_ab[p][q] += sum_i A^i_p B^i_q   (int32, exact; N_TOT < 2^31)
 * on the device: bits are expanded to K-major uint8 operands ("bit-unpacking") and
 * S_ab runs on tcgen05 kind::i8 (CPI_VARIANT_TC), kind::mxf4 (CPI_VARIANT_FP4) or popcount(AND)
 * (CPI_VARIANT_POPC).
 * If gamma_dev != NULL the GEMM epilogue also writes Gamma for the accumulated totals
 * (fused normalisation, see cpi_finalize for the formula) into gamma_dev [P_a][P_b].
 * Without CPI_KEEP_COUNTS only one correlate per cpi_reset is allowed (nothing to
 * accumulate into) and gamma_dev must be non-NULL.
 * Errors: STATE (nothing loaded; second batch without KEEP_COUNTS; no output at all),
 * CUDA. */
cpi_status cpi_correlate(cpi_ctx *ctx, float *gamma_dev, void *stream);

/* Row panel of cpi_correlate, for pipelining the multi-GPU reduction with the GEMM (SURVEY
 * §8(e): "panelise the GEMM over p_a row blocks and launch each panel's RS as soon as it is
 * done"): the same accumulation restricted to A pixels [row0, row0 + rows):
 *   S_ab[p][q] += sum_i A^i_p B^i_q  for row0 <= p < row0 + rows  (+ Gamma rows if gamma_dev)
 * The first cpi_correlate_rows of a loaded batch also expands it and adds its S_a, S_b and
 * N_TOT (so Gamma rows use the totals including this batch); later calls on the same batch
 * only run the GEMM.  The caller must cover every row exactly once per batch; rows not
 * covered miss that batch's pair sums.  gamma_dev, if non-NULL, is the full [P_a][P_b]
 * buffer (only the panel's rows are written).  row0 must be a multiple of
 * cpi_row_align(ctx); rows too unless row0 + rows == P_a.
 * Errors: STATE (nothing loaded; batch already consumed by cpi_correlate; no output),
 * INVALID_ARG (range / alignment), CUDA. */
cpi_status cpi_correlate_rows(cpi_ctx *ctx, int64_t row0, int64_t rows, float *gamma_dev, void *stream);

/* cpi_correlate_rows writing the panel's Gamma rows compactly: gamma_rows_dev (non-NULL) is
 * fp32 [rows][P_b] holding A pixels row0 .. row0 + rows - 1 (output-tile sharding: a rank
 * computes only the Gamma rows it owns, over all frames, without a full-size buffer).
 * Errors as cpi_correlate_rows. */
cpi_status cpi_correlate_rows_to(cpi_ctx *ctx, int64_t row0, int64_t rows, float *gamma_rows_dev, void *stream);

/* Row alignment (A pixels) of cpi_correlate_rows panels for this context's GEMM variant. */
int64_t cpi_row_align(const cpi_ctx *ctx);

/* Borrow the device pointers of the accumulated sums (valid until cpi_destroy; contents
 * change with every correlate / reset): s_ab int32 [P_a][P_b] (NULL without
 * CPI_KEEP_COUNTS; with CPI_FUSED_REDUCE this rank's reduced shard [owned A pixels][P_b], see
 * cpi_finalize for the row layout), s_a int32 [P_a], s_b int32 [P_b] (this rank's frames).  Lets a caller run collectives on the
 * library's buffers without copies.  Any out pointer may be NULL.  Errors: INVALID_ARG. */
cpi_status cpi_counts_dev(cpi_ctx *ctx, int32_t **s_ab, int32_t **s_a, int32_t **s_b);

/* Gamma of Eq. (1) from the accumulated sums:
 *   Gamma[p][q] = (N*S_ab[p][q] - S_a[p]*S_b[q]) / N^2   (= (1/N) S_ab - (S_a/N)(S_b/N))
 * with the numerator formed exactly (integer) and one rounding to fp32.
 * Single GPU: if the last cpi_correlate already wrote Gamma for the current totals and gamma_dev
 * is NULL or that same buffer, nothing is launched.  Otherwise needs CPI_KEEP_COUNTS; gamma_dev is
 * [P_a][P_b].  *row0 = 0, *rows = P_a.
 * Multi-GPU (cfg.world >= 2, or a one-rank group): the cross-rank reduction runs here, stream-ordered on
 * `stream` over the library's NCCL communicator: C2 all-reduce of [S_a | S_b | N] (int32) and C1
 * reduce-scatter of the int32 partial S_ab in row panels, so that this rank receives the exact
 * totals of its own A rows, which it finalises into gamma_dev (compact [rows][P_b], may be NULL:
 * a library workspace, then refocus with gamma_dev = NULL).  The owned rows are block-cyclic (load
 * balance of refocusing for alpha < 1): local Gamma row r is A pixel
 *   p(r) = (row0 / W_a + (r / W_a / row_block) * row_stride + (r / W_a) % row_block) * W_a + r % W_a
 * with row_block, row_stride from cpi_shard_layout; *row0 = first owned A pixel, *rows = owned
 * A pixels.  Integer sums: Gamma is bit-identical for any world size.
 * Outputs n_tot (global N_TOT), row0, rows are optional.  Errors: ZERO_FRAMES, STATE, INVALID_ARG,
 * CUDA, NCCL. */
cpi_status cpi_finalize(cpi_ctx *ctx, float *gamma_dev, int64_t *n_tot, int64_t *row0, int64_t *rows,
                        void *stream);

/* Block-cyclic ownership of this rank's Gamma rows (see cpi_finalize): blocks of row_block A rows
 * every row_stride A rows, starting at A row row0 / W_a.  Single GPU: row_block = row_stride = H_a.
 * Either pointer may be NULL.  Errors: INVALID_ARG. */
cpi_status cpi_shard_layout(const cpi_ctx *ctx, int32_t *row_block, int32_t *row_stride);

/* CPI_FUSED_REDUCE: the CUDA IPC handle (CPI_SHARD_HANDLE_BYTES bytes) of this rank's shard of
 * the pair sums ([owned A pixels][P_b] int32), for cpi_open_peer_shards on the other ranks.
 * Errors: INVALID_ARG, STATE (not fused), CUDA. */
cpi_status cpi_shard_ipc_handle(cpi_ctx *ctx, uint8_t *handle);

/* CPI_FUSED_REDUCE, external mode: map every rank's shard (handles[r * CPI_SHARD_HANDLE_BYTES ..]
 * from cpi_shard_ipc_handle of rank r; this rank's own entry is ignored) so that the GEMM
 * epilogue can add into it.  Once per context.  Errors: INVALID_ARG, STATE, CUDA. */
cpi_status cpi_open_peer_shards(cpi_ctx *ctx, const uint8_t *handles);

/* A new NCCL unique id (CPI_NCCL_ID_BYTES bytes into id) for the cpi_config.nccl_id of a
 * multi-GPU group: call on one rank, share the bytes with the others (any out-of-band channel).
 * Errors: INVALID_ARG, NCCL (libnccl.so.2 unavailable). */
cpi_status cpi_nccl_unique_id(uint8_t *id);

/* Stateless finalisation of an externally reduced row shard (frame-sharded multi-GPU:
 * SURVEY §8(e), after an all-reduce of S_a/S_b/N and a reduce-scatter of S_ab rows):
 *   gamma_rows[r][q] = Gamma(s_ab_rows[r][q], s_a[row0 + r], s_b[q], n_tot)
 * s_ab_rows: device int32 [rows][P_b]; s_a: device int32 [P_a]; s_b: device int32 [P_b];
 * gamma_rows: device fp32 [rows][P_b].  Errors: INVALID_ARG, ZERO_FRAMES, CUDA. */
cpi_status cpi_finalize_counts(cpi_ctx *ctx, const int32_t *s_ab_rows, int64_t row0, int64_t rows,
                               const int32_t *s_a, const int32_t *s_b, int64_t n_tot,
                               float *gamma_rows, void *stream);

/* Copy the accumulated sums to caller device buffers (audit / bit-exact tests / multi-GPU
 * reduction).  Any pointer may be NULL.  s_ab_dev (int32 [P_a][P_b]) needs
 * CPI_KEEP_COUNTS.  *n_tot receives N_TOT.  Errors: STATE, CUDA. */
cpi_status cpi_get_counts(cpi_ctx *ctx, int32_t *s_ab_dev, int32_t *s_a_dev, int32_t *s_b_dev,
                          int64_t *n_tot, void *stream);

/* Zero the accumulated sums (start a new acquisition). */
cpi_status cpi_reset(cpi_ctx *ctx, void *stream);

/* Refocus Gamma into a stack of planes ("Refocusing").
 * Multi-GPU contexts with spec->gamma_dev = NULL refocus this rank's own Gamma rows (those the
 * last cpi_finalize produced) and all-reduce the planes in fp64, so every rank
 * returns the whole stack (each rank's fp32 share is within 2^-24 of its own M, M is additive over
 * row shards, so the sum meets the single-GPU 1e-6 M bar).  With an explicit gamma_dev a
 * multi-GPU context refocuses that shard only (no reduction), as a single-GPU context does.
 * For plane alpha and output pixel (x, y) of the A lattice,
 *   R(x,y) = (1/count) * sum over B lattice (u, v) of the multilinear interpolation of
 *            Gamma at A coordinates
 *              c_x = alpha*(x - c_ax) + (1 - alpha)*(u - c_bx) + c_ax
 *              c_y = alpha*(y - c_ay) + (1 - alpha)*(v - c_by) + c_ay
 *            and B coordinates (u, v)  (SPEC default map S:274, centres c = (W-1)/2),
 *   samples outside [0, W_a-1] x [0, H_a-1] skipped (CPI_SKIP_RENORMALIZE) or clamped,
 *   count = number of samples used, R = 0 when count = 0.
 * The B coordinates are integers, so the 16-corner interpolation is the bilinear one on
 * the A axes; the kernels evaluate it separably (stage 1 over x, stage 2 over y), fp64
 * coordinates, fp32 taps summed in fp64.
 * planes_dev: device fp32 [n_planes][H_a][W_a].  Needs W_a, H_a >= 2.
 * Errors: INVALID_ARG, DEGENERATE_ALPHA, EMPTY_ANGULAR_GRID, UNSUPPORTED, OOM, CUDA. */
cpi_status cpi_refocus(cpi_ctx *ctx, const cpi_refocus_spec *spec, float *planes_dev,
                       void *stream);

/* Number of kernels this context has launched so far (for launch accounting). */
int64_t cpi_launch_count(const cpi_ctx *ctx);

/* Per-kernel timing: when enabled, the library records CUDA events around its main
 * kernels on the launching stream; cpi_kernel_time_ms returns the accumulated device time
 * of one kernel class since the last reset (0 = GEMM, 1 = expand, 2 = refocus stage 1,
 * 3 = refocus stage 2, 4 = finalize, 5 = refocus coords, 6 = fractional-B resample) and its
 * launch count.
 * Enabling timing synchronises each timed launch's end event lazily (at query time). */
cpi_status cpi_set_timing(cpi_ctx *ctx, int32_t enable);
cpi_status cpi_kernel_time_ms(cpi_ctx *ctx, int32_t kernel_class, double *ms, int64_t *launches);

/* ABI version (major * 100 + minor): 201 = 2.01 (2.00 + cpi_bin_frames / cpi_read_bin and
 * CPI_VARIANT_TC_BITS). */
int32_t cpi_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPI_H_ */
