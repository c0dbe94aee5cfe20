// kernels.h — host-side launchers of the CPI device kernels (internal to libcpi).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>   // types of the run-time loaded NCCL (comm.cu); libcpi does not link it

namespace cpi {

struct RoiDev {
    int x0, y0, w, h;
};

// Epilogue of the pair-sum GEMMs: exact Eq. (1) normalisation and/or int32 counts.
struct Epilogue {
    const int32_t* s_a;   // [P_a] totals (including this batch)
    const int32_t* s_b;   // [P_b]
    float* gamma;         // [P_a][ldg] or nullptr
    int64_t ldg;
    int32_t* counts;      // [P_a][ldc] or nullptr
    int64_t ldc;
    int accumulate;       // add the existing counts before storing / normalising
    int p_a, p_b;         // valid rows / columns
    int vec;              // 16-byte vector stores allowed (ldg, ldc, p_b multiples of 4)
    double n;             // N_TOT (all batches)
    double inv_n2;        // 1 / N_TOT^2 (kept for reference; kernels use make_gamma_scale(n))
    int cache;            // bit 0: Gamma stores evict-first (st.global.cs); bit 1: operand loads L2 evict_last
    int m_tile0;          // first M tile of this launch (row panels: cpi_correlate_rows)
    // fused cross-rank reduction (CPI_FUSED_REDUCE): when peers != nullptr the
    // epilogue adds each partial pair sum into the shard of the rank that owns its A row (peer
    // memory, red.global.add.s32) instead of writing local counts: A pixel row is owned by rank
    // (row / chunk_rows) % world, at local row (row / panel_rows) * chunk_rows + row % chunk_rows
    // of that rank's shard [rows][ldc].
    int32_t* const* peers;
    int world;
    int64_t chunk_rows, panel_rows;
    // symmetric pair sums (SYRK, roi_a == roi_b): tiles entirely below the diagonal
    // are skipped; a computed element (r, c) with c > r is written at (r, c) and (c, r), c < r not
    int symmetric;
};

// KB1: expand one RoI of packed frames into a K-major operand, zero-filling frames [n, k_pad),
// and accumulate the single-pixel sums into s[P].  mode: kExpandU8 bytes 0/1 (kind::i8),
// kExpandBits pixel-major 32-bit bit streams (popcount), kExpandE2M1 nibbles 0x0 / 0x2
// (E2M1 0.0 / 1.0, frame 2i in the low nibble of byte i; kind::mxf4).
enum { kExpandU8 = 0, kExpandBits = 1, kExpandE2M1 = 2 };
// order: operand row / sum slot of RoI pixel (m, j): kOrderRowMajor m * roi.w + j, kOrderUBlocked
// (j / 8) * (8 * roi.h) + 8 * m + j % 8 (CPI_GAMMA_UBLOCKED), kOrderVMajor j * roi.h + m
// (CPI_GAMMA_VMAJOR); the B arm follows the context's order, the A arm is always row-major.
enum { kOrderRowMajor = 0, kOrderUBlocked = 1, kOrderVMajor = 2 };
// v-major order (CPI_GAMMA_VMAJOR): B rows in blocks of kVMajorBlock (all H_b rows if H_b <= 128):
// pixel (u, v) -> (v / VB) * (W_b * VB) + u * VB + v % VB, VB = min(H_b, kVMajorBlock).  For one A
// pixel and one v block, every column u is one contiguous VB-row segment, and consecutive u are
// adjacent (DRAM pages stay open across consecutive refocus stages).
constexpr int kVMajorBlock = 128;
__host__ __device__ inline int vmajor_block(int Hb) { return Hb < kVMajorBlock ? Hb : kVMajorBlock; }
__host__ __device__ inline int64_t vmajor_slot(int u, int v, int Wb, int Hb) {
    const int vb = vmajor_block(Hb);
    return static_cast<int64_t>(v / vb) * Wb * vb + static_cast<int64_t>(u) * vb + v % vb;
}
void launch_expand(const uint8_t* frames, int64_t n, int row_bytes, int frame_h, int msb,
                   RoiDev roi, void* op, int64_t ld, int64_t k_pad, int32_t* s, int mode,
                   int order, cudaStream_t st);

// KB2: persistent tcgen05 kind::i8 GEMM  S = A^T B  (A: [M_pad][K] u8, B: [N_pad][K] u8,
// both K-major) with the fused epilogue.  k_blocks = K / 128.
cudaError_t launch_gemm_tc(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                           int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                           cudaStream_t st);
int gemm_tc_block_m();
int gemm_tc_block_n();
// KB2 CTA-pair variant (cta_group::2, M = N = 256 per pair, 6 stages).  Operand maps with
// 128-row boxes for both A and B; M_pad and N_pad multiples of 256.
cudaError_t launch_gemm_tc2(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                            int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                            cudaStream_t st);
int gemm_tc2_block_m();
int gemm_tc2_block_n();
int gemm_tc2_box_rows();
// KB2 FP4 variant (tcgen05 kind::mxf4, all block scales 2^0): E2M1 operands with 2 frames
// per byte, K-major, 128-B swizzle; M = 256, N = 224 per pair; k_blocks of 256 frames.
cudaError_t launch_gemm_f4(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                           int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                           cudaStream_t st);
int gemm_f4_block_n();
// f1: the CTA-pair kind::i8 GEMM fed with packed bit streams (uint32 [rows][k_pad / 32], KB1's
// popcount layout) that expansion warps unpack into the swizzled u8 stages in shared memory.
// Tensor maps: 2D uint32 (k_pad / 32 words, rows) with box (4, 128).  Plain epilogue only.
cudaError_t launch_gemm_bits(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles, int n_tiles,
                             int k_blocks, const Epilogue& epi, int num_sms, cudaStream_t st);
int gemm_f4_box_rows_b();

// KB3: popcount(AND) GEMM on CUDA cores over 32-bit bit streams [rows][ldw].
cudaError_t launch_gemm_popc(const uint32_t* a, const uint32_t* b, int64_t ldw, int64_t kw,
                             const Epilogue& epi, cudaStream_t st);
int gemm_popc_block();

// KB4: Gamma rows from int32 counts.
cudaError_t launch_finalize(const int32_t* counts, int64_t ldc, int64_t rows, int64_t p_b,
                            const int32_t* s_a_rows, const int32_t* s_b, double n, float* gamma,
                            int64_t ldg, cudaStream_t st);

// KB5/KB6 refocusing.  T (the stage-1 output, [W_a][H_a][H_b] per plane) is stored in fp32:
// the taps accumulate in fp32 per chunk and fp64 across chunks, and one rounding of the
// finished sum adds <= 2^-24 of T(|Gamma|) <= 2^-24 M to a plane; it halves
// the T traffic of both stages.
using TElem = float;
struct AxisTables {           // one axis (x with B-axis u, or y with B-axis v)
    int32_t* i0;              // [Wb][W]  lower interpolation index, -1 = sample skipped
    double* t;                // [Wb][W]  interpolation fraction
    int32_t* cnt;             // [W]      number of used samples per output coordinate
    int32_t* lo;              // [Wb]     min used i0 over outputs (INT_MAX if none)
    int32_t* hi;              // [Wb]     max used i0 + 1 over outputs (-1 if none)
};
// All coordinate tables of a fused plane group in two launches (tables + counts);
// map[f] = {ax, bx, cx, ay, by, cy} of plane f's A-axis maps.
struct CoordsGroupArgs {
    int Wa, Ha, Wb, Hb, boundary;
    double map[4][6];
    AxisTables xs[4], ys[4];
    double bmap[4][4];          // B-axis maps (ex, fx, ey, fy): c_B = ((e (u - c_b)) + f) + c_b;
                                // (1, 0, 1, 0) = integral B lattice (default).  A sample whose B
                                // coordinate leaves [0, W_b - 1] is skipped (skip policy).
    AxisTables bx[4], by[4];    // fractional-B path only: B support per u / v (i0 [W_b], t [W_b])
    int genb;                   // fill bx / by
};
cudaError_t launch_refocus_coords_group(const CoordsGroupArgs& g, int n_fuse, cudaStream_t st);
// General-B refocus (maps with fractional B coordinates that depend on u / v only): plain
// staged stage 1 with 2 x 2 corners per sample into T[x][m][n] for every (m, n), and a
// warp-per-pixel stage 2 with 2 x 2 corners.  Row-major Gamma, contiguous row shards.
cudaError_t launch_refocus_stage1_genb(const float* gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb,
                                       int m_base, int m_count, AxisTables xs, AxisTables bx, TElem* T,
                                       cudaStream_t st);
cudaError_t launch_refocus_stage2_genb(const TElem* T, int Wa, int Ha, int Hb, int m_base, int m_count,
                                       AxisTables xs, AxisTables ys, AxisTables by, float* plane, cudaStream_t st);
// General-B pre-pass (default route for fractional B): Gamma'(p; v, u) = bilinear of Gamma(p; ., .)
// at the B support (by[v], bx[u]) for rows A pixels of P_b slots each (B order row-major or
// u-blocked), so that the separable fast path runs Gamma' with the identity B map.  ey = the
// map's B-row scale (bounds the B support rows of a band: banded shared-memory form if small).
cudaError_t launch_resample_b(const float* src, float* dst, int64_t rows, int Wb, int Hb, int order, double ey,
                              AxisTables bx, AxisTables by, cudaStream_t st);
// plain staged stage 1 (fallback): row-major B order, or v-major with vmajor = 1
cudaError_t launch_refocus_stage1(const float* gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb,
                                  int m_base, int m_count, AxisTables xs, AxisTables ys,
                                  TElem* T, cudaStream_t st, int vmajor = 0);
// KB5 (TMA variant): warp-specialised, persistent, TMA-fed stage 1 over n_fuse (<= 4) planes
// sharing one pass over Gamma.  Needs W_a <= 256 with W_a % 4 == 0, W_b % 4 == 0, W_b <= 512, H_b <= 256, the tensor maps of
// Gamma (4D: u, v, j, m) and of the packed x-tables (3D uint32: x, u, plane slot).
constexpr int kRefocusMaxFuse = 4;
constexpr int kStage1MaxFuse = 2;   // planes per KB5 launch: x-tables and their fp32 weights share the ring
constexpr int kS2MaxPlanes = 16;   // planes per staged stage-2 launch (more CTAs in flight over T)
struct Stage1Maps {
    CUtensorMap gamma;       // 4D (u, v, j, m) row-major Gamma, or 5D (u%8, v, u/8, j, m) u-blocked
    CUtensorMap xtab;
    CUtensorMap xwtab;       // the x-tables' fp32 near-t weights (same shape)
    int gamma_5d = 0;
};
bool stage1_tma_supported(int Wa, int Wb, int Hb);
int stage1_vgroup(int Wa);   // B rows v per stage-1 tile (Gamma tensor-map box height)
cudaError_t launch_refocus_stage1_tma(const Stage1Maps* maps, int n_fuse, int Wa, int Ha, int Wb, int Hb,
                                      int m_base, int m_count, int m_block, int m_stride, const AxisTables* xs,
                                      const AxisTables* ys, TElem* const* T, const uint32_t* xblk, int num_sms,
                                      cudaStream_t st);
// x-tables of a fused group packed for the TMA stage 1: uint32 j_rel << 23 | round(t * 2^23),
// [n_fuse][Wb][Wa] (see refocus.cu), and xblk[n_fuse][ceil(Wb / 8)]: bit b set if some
// x in [16 b, 16 b + 16) has a used sample for some u of the 8-column chunk.
struct PackGroupArgs {
    int n;
    const int32_t* i0[kRefocusMaxFuse];
    const double* t[kRefocusMaxFuse];
    const int32_t* lo[kRefocusMaxFuse];
};
cudaError_t launch_pack_xtable_group(const AxisTables* xs, int n_fuse, int Wa, int Wb, uint32_t* xpack, float* xwpack,
                                     uint32_t* xblk, cudaStream_t st);
// General maps with output-dependent B coordinates (refocus_gen.cu, SPEC.md:273 with d != 0):
// per-axis tables [n_out][n_samp] of both supports, then two image-sampling stages.
struct GenMap { double a, b, c, d, e, f; };   // c_A = a (o - c) + b (s - c') + c ..., c_B = d (o - c) + e (s - c') + f ...
struct GenTables {
    int32_t* a0;   // A-lattice support (-1: sample skipped)
    float* at;
    int32_t* b0;   // B-lattice support
    float* bt;
    int32_t* cnt;  // [n_out] used samples
};
bool refocus_gen_supported(int Wa, int Ha, int Wb, int Hb);
cudaError_t launch_gen_axis(const GenMap& mp, int WA, int WB, int boundary, const GenTables& tab, cudaStream_t st);
// one plane: T (W_a H_a H_b fp32 workspace) from Gamma rows [m_base, m_base + m_count) (row-major B
// order, gamma points at the shard's first row), then the plane [H_a][W_a]
cudaError_t launch_refocus_gen(const float* gamma, int64_t pb, int Wa, int Ha, int Wb, int Hb, int m_base, int m_count,
                               const GenTables& xt, const GenTables& yt, TElem* T, float* plane, cudaStream_t st);
// KB5w (refocus_w.cu): stage 1 with window reuse along x, for Gamma in the v-major B order
// (CPI_GAMMA_VMAJOR).  One launch refocuses a batch of n_planes planes (groups of 4 share each
// staged slab); fp64 accumulators in TMEM.  Tensor maps: Gamma 4D (v, u, j, local m) with box
// (64, 1, 16, 1); step entries 3D uint32 (2 words per x, x padded to 128, u, plane) with box
// (256, 1, 4).  launch_pack_w fills ent (32-bit j0 | t table [plane][u][x_pad]), the spans, the
// m bands and the 64-bit step entries [plane][u][x_pad] from the coordinate tables.
struct S1WArgs {
    int Wa, Ha, Wb, Hb;
    int m_base, m_count, m_block, m_stride;   // shard rows (see S1Args)
    int n_planes;
    int n_groups, n_xt, n_vb;                 // filled by the launcher
    const int2* span;                         // [n_groups][n_xt][W_b] union j span per (group, x tile, u)
    const int2* mband;                        // [n_groups][n_vb] union A-row band read by stage 2
    float* T;                                 // plane p at T + p * t_plane: [W_a][H_a][H_b]
    int64_t t_plane;
    int probe;                                // timing probes (CPI_S1W_PROBE; 1/4/16 give wrong
                                              // values): 1 = no Gamma loads, 4 = no fp64 flushes,
                                              // 8 = non-suspending barrier waits, 16 = no step work
};
bool stage1_w_supported(int Wa, int Hb);
int stage1_w_xtile();      // outputs x per tile (entry table x padding)
int stage1_w_vblock();     // B rows v per tile (Gamma box width)
int stage1_w_group();      // planes per group (entry box depth)
int stage1_w_jbox();       // j rows per Gamma box
int stage1_w_max_span();   // staged j rows per stage (plane groups with a longer span use refocus.cu)
cudaError_t launch_pack_w(const int32_t* const* i0s_dev, const double* const* ts_dev, const int32_t* const* ylo_dev,
                          const int32_t* const* yhi_dev, int n_planes, int Wa, int Wb, int Hb, uint32_t* ent,
                          uint4* steps, int2* span, int2* mband, cudaStream_t st);
cudaError_t launch_refocus_stage1_w(const CUtensorMap* tm_gamma, const CUtensorMap* tm_ent, const S1WArgs& a,
                                    int num_sms, cudaStream_t st);
// driver entry point cuTensorMapEncodeTiled (nullptr if unavailable)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn();

cudaError_t launch_refocus_stage2(const TElem* T, int Wa, int Ha, int Hb, int m_base,
                                  int m_count, AxisTables xs, AxisTables ys, float* plane,
                                  cudaStream_t st);
// Shard A rows (both stages): local A row l is global row m_base + (l / m_block) * m_stride
// + l % m_block, l < m_count (m_block <= 0: contiguous).
// staged stage 2 (KB6'): one launch for n_fuse planes written to planes[f * Ha * Wa]; rows of
// T outside the shard count as 0.  Needs the packed y-tables [n_fuse][Hb][Ha] (H_a <= 256).
bool stage2_staged_supported(int Ha);
cudaError_t launch_pack_ytable_group(const AxisTables* ys, int n_fuse, int Ha, int Hb, uint2* ypack,
                                     cudaStream_t st);
cudaError_t launch_refocus_stage2_group(TElem* const* T, int n_fuse, int Wa, int Ha, int Hb, int m_base, int m_count,
                                        int m_block, int m_stride, const AxisTables* xs, const AxisTables* ys,
                                        const uint2* ypack, float* planes, cudaStream_t st);

// NCCL entry points, resolved from libnccl.so.2 at run time (comm.cu); nullptr if unavailable.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*);
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    const char* (*error_string)(ncclResult_t);
};
const NcclApi* nccl_api();
cudaError_t launch_f32_to_f64(const float* a, double* b, int64_t n, cudaStream_t st);
cudaError_t launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t st);

}  // namespace cpi
