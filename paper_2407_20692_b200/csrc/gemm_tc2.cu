// gemm_tc2.cu — KB2 (CTA-pair variant): S_ab = A^T B of Eq. (1) on
// tcgen05 tensor cores with two SMs per MMA (cta_group::2), fused exact normalisation
// (P:100-111).
//
// A pair of CTAs (cluster of 2) owns a 256 x 256 output tile.  Each CTA TMA-loads its own
// 128-row half of the A panel and its own 128-row half of the B panel (128 B of K each) into
// a 6-stage ring; the transaction bytes of both halves are counted on the leader CTA's
// barrier.  The leader's single MMA thread issues tcgen05.mma.cta_group::2.kind::i8 with
// M = 256, N = 256, K = 32: the tensor cores of both SMs read A rows from their own smem and
// the two B halves from both, and each CTA's TMEM receives its 128 rows x 256 columns.
// Commits are multicast to both CTAs (smem slots free, accumulator full); both CTAs'
// epilogue warps release an accumulator on the leader's barrier.  Per SM this halves the
// B-panel L2->SMEM traffic of the 1-CTA kernel (32 KB instead of 48 KB per 512 MMA
// cycles) and leaves room for 6 stages.
#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

// kF4 = false: kind::i8, u8 operands (1 frame per byte), BN = 256, accumulators in TMEM
//              columns [0, 512).
// kF4 = true:  kind::mxf4 block-scaled, E2M1 operands (2 frames per byte), BN = 224 so that
//              the two accumulators (448 columns) leave room for the scale factors (all
//              2^0 = UE8M0 127) in columns [448, 480); fp32 accumulators hold exact integers.
// BK = 128 bytes of K per stage in both (128 frames i8, 256 frames fp4); each MMA consumes
// 32 bytes of K (K = 32 u8 or K = 64 e2m1).
template <bool kF4>
struct Tc2 {
    static constexpr int BM = 256, BN = kF4 ? 224 : 256, BK = 128;
    static constexpr int HM = BM / 2, HN = BN / 2;          // per-CTA halves
    static constexpr int kStages = 6;
    static constexpr int kABytes = HM * BK;                 // 16 KB
    static constexpr int kBBytes = HN * BK;                 // 16 / 14 KB
    static constexpr int kStageBytes = kABytes + kBBytes;   // per CTA
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256 + 2 * BN * 4;
    static constexpr uint32_t kSfCol = 448;                 // fp4: SFA at 448, SFB at 464
    // f1 (bits mode, kind::i8 only): the packed bit streams of a stage (16 B per operand row) land
    // by TMA in a small ring after the S_b staging; expansion warps write the u8 operand stage
    static constexpr int kOffBits = kStages * kStageBytes + 256 + 2 * BN * 4;
    static constexpr int kBitsStage = (HM + HN) * 16;       // 4 KB
    static constexpr int kBitsSmem = kSmemBytes + kStages * kBitsStage;
};
constexpr int BM = 256, BK = 128;
constexpr int kThreads = 192;
constexpr int kExpGroups = 4;                     // f1: groups of 4 expansion warps, stage s to group s % kExpGroups
constexpr int kExpWarps = 4 * kExpGroups;
constexpr int kThreadsBits = kThreads + 32 * kExpWarps;
constexpr int kTmemCols = 512;
constexpr int kGroupM = 8;                        // pair-tile rows per raster group

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& tm, int& tn) {
    const int group = kGroupM * n_tiles;
    const int g = t / group;
    const int first_m = g * kGroupM;
    const int gm = min(m_tiles - first_m, kGroupM);
    const int r = t - g * group;
    tm = first_m + r % gm;
    tn = r / gm;
}

// Epilogue modes, compiled separately so the plain kernel carries none of the others' code:
// plain (counts / fused Gamma), f2 peer reduction (epi.peers), SYRK (epi.symmetric).
enum EpiMode { kEpiPlain = 0, kEpiPeers = 1, kEpiSyrk = 2 };

// SYRK: a tile with no element on or above the diagonal (every column < every row) is not computed
template <int kMode>
__device__ __forceinline__ bool below_diagonal(int tm, int tn, int bn) {
    return kMode == kEpiSyrk && (tn + 1) * bn - 1 < tm * BM;
}

// f1: 16 packed frames (16 bits) of one operand row -> 16 u8 bytes (0 / 1), frame f in byte f
__device__ __forceinline__ uint4 bits_to_u8(uint32_t b16) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = (((b16 >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;   // bit k -> byte k
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// kBits (f1, SURVEY §8(f) "unpack fused into the GEMM producer"): the operands arrive as
// pixel-major bit streams (bit f % 32 of word f / 32 = frame f, KB1's popcount layout); per stage
// the producer TMA-loads 16 B of bits per operand row and kExpWarps expansion warps write the
// 128-B swizzled u8 rows the MMA reads (fence.proxy.async, then an arrive on the leader's stage
// barrier: 2 CTAs x kExpWarps arrivals instead of TMA transaction bytes).
template <bool kF4, int kMode, bool kBits = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kBits ? kThreadsBits : kThreads, 1)
gemm_i8_tc2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   int m_tiles, int n_tiles, int k_blocks, Epilogue epi) {
    using P = Tc2<kF4>;
    constexpr int BN = P::BN, HM = P::HM, HN = P::HN, kStages = P::kStages;
    constexpr int kABytes = P::kABytes, kBBytes = P::kBBytes, kStageBytes = P::kStageBytes;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint64_t* bfull = reinterpret_cast<uint64_t*>(tmem_slot + 2);   // f1: bits stage landed (this CTA)
    int32_t* sb_stage = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 256);   // [2][BN]
    uint8_t* sbits = smem + P::kOffBits;                             // f1: [kStages][HM + HN][16 B]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    constexpr int kProdWarp = 4, kMmaWarp = 5;   // highest warp ids win the issue arbiter
    if (warp == kProdWarp && lane == 0) {
        tma_prefetch_desc(&tma_a);
        tma_prefetch_desc(&tma_b);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], kBits ? 8 : 1);   // leader: arrive.expect_tx (TMA), or 4 expansion warps x 2 CTAs
            mbar_init(&empty[s], 1);     // one multicast commit per stage
            if (kBits) mbar_init(&bfull[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);     // one multicast commit per tile
            mbar_init(&tempty[a], 8);    // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc_2sm(tmem_slot, kTmemCols);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if constexpr (kF4) {
        // block scale factors 2^0 (UE8M0 127) in every lane of the SF columns of both CTAs
        if (warp < 4) {
            const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(32 * warp) << 16) + P::kSfCol;
            tmem_fill_x16(lane_base, 0x7F7F7F7Fu);
            tmem_fill_x16(lane_base + 16, 0x7F7F7F7Fu);
        }
        tc_fence_before();
        cluster_sync();
        tc_fence_after();
    }
    const int num_tiles = m_tiles * n_tiles;
    const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

    if (warp == kProdWarp) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol = l2_policy_evict_last();
            for (int t = pair; t < num_tiles; t += num_pairs) {
                int tm, tn;
                tile_coords(t, m_tiles, n_tiles, tm, tn);
                tm += epi.m_tile0;
                if (below_diagonal<kMode>(tm, tn, BN)) continue;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if constexpr (kBits) {   // this CTA's rows of the packed bits (4 words = 128 frames each)
                        uint8_t* dst = sbits + stage * P::kBitsStage;
                        mbar_expect_tx(&bfull[stage], P::kBitsStage);
                        tma_load_2d(dst, &tma_a, &bfull[stage], kb * 4, tm * BM + rank * HM);
                        tma_load_2d(dst + HM * 16, &tma_b, &bfull[stage], kb * 4, tn * BN + rank * HN);
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (leader) mbar_expect_tx(&full[stage], 2 * kStageBytes);
                    if (epi.cache & 2) {
                        tma_load_2d_2sm_hint(sA + stage * kABytes, &tma_a, &full[stage], kb * BK, tm * BM + rank * HM, pol);
                        tma_load_2d_2sm_hint(sB + stage * kBBytes, &tma_b, &full[stage], kb * BK, tn * BN + rank * HN, pol);
                    } else {
                        tma_load_2d_2sm(sA + stage * kABytes, &tma_a, &full[stage], kb * BK, tm * BM + rank * HM);
                        tma_load_2d_2sm(sB + stage * kBBytes, &tma_b, &full[stage], kb * BK, tn * BN + rank * HN);
                    }
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (leader && lane == 0) {
            constexpr uint32_t idesc = kF4 ? idesc_mxf4(BM, BN) : idesc_u8_s32(BM, BN);
            const uint32_t sfa = tmem_base + P::kSfCol, sfb = tmem_base + P::kSfCol + 16;
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = pair; t < num_tiles; t += num_pairs) {
                {
                    int tm, tn;
                    tile_coords(t, m_tiles, n_tiles, tm, tn);
                    if (below_diagonal<kMode>(tm + epi.m_tile0, tn, BN)) continue;
                }
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ++local;
                mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * kABytes);
                    const uint32_t b0 = smem_u32(sB + stage * kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k) {
                        if constexpr (kF4)
                            mma_mxf4_2sm(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), idesc, sfa, sfb,
                                         (kb | k) != 0);
                        else
                            mma_i8_2sm(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), idesc,
                                       (kb | k) != 0);
                    }
                    mma_commit_2sm(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm(&tfull[acc]);
            }
        }
    } else if (kBits && warp >= kThreads / 32) {
        // f1 expansion warps: kExpGroups groups of 4 take stages in turn (several stages expanded at once);
        // thread t of a group expands row t of this CTA's A half and of its B half
        const int t = (threadIdx.x - kThreads) & 127, grp = (threadIdx.x - kThreads) >> 7;
        const uint32_t full_leader0 = leader_addr(&full[0]);
        int stage = 0, seq = 0;
        uint32_t phase = 0;
        for (int tt = pair; tt < num_tiles; tt += num_pairs) {
            for (int kb = 0; kb < k_blocks; ++kb, ++seq) {
                if (seq % kExpGroups == grp) {
                    mbar_wait(&bfull[stage], phase);
                    const uint8_t* src = sbits + stage * P::kBitsStage;
#pragma unroll
                    for (int op = 0; op < 2; ++op) {
                        const uint4 b = *reinterpret_cast<const uint4*>(src + (op ? HM * 16 : 0) + t * 16);
                        uint8_t* row = (op ? sB + stage * kBBytes : sA + stage * kABytes) + (t >> 3) * 1024 + (t & 7) * 128;
                        const uint32_t wv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int c = 0; c < 8; ++c)   // 16-B chunk c = frames 16 c .. 16 c + 15, 128-B swizzle
                            *reinterpret_cast<uint4*>(row + ((c ^ (t & 7)) << 4)) =
                                bits_to_u8(wv[c >> 1] >> (16 * (c & 1)));
                    }
                    fence_proxy_async_smem();   // generic-proxy writes -> the tensor cores' async-proxy reads
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(full_leader0 + stage * 8);
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // epilogue warps 0..3 of both CTAs -> TMEM lane quadrant (warp % 4) of this CTA
        const int q = warp & 3;
        const GammaScale gs = make_gamma_scale(epi.n);
        const uint32_t tempty_leader0 = leader_addr(&tempty[0]), tempty_leader1 = leader_addr(&tempty[1]);
        int local = 0;
        for (int t = pair; t < num_tiles; t += num_pairs) {
            int tm, tn;
            tile_coords(t, m_tiles, n_tiles, tm, tn);
            tm += epi.m_tile0;
            if (below_diagonal<kMode>(tm, tn, BN)) continue;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            ++local;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            // this tile's S_b slice -> smem once (coalesced), read back as broadcast LDS
            int32_t* sbs = sb_stage + acc * BN;
            for (int j = threadIdx.x; j < BN; j += 128) {
                const int col = tn * BN + j;
                sbs[j] = col < epi.p_b ? __ldg(epi.s_b + col) : 0;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int row = tm * BM + rank * HM + 32 * q + lane;
            const bool row_ok = row < epi.p_a;
            const int32_t sa = row_ok ? __ldg(epi.s_a + row) : 0;
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(taddr + 32 * c, r);
                tmem_wait_ld();
                if constexpr (kF4) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = static_cast<uint32_t>(__float2int_rn(__uint_as_float(r[e])));
                }
                const int col0 = tn * BN + 32 * c;
                if (kMode == kEpiPeers) {
                  if (row_ok && col0 < epi.p_b) {
                    // f2: this tile row's partial sums go straight to the owning rank's shard
                    const int64_t ch = row / epi.chunk_rows;
                    const int owner = static_cast<int>(ch % epi.world);
                    const int64_t lrow = (row / epi.panel_rows) * epi.chunk_rows + row % epi.chunk_rows;
                    int32_t* dp = epi.peers[owner] + lrow * epi.ldc + col0;
                    const int nc = min(32, epi.p_b - col0);
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (e < nc && r[e] != 0u) atomicAdd(dp + e, static_cast<int>(r[e]));   // RED.ADD (no return)
                  }
                } else if (kMode == kEpiSyrk) {
                  if (row_ok && col0 < epi.p_b && col0 + 31 >= row) {   // chunks below the diagonal: mirrored elsewhere
                    // SYRK: element (row, col) for col >= row, mirrored to (col, row) for col > row;
                    // per column the warp's 32 rows are consecutive, so the mirrored stores coalesce
                    const int nc = min(32, epi.p_b - col0);
                    if (col0 > row && epi.vec && nc == 32) {   // whole chunk above the diagonal
                        int32_t* cp = epi.counts ? epi.counts + static_cast<int64_t>(row) * epi.ldc + col0 : nullptr;
                        float* gp = epi.gamma ? epi.gamma + static_cast<int64_t>(row) * epi.ldg + col0 : nullptr;
                        const int32_t* sbc = sbs + 32 * c;
                        if (gs.small) epilogue_chunk_vec<true>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                        else epilogue_chunk_vec<false>(r, cp, epi.accumulate, gp, sbc, sa, gs);
#pragma unroll 4
                        for (int e = 0; e < 32; ++e) {   // r[] now holds the accumulated sums
                            const int64_t mi = static_cast<int64_t>(col0 + e);
                            if (epi.counts) epi.counts[mi * epi.ldc + row] = static_cast<int>(r[e]);
                            if (epi.gamma) epi.gamma[mi * epi.ldg + row] = gamma_entry(static_cast<int>(r[e]), sa, sbc[e], gs);
                        }
                    } else
#pragma unroll 4
                    for (int e = 0; e < 32; ++e) {
                        const int col = col0 + e;
                        if (e >= nc || col < row) continue;
                        int v = static_cast<int>(r[e]);
                        if (epi.counts) {
                            int32_t* cp = epi.counts + static_cast<int64_t>(row) * epi.ldc + col;
                            if (epi.accumulate) v += *cp;
                            *cp = v;
                            if (col != row) epi.counts[static_cast<int64_t>(col) * epi.ldc + row] = v;
                        }
                        if (epi.gamma) {
                            const float gv = gamma_entry(v, sa, sbs[32 * c + e], gs);
                            epi.gamma[static_cast<int64_t>(row) * epi.ldg + col] = gv;
                            if (col != row) epi.gamma[static_cast<int64_t>(col) * epi.ldg + row] = gv;
                        }
                    }
                  }
                } else if (row_ok && col0 < epi.p_b) {
                    int32_t* cp = epi.counts ? epi.counts + static_cast<int64_t>(row) * epi.ldc + col0 : nullptr;
                    float* gp = epi.gamma ? epi.gamma + static_cast<int64_t>(row) * epi.ldg + col0 : nullptr;
                    const int32_t* sbc = sbs + 32 * c;
                    if (epi.vec && col0 + 32 <= epi.p_b) {
                        if (epi.cache & 1) {
                            if (gs.small) epilogue_chunk_vec<true, true>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                            else epilogue_chunk_vec<false, true>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                        } else {
                            if (gs.small) epilogue_chunk_vec<true>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                            else epilogue_chunk_vec<false>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                        }
                    } else {
                        epilogue_chunk_tail(r, min(32, epi.p_b - col0), cp, epi.accumulate, gp, sbc, sa, gs);
                    }
                }
                __syncwarp();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
        }
        if (kMode == kEpiPeers) __threadfence_system();   // peer-memory reductions visible beyond this GPU
    }
    __syncwarp();
    tc_fence_before();
    cluster_sync();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc_2sm(tmem_base, kTmemCols);
    }
}

}  // namespace

int gemm_tc2_block_m() { return BM; }
int gemm_tc2_block_n() { return Tc2<false>::BN; }
int gemm_tc2_box_rows() { return Tc2<false>::HM; }
int gemm_f4_block_n() { return Tc2<true>::BN; }
int gemm_f4_box_rows_b() { return Tc2<true>::HN; }

template <bool kF4, int kMode>
static cudaError_t launch_tc2_mode(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles, int n_tiles,
                                   int k_blocks, const Epilogue& epi, int num_sms, cudaStream_t st) {
    // the attribute is per device: set it before every launch (a host-side call, negligible)
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_tc2_kernel<kF4, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Tc2<kF4>::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int tiles = m_tiles * n_tiles;
    int pairs = num_sms / 2;
    if (tiles < pairs) pairs = tiles;
    gemm_i8_tc2_kernel<kF4, kMode><<<2 * pairs, kThreads, Tc2<kF4>::kSmemBytes, st>>>(*tma_a, *tma_b, m_tiles,
                                                                                    n_tiles, k_blocks, epi);
    return cudaGetLastError();
}
template <bool kF4>
static cudaError_t launch_tc2(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles, int n_tiles,
                              int k_blocks, const Epilogue& epi, int num_sms, cudaStream_t st) {
    if (epi.peers) return launch_tc2_mode<kF4, kEpiPeers>(tma_a, tma_b, m_tiles, n_tiles, k_blocks, epi, num_sms, st);
    if (epi.symmetric)
        return launch_tc2_mode<kF4, kEpiSyrk>(tma_a, tma_b, m_tiles, n_tiles, k_blocks, epi, num_sms, st);
    return launch_tc2_mode<kF4, kEpiPlain>(tma_a, tma_b, m_tiles, n_tiles, k_blocks, epi, num_sms, st);
}

cudaError_t launch_gemm_tc2(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                            int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                            cudaStream_t st) {
    return launch_tc2<false>(tma_a, tma_b, m_tiles, n_tiles, k_blocks, epi, num_sms, st);
}

cudaError_t launch_gemm_f4(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                           int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                           cudaStream_t st) {
    return launch_tc2<true>(tma_a, tma_b, m_tiles, n_tiles, k_blocks, epi, num_sms, st);
}

cudaError_t launch_gemm_bits(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles, int n_tiles,
                             int k_blocks, const Epilogue& epi, int num_sms, cudaStream_t st) {
    if (epi.peers || epi.symmetric) return cudaErrorInvalidValue;   // plain epilogue only
    auto kern = gemm_i8_tc2_kernel<false, kEpiPlain, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc2<false>::kBitsSmem);
    if (e != cudaSuccess) return e;
    const int tiles = m_tiles * n_tiles;
    int pairs = num_sms / 2;
    if (tiles < pairs) pairs = tiles;
    kern<<<2 * pairs, kThreadsBits, Tc2<false>::kBitsSmem, st>>>(*tma_a, *tma_b, m_tiles, n_tiles, k_blocks, epi);
    return cudaGetLastError();
}

}  // namespace cpi
