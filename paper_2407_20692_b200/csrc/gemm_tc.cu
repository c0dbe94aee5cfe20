// gemm_tc.cu — KB2: pair sums S_ab = A^T B of Eq. (1) ("cross-correlation
// ... computed by matrix multiplication") on 5th-generation tensor cores, with the
// single-pixel sums and the exact normalisation fused into the epilogue.
//
// A = expanded arm-A operand [M_pad][K] u8 (row p = A pixel, column i = frame, 0/1),
// B = expanded arm-B operand [N_pad][K] u8; both K-major.  S_ab[p][q] = sum_i A[p][i] B[q][i]
// is exact in int32 (S_ab <= N < 2^31).
//
// Design (sm_100a, one CTA per SM, persistent):
//   warp 4      : TMA producer — 128x128 B A-tile + 256x128 B B-tile per stage into a
//                 4-stage shared-memory ring (128-byte swizzle), mbarrier full/empty.
//   warp 5      : TMEM allocator + single-thread MMA issuer — tcgen05.mma.cta_group::1
//                 .kind::i8, M=128 N=256 K=32, 4 per stage, into one of two TMEM
//                 accumulators (2 x 256 columns), tcgen05.commit -> mbarriers.
//   warps 0..3  : epilogue — tcgen05.ld 32x32b.x32, then Gamma = (N s - S_a S_b)/N^2
//                 (exact numerator in fp64) and/or int32 counts, straight to global.
// The double-buffered accumulator lets the epilogue of tile t overlap the MMAs of t+1.
// Tiles are rasterised in groups of kGroupM M-tiles so concurrently running CTAs share
// A and B panels in L2.
#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

constexpr int BM = 128, BN = 256, BK = 128;  // BK in bytes (= u8 elements)
constexpr int kStages = 4;
constexpr int kABytes = BM * BK;              // 16 KB
constexpr int kBBytes = BN * BK;              // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kTmemCols = 512;                // 2 accumulators x 256 columns
constexpr int kGroupM = 16;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/ + 2 * BN * 4;

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& tm, int& tn) {
    const int group = kGroupM * n_tiles;
    const int g = t / group;
    const int first_m = g * kGroupM;
    const int gm = min(m_tiles - first_m, kGroupM);
    const int r = t - g * group;
    tm = first_m + r % gm;
    tn = r / gm;
}

__global__ void __launch_bounds__(kThreads, 1)
gemm_i8_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                  int m_tiles, int n_tiles, int k_blocks, Epilogue epi) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int32_t* sb_stage = reinterpret_cast<int32_t*>(sB + kStages * kBBytes + 256);   // [2][BN]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kProdWarp = 4, kMmaWarp = 5;   // highest warp ids win the issue arbiter
    if (warp == kProdWarp && lane == 0) {
        tma_prefetch_desc(&tma_a);
        tma_prefetch_desc(&tma_b);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);   // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_tiles = m_tiles * n_tiles;

    if (warp == kProdWarp) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int tm, tn;
                tile_coords(t, m_tiles, n_tiles, tm, tn);
                tm += epi.m_tile0;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], kStageBytes);
                    tma_load_2d(sA + stage * kABytes, &tma_a, &full[stage], kb * BK, tm * BM);
                    tma_load_2d(sB + stage * kBBytes, &tma_b, &full[stage], kb * BK, tn * BN);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_u8_s32(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * kABytes);
                    const uint32_t b0 = smem_u32(sB + stage * kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)
                        mma_i8(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), idesc,
                               (kb | k) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else {
        // epilogue warps 0..3 -> TMEM lane quadrant (warp % 4)
        const int q = warp & 3;
        const GammaScale gs = make_gamma_scale(epi.n);
        int local = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
            int tm, tn;
            tile_coords(t, m_tiles, n_tiles, tm, tn);
            tm += epi.m_tile0;
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            // this tile's S_b slice -> smem once (coalesced), read back as broadcast LDS
            int32_t* sbs = sb_stage + acc * BN;
            for (int j = threadIdx.x; j < BN; j += 128) {
                const int col = tn * BN + j;
                sbs[j] = col < epi.p_b ? __ldg(epi.s_b + col) : 0;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int row = tm * BM + 32 * q + lane;
            const bool row_ok = row < epi.p_a;
            const int32_t sa = row_ok ? __ldg(epi.s_a + row) : 0;
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(taddr + 32 * c, r);
                tmem_wait_ld();
                const int col0 = tn * BN + 32 * c;
                if (row_ok && col0 < epi.p_b) {
                    int32_t* cp = epi.counts ? epi.counts + static_cast<int64_t>(row) * epi.ldc + col0 : nullptr;
                    float* gp = epi.gamma ? epi.gamma + static_cast<int64_t>(row) * epi.ldg + col0 : nullptr;
                    const int32_t* sbc = sbs + 32 * c;
                    if (epi.vec && col0 + 32 <= epi.p_b) {
                        if (gs.small) epilogue_chunk_vec<true>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                        else epilogue_chunk_vec<false>(r, cp, epi.accumulate, gp, sbc, sa, gs);
                    } else {
                        epilogue_chunk_tail(r, min(32, epi.p_b - col0), cp, epi.accumulate, gp, sbc, sa, gs);
                    }
                }
                __syncwarp();   // reconverge before the next warp-collective tcgen05.ld
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

}  // namespace

int gemm_tc_block_m() { return BM; }
int gemm_tc_block_n() { return BN; }

cudaError_t launch_gemm_tc(const CUtensorMap* tma_a, const CUtensorMap* tma_b, int m_tiles,
                           int n_tiles, int k_blocks, const Epilogue& epi, int num_sms,
                           cudaStream_t st) {
    // the attribute is per device: set it before every launch (a host-side call, negligible)
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    const int tiles = m_tiles * n_tiles;
    const int grid = tiles < num_sms ? tiles : num_sms;
    gemm_i8_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(*tma_a, *tma_b, m_tiles, n_tiles,
                                                           k_blocks, epi);
    return cudaGetLastError();
}

}  // namespace cpi
