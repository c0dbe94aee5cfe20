// gemm_popc.cu — KB3: the paper's optimised correlation kernel re-expressed for CUDA cores:
// "bit-packing ... implementing the cross-correlation multiplication as a bit-by-bit AND
// operation" with unpack and correlation "jointly in the same kernel".
//   S_ab[p][q] = sum_w popc(a_p[w] AND b_q[w])   (pixel-major 32-bit frame bit streams)
// Kept as the measured comparison variant to the tcgen05 kind::i8 path (BASELINE north_star).
// Register-tiled: 64x64 outputs per CTA, 4x4 per thread, 32-word K chunks staged in smem.
#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

constexpr int T = 64;      // CTA tile (pixels x pixels)
constexpr int KW = 32;     // words per K chunk

__global__ void __launch_bounds__(256)
gemm_popc_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t ldw,
                 int64_t kw, Epilogue epi) {
    __shared__ uint32_t As[KW][T + 1];
    __shared__ uint32_t Bs[KW][T + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = static_cast<int64_t>(blockIdx.y + epi.m_tile0) * T;
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * T;
    int acc[4][4] = {};
    for (int64_t w0 = 0; w0 < kw; w0 += KW) {
#pragma unroll
        for (int i = 0; i < (T * KW) / 256; ++i) {
            const int idx = tid + 256 * i;
            const int p = idx / KW, w = idx % KW;
            const bool in = w0 + w < kw;
            As[w][p] = in ? __ldg(a + (row0 + p) * ldw + w0 + w) : 0u;
            Bs[w][p] = in ? __ldg(b + (col0 + p) * ldw + w0 + w) : 0u;
        }
        __syncthreads();
#pragma unroll 8
        for (int w = 0; w < KW; ++w) {
            uint32_t av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { av[i] = As[w][ty * 4 + i]; bv[i] = Bs[w][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += __popc(av[i] & bv[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = row0 + ty * 4 + i;
        if (row >= epi.p_a) continue;
        const int32_t sa = epi.s_a[row];
        const GammaScale gs = make_gamma_scale(epi.n);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t col = col0 + tx * 4 + j;
            if (col >= epi.p_b) continue;
            int s = acc[i][j];
            if (epi.counts) {
                int32_t* cp = epi.counts + row * epi.ldc + col;
                if (epi.accumulate) s += *cp;
                *cp = s;
            }
            if (epi.gamma)
                epi.gamma[row * epi.ldg + col] =
                    gamma_entry(s, sa, epi.s_b[col], gs);
        }
    }
}

__global__ void finalize_kernel(const int32_t* __restrict__ counts, int64_t ldc, int64_t rows,
                                int64_t p_b, const int32_t* __restrict__ s_a_rows,
                                const int32_t* __restrict__ s_b, double n,
                                float* __restrict__ gamma, int64_t ldg) {
    const GammaScale gs = make_gamma_scale(n);
    const int64_t total = rows * p_b;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / p_b, q = idx - r * p_b;
        gamma[r * ldg + q] = gamma_entry(counts[r * ldc + q], s_a_rows[r], s_b[q], gs);
    }
}

}  // namespace

int gemm_popc_block() { return T; }

cudaError_t launch_gemm_popc(const uint32_t* a, const uint32_t* b, int64_t ldw, int64_t kw,
                             const Epilogue& epi, cudaStream_t st) {
    dim3 grid(static_cast<unsigned>((epi.p_b + T - 1) / T),
              static_cast<unsigned>((epi.p_a - static_cast<int64_t>(epi.m_tile0) * T + T - 1) / T));
    gemm_popc_kernel<<<grid, 256, 0, st>>>(a, b, ldw, kw, epi);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const int32_t* counts, int64_t ldc, int64_t rows, int64_t p_b,
                            const int32_t* s_a_rows, const int32_t* s_b, double n, float* gamma,
                            int64_t ldg, cudaStream_t st) {
    const int64_t total = rows * p_b;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    finalize_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(counts, ldc, rows, p_b, s_a_rows,
                                                                   s_b, n, gamma, ldg);
    return cudaGetLastError();
}

}  // namespace cpi
