// expand.cu — KB1: on-device bit unpacking of SwissSPAD2 frames into GEMM operands,
// fused with the single-pixel sums S_a / S_b of Eq. (1).
//
// PAPER.md:265 (prototype: "bit-unpacking is performed" before the matrix product),
// PAPER.md:266-267 (bit-packed AND variant; unpack joint with correlation)
// (frame layout), P:104-109 (single-pixel sums).  SURVEY §8(a) row a2.
//
// One CTA = one RoI row m of one arm x 512 consecutive frames.  The row's bytes for 128
// frames are staged in shared memory; each warp then owns one pixel at a time and every
// lane produces 4 consecutive frames of it, so a warp stores 128 contiguous bytes of the
// pixel's K-major operand row (fully coalesced).  Frames in [n, k_pad) are written as
// zeros, so the GEMM's K tail is inert.  The bit-stream variant (KB3 operand) ballots the
// same bits into pixel-major 32-bit words (bit f%32 of word f/32 = frame f); the E2M1
// variant (FP4 GEMM operand) writes 4 frames as 4 nibbles (0x2 = 1.0), 64 B per warp.
#include "kernels.h"

namespace cpi {
namespace {

constexpr int kThreads = 256;

// operand row / sum slot of RoI pixel (m, j) (include/cpi.h B pixel orders): row-major m * w + j,
// u-blocked (j / 8) * (8 h) + 8 m + j % 8 (CPI_GAMMA_UBLOCKED), v-major vmajor_slot (CPI_GAMMA_VMAJOR)
__device__ __forceinline__ int64_t pixel_slot(int order, int m, int j, const RoiDev& roi) {
    if (order == kOrderUBlocked) return static_cast<int64_t>(j >> 3) * (8 * roi.h) + 8 * m + (j & 7);
    if (order == kOrderVMajor) return vmajor_slot(j, m, roi.w, roi.h);
    return static_cast<int64_t>(m) * roi.w + j;
}
constexpr int kSub = 128;       // frames per staged sub-block
constexpr int kFramesCta = 512; // frames per CTA
constexpr int kRowStride = 65;  // bytes per staged frame row: odd word stride -> no bank conflicts
constexpr int kMaxWidth = 512;

template <int kMode>
__global__ void __launch_bounds__(kThreads)
expand_kernel(const uint8_t* __restrict__ frames, int64_t n, int row_bytes, int frame_h, int msb,
              RoiDev roi, void* __restrict__ op, int64_t ld, int64_t k_pad, int32_t* __restrict__ s,
              int order) {
    __shared__ uint8_t sbits[kSub * kRowStride];
    __shared__ int cnt[kMaxWidth];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = blockIdx.y;
    const int b0 = roi.x0 >> 3;
    const int nb = ((roi.x0 + roi.w - 1) >> 3) - b0 + 1;
    for (int j = tid; j < roi.w; j += kThreads) cnt[j] = 0;
    const int64_t f_begin = static_cast<int64_t>(blockIdx.x) * kFramesCta;
    const int64_t row_off = static_cast<int64_t>(roi.y0 + m) * row_bytes + b0;
    for (int sub = 0; sub < kFramesCta / kSub; ++sub) {
        const int64_t f0 = f_begin + sub * kSub;
        if (f0 >= k_pad) break;
        __syncthreads();
        for (int idx = tid; idx < kSub * nb; idx += kThreads) {
            const int fl = idx / nb, b = idx - fl * nb;
            const int64_t f = f0 + fl;
            sbits[fl * kRowStride + b] =
                (f < n) ? __ldg(frames + f * frame_h * row_bytes + row_off + b) : uint8_t(0);
        }
        __syncthreads();
        for (int j = warp; j < roi.w; j += kThreads / 32) {
            const int col = roi.x0 + j;
            const int b = (col >> 3) - b0;
            const int sh = msb ? 7 - (col & 7) : (col & 7);
            const int64_t prow = pixel_slot(order, m, j, roi);
            int c;
            if constexpr (kMode == kExpandE2M1) {
                // 4 frames -> 4 nibbles (E2M1 1.0 = 0x2), frame f in nibble f % 2 of byte f / 2
                uint32_t word = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    word |= static_cast<uint32_t>((sbits[(4 * lane + k) * kRowStride + b] >> sh) & 1) << (4 * k + 1);
                *reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(op) + prow * ld + ((f0 + 4 * lane) >> 1)) =
                    static_cast<uint16_t>(word);
                c = __popc(word);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            } else if constexpr (kMode == kExpandU8) {
                uint32_t word = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    word |= static_cast<uint32_t>((sbits[(4 * lane + k) * kRowStride + b] >> sh) & 1)
                            << (8 * k);
                *reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(op) + prow * ld + f0 + 4 * lane) = word;
                c = __popc(word);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            } else {
                c = 0;
                uint32_t mine = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t bit = (sbits[(32 * q + lane) * kRowStride + b] >> sh) & 1;
                    const uint32_t w = __ballot_sync(0xffffffffu, bit);
                    c += __popc(w);
                    if (lane == q) mine = w;
                }
                if (lane < 4)
                    static_cast<uint32_t*>(op)[prow * ld + (f0 >> 5) + lane] = mine;
            }
            if (lane == 0) cnt[j] += c;   // pixel j is owned by this warp only
        }
    }
    __syncthreads();
    for (int j = tid; j < roi.w; j += kThreads)
        if (cnt[j])
            atomicAdd(s + pixel_slot(order, m, j, roi), cnt[j]);
}

// u8 / E2M1 operands, byte-column parallel: the sub-block's bytes are staged transposed,
// [byte column][frame], so one 32-bit shared load gives a lane 4 consecutive frames of 8 pixels.
// For bit s of the byte, x = (word >> s) & 0x01010101 holds the 4 frames' bits at byte positions
// 0, 8, 16, 24: that is the u8 operand word as is; for E2M1 the bits are folded onto nibbles
// 0..3 (frames 0, 2, 1, 3 of the group -- A and B use the same order, so the K sum is
// unchanged) and shifted to 0x2 = 1.0.  Pixel counts: popc + one warp REDUX per pixel.
constexpr int kTStride = kSub + 4;    // bytes per staged byte column (keeps 32-bit alignment)

template <int kMode>
__global__ void __launch_bounds__(kThreads)
expand_cols_kernel(const uint8_t* __restrict__ frames, int64_t n, int row_bytes, int frame_h, int msb,
                   RoiDev roi, void* __restrict__ op, int64_t ld, int64_t k_pad, int32_t* __restrict__ s,
                   int order, int words) {
    __shared__ __align__(16) uint8_t sbt[(kMaxWidth / 8 + 1) * kTStride];
    __shared__ int cnt[kMaxWidth];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = blockIdx.y;
    const int b0 = roi.x0 >> 3;
    const int nb = ((roi.x0 + roi.w - 1) >> 3) - b0 + 1;
    for (int j = tid; j < roi.w; j += kThreads) cnt[j] = 0;
    const int64_t f_begin = static_cast<int64_t>(blockIdx.x) * kFramesCta;
    const int64_t row_off = static_cast<int64_t>(roi.y0 + m) * row_bytes + b0;
    for (int sub = 0; sub < kFramesCta / kSub; ++sub) {
        const int64_t f0 = f_begin + sub * kSub;
        if (f0 >= k_pad) break;
        __syncthreads();
        if (words) {   // 4-byte loads of the word range covering the RoI's bytes
            const int wb0 = b0 & ~3, nw = (b0 + nb - wb0 + 3) >> 2;
            const int64_t row_w = static_cast<int64_t>(roi.y0 + m) * row_bytes + wb0;
            for (int idx = tid; idx < kSub * nw; idx += kThreads) {
                const int fl = idx / nw, w = idx - fl * nw;
                const int64_t f = f0 + fl;
                const uint32_t v = (f < n) ? __ldg(reinterpret_cast<const uint32_t*>(frames + f * frame_h * row_bytes + row_w) + w)
                                           : 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int b = 4 * w + k - (b0 - wb0);
                    if (b >= 0 && b < nb) sbt[b * kTStride + fl] = static_cast<uint8_t>(v >> (8 * k));
                }
            }
        } else {
            for (int idx = tid; idx < kSub * nb; idx += kThreads) {
                const int fl = idx / nb, b = idx - fl * nb;
                const int64_t f = f0 + fl;
                sbt[b * kTStride + fl] = (f < n) ? __ldg(frames + f * frame_h * row_bytes + row_off + b) : uint8_t(0);
            }
        }
        __syncthreads();
        for (int b = warp; b < nb; b += kThreads / 32) {
            const uint32_t w4 = *reinterpret_cast<const uint32_t*>(sbt + b * kTStride + 4 * lane);   // frames 4 lane + 0..3
#pragma unroll
            for (int bit = 0; bit < 8; ++bit) {
                const int col = (b0 + b) * 8 + (msb ? 7 - bit : bit);
                const int j = col - roi.x0;
                if (j < 0 || j >= roi.w) continue;          // warp-uniform
                const uint32_t x = (w4 >> bit) & 0x01010101u;
                const int64_t prow = pixel_slot(order, m, j, roi);
                if constexpr (kMode == kExpandE2M1) {
                    const uint32_t nib = ((x | (x >> 12)) & 0x1111u) << 1;   // 4 nibbles, 0x2 = 1.0
                    *reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(op) + prow * ld + ((f0 + 4 * lane) >> 1)) =
                        static_cast<uint16_t>(nib);
                } else {
                    *reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(op) + prow * ld + f0 + 4 * lane) = x;
                }
                const int c = __reduce_add_sync(0xffffffffu, __popc(x));
                if (lane == 0) cnt[j] += c;                 // pixel j belongs to this warp only
            }
        }
    }
    __syncthreads();
    for (int j = tid; j < roi.w; j += kThreads)
        if (cnt[j])
            atomicAdd(s + pixel_slot(order, m, j, roi), cnt[j]);
}

}  // namespace

void launch_expand(const uint8_t* frames, int64_t n, int row_bytes, int frame_h, int msb,
                   RoiDev roi, void* op, int64_t ld, int64_t k_pad, int32_t* s, int mode,
                   int order, cudaStream_t st) {
    if (k_pad <= 0) return;
    dim3 grid(static_cast<unsigned>((k_pad + kFramesCta - 1) / kFramesCta), roi.h);
    if (mode == kExpandBits)
        expand_kernel<kExpandBits><<<grid, kThreads, 0, st>>>(frames, n, row_bytes, frame_h, msb, roi, op,
                                                              ld, k_pad, s, order);
    else {
        // word loads need 4-byte aligned frame rows
        const int words = (row_bytes % 4 == 0 && (reinterpret_cast<uintptr_t>(frames) & 3) == 0) ? 1 : 0;
        if (mode == kExpandE2M1)
            expand_cols_kernel<kExpandE2M1><<<grid, kThreads, 0, st>>>(frames, n, row_bytes, frame_h, msb, roi, op,
                                                                       ld, k_pad, s, order, words);
        else
            expand_cols_kernel<kExpandU8><<<grid, kThreads, 0, st>>>(frames, n, row_bytes, frame_h, msb, roi, op,
                                                                     ld, k_pad, s, order, words);
    }
}

}  // namespace cpi
