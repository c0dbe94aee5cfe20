// b1_mma_probe.cu — one-off measurement (SURVEY §8(f) "Legacy mma.sync ... .b1 .and.popc: rate
// on sm_100 unknown"): the register-only throughput of the warp-level binary MMA
//   mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc
// on B200, to compare with the tcgen05 kinds the GEMM uses (each b1 MAC is one frame pair,
// like one kind::i8 / kind::mxf4 MAC on 0/1 operands).  No memory traffic: operands live in
// registers, 8 independent accumulator chains per warp.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/b1_mma_probe tools/b1_mma_probe.cu
// Run:   /tmp/b1_mma_probe   -> one JSON line
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void b1_mma_kernel(int iters, uint32_t seed, int* out) {
    uint32_t a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = (seed * 2654435761u) ^ (threadIdx.x * 40503u + i * 977u);
#pragma unroll
    for (int i = 0; i < 2; ++i) b[i] = (seed * 362437u) ^ (threadIdx.x * 69069u + i * 131u);
    int c[kChains][4];
#pragma unroll
    for (int k = 0; k < kChains; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) c[k][i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) {
            asm volatile(
                "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
                : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    if (s == 0x7fffffff) out[0] = s;   // keep the chains alive
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    int* out;
    cudaMalloc(&out, sizeof(int));
    const int iters = 4096;
    double best_tops = 0, best_ms = 0;
    int best_warps = 0;
    for (int warps = 4; warps <= 32; warps *= 2) {
        const dim3 grid(sms * 2), block(32 * warps / 2);
        b1_mma_kernel<<<grid, block>>>(16, 1u, out);   // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        b1_mma_kernel<<<grid, block>>>(iters, 2u, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = double(grid.x) * (block.x / 32) * iters * kChains;
        const double ops = mmas * 2.0 * 16 * 8 * 256;   // 2 ops per binary MAC
        const double tops = ops / (ms * 1e-3) / 1e12;
        if (tops > best_tops) { best_tops = tops; best_ms = ms; best_warps = warps; }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"probe\": \"mma.sync.m16n8k256.b1.and.popc, register operands\", \"sms\": %d, "
           "\"warps_per_sm\": %d, \"ms\": %.3f, \"tops\": %.1f, \"per_sm_macs_per_clk_at_max_clock\": %.1f, "
           "\"max_clock_mhz\": %d, \"cuda\": \"%s\"}\n",
           sms, best_warps, best_ms, best_tops, best_tops * 1e12 / 2.0 / sms / (clk_khz * 1e3), clk_khz / 1000,
           cudaGetErrorString(err));
    return 0;
}
