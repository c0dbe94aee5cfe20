// refocus_gen.cu — refocusing under a general RefocusMap whose B coordinates depend on the output
// pixel (SPEC.md:273 RefocusMap, d != 0: c_Bx = dx (x - c_ax) + ex (u - c_bx) + fx + c_bx; SURVEY
// §8(f) f3 "general maps"; PAPER.md:114-116, P:270 16-corner interpolation).
//
// The sample weight of the 16-corner interpolation factorises per axis, and the skip rule is a
// conjunction of per-axis tests, so with both coordinates of an axis depending on
// (output, B index) the sum still splits in two stages:
//   T(x, m, n) = sum_u valid_x(x, u) bilinear(Gamma(., m; ., n); c_Ax(x, u), c_Bx(x, u))
//   R(x, y)    = sum_v valid_y(y, v) bilinear(T(x, ., .); c_Ay(y, v), c_By(y, v)) / (cnt_x(x) cnt_y(y))
// Both are the same operation: every output o of a 2D image I (R rows x C columns) sums the
// bilinear samples of I at its table's points (a0 + ta, b0 + tb) over the B index s.  One CTA per
// image stages the image in shared memory (column windows of 129 when C > 160) and one thread per
// output walks its samples: 4 shared-memory taps per sample in fp32, summed in fp64.
//   stage 1: images (m, n) = Gamma[(m W_a + j)][n W_b + k] (rows j, columns k), outputs x
//   stage 2: images x = T[x][m][n] (rows m, columns n), outputs y
// Gamma must be in the row-major B order; contiguous row shards (T rows outside them are zero).
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

// A corner offset t in [0, 1] is stored in fp32 as t (t <= 1/2) or -(1 - t) (exact in fp64), so
// the smaller corner weight keeps its relative precision when rounded; gen_weights recovers
// (1 - t, t) with each weight's relative error <= 2^-24.
// (t = 1 is stored as -0.0: the sign bit, not the value, says which corner s belongs to.)
__device__ __forceinline__ float gen_near_t(double t) { return __double2float_rn(t > 0.5 ? -(1.0 - t) : t); }
__device__ __forceinline__ void gen_weights(float s, float& w0, float& w1) {
    const bool up = signbit(s);
    w0 = up ? -s : 1.f - s;
    w1 = up ? 1.f + s : s;
}

constexpr int kGenMaxR = 256, kGenWin = 128, kGenPitch = kGenWin + 1;   // staged columns per window (+1 overlap)
constexpr int kGenThreads = 256;

// axis tables of one plane: output o (A lattice, size WA), B index s (size WB).  fp64 in the
// oracle's operation order (oracle/cpi_oracle.c refocus_pixel_affine):
//   c_A = (((a (o - c_A0)) + (b (s - c_B0))) + c) + c_A0,  c_B = (((d (o - c_A0)) + (e (s - c_B0))) + f) + c_B0
// skip: both in their closed lattice intervals; clamp: both clamped.  support i0 = min(floor(c), W - 2),
// t = c - i0 (R10).  a0 = -1 marks a skipped sample; cnt[o] = number of used samples.
__global__ void gen_axis_kernel(GenMap mp, int WA, int WB, int boundary, GenTables tab) {
    const int o = blockIdx.x;
    const double cA0 = (WA - 1) / 2.0, cB0 = (WB - 1) / 2.0;
    const double orr = __dadd_rn(static_cast<double>(o), -cA0);
    int used = 0;
    for (int s = threadIdx.x; s < WB; s += blockDim.x) {
        const double sr = __dadd_rn(static_cast<double>(s), -cB0);
        double cA = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(mp.a, orr), __dmul_rn(mp.b, sr)), mp.c), cA0);
        double cB = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(mp.d, orr), __dmul_rn(mp.e, sr)), mp.f), cB0);
        bool ok;
        if (boundary == 0) {
            ok = cA >= 0.0 && cA <= static_cast<double>(WA - 1) && cB >= 0.0 && cB <= static_cast<double>(WB - 1);
        } else {
            cA = fmin(fmax(cA, 0.0), static_cast<double>(WA - 1));
            cB = fmin(fmax(cB, 0.0), static_cast<double>(WB - 1));
            ok = true;
        }
        const int64_t idx = static_cast<int64_t>(o) * WB + s;
        if (ok) {
            double fa = floor(cA), fb = floor(cB);
            if (fa > static_cast<double>(WA - 2)) fa = static_cast<double>(WA - 2);
            if (fb > static_cast<double>(WB - 2)) fb = static_cast<double>(WB - 2);
            tab.a0[idx] = static_cast<int>(fa);
            tab.at[idx] = gen_near_t(__dadd_rn(cA, -fa));
            tab.b0[idx] = static_cast<int>(fb);
            tab.bt[idx] = gen_near_t(__dadd_rn(cB, -fb));
            ++used;
        } else {
            tab.a0[idx] = -1;
            tab.at[idx] = 0.f;
            tab.b0[idx] = 0;
            tab.bt[idx] = 0.f;
        }
    }
    __shared__ int sw[kGenThreads / 32];
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) used += __shfl_xor_sync(0xffffffffu, used, k);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = used;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sw[w];
        tab.cnt[o] = t;
    }
}

struct GenSumArgs {
    const float* src;
    int R, C;                 // image rows / columns (R <= 256)
    int64_t row_stride;       // floats between image rows
    int n_out, n_samp;        // outputs o (threads), samples s per output
    GenTables tab;            // [n_out][n_samp]
    // stage 1 (mode 0): image i = (local A row l, n): base l W_a P_b + n W_b, output T[(o H_a + m) H_b + n]
    // stage 2 (mode 1): image i = x: base x H_a H_b, output plane[o W_a + x] / (cnt_x[x] cnt_y[o])
    int mode;
    int Wa, Ha, Hb, Wb, m0;   // m = m0 + l in mode 0
    int64_t pb;
    float* out;
    const int32_t* cnt_x;
};

__global__ void __launch_bounds__(kGenThreads) gen_sum_kernel(GenSumArgs g) {
    extern __shared__ float simg[];   // [R][kGenPitch]
    const int i = blockIdx.x;
    int64_t base;
    if (g.mode == 0) {
        const int l = i / g.Hb, n = i - l * g.Hb;
        base = static_cast<int64_t>(l) * g.Wa * g.pb + static_cast<int64_t>(n) * g.Wb;
    } else {
        base = static_cast<int64_t>(i) * g.Ha * g.Hb;
    }
    const float* img = g.src + base;
    const int o = threadIdx.x;
    double sum = 0.0;
    const int n_win = g.C <= 160 ? 1 : (g.C - 2) / kGenWin + 1;
    const int pitch = g.C <= 160 ? g.C + 1 : kGenPitch;
    for (int w = 0; w < n_win; ++w) {
        const int c_lo = n_win == 1 ? 0 : w * kGenWin;
        const int nc = n_win == 1 ? g.C : min(kGenPitch, g.C - c_lo);
        __syncthreads();
        for (int e = threadIdx.x; e < g.R * nc; e += blockDim.x) {
            const int r = e / nc, cc = e - r * nc;
            simg[r * pitch + cc] = __ldg(img + r * g.row_stride + c_lo + cc);
        }
        __syncthreads();
        if (o < g.n_out) {
            const int64_t t0 = static_cast<int64_t>(o) * g.n_samp;
            for (int s = 0; s < g.n_samp; ++s) {
                const int a0 = __ldg(g.tab.a0 + t0 + s);
                if (a0 < 0) continue;
                const int b0 = __ldg(g.tab.b0 + t0 + s);
                if (n_win > 1 && min(b0 / kGenWin, n_win - 1) != w) continue;   // sample's window
                const float ta = __ldg(g.tab.at + t0 + s), tb = __ldg(g.tab.bt + t0 + s);
                const float* p = simg + a0 * pitch + (b0 - c_lo);
                float wa0, wa1, wb0, wb1;
                gen_weights(ta, wa0, wa1);
                gen_weights(tb, wb0, wb1);
                const float lo = fmaf(wb1, p[1], wb0 * p[0]);
                const float hi = fmaf(wb1, p[pitch + 1], wb0 * p[pitch]);
                sum += static_cast<double>(fmaf(wa1, hi, wa0 * lo));
            }
        }
    }
    if (o >= g.n_out) return;
    if (g.mode == 0) {
        const int l = i / g.Hb, n = i - l * g.Hb;
        g.out[(static_cast<int64_t>(o) * g.Ha + g.m0 + l) * g.Hb + n] = static_cast<float>(sum);
    } else {
        const int64_t cnt = static_cast<int64_t>(__ldg(g.cnt_x + i)) * __ldg(g.tab.cnt + o);
        g.out[static_cast<int64_t>(o) * g.Wa + i] = cnt ? static_cast<float>(sum / static_cast<double>(cnt)) : 0.f;
    }
}

}  // namespace

bool refocus_gen_supported(int Wa, int Ha, int Wb, int Hb) {
    return Wa >= 2 && Ha >= 2 && Wb >= 2 && Hb >= 2 && Wa <= kGenMaxR && Ha <= kGenMaxR && Wb <= 512 && Hb <= 512;
}

cudaError_t launch_gen_axis(const GenMap& mp, int WA, int WB, int boundary, const GenTables& tab, cudaStream_t st) {
    gen_axis_kernel<<<WA, kGenThreads, 0, st>>>(mp, WA, WB, boundary, tab);
    return cudaGetLastError();
}

static size_t gen_smem(int R, int C) { return sizeof(float) * size_t(R) * (C <= 160 ? C + 1 : kGenPitch); }

cudaError_t launch_refocus_gen(const float* gamma, int64_t pb, int Wa, int Ha, int Wb, int Hb, int m_base, int m_count,
                               const GenTables& xt, const GenTables& yt, TElem* T, float* plane, cudaStream_t st) {
    if (!refocus_gen_supported(Wa, Ha, Wb, Hb)) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    if (m_count < Ha) e = cudaMemsetAsync(T, 0, sizeof(TElem) * size_t(Wa) * Ha * Hb, st);   // rows outside the shard
    if (e != cudaSuccess) return e;
    GenSumArgs a{};
    a.Wa = Wa; a.Ha = Ha; a.Hb = Hb; a.Wb = Wb; a.m0 = m_base; a.pb = pb;
    // stage 1
    a.src = gamma; a.R = Wa; a.C = Wb; a.row_stride = pb; a.n_out = Wa; a.n_samp = Wb; a.tab = xt; a.mode = 0; a.out = T;
    size_t smem = gen_smem(a.R, a.C);
    e = cudaFuncSetAttribute(gen_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    gen_sum_kernel<<<m_count * Hb, kGenThreads, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // stage 2
    a.src = T; a.R = Ha; a.C = Hb; a.row_stride = Hb; a.n_out = Ha; a.n_samp = Hb; a.tab = yt; a.mode = 1; a.out = plane;
    a.cnt_x = xt.cnt;
    smem = gen_smem(a.R, a.C);
    gen_sum_kernel<<<Wa, kGenThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace cpi
