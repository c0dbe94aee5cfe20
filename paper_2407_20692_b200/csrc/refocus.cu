// refocus.cu — KB5/KB6: refocusing of Gamma into a stack of planes (PAPER.md:114-116,
// P:269-272; SPEC.md:274 default map).
//
// For plane alpha the output pixel (x, y) is the mean, over the B lattice (u, v), of Gamma
// interpolated at A coordinates c_x(x,u), c_y(y,v) and B coordinates (u, v).  Because the
// B coordinates are integers the 4D multilinear interpolation reduces exactly to
// bilinear interpolation over the A axes, and the sum separates:
//   stage 1 (KB5):  T[x][m][v] = sum_u [(1-t_x) G(m, j0; v, u) + t_x G(m, j0+1; v, u)]
//   stage 2 (KB6):  R[y][x]    = sum_v [(1-t_y) T[x][m0][v] + t_y T[x][m0+1][v]] / (cnt_x cnt_y)
// with (j0, t_x) = support of c_x(x,u) and (m0, t_y) of c_y(y,v), and skipped samples
// removed from both the sums and the counts (skip rule is per axis, so counts factorise).
// The interpolation coordinates are computed on the device for each plane ("computed
// on-the-fly in the main refocusing kernel") by KB5a in fp64 with the operation
// order of the declared convention, so skip / index decisions are exact.
//
// Stage 1 streams Gamma from HBM once per plane: a CTA owns one A row m and 8 B rows v,
// stages 8-column (u) slabs of the rows j it needs into padded shared memory (odd word
// stride -> conflict-free gathers), and each thread owns one output x.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

constexpr int kVG = 8;     // B rows v per stage-1 CTA
constexpr int kUC = 8;     // B columns u per staged slab
constexpr int kPad = 9;    // smem words per staged (v, j) row (odd -> no bank conflicts)
constexpr int kS1Threads = 256;

// ---- KB5a: per-axis interpolation tables ------------------------------------------
// Block per B coordinate ub (u or v), threads over the output coordinate x (or y).
// A-axis map c = ((a (x - c_a)) + (b (u - c_b))) + c_off + c_a: the default map is a = alpha,
// b = 1 - alpha, c_off = 0 (adding +0.0 leaves the default's value unchanged), a general
// RefocusMap row supplies (ax, bx, cx) / (ay, by, cy) (include/cpi.h cpi_refocus_spec.affine).
__device__ __forceinline__ void coords_block(double a, double b, double c_off, int boundary, int W, int Wb,
                                             AxisTables tab, int ub, bool b_ok);
// B coordinate of lattice index ub: c_B = ((e (ub - c_b)) + f) + c_b (fp64, oracle order); the
// integral map (1, 0) gives ub exactly.
__device__ __forceinline__ double b_coord(double e, double f, int Wb, int ub) {
    const double c_b = (Wb - 1) / 2.0;
    return __dadd_rn(__dadd_rn(__dmul_rn(e, __dadd_rn(static_cast<double>(ub), -c_b)), f), c_b);
}
// One launch for a fused group: blockIdx = (B coordinate, plane, axis 0 = x / 1 = y); the
// per-output counts are left to count_kernel (no atomics, no memsets).
__global__ void coords_group_kernel(CoordsGroupArgs g) {
    const int ax = blockIdx.z, f = blockIdx.y, ub = blockIdx.x;
    const int W = ax ? g.Ha : g.Wa, Wb = ax ? g.Hb : g.Wb;
    if (ub >= Wb) return;
    // the sample needs its B coordinate on the lattice too (skip policy)
    const double e = g.bmap[f][2 * ax], fo = g.bmap[f][2 * ax + 1];
    const double cb = b_coord(e, fo, Wb, ub);
    const bool b_ok = g.boundary != 0 || (cb >= 0.0 && cb <= static_cast<double>(Wb - 1));
    coords_block(g.map[f][3 * ax], g.map[f][3 * ax + 1], g.map[f][3 * ax + 2], g.boundary, W, Wb,
                 ax ? g.ys[f] : g.xs[f], ub, b_ok);
    if (g.genb && threadIdx.x == 0) {   // B support of this lattice index (clamped under CPI_CLAMP)
        const double c = fmin(fmax(cb, 0.0), static_cast<double>(Wb - 1));
        double fl = floor(c);
        if (fl > static_cast<double>(Wb - 2)) fl = static_cast<double>(Wb - 2);
        const AxisTables& bt = ax ? g.by[f] : g.bx[f];
        bt.i0[ub] = static_cast<int>(fl);
        bt.t[ub] = __dadd_rn(c, -fl);
    }
}
// cnt[x] = number of B coordinates with a used sample at output coordinate x.  CTA = (32
// outputs x, plane, axis); its 8 warps split the B coordinates and reduce in smem.
__global__ void count_kernel(CoordsGroupArgs g) {
    const int ax = blockIdx.z, f = blockIdx.y;
    const int W = ax ? g.Ha : g.Wa, Wb = ax ? g.Hb : g.Wb;
    const AxisTables& t = ax ? g.ys[f] : g.xs[f];
    const int x = blockIdx.x * 32 + (threadIdx.x & 31), part = threadIdx.x >> 5, parts = blockDim.x >> 5;
    __shared__ int sc[32][33];
    int c = 0;
    if (x < W)
        for (int ub = part; ub < Wb; ub += parts) c += __ldg(t.i0 + static_cast<int64_t>(ub) * W + x) >= 0;
    sc[threadIdx.x & 31][part] = c;
    __syncthreads();
    if (part == 0 && x < W) {
        int s = 0;
        for (int p = 0; p < parts; ++p) s += sc[threadIdx.x][p];
        t.cnt[x] = s;
    }
}
__device__ __forceinline__ void coords_block(double a, double b, double c_off, int boundary, int W, int Wb,
                                             AxisTables tab, int ub, bool b_ok) {
    const double c_a = (W - 1) / 2.0, c_b = (Wb - 1) / 2.0;
    const double bu = __dmul_rn(b, __dadd_rn(static_cast<double>(ub), -c_b));
    int lo = INT_MAX, hi = -1;
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
        // c = ((a*(x - c_a)) + (b*(u - c_b))) + c_off + c_a, each op rounded, no FMA
        double c = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, __dadd_rn(static_cast<double>(x), -c_a)), bu), c_off), c_a);
        bool ok;
        if (boundary == 0) {
            ok = b_ok && (c >= 0.0) && (c <= static_cast<double>(W - 1));
        } else {
            c = fmin(fmax(c, 0.0), static_cast<double>(W - 1));
            ok = true;
        }
        int i0 = 0;
        double t = 0.0;
        if (ok) {
            double f = floor(c);
            if (f > static_cast<double>(W - 2)) f = static_cast<double>(W - 2);
            i0 = static_cast<int>(f);
            t = __dadd_rn(c, -f);
            lo = min(lo, i0);
            hi = max(hi, i0 + 1);
        }
        tab.i0[static_cast<int64_t>(ub) * W + x] = ok ? i0 : -1;
        tab.t[static_cast<int64_t>(ub) * W + x] = t;
    }
    // block min / max
    __shared__ int slo[32], shi[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) { slo[warp] = lo; shi[warp] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) { lo = min(lo, slo[w]); hi = max(hi, shi[w]); }
        tab.lo[ub] = lo;
        tab.hi[ub] = hi;
    }
}

// ---- KB5: stage 1 -----------------------------------------------------------------
// grid (ceil(Hb / kVG), m_count, ceil(Wa / 256)); thread = output x.
__global__ void __launch_bounds__(kS1Threads)
stage1_kernel(const float* __restrict__ gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb,
              int m_base, AxisTables xs, AxisTables ys, TElem* __restrict__ T, int vmajor) {
    extern __shared__ float sm[];   // [kVG][nj][kPad]
    const int v0 = blockIdx.x * kVG;
    const int m = m_base + blockIdx.y;
    const int x = blockIdx.z * kS1Threads + threadIdx.x;
    const int nv = min(kVG, Hb - v0);
    // which of this CTA's v rows need A row m (stage 2 reads m in [lo_y(v), hi_y(v)])
    unsigned need = 0;
    for (int v = 0; v < nv; ++v) {
        const int lo = __ldg(ys.lo + v0 + v), hi = __ldg(ys.hi + v0 + v);
        if (m >= lo && m <= hi) need |= 1u << v;
    }
    if (!need) return;
    double acc[kVG];
#pragma unroll
    for (int v = 0; v < kVG; ++v) acc[v] = 0.0;
    const float* g_m = gamma + static_cast<int64_t>(m - m_base) * Wa * ldg;   // row (m, j=0) of the shard
    for (int u0 = 0; u0 < Wb; u0 += kUC) {
        const int nu = min(kUC, Wb - u0);
        int jlo = INT_MAX, jhi = -1;
        for (int k = 0; k < nu; ++k) {
            jlo = min(jlo, __ldg(xs.lo + u0 + k));
            jhi = max(jhi, __ldg(xs.hi + u0 + k));
        }
        if (jhi < jlo) continue;              // no x uses these u (block-uniform)
        const int nj = jhi - jlo + 1;
        __syncthreads();
        // stage rows (v, j), columns [u0, u0+nu): Gamma[(m, j)][(v0+v, u)]
        for (int rr = threadIdx.x; rr < nv * nj; rr += kS1Threads) {
            const int v = rr / nj, jj = rr - v * nj;
            float* dst = sm + (v * nj + jj) * kPad;
            if (vmajor) {   // B pixel (u, v) at column vmajor_slot(u, v) (CPI_GAMMA_VMAJOR)
                const float* row = g_m + static_cast<int64_t>(jlo + jj) * ldg;
                for (int k = 0; k < nu; ++k) dst[k] = __ldg(row + vmajor_slot(u0 + k, v0 + v, Wb, Hb));
                continue;
            }
            const float* src = g_m + static_cast<int64_t>(jlo + jj) * ldg + static_cast<int64_t>(v0 + v) * Wb + u0;
            if (nu == kUC && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
                const float4 p0 = __ldg(reinterpret_cast<const float4*>(src));
                const float4 p1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
                dst[0] = p0.x; dst[1] = p0.y; dst[2] = p0.z; dst[3] = p0.w;
                dst[4] = p1.x; dst[5] = p1.y; dst[6] = p1.z; dst[7] = p1.w;
            } else {
                for (int k = 0; k < nu; ++k) dst[k] = __ldg(src + k);
            }
        }
        __syncthreads();
        if (x < Wa) {
            float part[kVG];
#pragma unroll
            for (int v = 0; v < kVG; ++v) part[v] = 0.f;
            for (int k = 0; k < nu; ++k) {
                const int64_t ti = static_cast<int64_t>(u0 + k) * Wa + x;
                const int j0 = __ldg(xs.i0 + ti);
                if (j0 < 0) continue;
                // both corner weights rounded once from fp64 (the small one keeps its relative
                // precision)
                const double td = __ldg(xs.t + ti);
                const float t = __double2float_rn(td);
                const float w0 = __double2float_rn(1.0 - td);
                const float* s0 = sm + (j0 - jlo) * kPad + k;
#pragma unroll
                for (int v = 0; v < kVG; ++v) {
                    if (v < nv) {
                        const float g0 = s0[v * nj * kPad];
                        const float g1 = s0[v * nj * kPad + kPad];
                        part[v] = fmaf(t, g1, fmaf(w0, g0, part[v]));
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < kVG; ++v) acc[v] += static_cast<double>(part[v]);
        }
    }
    if (x < Wa) {
        TElem* dst = T + (static_cast<int64_t>(x) * Ha + m) * Hb + v0;
        for (int v = 0; v < nv; ++v)
            if (need & (1u << v)) dst[v] = acc[v];
    }
}

// ---- KB6: stage 2 -----------------------------------------------------------------
// One warp per output pixel (x, y); lanes stride over v; warp-shuffle fp64 reduction.
__global__ void stage2_kernel(const TElem* __restrict__ T, int Wa, int Ha, int Hb, int m_lo,
                              int m_hi, AxisTables xs, AxisTables ys, float* __restrict__ plane) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= static_cast<int64_t>(Wa) * Ha) return;
    const int x = static_cast<int>(gw % Wa), y = static_cast<int>(gw / Wa);
    const TElem* Tx = T + static_cast<int64_t>(x) * Ha * Hb;
    double sum = 0.0;
    for (int v = lane; v < Hb; v += 32) {
        const int64_t ti = static_cast<int64_t>(v) * Ha + y;
        const int m0 = __ldg(ys.i0 + ti);
        if (m0 < 0) continue;
        const double t = __ldg(ys.t + ti);
        const double t0 = (m0 >= m_lo && m0 < m_hi) ? Tx[static_cast<int64_t>(m0) * Hb + v] : 0.0;
        const double t1 = (m0 + 1 >= m_lo && m0 + 1 < m_hi) ? Tx[static_cast<int64_t>(m0 + 1) * Hb + v] : 0.0;
        sum += __dadd_rn(1.0, -t) * t0 + t * t1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
        const int64_t c = static_cast<int64_t>(__ldg(xs.cnt + x)) * __ldg(ys.cnt + y);
        plane[static_cast<int64_t>(y) * Wa + x] = c ? static_cast<float>(sum / static_cast<double>(c)) : 0.f;
    }
}


// ---- KB5 (TMA variant, F fused planes) --------------------------------------------
// Persistent, warp-specialised.  Tile = (A row m, 8 B rows v); the tile's Gamma is streamed
// in chunks of 8 B columns u: warp 8 (one elected lane) issues, per chunk, TMA boxes of
// 32 j-rows x 8 v x 8 u of Gamma covering only the union of the j spans the chunk's outputs
// touch in the F planes of the group, plus the 8 x W_a packed x-table rows of each plane,
// into a ring of mbarrier-guarded stages.  One HBM read of the span feeds F planes.
// Warps 0..7 consume: lane = (vq = lane/16, xl = lane%16), thread owns
// x = 16*warp + xl + 128*i (i < 2) and v = vq + 2*((s + xl/8) % 4) for slot s < 4.  At step k
// a lane reads column u' = (k + xl) % 8, so the 32 lanes hit 32 distinct banks
// (bank = 8 v + u') for any j0.  fp32 taps per 8-u chunk, fp64 across chunks.
constexpr int kTVG = 8, kTUC = 8, kTJBox = 32, kTMaxJ = 256;
constexpr int kTRow = kTVG * kTUC;                     // floats per staged j row (64)
constexpr int kTGFloats = (kTMaxJ + 2) * kTRow;        // 64.5 KB per stage; rows 256-257 stay zero
constexpr int kTXEntries = kTUC * 256;                 // 8 KB per plane per stage (uint32 entries)
constexpr int kTMaxChunks = 64;                        // W_b <= 512
// staged j rows of the TMA stage 1 for an A RoI of width W_a (the zero rows follow them)
__host__ __device__ constexpr int stage1_rows(int Wa) { return Wa <= 128 ? 128 : kTMaxJ; }
// B rows v per stage-1 tile: 16 for A RoIs up to 128 wide (their 130-row stages leave room), else 8
__host__ __device__ constexpr int stage1_vg(int kJ) { return kJ <= 128 ? 16 : kTVG; }
constexpr int kTConsumers = 8;
constexpr int kTThreads = 32 * (kTConsumers + 1);

// packed fp32 pairs for FFMA2 (sm_100a fma.rn.f32x2): lo = first, hi = second
__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float unpack_f32x2(uint64_t v, int hi) {
    float lo_f, hi_f;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo_f), "=f"(hi_f) : "l"(v));
    return hi ? hi_f : lo_f;
}
// d = (w, w) * g + c on both halves; w2 is the pre-packed broadcast of w
__device__ __forceinline__ uint64_t ffma2(float, uint64_t g, uint64_t c, uint64_t w2) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(w2), "l"(g), "l"(c));
    return d;
}

// The 8 taps of one packed x-table entry for one lane: 4 v slots x 2 corners, as FFMA2 pairs
// (lane-wise identical to scalar fmaf in the same order).  entry = j_rel << 23 (| a 2^-23 t the
// taps do not use), j_rel = smem row of j0 relative to the chunk's staged span (the zero rows for
// a skipped sample); sn = the sample's corner offset in the near-t form of the weight table
// (t for t <= 1/2, -(1 - t) above, 0 for a skipped sample), so both weights keep their relative
// precision (a t on the 2^-23 grid erred by up to 2^-24 |Gamma(j0 + 1) - Gamma(j0)|).
template <int NS, int kRow>
__device__ __forceinline__ void s1_taps(uint64_t (&part)[NS / 2], uint32_t e, float sn, const float* Gu,
                                        const int (&voff)[NS]) {
    const bool up = signbit(sn);
    const float w0 = up ? -sn : 1.f - sn;
    const float t = up ? 1.f + sn : sn;
    const float* gp = Gu + (e >> 23) * kRow;
    const uint64_t t2 = pack_f32x2(t, t), w2 = pack_f32x2(w0, w0);
#pragma unroll
    for (int p = 0; p < NS / 2; ++p) {
        const uint64_t g0 = pack_f32x2(gp[voff[2 * p]], gp[voff[2 * p + 1]]);
        const uint64_t g1 = pack_f32x2(gp[voff[2 * p] + kRow], gp[voff[2 * p + 1] + kRow]);
        part[p] = ffma2(t, g1, ffma2(w0, g0, part[p], w2), t2);
    }
}

// kJ = staged j rows (W_a <= kJ): 256, or 128 for A RoIs up to 128 wide, whose smaller stages
// give a 4-deep ring; rows kJ, kJ + 1 of every stage stay zero (skipped samples).
template <int F, int kJ = kTMaxJ>
struct S1Cfg {
    static constexpr int kVG = stage1_vg(kJ), kRow = kVG * kTUC;   // staged j row: kVG v x 8 u
    static constexpr int kGFloats = (kJ + 2) * kRow;
    // both row capacities: ~66 KB Gamma stages (three fit next to one plane's x-tables, two next
    // to 2-4 planes' tables)
    static constexpr int kStages = 2;   // (3 for F = 1 before the weight tables joined the ring)
    // smem map (bytes): [Gamma stages (258 rows each)][x-table stages x F][span table]
    //                   [x-block masks][barriers]
    static constexpr int kOffX = kStages * kGFloats * 4;
    static constexpr int kXEntries = kTUC * kJ;             // x-table entries per (stage, plane) slot
    static constexpr int kOffW = kOffX + kStages * F * kXEntries * 4;    // the x-tables' near-t weights
    static constexpr int kOffSpan = kOffW + kStages * F * kXEntries * 4;
    static constexpr int kOffXblk = kOffSpan + kTMaxChunks * 8;
    static constexpr int kOffYb = kOffXblk + kTMaxChunks * 4;   // int2 [F][H_b <= 256] y bands
    static constexpr int kOffBar = kOffYb + F * 256 * 8;
    static constexpr int kSmem = kOffBar + 4 * kStages * 8 + 64;
};

struct S1Args {
    int Wa, Ha, Wb, Hb, m_base, m_count, n_vg, n_chunks;
    int m_block, m_stride;                   // shard A-row l -> m_base + (l / m_block) * m_stride + l % m_block
    const int32_t* xlo[kRefocusMaxFuse];
    const int32_t* xhi[kRefocusMaxFuse];
    const int32_t* ylo[kRefocusMaxFuse];
    const int32_t* yhi[kRefocusMaxFuse];
    TElem* T[kRefocusMaxFuse];
    const uint32_t* xblk;                    // [F][n_chunks] x-block masks (OR-ed over F in smem)
    int gamma_5d;                            // Gamma map is 5D u-blocked (u%8, v, u/8, j, m)
};

// global A row of the shard's local A row l (block-cyclic row ownership)
__device__ __forceinline__ int shard_row(const S1Args& a, int l) {
    return a.m_base + (l / a.m_block) * a.m_stride + l % a.m_block;
}

// v rows of the tile (m, v0..v0+7) that plane f needs: m inside the used band [lo_y(v), hi_y(v)]
// of stage 2 (bands staged in smem once per CTA)
__device__ __forceinline__ unsigned tile_mask(const int2* yband, int Hb, int m, int v0, int f, int vgs) {
    unsigned need = 0;
    const int nv = min(vgs, Hb - v0);
    for (int v = 0; v < nv; ++v) {
        const int2 b = yband[f * 256 + v0 + v];
        if (m >= b.x && m <= b.y) need |= 1u << v;
    }
    return need;
}

#define C_SMEM_OK(F, kJ) (S1Cfg<F, kJ>::kSmem <= 232448)
template <bool kFullX, int F, bool kSkip, int kJ>
__global__ void __launch_bounds__(kTThreads, 1)
stage1_tma_kernel(const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_x,
                  const __grid_constant__ CUtensorMap tm_w, S1Args a) {
    static_assert(C_SMEM_OK(F, kJ), "stage-1 shared memory exceeds 227 KB");
    using C = S1Cfg<F, kJ>;
    extern __shared__ __align__(1024) uint8_t s1_smem[];
    float* sg = reinterpret_cast<float*>(s1_smem);
    const uint32_t* sx = reinterpret_cast<const uint32_t*>(s1_smem + C::kOffX);
    const float* swt = reinterpret_cast<const float*>(s1_smem + C::kOffW);
    int2* span = reinterpret_cast<int2*>(s1_smem + C::kOffSpan);
    uint64_t* full = reinterpret_cast<uint64_t*>(s1_smem + C::kOffBar);
    uint64_t* empty = full + C::kStages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTConsumers);
        }
        fence_mbar_init();
    }
    // zero every staged Gamma row once: rows 256-257 of each stage are the skipped-sample
    // rows, and a zero-weight tap past a chunk's span then reads 0 or an earlier finite value
    for (int i = threadIdx.x; i < C::kStages * C::kGFloats; i += blockDim.x) sg[i] = 0.f;
    fence_proxy_async_smem();   // the zeros must land before the first TMA writes these rows
    // union j span [lo, hi] over the F planes of every u chunk (lo > hi: chunk unused)
    for (int c = threadIdx.x; c < a.n_chunks; c += blockDim.x) {
        int lo = INT_MAX, hi = -1;
#pragma unroll
        for (int f = 0; f < F; ++f)
            for (int k = 0; k < kTUC && c * kTUC + k < a.Wb; ++k) {
                lo = min(lo, __ldg(a.xlo[f] + c * kTUC + k));
                hi = max(hi, __ldg(a.xhi[f] + c * kTUC + k));
            }
        span[c] = make_int2(lo, hi);
    }
    int2* yband = reinterpret_cast<int2*>(s1_smem + C::kOffYb);
    for (int i = threadIdx.x; i < F * a.Hb; i += blockDim.x) {
        const int f = i / a.Hb, v = i - f * a.Hb;
        yband[f * 256 + v] = make_int2(__ldg(a.ylo[f] + v), __ldg(a.yhi[f] + v));
    }
    uint32_t* xblk = reinterpret_cast<uint32_t*>(s1_smem + C::kOffXblk);
    for (int c = threadIdx.x; c < a.n_chunks; c += blockDim.x) {   // OR over the group's planes
        uint32_t b = 0;
#pragma unroll
        for (int f = 0; f < F; ++f) b |= __ldg(a.xblk + f * a.n_chunks + c);
        xblk[c] = b;
    }
    __syncthreads();
    const int n_tiles = a.m_count * a.n_vg;
    const int t_first = blockIdx.x, t_step = gridDim.x, t_end = n_tiles;   // persistent tile loop

    if (warp == kTConsumers) {
        if (lane == 0) {
            tma_prefetch_desc(&tm_g);
            tma_prefetch_desc(&tm_x);
            tma_prefetch_desc(&tm_w);
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = t_first; tile < t_end; tile += t_step) {
                const int ml = tile / a.n_vg, vg = tile - ml * a.n_vg;
                unsigned any = 0;
#pragma unroll
                for (int f = 0; f < F; ++f) any |= tile_mask(yband, a.Hb, shard_row(a, ml), vg * C::kVG, f, C::kVG);
                if (!any) continue;
                for (int c = 0; c < a.n_chunks; ++c) {
                    const int2 sp = span[c];
                    if (sp.y < sp.x) continue;
                    const int nb = (sp.y - sp.x + kTJBox) / kTJBox;
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], nb * kTJBox * C::kRow * 4 + 2 * F * kTUC * a.Wa * 4);
                    float* dst = sg + stage * C::kGFloats;
                    for (int b = 0; b < nb; ++b) {
                        if (a.gamma_5d)   // u-blocked Gamma: one 256-B segment per (j, chunk)
                            tma_load_5d(dst + b * kTJBox * C::kRow, &tm_g, &full[stage], 0, vg * C::kVG, c,
                                        sp.x + b * kTJBox, ml);
                        else
                            tma_load_4d(dst + b * kTJBox * C::kRow, &tm_g, &full[stage], c * kTUC, vg * C::kVG,
                                        sp.x + b * kTJBox, ml);
                    }
#pragma unroll
                    for (int f = 0; f < F; ++f)
                            tma_load_3d(s1_smem + C::kOffX + (stage * F + f) * C::kXEntries * 4, &tm_x, &full[stage], 0,
                                        c * kTUC, f);
#pragma unroll
                    for (int f = 0; f < F; ++f)
                            tma_load_3d(s1_smem + C::kOffW + (stage * F + f) * C::kXEntries * 4, &tm_w, &full[stage], 0,
                                        c * kTUC, f);
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
        return;
    }

    const int vq = lane >> 4, xl = lane & 15, hi = xl >> 3;
    const int xbase = warp * 16 + xl;
    constexpr int NS = C::kVG / 2, NI = kJ <= 128 ? 1 : 2;   // v slots per lane, x blocks per lane
    int voff[NS];                                          // float offset of slot s's v row
#pragma unroll
    for (int s = 0; s < NS; ++s) voff[s] = (vq + 2 * ((s + hi) & (NS - 1))) * kTUC;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = t_first; tile < t_end; tile += t_step) {
        const int ml = tile / a.n_vg, vg = tile - ml * a.n_vg;
        const int m = shard_row(a, ml), v0 = vg * C::kVG;
        unsigned mask[F], any = 0;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            mask[f] = tile_mask(yband, a.Hb, m, v0, f, C::kVG);
            any |= mask[f];
        }
        if (!any) continue;
        double acc[F][NI][NS];
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
            for (int i = 0; i < NI; ++i)
#pragma unroll
                for (int s = 0; s < NS; ++s) acc[f][i][s] = 0.0;
        for (int c = 0; c < a.n_chunks; ++c) {
            const int2 sp = span[c];
            if (sp.y < sp.x) continue;
            mbar_wait(&full[stage], phase);
            const float* G = sg + stage * C::kGFloats;
            // fp32 partial sums of this chunk as packed pairs (slots s = 2p, 2p + 1): the taps run
            // on FFMA2 (fma.rn.f32x2), lane-wise identical to two scalar fmaf in the same order
            uint64_t part[F][NI][NS / 2];
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int i = 0; i < NI; ++i)
#pragma unroll
                    for (int p = 0; p < NS / 2; ++p) part[f][i][p] = 0ull;
            const uint32_t* sxs = sx + stage * F * C::kXEntries + xbase;
            const float* swx = swt + stage * F * C::kXEntries + xbase;   // the same entries' weights
            if constexpr (kSkip) {
                // i-outer order with a warp-uniform skip of a 16-wide x block that has no used
                // sample in this chunk for any plane of the group
                const uint32_t xb = xblk[c] >> warp;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    if (!((xb >> (8 * i)) & 1u)) continue;
                    if (!kFullX && xbase + 128 * i >= a.Wa) continue;
                    // all x-table entries of this x block first, so entry decode overlaps taps
                    uint32_t ent[kTUC][F];
                    float sn[kTUC][F];
#pragma unroll
                    for (int k = 0; k < kTUC; ++k) {
                        const int uu = (k + xl) & (kTUC - 1);
#pragma unroll
                        for (int f = 0; f < F; ++f) {
                            ent[k][f] = sxs[f * C::kXEntries + uu * a.Wa + 128 * i];
                            sn[k][f] = swx[f * C::kXEntries + uu * a.Wa + 128 * i];
                        }
                    }
#pragma unroll
                    for (int k = 0; k < kTUC; ++k) {
                        const int uu = (k + xl) & (kTUC - 1);
#pragma unroll
                        for (int f = 0; f < F; ++f) s1_taps<NS, C::kRow>(part[f][i], ent[k][f], sn[k][f], G + uu, voff);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < kTUC; ++k) {
                    const int uu = (k + xl) & (kTUC - 1);
#pragma unroll
                    for (int f = 0; f < F; ++f)
#pragma unroll
                        for (int i = 0; i < NI; ++i)
                            if (kFullX || xbase + 128 * i < a.Wa) {
                                const float sn = swx[f * C::kXEntries + uu * a.Wa + 128 * i];
                                s1_taps<NS, C::kRow>(part[f][i], sxs[f * C::kXEntries + uu * a.Wa + 128 * i], sn,
                                                     G + uu, voff);
                            }
                }
            }
            // Release the stage to the TMA producer.  The reads above are generic-proxy loads and
            // the refill is an async-proxy write: order them with a proxy fence before the arrive
            // (without it the refill could land while loads of this stage are still in flight).
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int i = 0; i < NI; ++i)
#pragma unroll
                    for (int s = 0; s < NS; ++s) acc[f][i][s] += static_cast<double>(unpack_f32x2(part[f][i][s >> 1], s & 1));
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int x = xbase + 128 * i;
                if (!kFullX && x >= a.Wa) continue;
                TElem* dst = a.T[f] + (static_cast<int64_t>(x) * a.Ha + m) * a.Hb + v0;
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const int v = vq + 2 * ((s + hi) & (NS - 1));
                    if (mask[f] & (1u << v)) dst[v] = acc[f][i][s];
                }
            }
    }
}

// Packed x-tables of a fused group of F planes for the TMA stage 1 (W_a <= 256):
//   entry(f, u, x) = j_rel << 23 | round(t * 2^23)
// where j_rel = j0 - j_lo(chunk of u) is the smem row of the lower tap inside the chunk's
// staged union span (the same union the producer stages), t in [0, 1) (a t that rounds to
// 1 moves to the next row with t = 0), and skipped samples point at the zero rows
// (j_rel = zrow = the stage's row capacity, t = 0).  t keeps 2^-23 resolution; t = 0 stays exact.
__global__ void pack_xtable_group_kernel(PackGroupArgs g, int Wa, int Wb, uint32_t zrow, uint32_t* __restrict__ out,
                                         float* __restrict__ outw, uint32_t* __restrict__ xblk) {
    const int c = blockIdx.x, f = blockIdx.y, c0 = c * 8, n_chunks = gridDim.x;
    __shared__ uint32_t sblk;
    if (threadIdx.x == 0) sblk = 0;
    int jlo = INT_MAX;
    for (int ff = 0; ff < g.n; ++ff)
        for (int k = c0; k < c0 + 8 && k < Wb; ++k) jlo = min(jlo, __ldg(g.lo[ff] + k));
    __syncthreads();
    for (int x = threadIdx.x; x < Wa; x += blockDim.x) {
        bool used = false;
        for (int u = c0; u < c0 + 8 && u < Wb; ++u) {
            const int64_t idx = static_cast<int64_t>(u) * Wa + x;
            const int j = __ldg(g.i0[f] + idx);
            uint32_t e = zrow << 23;
            float sn = 0.f;
            if (j >= 0) {
                const double t = __ldg(g.t[f] + idx);
                e = static_cast<uint32_t>(j - jlo) << 23;
                // near-t form (s1_taps): -(1 - t) is exact in fp64 for t > 1/2; t = 1 -> -0.0
                sn = __double2float_rn(t > 0.5 ? -(1.0 - t) : t);
                used = true;
            }
            out[(static_cast<int64_t>(f) * Wb + u) * Wa + x] = e;
            outw[(static_cast<int64_t>(f) * Wb + u) * Wa + x] = sn;
        }
        if (used) atomicOr(&sblk, 1u << (x >> 4));
    }
    __syncthreads();
    if (threadIdx.x == 0) xblk[f * n_chunks + c] = sblk;
}

// ---- KB6 (staged): stage 2 for a fused group of planes -------------------------------
// grid (ceil(W_a / 2), F); CTA = 2 output columns x of one plane, thread = output row y
// (H_a <= 256).  The CTA walks v in chunks of 16: it stages T[x][m][v0..v0+15] for every m
// (64-byte coalesced fp32 row segments; rows outside the used band [lo_y(v), hi_y(v)] and outside
// the caller's row shard [m_lo, m_hi) are stored as 0) transposed to [x][v][m], plus the
// chunk's packed y-table rows; every thread then gathers its two taps per (x, v) from shared
// memory (the pair interpolated in fp32, accumulated over v in fp64).  The next chunk's loads
// are issued into registers before the current chunk is consumed, so HBM latency overlaps
// the gathers.  T is read from HBM once per plane.
constexpr int kS2VC = 16, kS2XB = 2, kS2Threads = 256, kS2MI = 256 / (kS2Threads / kS2VC);

struct S2Args {
    int Wa, Ha, Hb;
    int m_base, m_count, m_block, m_stride;      // rows of T present: the shard's A rows (see S1Args)
    const TElem* T[kS2MaxPlanes];
    const int32_t* xcnt[kS2MaxPlanes];
    const int32_t* ycnt[kS2MaxPlanes];
    const int32_t* ylo[kS2MaxPlanes];
    const int32_t* yhi[kS2MaxPlanes];
    const uint2* ypack;                          // [F][H_b][H_a] (m_near, delta) entries
    float* plane[kS2MaxPlanes];
};

__global__ void __launch_bounds__(kS2Threads, 2)
stage2_staged_kernel(S2Args a) {
    extern __shared__ __align__(16) uint8_t s2_smem[];
    const int f = blockIdx.y, x0 = blockIdx.x * kS2XB;
    const int Ha = a.Ha, Hb = a.Hb, P = Ha + 2;           // staged row pitch (rows Ha, Ha+1 = 0)
    TElem* ts = reinterpret_cast<TElem*>(s2_smem);                       // [kS2XB][kS2VC][P]
    uint2* tab = reinterpret_cast<uint2*>(ts + kS2XB * kS2VC * P);        // [kS2VC][Ha]
    const TElem* T = a.T[f];
    const uint2* yp = a.ypack + static_cast<int64_t>(f) * Hb * Ha;
    const int32_t* ylo = a.ylo[f];
    const int32_t* yhi = a.yhi[f];
    for (int i = threadIdx.x; i < kS2XB * kS2VC * 2; i += blockDim.x) ts[(i >> 1) * P + Ha + (i & 1)] = 0.f;
    // loader role: thread = (vv = tid % 8, m = tid / 8 + 32 k), both x of the CTA
    const int vl = threadIdx.x & (kS2VC - 1), ml = threadIdx.x / kS2VC;
    TElem pre[kS2XB][kS2MI];
    uint2 ptab[kS2MI];
    uint32_t present = 0;                          // bit k: this thread's row m = ml + 32 k is in the shard
#pragma unroll
    for (int k = 0; k < kS2MI; ++k) {
        const int rel = ml + k * (kS2Threads / kS2VC) - a.m_base;
        if (rel >= 0) {
            const int blk = rel / a.m_stride, off = rel - blk * a.m_stride;
            if (off < a.m_block && blk * a.m_block + off < a.m_count) present |= 1u << k;
        }
    }
    auto prefetch = [&](int v0) {
        const int v = v0 + vl, nvalid = min(kS2VC, Hb - v0) * Ha;   // table entries of real v rows
        int lo = 1, hi = 0;
        if (v < Hb) { lo = __ldg(ylo + v); hi = __ldg(yhi + v); }
#pragma unroll
        for (int k = 0; k < kS2MI; ++k) {
            const int m = ml + k * (kS2Threads / kS2VC);
            const bool ok = m >= lo && m <= hi && ((present >> k) & 1u);
#pragma unroll
            for (int xb = 0; xb < kS2XB; ++xb) {
                const int x = x0 + xb;
                pre[xb][k] = ok && x < a.Wa ? __ldg(T + (static_cast<int64_t>(x) * Ha + m) * Hb + v) : 0.f;
            }
            const int i = threadIdx.x + k * kS2Threads;               // table entry (vv, y)
            ptab[k] = i < nvalid ? __ldg(yp + static_cast<int64_t>(v0) * Ha + i) : make_uint2(static_cast<uint32_t>(Ha), 0u);
        }
    };
    double sum[kS2XB];
#pragma unroll
    for (int xb = 0; xb < kS2XB; ++xb) sum[xb] = 0.0;
    const int y = threadIdx.x;
    prefetch(0);
    for (int v0 = 0; v0 < Hb; v0 += kS2VC) {
        __syncthreads();                                  // previous chunk consumed
#pragma unroll
        for (int k = 0; k < kS2MI; ++k) {
            const int m = ml + k * (kS2Threads / kS2VC);
            if (m < Ha) {
#pragma unroll
                for (int xb = 0; xb < kS2XB; ++xb) ts[(xb * kS2VC + vl) * P + m] = pre[xb][k];
            }
            const int i = threadIdx.x + k * kS2Threads;
            if (i < kS2VC * Ha) tab[i] = ptab[k];
        }
        __syncthreads();
        if (v0 + kS2VC < Hb) prefetch(v0 + kS2VC);        // in flight while this chunk is gathered
        if (y < Ha) {
#pragma unroll
            for (int vv = 0; vv < kS2VC; ++vv) {
                // entry = (nearest row m_near, delta = c - m_near in fp32): the small weight |delta|
                // is exact to 2^-24 relative, the large one 1 - |delta| >= 1/2 likewise, so each
                // corner's weight carries a relative error <= 2^-24
                const uint2 e = tab[vv * Ha + y];
                const float d = __uint_as_float(e.y), s = fabsf(d), big = 1.f - s;
                const bool below = d < 0.f;   // c lies in [m_near - 1, m_near]
                const int m0 = static_cast<int>(e.x) - (below ? 1 : 0);
                const float w0 = below ? s : big, w1 = below ? big : s;
#pragma unroll
                for (int xb = 0; xb < kS2XB; ++xb) {
                    const TElem* row = ts + (xb * kS2VC + vv) * P + m0;
                    sum[xb] += static_cast<double>(fmaf(w1, row[1], w0 * row[0]));
                }
            }
        }
    }
    if (y < Ha) {
        const int64_t cy = __ldg(a.ycnt[f] + y);
#pragma unroll
        for (int xb = 0; xb < kS2XB; ++xb) {
            const int x = x0 + xb;
            if (x >= a.Wa) continue;
            const int64_t c = cy * __ldg(a.xcnt[f] + x);
            a.plane[f][static_cast<int64_t>(y) * a.Wa + x] = c ? static_cast<float>(sum[xb] / static_cast<double>(c)) : 0.f;
        }
    }
}

// Packed y-tables of a group: entry(f, v, y) = (m_near, delta) with c = i0 + t, m_near = i0 and
// delta = t for t <= 1/2, else m_near = i0 + 1 and delta = t - 1 (exact in fp64), delta rounded
// once to fp32 -- relative, not absolute, precision for the small corner weight (a fixed-point t
// on a 2^-23 grid loses it when t or 1 - t is tiny: |error| up to 2^-24 |T(i0 + 1) - T(i0)|,
// beyond 1e-6 M when the two corners differ widely).  Skipped samples point at the zero rows
// (m_near = H_a, delta = 0).
__global__ void pack_ytable_kernel(PackGroupArgs g, int Ha, int Hb, uint2* __restrict__ out) {
    const int v = blockIdx.x, f = blockIdx.y;
    for (int y = threadIdx.x; y < Ha; y += blockDim.x) {
        const int64_t idx = static_cast<int64_t>(v) * Ha + y;
        const int m0 = __ldg(g.i0[f] + idx);
        uint2 e = make_uint2(static_cast<uint32_t>(Ha), 0u);
        if (m0 >= 0) {
            const double t = __ldg(g.t[f] + idx);
            const bool up = t > 0.5;
            e = make_uint2(static_cast<uint32_t>(m0 + (up ? 1 : 0)), __float_as_uint(__double2float_rn(up ? t - 1.0 : t)));
        }
        out[(static_cast<int64_t>(f) * Hb + v) * Ha + y] = e;
    }
}

// ---- general-B refocus (fractional B coordinates depending on u / v only) ----------------
// Stage 1: CTA = (8 B rows n, A row m, 256 x); u is walked in chunks whose B supports span at
// most kGbCols columns; the chunk's Gamma rows (n, j in span) x those columns are staged in
// padded smem and each thread (x) takes 2 x 2 corners per (u, n).
constexpr int kGbCols = 10, kGbPad = 11, kGbMaxU = 8;

__global__ void __launch_bounds__(kS1Threads)
stage1_genb_kernel(const float* __restrict__ gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb, int m_base,
                   AxisTables xs, AxisTables bx, TElem* __restrict__ T) {
    extern __shared__ float sgb[];   // [kVG][nj][kGbPad]
    const int n0 = blockIdx.x * kVG;
    const int m = m_base + blockIdx.y;
    const int x = blockIdx.z * kS1Threads + threadIdx.x;
    const int nv = min(kVG, Hb - n0);
    double acc[kVG];
#pragma unroll
    for (int v = 0; v < kVG; ++v) acc[v] = 0.0;
    const float* g_m = gamma + static_cast<int64_t>(m - m_base) * Wa * ldg;
    int u0 = 0;
    while (u0 < Wb) {
        // grow the chunk while its B supports fit kGbCols columns (block-uniform)
        int klo = INT_MAX, khi = -1, jlo = INT_MAX, jhi = -1, nu = 0;
        while (u0 + nu < Wb && nu < kGbMaxU) {
            const int k = __ldg(bx.i0 + u0 + nu);
            const int l = min(klo, k), h = max(khi, k + 1);
            if (h - l + 1 > kGbCols) break;
            klo = l; khi = h;
            jlo = min(jlo, __ldg(xs.lo + u0 + nu));
            jhi = max(jhi, __ldg(xs.hi + u0 + nu));
            ++nu;
        }
        const int nk = khi - klo + 1;
        if (jhi >= jlo) {
            const int nj = jhi - jlo + 1;
            __syncthreads();
            for (int rr = threadIdx.x; rr < nv * nj * nk; rr += kS1Threads) {
                const int v = rr / (nj * nk), rem = rr - v * nj * nk, jj = rem / nk, kk = rem - jj * nk;
                sgb[(v * nj + jj) * kGbPad + kk] =
                    __ldg(g_m + static_cast<int64_t>(jlo + jj) * ldg + static_cast<int64_t>(n0 + v) * Wb + klo + kk);
            }
            __syncthreads();
            if (x < Wa) {
                float part[kVG];
#pragma unroll
                for (int v = 0; v < kVG; ++v) part[v] = 0.f;
                for (int q = 0; q < nu; ++q) {
                    const int u = u0 + q;
                    const int64_t ti = static_cast<int64_t>(u) * Wa + x;
                    const int j0 = __ldg(xs.i0 + ti);
                    if (j0 < 0) continue;
                    const double td = __ldg(xs.t + ti), tkd = __ldg(bx.t + u);
                    const float t = __double2float_rn(td), w0 = __double2float_rn(1.0 - td);
                    const float tk = __double2float_rn(tkd), wk0 = __double2float_rn(1.0 - tkd);
                    const int kk = __ldg(bx.i0 + u) - klo;
                    const float* s0 = sgb + (j0 - jlo) * kGbPad + kk;
#pragma unroll
                    for (int v = 0; v < kVG; ++v) {
                        if (v < nv) {
                            const float* r = s0 + v * nj * kGbPad;
                            const float lo = fmaf(tk, r[1], wk0 * r[0]);
                            const float hi = fmaf(tk, r[kGbPad + 1], wk0 * r[kGbPad]);
                            part[v] = fmaf(t, hi, fmaf(w0, lo, part[v]));
                        }
                    }
                }
#pragma unroll
                for (int v = 0; v < kVG; ++v) acc[v] += static_cast<double>(part[v]);
            }
        }
        u0 += nu;
    }
    if (x < Wa) {
        TElem* dst = T + (static_cast<int64_t>(x) * Ha + m) * Hb + n0;
        for (int v = 0; v < nv; ++v) dst[v] = acc[v];
    }
}

// Stage 2: one warp per output pixel (x, y); lanes over v; 2 x 2 corners (m, n) of T.
__global__ void stage2_genb_kernel(const TElem* __restrict__ T, int Wa, int Ha, int Hb, int m_lo, int m_hi,
                                   AxisTables xs, AxisTables ys, AxisTables by, float* __restrict__ plane) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= static_cast<int64_t>(Wa) * Ha) return;
    const int x = static_cast<int>(gw % Wa), y = static_cast<int>(gw / Wa);
    const TElem* Tx = T + static_cast<int64_t>(x) * Ha * Hb;
    double sum = 0.0;
    for (int v = lane; v < Hb; v += 32) {
        const int64_t ti = static_cast<int64_t>(v) * Ha + y;
        const int m0 = __ldg(ys.i0 + ti);
        if (m0 < 0) continue;
        const double t = __ldg(ys.t + ti);
        const int n = __ldg(by.i0 + v);
        const double tn = __ldg(by.t + v);
        double c[2];
        for (int dm = 0; dm < 2; ++dm) {
            const int mm = m0 + dm;
            const bool in = mm >= m_lo && mm < m_hi;
            const double a0 = in ? Tx[static_cast<int64_t>(mm) * Hb + n] : 0.0;
            const double a1 = in ? Tx[static_cast<int64_t>(mm) * Hb + n + 1] : 0.0;
            c[dm] = __dadd_rn(1.0, -tn) * a0 + tn * a1;
        }
        sum += __dadd_rn(1.0, -t) * c[0] + t * c[1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
        const int64_t cnt = static_cast<int64_t>(__ldg(xs.cnt + x)) * __ldg(ys.cnt + y);
        plane[static_cast<int64_t>(y) * Wa + x] = cnt ? static_cast<float>(sum / static_cast<double>(cnt)) : 0.f;
    }
}

// ---- general-B pre-pass: resample Gamma onto the B lattice -------------------------------
// With B coordinates that depend on u / v only (dx = dy = 0), the 16-corner multilinear weight
// of a sample factorises into (A corners) x (B corners), so
//   sum_A w_A sum_B w_B Gamma(A corner; B corner) = sum_A w_A Gamma'(A corner; v, u),
//   Gamma'(p; v, u) = (1 - t_v) [(1 - t_u) G(n, k) + t_u G(n, k + 1)] + t_v [(1 - t_u) G(n + 1, k) + t_u G(n + 1, k + 1)]
// with (k, t_u) = bx[u], (n, t_v) = by[v] the B support of the map (skipped samples are
// removed by the A tables, which carry the B lattice test).  Gamma' then runs through the
// separable fast path with the identity B map.  grid (rows, ceil(P_b / (kV * 256))); thread =
// kV consecutive B slots of one A pixel (same v, consecutive u in both B orders).
template <int kV>
__global__ void __launch_bounds__(256)
resample_b_kernel(const float* __restrict__ src, float* __restrict__ dst, int Wb, int Hb, int ub,
                  const int32_t* __restrict__ bxi, const double* __restrict__ bxt, const int32_t* __restrict__ byi,
                  const double* __restrict__ byt) {
    const int64_t pb = static_cast<int64_t>(Wb) * Hb;
    const int q = (blockIdx.y * 256 + threadIdx.x) * kV;
    if (q >= pb) return;
    const int64_t p = blockIdx.x;
    int v, u0;
    if (ub) {
        const int u8 = q / (8 * Hb), r = q - u8 * 8 * Hb;
        v = r >> 3;
        u0 = u8 * 8 + (r & 7);
    } else {
        v = q / Wb;
        u0 = q - v * Wb;
    }
    const float* s = src + p * pb;
    const int n = __ldg(byi + v);
    const double tv = __ldg(byt + v), wv = __dadd_rn(1.0, -tv);
    float out[kV];
#pragma unroll
    for (int i = 0; i < kV; ++i) {
        const int u = u0 + i;
        const int k = __ldg(bxi + u);
        const double tu = __ldg(bxt + u), wu = __dadd_rn(1.0, -tu);
        int64_t i00, i01, i10, i11;
        if (ub) {
            const int64_t c0 = static_cast<int64_t>(k >> 3) * 8 * Hb + (k & 7);
            const int64_t c1 = static_cast<int64_t>((k + 1) >> 3) * 8 * Hb + ((k + 1) & 7);
            i00 = c0 + 8 * n; i01 = c1 + 8 * n; i10 = c0 + 8 * (n + 1); i11 = c1 + 8 * (n + 1);
        } else {
            i00 = static_cast<int64_t>(n) * Wb + k; i01 = i00 + 1; i10 = i00 + Wb; i11 = i10 + 1;
        }
        const double lo = wu * static_cast<double>(__ldg(s + i00)) + tu * static_cast<double>(__ldg(s + i01));
        const double hi = wu * static_cast<double>(__ldg(s + i10)) + tu * static_cast<double>(__ldg(s + i11));
        out[i] = static_cast<float>(wv * lo + tv * hi);
    }
    float* d = dst + p * pb + q;
    if constexpr (kV == 4) {
        __stcs(reinterpret_cast<float4*>(d), make_float4(out[0], out[1], out[2], out[3]));
    } else {
        d[0] = out[0];
    }
}

// v-major B order (CPI_GAMMA_VMAJOR, slot q = vmajor_slot(u, v)): thread = one slot; consecutive
// threads take consecutive v of one u and v block, so the corner reads (rows n(v), n(v) + 1 of
// columns k(u), k(u) + 1) and the stores are coalesced.
__global__ void __launch_bounds__(256)
resample_b_vmajor_kernel(const float* __restrict__ src, float* __restrict__ dst, int Wb, int Hb,
                         const int32_t* __restrict__ bxi, const double* __restrict__ bxt,
                         const int32_t* __restrict__ byi, const double* __restrict__ byt) {
    const int64_t pb = static_cast<int64_t>(Wb) * Hb;
    const int64_t q = static_cast<int64_t>(blockIdx.y) * 256 + threadIdx.x;
    if (q >= pb) return;
    const int64_t p = blockIdx.x;
    const int vbs = vmajor_block(Hb);
    const int64_t blk = q / (static_cast<int64_t>(Wb) * vbs), r = q - blk * Wb * vbs;
    const int u = static_cast<int>(r / vbs), v = static_cast<int>(blk * vbs + r % vbs);
    const float* s = src + p * pb;
    const int n = __ldg(byi + v), k = __ldg(bxi + u);
    const double tv = __ldg(byt + v), wv = __dadd_rn(1.0, -tv);
    const double tu = __ldg(bxt + u), wu = __dadd_rn(1.0, -tu);
    const double lo = wu * static_cast<double>(__ldg(s + vmajor_slot(k, n, Wb, Hb))) +
                      tu * static_cast<double>(__ldg(s + vmajor_slot(k + 1, n, Wb, Hb)));
    const double hi = wu * static_cast<double>(__ldg(s + vmajor_slot(k, n + 1, Wb, Hb))) +
                      tu * static_cast<double>(__ldg(s + vmajor_slot(k + 1, n + 1, Wb, Hb)));
    __stcs(dst + p * pb + q, static_cast<float>(wv * lo + tv * hi));
}

// Banded form (the default): CTA = (A pixel p, band of kRsV B rows v).  The band's B support
// rows n in [lo, hi + 1] (n(v) is monotone in v, so the band ends bound it) are staged in
// shared memory with coalesced 16-byte loads, de-blocked to row-major [n][k] with a padded row
// stride; each thread then owns B columns u (weights loaded once) and walks the band's rows v,
// four shared-memory taps and three FMAs per output, stores coalesced across the warp.  The
// host sizes the stage to the map's bound on the support rows (cap = ceil(|ey| (kRsV - 1)) + 4,
// 20 rows for |ey| <= 1, so several CTAs per SM keep loads in flight) and launches this form
// only when cap <= kRsCap, else the gather form above.
constexpr int kRsV = 16, kRsCap = 40;
__host__ __device__ constexpr int rs_pitch(int Wb) { return Wb + 8; }
template <bool kUB>
__global__ void __launch_bounds__(256)
resample_b_band_kernel(const float* __restrict__ src, float* __restrict__ dst, int Wb, int Hb, int cap,
                       const int32_t* __restrict__ bxi, const double* __restrict__ bxt,
                       const int32_t* __restrict__ byi, const double* __restrict__ byt) {
    extern __shared__ float4 rs_sm4[];
    float* s_g = reinterpret_cast<float*>(rs_sm4);   // [kRsCap][pitch]
    __shared__ int s_vr[kRsV];                       // support row of v0 + i, relative to lo
    __shared__ float s_vt[kRsV], s_vw[kRsV];         // its weights t and 1 - t (each rounded once)
    const int pitch = rs_pitch(Wb);
    const int64_t pb = static_cast<int64_t>(Wb) * Hb;
    const int64_t p = blockIdx.x;
    const int v0 = blockIdx.y * kRsV, nv = min(kRsV, Hb - v0);
    const int na = __ldg(byi + v0), nz = __ldg(byi + v0 + nv - 1);
    const int lo = min(na, nz), rows = max(na, nz) + 2 - lo;   // support rows [lo, lo + rows)
    if (threadIdx.x < nv) {
        s_vr[threadIdx.x] = (__ldg(byi + v0 + threadIdx.x) - lo) * pitch;
        const double tvd = __ldg(byt + v0 + threadIdx.x);
        s_vt[threadIdx.x] = __double2float_rn(tvd);
        s_vw[threadIdx.x] = __double2float_rn(1.0 - tvd);
    }
    const float* s = src + p * pb;
    if (rows > cap) {   // cannot happen for the host's cap; kept as a safe global-memory path
        for (int w = threadIdx.x; w < nv * Wb; w += 256) {
            const int v = v0 + w / Wb, u = w % Wb;
            const int n = __ldg(byi + v), k = __ldg(bxi + u);
            const double tud = __ldg(bxt + u), tvd = __ldg(byt + v);
            const float tu = __double2float_rn(tud), wu = __double2float_rn(1.0 - tud);
            const float tv = __double2float_rn(tvd), wv = __double2float_rn(1.0 - tvd);
            auto at = [&](int nn, int kk) {
                return __ldg(s + (kUB ? static_cast<int64_t>(kk >> 3) * 8 * Hb + 8 * nn + (kk & 7)
                                      : static_cast<int64_t>(nn) * Wb + kk));
            };
            const float a = fmaf(tu, at(n, k + 1), wu * at(n, k));
            const float b = fmaf(tu, at(n + 1, k + 1), wu * at(n + 1, k));
            dst[p * pb + (kUB ? static_cast<int64_t>(u >> 3) * 8 * Hb + 8 * v + (u & 7) : static_cast<int64_t>(v) * Wb + u)] =
                fmaf(tv, b, wv * a);
        }
        return;
    }
    if constexpr (kUB) {
        // (k / 8, n, k % 8): per 8-column block the support rows are one run of 8 rows floats
        const int per = 2 * rows;   // float4 per 8-column block
        for (int i = threadIdx.x; i < (Wb / 8) * per; i += 256) {
            const int kb = i / per, r4 = i - kb * per;
            const float4 x = __ldg(reinterpret_cast<const float4*>(s + static_cast<int64_t>(kb) * 8 * Hb + 8 * lo) + r4);
            *reinterpret_cast<float4*>(s_g + (r4 >> 1) * pitch + kb * 8 + (r4 & 1) * 4) = x;
        }
    } else {
        const int q4 = Wb / 4;
        const float4* g4 = reinterpret_cast<const float4*>(s + static_cast<int64_t>(lo) * Wb);
        for (int i = threadIdx.x; i < rows * q4; i += 256) {
            const int r = i / q4, c4 = i - r * q4;
            *reinterpret_cast<float4*>(s_g + r * pitch + 4 * c4) = __ldg(g4 + i);
        }
    }
    __syncthreads();
    float* d = dst + p * pb;
    for (int u = threadIdx.x; u < Wb; u += 256) {
        const int k = __ldg(bxi + u);
        const double tud = __ldg(bxt + u);
        const float tu = __double2float_rn(tud), wu = __double2float_rn(1.0 - tud);
        const float* col = s_g + k;
        float* o = d + (kUB ? static_cast<int64_t>(u >> 3) * 8 * Hb + 8 * v0 + (u & 7) : static_cast<int64_t>(v0) * Wb + u);
        const int ostep = kUB ? 8 : Wb;
#pragma unroll 4
        for (int i = 0; i < nv; ++i) {
            const float* r0 = col + s_vr[i];
            const float tv = s_vt[i], wv = s_vw[i];
            const float a = fmaf(tu, r0[1], wu * r0[0]);
            const float b = fmaf(tu, r0[pitch + 1], wu * r0[pitch]);
            __stcs(o + i * ostep, fmaf(tv, b, wv * a));
        }
    }
}

}  // namespace

cudaError_t launch_resample_b(const float* src, float* dst, int64_t rows, int Wb, int Hb, int order, double ey,
                              AxisTables bx, AxisTables by, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    if (rows > 0x7fffffffLL || Wb < 2 || Hb < 2) return cudaErrorInvalidValue;
    const int64_t pb = static_cast<int64_t>(Wb) * Hb;
    if (order == kOrderVMajor) {
        const dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>((pb + 255) / 256));
        resample_b_vmajor_kernel<<<grid, 256, 0, st>>>(src, dst, Wb, Hb, bx.i0, bx.t, by.i0, by.t);
        return cudaGetLastError();
    }
    const int ublocked = order == kOrderUBlocked ? 1 : 0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    // support rows of a band: |n(v0 + kRsV - 1) - n(v0)| + 2 <= ceil(|ey| (kRsV - 1)) + 3 (+1 margin)
    const double span = std::ceil(std::fabs(ey) * (kRsV - 1)) + 4;
    const bool band = aligned && Wb % 4 == 0 && (!ublocked || Wb % 8 == 0) && span <= kRsCap &&
                      getenv("CPI_RESAMPLE_GATHER") == nullptr;
    if (band) {
        const int cap = static_cast<int>(span);
        const size_t smem = size_t(cap) * rs_pitch(Wb) * 4;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(ublocked ? resample_b_band_kernel<true> : resample_b_band_kernel<false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        const dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>((Hb + kRsV - 1) / kRsV));
        if (ublocked)
            resample_b_band_kernel<true><<<grid, 256, smem, st>>>(src, dst, Wb, Hb, cap, bx.i0, bx.t, by.i0, by.t);
        else
            resample_b_band_kernel<false><<<grid, 256, smem, st>>>(src, dst, Wb, Hb, cap, bx.i0, bx.t, by.i0, by.t);
        return cudaGetLastError();
    }
    const bool vec = Wb % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    const int per = vec ? 4 * 256 : 256;
    const dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>((pb + per - 1) / per));
    if (vec)
        resample_b_kernel<4><<<grid, 256, 0, st>>>(src, dst, Wb, Hb, ublocked, bx.i0, bx.t, by.i0, by.t);
    else
        resample_b_kernel<1><<<grid, 256, 0, st>>>(src, dst, Wb, Hb, ublocked, bx.i0, bx.t, by.i0, by.t);
    return cudaGetLastError();
}

bool stage2_staged_supported(int Ha) { return Ha >= 2 && Ha <= kS2Threads; }

cudaError_t launch_pack_ytable_group(const AxisTables* ys, int n_fuse, int Ha, int Hb, uint2* ypack,
                                     cudaStream_t st) {
    PackGroupArgs g{};
    g.n = n_fuse;
    for (int f = 0; f < n_fuse; ++f) { g.i0[f] = ys[f].i0; g.t[f] = ys[f].t; g.lo[f] = ys[f].lo; }
    pack_ytable_kernel<<<dim3(Hb, n_fuse), Ha >= 256 ? 256 : ((Ha + 31) / 32) * 32, 0, st>>>(g, Ha, Hb, ypack);
    return cudaGetLastError();
}

cudaError_t launch_refocus_stage2_group(TElem* const* T, int n_fuse, int Wa, int Ha, int Hb, int m_base, int m_count,
                                        int m_block, int m_stride, const AxisTables* xs, const AxisTables* ys,
                                        const uint2* ypack, float* planes, cudaStream_t st) {
    if (n_fuse < 1 || n_fuse > kS2MaxPlanes || !stage2_staged_supported(Ha)) return cudaErrorInvalidValue;
    S2Args a{};
    a.Wa = Wa; a.Ha = Ha; a.Hb = Hb; a.ypack = ypack;
    a.m_base = m_base; a.m_count = m_count;
    a.m_block = m_block > 0 ? m_block : (m_count > 0 ? m_count : 1);
    a.m_stride = m_block > 0 ? m_stride : a.m_block;
    for (int f = 0; f < n_fuse; ++f) {
        a.T[f] = T[f]; a.xcnt[f] = xs[f].cnt; a.ycnt[f] = ys[f].cnt; a.ylo[f] = ys[f].lo; a.yhi[f] = ys[f].hi;
        a.plane[f] = planes + static_cast<int64_t>(f) * Ha * Wa;
    }
    const size_t smem = sizeof(TElem) * kS2XB * kS2VC * (Ha + 2) + sizeof(uint2) * kS2VC * Ha;
    if (smem > 48 * 1024) {   // per-device attribute: set before every launch
        cudaError_t e = cudaFuncSetAttribute(stage2_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    stage2_staged_kernel<<<dim3((Wa + kS2XB - 1) / kS2XB, n_fuse), kS2Threads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_refocus_coords_group(const CoordsGroupArgs& g, int n_fuse, cudaStream_t st) {
    const int nub = g.Wb > g.Hb ? g.Wb : g.Hb;
    const int wmax = g.Wa > g.Ha ? g.Wa : g.Ha;
    const int threads = wmax >= 256 ? 256 : ((wmax + 31) / 32) * 32;
    coords_group_kernel<<<dim3(nub, n_fuse, 2), threads, 0, st>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    count_kernel<<<dim3((wmax + 31) / 32, n_fuse, 2), 256, 0, st>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_refocus_stage1(const float* gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb,
                                  int m_base, int m_count, AxisTables xs, AxisTables ys, TElem* T,
                                  cudaStream_t st, int vmajor) {
    const size_t smem = static_cast<size_t>(kVG) * Wa * kPad * sizeof(float);
    if (smem > 48 * 1024) {   // per-device attribute: set before every launch
        cudaError_t e = cudaFuncSetAttribute(stage1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((Hb + kVG - 1) / kVG, m_count, (Wa + kS1Threads - 1) / kS1Threads);
    stage1_kernel<<<grid, kS1Threads, smem, st>>>(gamma, ldg, Wa, Ha, Wb, Hb, m_base, xs, ys, T, vmajor);
    return cudaGetLastError();
}

int stage1_vgroup(int Wa) { return stage1_vg(stage1_rows(Wa)); }

bool stage1_tma_supported(int Wa, int Wb, int Hb) {
    // 16-byte TMA strides: W_a (x-table rows) and W_b (Gamma rows) multiples of 4 floats
    return Wa <= 256 && Wa >= 4 && (Wa % 4) == 0 && (Wb % 4) == 0 && Wb <= 8 * kTMaxChunks && Hb <= 256;
}

cudaError_t launch_pack_xtable_group(const AxisTables* xs, int n_fuse, int Wa, int Wb, uint32_t* xpack, float* xwpack,
                                     uint32_t* xblk, cudaStream_t st) {
    PackGroupArgs g{};
    g.n = n_fuse;
    for (int f = 0; f < n_fuse; ++f) { g.i0[f] = xs[f].i0; g.t[f] = xs[f].t; g.lo[f] = xs[f].lo; }
    pack_xtable_group_kernel<<<dim3((Wb + 7) / 8, n_fuse), Wa >= 256 ? 256 : ((Wa + 31) / 32) * 32, 0, st>>>(
        g, Wa, Wb, static_cast<uint32_t>(stage1_rows(Wa)), xpack, xwpack, xblk);
    return cudaGetLastError();
}

template <bool kFullX, int F, bool kSkip, int kJ>
static cudaError_t launch_s1(const Stage1Maps* maps, const S1Args& a, int grid, cudaStream_t st) {
    using C = S1Cfg<F, kJ>;
    auto kern = stage1_tma_kernel<kFullX, F, kSkip, kJ>;
    // the attribute is per device: set it before every launch (a host-side call, negligible)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kTThreads, C::kSmem, st>>>(maps->gamma, maps->xtab, maps->xwtab, a);
    return cudaGetLastError();
}

template <bool kFullX, bool kSkip, int kJ>
static cudaError_t launch_s1_f(int F, const Stage1Maps* maps, const S1Args& a, int grid, cudaStream_t st) {
    switch (F) {
        case 1: return launch_s1<kFullX, 1, kSkip, kJ>(maps, a, grid, st);
        case 2: return launch_s1<kFullX, 2, kSkip, kJ>(maps, a, grid, st);
        default: return launch_s1<kFullX, 2, kSkip, kJ>(maps, a, grid, st);   // F <= 2 (kStage1MaxFuse)
    }
}

cudaError_t launch_refocus_stage1_tma(const Stage1Maps* maps, int n_fuse, int Wa, int Ha, int Wb, int Hb,
                                      int m_base, int m_count, int m_block, int m_stride, const AxisTables* xs,
                                      const AxisTables* ys, TElem* const* T, const uint32_t* xblk, int num_sms,
                                      cudaStream_t st) {
    if (n_fuse < 1 || n_fuse > kRefocusMaxFuse) return cudaErrorInvalidValue;
    S1Args a{};
    a.Wa = Wa; a.Ha = Ha; a.Wb = Wb; a.Hb = Hb; a.m_base = m_base; a.m_count = m_count;
    a.m_block = m_block > 0 ? m_block : (m_count > 0 ? m_count : 1);
    a.m_stride = m_block > 0 ? m_stride : a.m_block;
    a.n_vg = (Hb + stage1_vg(stage1_rows(Wa)) - 1) / stage1_vg(stage1_rows(Wa));
    a.n_chunks = (Wb + kTUC - 1) / kTUC;
    a.xblk = xblk;
    a.gamma_5d = maps->gamma_5d;
    for (int f = 0; f < n_fuse; ++f) {
        a.xlo[f] = xs[f].lo; a.xhi[f] = xs[f].hi; a.ylo[f] = ys[f].lo; a.yhi[f] = ys[f].hi; a.T[f] = T[f];
    }
    const int tiles = m_count * a.n_vg;
    const int grid = tiles < num_sms ? tiles : num_sms;
    const bool skip = getenv("CPI_S1_NOSKIP") == nullptr;   // A/B knob for the x-block skip (read per launch)
    if (stage1_rows(Wa) == 128)
        return skip ? launch_s1_f<false, true, 128>(n_fuse, maps, a, grid, st)
                    : launch_s1_f<false, false, 128>(n_fuse, maps, a, grid, st);
    if (skip)
        return Wa == 256 ? launch_s1_f<true, true, 256>(n_fuse, maps, a, grid, st)
                         : launch_s1_f<false, true, 256>(n_fuse, maps, a, grid, st);
    return Wa == 256 ? launch_s1_f<true, false, 256>(n_fuse, maps, a, grid, st)
                     : launch_s1_f<false, false, 256>(n_fuse, maps, a, grid, st);
}

cudaError_t launch_refocus_stage2(const TElem* T, int Wa, int Ha, int Hb, int m_base, int m_count,
                                  AxisTables xs, AxisTables ys, float* plane, cudaStream_t st) {
    const int64_t warps = static_cast<int64_t>(Wa) * Ha;
    const int64_t blocks = (warps * 32 + 255) / 256;
    stage2_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(T, Wa, Ha, Hb, m_base, m_base + m_count,
                                                                 xs, ys, plane);
    return cudaGetLastError();
}

cudaError_t launch_refocus_stage1_genb(const float* gamma, int64_t ldg, int Wa, int Ha, int Wb, int Hb,
                                       int m_base, int m_count, AxisTables xs, AxisTables bx, TElem* T,
                                       cudaStream_t st) {
    const size_t smem = static_cast<size_t>(kVG) * Wa * kGbPad * sizeof(float);
    if (smem > 48 * 1024) {   // per-device attribute: set before every launch
        cudaError_t e = cudaFuncSetAttribute(stage1_genb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((Hb + kVG - 1) / kVG, m_count, (Wa + kS1Threads - 1) / kS1Threads);
    stage1_genb_kernel<<<grid, kS1Threads, smem, st>>>(gamma, ldg, Wa, Ha, Wb, Hb, m_base, xs, bx, T);
    return cudaGetLastError();
}

cudaError_t launch_refocus_stage2_genb(const TElem* T, int Wa, int Ha, int Hb, int m_base, int m_count,
                                       AxisTables xs, AxisTables ys, AxisTables by, float* plane, cudaStream_t st) {
    const int64_t warps = static_cast<int64_t>(Wa) * Ha;
    const int64_t blocks = (warps * 32 + 255) / 256;
    stage2_genb_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(T, Wa, Ha, Hb, m_base, m_base + m_count, xs,
                                                                      ys, by, plane);
    return cudaGetLastError();
}

}  // namespace cpi
