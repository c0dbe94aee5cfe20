// refocus_w.cu — KB5w: refocus stage 1 with window reuse along x (
// SPEC.md:274 default map).
//
//   T_p[x][m][v] = sum_u [(1 - t(x,u)) Gamma(m, j0(x,u); v, u) + t(x,u) Gamma(m, j0(x,u) + 1; v, u)]
//
// The TMA stage 1 of refocus.cu gives every lane its own (x, v) samples, so every tap costs one
// 4-byte shared-memory load and the shared-memory pipe bounds it.  Here the 16
// lanes of a half-warp work on the SAME (plane, x, u) sample and on 128 different B rows v (eight
// per lane), so the support (j0, t) is uniform across the half (one entry decode per 8 v), and a
// warp walks 8 consecutive outputs x for one u (its two halves: two planes): the lower tap row of
// output x + 1 is j0(x) + d with d = 0 or 1 for alpha <= 1 (1 or 2 for 1 < alpha <= 2), so the
// two rows (j0, j0 + 1) of consecutive outputs overlap and stay in registers.  A half-step is
// 128 v x 2 corners = 256 taps for d loads of 512 B (two 16-B loads per lane, each half reading
// 256 contiguous bytes: conflict-free), i.e. alpha / 2 shared-memory bytes per tap instead of 4.  Skipped
// samples and outputs outside the RoI add exact zeros without loads.
//
// The per-step logic is precomputed (pack_w_steps_kernel): an 80-byte walk entry per (plane, u,
// 8 outputs x) holds the stage rows of every step (a slot reloads when its row changes) and both
// corner weights in fp32, each rounded once from fp64 (relative precision).
//
// Layout: Gamma with the B pixels in v-major order (include/cpi.h CPI_GAMMA_VMAJOR): column
// q = u * H_b + v, so for one (A pixel (m, j), u) the v are contiguous.  A tile = (A row m, 128 B
// rows v, 32 outputs x, group of 8 planes); warp w takes planes 2 (w / 4) + {0, 1} of the group and
// outputs 8 (w % 4) + {0..7}.  Per u the group's union j span of Gamma[(m, j)][(u, v0 .. v0 + 127)]
// (<= 96 rows of 512 B: 80 for the 64-plane grid) and the step entries of the tile are TMA-loaded
// into a 4-deep ring (the last warp to release a slot refills it).  8 planes share each staged
// slab, so Gamma crosses HBM ~0.62x as often as with 4-plane groups over 64 outputs.  fp32 partials stay in registers for 8 u and are then added into fp64 accumulators
// that live in TMEM (64 per lane, 512 columns per CTA).  Tiles are ordered (m, v-block) outer and
// (plane group, x tile) inner, so the Gamma slab of the tiles in flight (32 MB per (m, v-block)) is
// reused from L2 by every plane group: Gamma crosses HBM about once per launch for the whole stack.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace cpi {
namespace {

constexpr int kWX = 32;                            // outputs x per tile
constexpr int kWV = 128;                           // B rows v per tile (4 per lane)
constexpr int kWWarps = 16;
constexpr int kWXW = 8;                            // outputs x per warp
constexpr int kWF = 8;                             // planes per group
constexpr int kWFW = 2;                            // planes per warp
constexpr int kWBox = 8;                           // j rows per Gamma TMA box
constexpr int kWRows = 96;                         // staged j rows (6 boxes); larger spans -> plain stage 1
constexpr int kWStages = 4;
constexpr int kWFlush = 8;                         // u per fp32 partial before the fp64 flush
// Timing probes (CPI_S1W_PROBE) are compiled in only with -DCPI_S1W_PROBES: the
// consumer loop of the product kernel carries no probe tests.
#ifdef CPI_S1W_PROBES
#define W_PROBE(a, bit) (((a).probe & (bit)) != 0)
#else
#define W_PROBE(a, bit) false
#endif
// A producer warpgroup (warps 16-19; warp 16 issues, the others exit) next to the 16 consumer
// warps: a 17th warp alone would put 5 warps on one SM sub-partition and cap the registers at 96,
// so the producers drop to kWProdRegs with setmaxnreg and the consumers rise to kWConsRegs
// (the CTA launches with 96 per thread for 640 threads: 4 x 32 x 32 + 16 x 32 x 112 = 61,440).
constexpr int kWProdWarps = 4;
constexpr int kWProdRegs = 32, kWConsRegs = 112;
constexpr int kWThreads = 32 * (kWWarps + kWProdWarps);
constexpr int kWRowBytes = kWV * 4;                // 512 B per staged row
constexpr int kWGBytes = kWRows * kWRowBytes;      // 72 KB of Gamma per stage
constexpr int kWWalkU4 = 5;                        // uint4 per walk: a row header + 4 x 2 steps' weights
constexpr int kWEBytes = kWF * (kWX / kWXW) * kWWalkU4 * 16;   // 2.5 KB of walk entries per stage
constexpr int kWStageBytes = kWGBytes + kWEBytes;
constexpr int kWOffBar = kWStages * kWStageBytes;              // full barriers, then empty barriers
constexpr int kWOffHdr = kWOffBar + 2 * kWStages * 8;           // stage headers (16 B each)
constexpr int kWOffTmem = kWOffHdr + kWStages * 16;             // TMEM base slot
constexpr int kWMaxWb = 512;                                    // B columns (tile span row copy)
constexpr int kWOffSpan = (kWOffTmem + 16 + 15) / 16 * 16;      // the issuing cursor's tile span row
constexpr int kWOffUList = kWOffSpan + kWMaxWb * 8;                // the tile's used u, in order
constexpr int kWSmem = kWOffUList + kWMaxWb * 4;
constexpr uint32_t kWInvalid = 0xFFFFFFFFu;        // 32-bit (j0 | t) table: skipped sample / padding x
// Walk entry of (plane, u, block of 8 outputs x) for a warp walking its 8 outputs in order: 80 B.
// The warp keeps two row registers, slot A for the even and slot B for the odd stage row of the
// pair (j0, j0 + 1).
//   uint4 0 (header): byte 2k = 2 x the even row of step k, byte 2k + 1 = 2 x its odd row; a
//       row equal to the previous step's is not reloaded (a skipped sample repeats the previous
//       rows, 0xFF before the first used one: no load);
//   uint4 1 + q: (even weight, odd weight) of steps 2q and 2q + 1 (fp32, each rounded once from
//       its fp64 value 1 - t or t, so the small one keeps its relative precision; 0, 0 for a
//       skipped sample: its taps add exact zeros).
// (A 64-bit step entry with t on a 2^-23 grid and the odd weight derived as 1 - even lost the
// small weight's relative precision: an error up to 2^-24 |Gamma(j0 + 1) - Gamma(j0)|, beyond
// 1e-6 M when t or 1 - t is tiny.)
constexpr uint32_t kWTmemCols = 512;

static_assert(kWSmem <= 232448, "stage-1 window kernel exceeds the 227 KB shared-memory limit");
static_assert(2 * (kWRows - 1) < 256, "step entries keep 2 x row in one byte");
static_assert(kWRowBytes == 512, "step entries encode a row's offset as 2 x row << 8");
static_assert(kWWarps * kWXW == kWX * (kWF / kWFW), "warps x outputs x planes must cover the tile");
static_assert(kWWarps * kWFW * kWXW * 4 * 2 <= 4 * 128 * 32 * 4, "fp64 accumulators exceed TMEM");

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 upk2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
// d = w * g + c on both fp32 halves (sm_100a fma.rn.f32x2), w = (w, w) pre-packed
__device__ __forceinline__ uint64_t fma2(uint64_t w, uint64_t g, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(w), "l"(g), "l"(c));
    return d;
}

// Both 16-byte halves of one staged row (addr, addr + 256) if flag != 0, one predicate for the pair
__device__ __forceinline__ void w_lds2_if(uint4& g0, uint4& g1, uint32_t addr, uint32_t flag) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %8, 0;\n\t"
        "@p ld.shared.v4.u32 {%0, %1, %2, %3}, [%9];\n\t"
        "@p ld.shared.v4.u32 {%4, %5, %6, %7}, [%9+256];\n\t}"
        : "+r"(g0.x), "+r"(g0.y), "+r"(g0.z), "+r"(g0.w), "+r"(g1.x), "+r"(g1.y), "+r"(g1.z), "+r"(g1.w)
        : "r"(flag), "r"(addr));
}

// The same pair load if x != y (the row offset changed since the previous step)
__device__ __forceinline__ void w_lds2_ifne(uint4& g0, uint4& g1, uint32_t addr, uint32_t x, uint32_t y) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %8, %9;\n\t"
        "@p ld.shared.v4.u32 {%0, %1, %2, %3}, [%10];\n\t"
        "@p ld.shared.v4.u32 {%4, %5, %6, %7}, [%10+256];\n\t}"
        : "+r"(g0.x), "+r"(g0.y), "+r"(g0.z), "+r"(g0.w), "+r"(g1.x), "+r"(g1.y), "+r"(g1.z), "+r"(g1.w)
        : "r"(x), "r"(y), "r"(addr));
}

// Compiler-level pin: every partial (hence every load feeding it) is computed before this point.
__device__ __forceinline__ void w_pin(const uint64_t (&part)[kWFW][kWXW][2]) {
#pragma unroll
    for (int pl = 0; pl < kWFW; ++pl)
#pragma unroll
        for (int i = 0; i < kWXW; ++i) asm volatile("" ::"l"(part[pl][i][0]), "l"(part[pl][i][1]) : "memory");
}
// part (4 v as two fp32 pairs) += wa * ga + wb * gb, in that order (FFMA2)
__device__ __forceinline__ void w_taps(uint64_t (&pp)[2], float wa, const uint4& ga, float wb, const uint4& gb) {
    const uint64_t wa2 = pk2(wa, wa), wb2 = pk2(wb, wb);
    pp[0] = fma2(wb2, pk2(__uint_as_float(gb.x), __uint_as_float(gb.y)),
                 fma2(wa2, pk2(__uint_as_float(ga.x), __uint_as_float(ga.y)), pp[0]));
    pp[1] = fma2(wb2, pk2(__uint_as_float(gb.z), __uint_as_float(gb.w)),
                 fma2(wa2, pk2(__uint_as_float(ga.z), __uint_as_float(ga.w)), pp[1]));
}

__device__ __forceinline__ int w_shard_row(const S1WArgs& a, int l) {
    return a.m_base + (l / a.m_block) * a.m_stride + l % a.m_block;
}

// tile t -> (local A row, v block, x tile) outer, plane group inner: the groups of one (m, v block,
// x tile) run on neighbouring CTAs at the same time and walk u in near lockstep, so the Gamma rows
// their spans share are read from L2
struct WTile { int ml, vb, g, xt; };
__device__ __forceinline__ WTile w_tile(const S1WArgs& a, int t) {
    const int o = t / a.n_groups;
    WTile w;
    w.g = t - o * a.n_groups;
    const int o2 = o / a.n_xt;
    w.xt = o - o2 * a.n_xt;
    w.ml = o2 / a.n_vb;
    w.vb = o2 - w.ml * a.n_vb;
    return w;
}
__device__ __forceinline__ bool w_needed(const S1WArgs& a, const WTile& w, int m) {
    const int2 b = __ldg(a.mband + w.g * a.n_vb + w.vb);
    return m >= b.x && m <= b.y;
}

// Stage ring protocol.  A dedicated producer warp (warp 16; its warpgroup gives its registers to
// the consumers) walks the CTA's tiles and their used u in order and refills ring slot s once all
// 16 consumer warps released it (empty[s]).  Each refill writes a header into the slot -- which
// tile the stage belongs to and whether it is the tile's first / last stage -- so the consumers
// only follow headers (no tile or span logic of their own); tile = -1 ends the CTA.  (The first
// version had no producer warp: the last warp to release a slot issued its refill, and that warp,
// late by the issue, tended to be the last releaser again, serialising issue and compute: 90.6 ms
// vs 66.9 ms with the producer warp.)
struct WHeader {
    int tile;    // -1: no more stages
    int flags;   // bit 0: first stage of the tile, bit 1: last stage of the tile
    int pad[2];
};

// Producer loop (warp 16).  Per tile the warp copies the tile's span row and compacts its used u
// (non-empty spans) into a list with ballots; lane 0 then issues the tile's stages straight from
// the list, so a stage costs lane 0 two shared loads, the header and the TMA instructions.
__device__ __forceinline__ void w_produce(int2* tspan, int* ulist, WHeader* hdr, const S1WArgs& a, int n_tiles,
                                          const CUtensorMap* tm_g, const CUtensorMap* tm_e, uint8_t* smem,
                                          uint64_t* full, uint64_t* empty, int lane) {
    int s = 0, k = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x;; t += gridDim.x) {
        int cnt = 0;
        WTile w{};
        for (; t < n_tiles; t += gridDim.x) {
            w = w_tile(a, t);
            if (!w_needed(a, w, w_shard_row(a, w.ml))) continue;
            const int2* sp_row = a.span + static_cast<int64_t>(w.g * a.n_xt + w.xt) * a.Wb;
            __syncwarp();
            for (int base = 0; base < a.Wb; base += 32) {
                const int u = base + lane;
                int2 sp = make_int2(1, 0);
                if (u < a.Wb) sp = __ldg(sp_row + u);
                const bool ne = sp.y >= sp.x;
                const unsigned m = __ballot_sync(0xffffffffu, ne);
                if (ne) {
                    const int pos = cnt + __popc(m & ((1u << lane) - 1u));
                    ulist[pos] = u;
                    tspan[pos] = sp;
                }
                cnt += __popc(m);
            }
            __syncwarp();
            if (cnt > 0) break;
        }
        if (lane == 0) {
            if (t >= n_tiles) {   // end marker
                if (k >= kWStages) mbar_wait(&empty[s], ph ^ 1);
                hdr[s].tile = -1;
                hdr[s].flags = 0;
                mbar_arrive(&full[s]);
            } else {
                for (int i = 0; i < cnt; ++i) {
                    if (k >= kWStages) mbar_wait(&empty[s], ph ^ 1);
                    const int u = ulist[i];
                    const int2 sp = tspan[i];
                    hdr[s].tile = t;
                    hdr[s].flags = (i == 0 ? 1 : 0) | (i == cnt - 1 ? 2 : 0);
                    const int nb = W_PROBE(a, 1) ? 0 : (sp.y - sp.x + kWBox) / kWBox;
                    mbar_expect_tx(&full[s], nb * kWBox * kWRowBytes + kWEBytes);
                    uint8_t* dst = smem + s * kWStageBytes;
                    for (int b = 0; b < nb; ++b)
                        tma_load_5d(dst + b * kWBox * kWRowBytes, tm_g, &full[s], 0, u, w.vb, sp.x + b * kWBox, w.ml);
                    tma_load_3d(dst + kWGBytes, tm_e, &full[s], w.xt * (kWX / kWXW) * kWWalkU4 * 4, u, w.g * kWF);
                    ++k;
                    if (++s == kWStages) { s = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
        if (t >= n_tiles) return;
    }
}

// fp64 accumulators of a lane in TMEM: v half h (of the lane's two 4-v groups), output i, v slot
// k at columns 64 h + 8 i + 2 k (+1: high word).  r holds columns [16 qt, +16) of one v half
// (outputs 2 qt, 2 qt + 1); adds the fp32 partials (r ignored when first).  16 columns at a time
// keep the temporaries small (the consumers run at the 112-register cap).
__device__ __forceinline__ void w_combine(const uint64_t (&pp)[kWXW][2], uint32_t (&r)[16], int qt, bool first) {
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
        const int i = 2 * qt + ii;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const float2 p = upk2(pp[i][q]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = 8 * ii + 4 * q + 2 * h;
                double d = static_cast<double>(h ? p.y : p.x);
                if (!first) d += __hiloint2double(static_cast<int>(r[c + 1]), static_cast<int>(r[c]));
                r[c] = static_cast<uint32_t>(__double2loint(d));
                r[c + 1] = static_cast<uint32_t>(__double2hiint(d));
            }
        }
    }
}
// Add the fp32 partials into the fp64 accumulators in TMEM and zero them.
__device__ __forceinline__ void w_flush(uint64_t (&part)[kWFW][kWXW][2], uint32_t tbase, bool first) {
#pragma unroll
    for (int pl = 0; pl < kWFW; ++pl)
#pragma unroll
        for (int qt = 0; qt < 4; ++qt) {
            uint32_t r[16];
            const uint32_t col = tbase + 64 * pl + 16 * qt;
            if (!first) {
                tmem_ld_32x32b_x16(col, r);
                tmem_wait_ld();
            }
            w_combine(part[pl], r, qt, first);
            tmem_st_32x32b_x16(col, r);
        }
    tmem_wait_st();
#pragma unroll
    for (int pl = 0; pl < kWFW; ++pl)
#pragma unroll
        for (int i = 0; i < kWXW; ++i) part[pl][i][0] = part[pl][i][1] = 0ull;
}

__global__ void __launch_bounds__(kWThreads, 1)
stage1_w_kernel(const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_e, S1WArgs a) {
    extern __shared__ __align__(1024) uint8_t w_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(w_smem + kWOffBar);
    WHeader* hdr = reinterpret_cast<WHeader*>(w_smem + kWOffHdr);
    int2* tspan = reinterpret_cast<int2*>(w_smem + kWOffSpan);
    uint64_t* empty = full + kWStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(w_smem + kWOffTmem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = a.m_count * a.n_vb * a.n_groups * a.n_xt;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWWarps);   // lane 0 of every consumer warp
        }
        fence_mbar_init();
        tma_prefetch_desc(&tm_g);
        tma_prefetch_desc(&tm_e);
    }
    if (warp == 0) tmem_alloc(tslot, kWTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp >= kWWarps) {   // producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWProdRegs));
        if (warp != kWWarps) return;
        // stages in order; slot s is refilled once all consumer warps released it
        w_produce(tspan, reinterpret_cast<int*>(w_smem + kWOffUList), hdr, a, n_tiles, &tm_g, &tm_e, w_smem, full,
                  empty, lane);
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWConsRegs));
    const uint32_t tmem = *tslot;

    // warp: planes 2 (warp / 4) + {0, 1} of the group, outputs x = x tile + 8 (warp % 4) + i;
    // lane: plane 2 (warp / 4) + lane / 16, B rows v = v block + 64 h + 4 (lane % 16) + {0..3} for
    // h = 0, 1 (each 16-lane half reads 256 contiguous bytes of a row per load: conflict-free)
    const int wp = warp >> 2, wx = warp & 3, lpl = lane >> 4;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(warp >> 2) * 128u;
    const uint32_t lane16 = 16u * (lane & 15);
    uint64_t part[kWFW][kWXW][2];
    // loop state kept small (the consumers run at the 112-register cap): kst = stages of the current
    // tile so far (a flush every kWFlush; no fp64 partial in TMEM while kst < kWFlush), ring position
    // sp = slot | phase << 2
    int kst = 0;
    uint32_t sp = 0;
    static_assert(kWStages == 4, "ring position packing assumes 4 slots");
    for (;;) {
        const int stage = static_cast<int>(sp & 3u);
        const uint32_t phase = sp >> 2;
        if (W_PROBE(a, 8)) mbar_wait_spin(&full[stage], phase);   // probe 8: non-suspending wait
        else mbar_wait(&full[stage], phase);
        const WHeader h = hdr[stage];
        if (h.tile < 0) break;
        if (h.flags & 1) {   // first stage of a tile
#pragma unroll
            for (int pl = 0; pl < kWFW; ++pl)
#pragma unroll
                for (int i = 0; i < kWXW; ++i) part[pl][i][0] = part[pl][i][1] = 0ull;
            kst = 0;
        }
        const uint8_t* sbase = w_smem + stage * kWStageBytes;
        const uint4* E = reinterpret_cast<const uint4*>(sbase + kWGBytes);
        const uint32_t gaddr = smem_u32(sbase) + lane16;   // this lane's 16 bytes (4 v) of row 0, half 0
        // each 16-lane half walks its own plane; entries of planes past the batch are the TMA's zero
        // fill: zero weights (exact zero taps)
        const uint4* Wk = E + ((kWFW * wp + lpl) * (kWX / kWXW) + wx) * kWWalkU4;   // this half's walk
        if (W_PROBE(a, 16)) {     // probe 16: no step work (ring / barrier / issue cost only)
        } else {   // window reuse (rows kept in registers, loads only when they change)
            uint4 ga[2], gb[2];   // even / odd row of the window, v halves h = 0, 1
            ga[0] = ga[1] = gb[0] = gb[1] = make_uint4(0u, 0u, 0u, 0u);
            const uint4 hd = Wk[0];
            uint32_t oa_prev = 0xFF00u, ob_prev = 0xFF00u;   // no rows in the slots yet
#pragma unroll
            for (int q = 0; q < kWXW / 2; ++q) {
                const uint32_t hw = q == 0 ? hd.x : q == 1 ? hd.y : q == 2 ? hd.z : hd.w;
                const uint4 wt = Wk[1 + q];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    // byte 2k / 2k + 1 of hw (2 x row) moved to byte 1 = the row's 512-B offset
                    const uint32_t oa = __byte_perm(hw, 0u, k ? 0x4424u : 0x4404u);
                    const uint32_t ob = __byte_perm(hw, 0u, k ? 0x4434u : 0x4414u);
                    w_lds2_ifne(ga[0], ga[1], gaddr + oa, oa, oa_prev);
                    w_lds2_ifne(gb[0], gb[1], gaddr + ob, ob, ob_prev);
                    oa_prev = oa;
                    ob_prev = ob;
                    const float wa = __uint_as_float(k ? wt.z : wt.x), wb = __uint_as_float(k ? wt.w : wt.y);
                    w_taps(part[0][2 * q + k], wa, ga[0], wb, gb[0]);
                    w_taps(part[1][2 * q + k], wa, ga[1], wb, gb[1]);
                }
            }
        }
        // release the slot to the producer (generic-proxy reads before the async-proxy refill,
        // DESIGN §14)
        w_pin(part);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        sp = (sp + 1u) & 7u;
        if (h.flags & 2) {   // last stage of the tile: fp64 sum (TMEM + partial) -> fp32 T
            const WTile w = w_tile(a, h.tile);
            const int m = w_shard_row(a, w.ml);
            const int x0 = w.xt * kWX + wx * kWXW;
            const bool first = kst < kWFlush;   // no fp64 partial in TMEM yet
            const bool lane_ok = kWFW * wp + lpl < a.n_planes - w.g * kWF;   // this lane's plane is in the batch
            float* Tf = a.T + static_cast<int64_t>(w.g * kWF + kWFW * wp + (lane_ok ? lpl : 0)) * a.t_plane;
#pragma unroll
            for (int hv = 0; hv < 2; ++hv) {   // v half (the accumulators' first index)
                const int v = w.vb * kWV + 64 * hv + 4 * (lane & 15);
#pragma unroll
                for (int qt = 0; qt < 4; ++qt) {   // outputs 2 qt, 2 qt + 1
                    uint32_t r[16];
                    if (!first) {   // warp-collective TMEM load (every lane, valid plane or not)
                        tmem_ld_32x32b_x16(tbase + 64 * hv + 16 * qt, r);
                        tmem_wait_ld();
                    }
                    w_combine(part[hv], r, qt, first);
#pragma unroll
                    for (int ii = 0; ii < 2; ++ii) {
                        const int x = x0 + 2 * qt + ii;
                        float o[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            o[k] = static_cast<float>(__hiloint2double(static_cast<int>(r[8 * ii + 2 * k + 1]),
                                                                       static_cast<int>(r[8 * ii + 2 * k])));
                        if (lane_ok && x < a.Wa && v < a.Hb)
                            *reinterpret_cast<float4*>(Tf + (static_cast<int64_t>(x) * a.Ha + m) * a.Hb + v) =
                                make_float4(o[0], o[1], o[2], o[3]);
                    }
                }
            }
        } else if ((++kst & (kWFlush - 1)) == 0 && !W_PROBE(a, 4)) {   // probe 4: no flushes (wrong values)
            w_flush(part, tbase, kst == kWFlush);
        }
    }
    // all consumer warps done with TMEM before warp 0 frees it (the producers have exited)
    tc_fence_before();
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kWWarps) : "memory");
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, kWTmemCols);
    }
}

// ---- pack: per-plane entries, per-(group, x tile, u) spans, step entries, m bands ----------
// entry(f, u, x) = j0 << 23 | min(round(t * 2^23), 2^23 - 1),
// kWInvalid for skipped samples and for the padding columns x >= W_a.
__global__ void pack_w_entries_kernel(const int32_t* const* i0s, const double* const* ts, int Wa, int Wb, int xpad,
                                      uint32_t* __restrict__ ent) {
    const int u = blockIdx.x, f = blockIdx.y;
    const int32_t* i0 = i0s[f];
    const double* tt = ts[f];
    for (int x = threadIdx.x; x < xpad; x += blockDim.x) {
        uint32_t e = kWInvalid;
        if (x < Wa) {
            const int64_t idx = static_cast<int64_t>(u) * Wa + x;
            const int j = __ldg(i0 + idx);
            if (j >= 0) {
                // t on a 2^-23 grid for the span logic only (the step weights come from the fp64 t)
                const uint32_t tq = min(static_cast<uint32_t>(__double2uint_rn(__ldg(tt + idx) * 8388608.0)), 8388607u);
                e = (static_cast<uint32_t>(j) << 23) | tq;
            }
        }
        ent[(static_cast<int64_t>(f) * Wb + u) * xpad + x] = e;
    }
}
// span(g, xt, u) = [min j0, max j0 + 1] over the group's planes and the tile's outputs (lo > hi: none)
__global__ void pack_w_span_kernel(const uint32_t* __restrict__ ent, int n_planes, int Wb, int xpad, int n_xt,
                                   int2* __restrict__ span) {
    const int u = blockIdx.x, g = blockIdx.y, xt = blockIdx.z;
    int lo = INT_MAX, hi = -1;
    for (int f = g * kWF; f < min(n_planes, g * kWF + kWF); ++f) {
        const uint32_t e = __ldg(ent + (static_cast<int64_t>(f) * Wb + u) * xpad + xt * kWX + threadIdx.x);
        if (e != kWInvalid) {
            const int j = static_cast<int>(e >> 23);
            lo = min(lo, j);
            hi = max(hi, j + 1);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ int slo[kWX / 32], shi[kWX / 32];
    if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kWX / 32; ++k) { lo = min(lo, slo[k]); hi = max(hi, shi[k]); }
        span[(static_cast<int64_t>(g) * n_xt + xt) * Wb + u] = hi >= lo ? make_int2(lo, hi) : make_int2(1, 0);
    }
}
// walk entries (see the layout above): one thread per (plane, u, warp block of 8 outputs x) scans
// the block in the warp's walk order, tracking which stage row each slot holds; rows are relative
// to the span of (group, x tile, u).
__global__ void pack_w_steps_kernel(const uint32_t* __restrict__ ent, const double* const* ts, const int2* __restrict__ span,
                                    int Wa, int Wb, int xpad, int n_xt, uint4* __restrict__ steps) {
    const int u = blockIdx.x, f = blockIdx.y, blk = threadIdx.x;
    if (blk >= xpad / kWXW) return;
    const int x0 = blk * kWXW, xt = x0 / kWX, g = f / kWF;
    const int2 sp = __ldg(span + (static_cast<int64_t>(g) * n_xt + xt) * Wb + u);
    const int64_t base = (static_cast<int64_t>(f) * Wb + u) * xpad + x0;
    uint32_t ra = 0xFFu, rb = 0xFFu;   // 2 x stage row in slots A (even) and B (odd); 0xFF: none yet
    uint32_t hdr[4] = {0u, 0u, 0u, 0u};
    uint32_t w[kWXW][2];
    for (int i = 0; i < kWXW; ++i) {
        const uint32_t e = __ldg(ent + base + i);
        w[i][0] = w[i][1] = 0u;
        if (e != kWInvalid) {
            const int r0 = static_cast<int>(e >> 23) - sp.x;               // stage row of j0 (< kWRows - 1)
            const double t = __ldg(ts[f] + static_cast<int64_t>(u) * Wa + x0 + i);
            const float w0 = __double2float_rn(1.0 - t), w1 = __double2float_rn(t);   // each rounded once
            const bool ev = (r0 & 1) == 0;
            ra = static_cast<uint32_t>(2 * (ev ? r0 : r0 + 1));
            rb = static_cast<uint32_t>(2 * (ev ? r0 + 1 : r0));
            w[i][0] = __float_as_uint(ev ? w0 : w1);
            w[i][1] = __float_as_uint(ev ? w1 : w0);
        }
        hdr[i / 2] |= (ra | (rb << 8)) << (16 * (i & 1));
    }
    uint4* out = steps + (static_cast<int64_t>(f) * Wb + u) * (xpad / kWXW) * kWWalkU4 + static_cast<int64_t>(blk) * kWWalkU4;
    out[0] = make_uint4(hdr[0], hdr[1], hdr[2], hdr[3]);
    for (int q = 0; q < kWXW / 2; ++q) out[1 + q] = make_uint4(w[2 * q][0], w[2 * q][1], w[2 * q + 1][0], w[2 * q + 1][1]);
}
// mband(g, vb) = union over the group's planes and the block's B rows v of the A rows stage 2
// reads, [lo_y(v), hi_y(v)] (tiles outside it are not computed)
__global__ void pack_w_mband_kernel(const int32_t* const* ylo, const int32_t* const* yhi, int n_planes, int Hb, int n_vb,
                                    int2* __restrict__ mband) {
    const int vb = blockIdx.x, g = blockIdx.y;
    int lo = INT_MAX, hi = -1;
    const int v = vb * kWV + threadIdx.x;
    if (v < Hb)
        for (int f = g * kWF; f < min(n_planes, g * kWF + kWF); ++f) {
            const int l = __ldg(ylo[f] + v), h = __ldg(yhi[f] + v);
            if (h >= l) { lo = min(lo, l); hi = max(hi, h); }
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ int slo[kWV / 32], shi[kWV / 32];
    if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kWV / 32; ++k) { lo = min(lo, slo[k]); hi = max(hi, shi[k]); }
        mband[g * n_vb + vb] = hi >= lo ? make_int2(lo, hi) : make_int2(1, 0);
    }
}

}  // namespace

int stage1_w_xtile() { return kWX; }
int stage1_w_vblock() { return kWV; }
int stage1_w_group() { return kWF; }
int stage1_w_jbox() { return kWBox; }
int stage1_w_max_span() { return kWRows; }
// the v-major block must be the kernel's v block (128 rows, or all of H_b <= 128)
bool stage1_w_supported(int Wa, int Hb) {
    return Wa >= 2 && Wa <= 256 && Hb >= 4 && Hb % 4 == 0 && (Hb <= kWV || Hb % kWV == 0) && kVMajorBlock == kWV;
}

cudaError_t launch_pack_w(const int32_t* const* i0s_dev, const double* const* ts_dev, const int32_t* const* ylo_dev,
                          const int32_t* const* yhi_dev, int n_planes, int Wa, int Wb, int Hb, uint32_t* ent,
                          uint4* steps, int2* span, int2* mband, cudaStream_t st) {
    const int xpad = ((Wa + kWX - 1) / kWX) * kWX, n_xt = xpad / kWX;
    const int n_groups = (n_planes + kWF - 1) / kWF, n_vb = (Hb + kWV - 1) / kWV;
    pack_w_entries_kernel<<<dim3(Wb, n_planes), 128, 0, st>>>(i0s_dev, ts_dev, Wa, Wb, xpad, ent);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    pack_w_span_kernel<<<dim3(Wb, n_groups, n_xt), kWX, 0, st>>>(ent, n_planes, Wb, xpad, n_xt, span);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    pack_w_steps_kernel<<<dim3(Wb, n_planes), ((xpad / kWXW + 31) / 32) * 32, 0, st>>>(ent, ts_dev, span, Wa, Wb, xpad,
                                                                                     n_xt, steps);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    pack_w_mband_kernel<<<dim3(n_vb, n_groups), kWV, 0, st>>>(ylo_dev, yhi_dev, n_planes, Hb, n_vb, mband);
    return cudaGetLastError();
}

cudaError_t launch_refocus_stage1_w(const CUtensorMap* tm_gamma, const CUtensorMap* tm_ent, const S1WArgs& a_in,
                                    int num_sms, cudaStream_t st) {
    S1WArgs a = a_in;
    a.n_xt = (a.Wa + kWX - 1) / kWX;
    a.n_vb = (a.Hb + kWV - 1) / kWV;
    a.n_groups = (a.n_planes + kWF - 1) / kWF;
    if (a.m_block <= 0) { a.m_block = a.m_count > 0 ? a.m_count : 1; a.m_stride = a.m_block; }
    const int64_t tiles = static_cast<int64_t>(a.m_count) * a.n_vb * a.n_groups * a.n_xt;
    if (tiles <= 0) return cudaSuccess;
    if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(stage1_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem);
    if (e != cudaSuccess) return e;
    const int grid = static_cast<int>(tiles < num_sms ? tiles : num_sms);
    stage1_w_kernel<<<grid, kWThreads, kWSmem, st>>>(*tm_gamma, *tm_ent, a);
    return cudaGetLastError();
}

}  // namespace cpi
