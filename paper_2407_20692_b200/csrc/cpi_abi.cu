// cpi_abi.cu — the C ABI of include/cpi.h: context, validation, workspaces, TMA
// descriptors, launch sequencing and timing.  All compute runs in the kernels of
// expand.cu / gemm_tc.cu / gemm_popc.cu / refocus.cu; nothing here touches pixel data.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cerrno>
#include <cstring>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/cpi.h"
#include "kernels.h"

namespace {

constexpr int64_t kKAlign = 128;   // frames per GEMM K block (bytes of one swizzle row)

enum KernelClass { KC_GEMM = 0, KC_EXPAND = 1, KC_STAGE1 = 2, KC_STAGE2 = 3, KC_FINALIZE = 4,
                   KC_COORDS = 5, KC_RESAMPLE = 6, KC_COUNT = 7 };

thread_local std::string g_create_error;

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace

struct cpi_ctx {
    cpi_config cfg{};
    int dev = 0;
    int num_sms = 148;
    bool popc = false, keep = false, pair = true;   // pair: cta_group::2 GEMM
    bool fp4 = false;                      // kind::mxf4 GEMM on E2M1 operands (2 frames per byte)
    bool bits = false;                     // f1: kind::i8 GEMM unpacking bit-stream operands in shared memory
    bool ublocked = false;                 // B pixels in u-blocked order (CPI_GAMMA_UBLOCKED)
    bool symmetric = false;                // roi_a == roi_b: one operand, SYRK GEMM (upper tiles, mirrored)
    int order = cpi::kOrderRowMajor;       // B pixel order (row-major / u-blocked / v-major)
    int64_t k_align = 128;                 // frames per GEMM K block
    int64_t p_a = 0, p_b = 0;
    int64_t rows_a = 0, rows_b = 0;        // padded operand rows
    int64_t k_cap = 0;                     // frames capacity rounded to 128
    int64_t ld_op = 0;                     // operand leading dimension (bytes or 32-bit words)
    int64_t frame_bytes = 0;
    uint8_t* frames_dev[2] = {nullptr, nullptr};   // double-buffered staging for host loads
    cudaStream_t copy_stream = nullptr;    // host->device copies overlap the previous batch's compute
    cudaEvent_t ev_loaded[2] = {nullptr, nullptr};    // copy into buffer b complete
    cudaEvent_t ev_consumed[2] = {nullptr, nullptr};  // expand of buffer b complete (buffer reusable)
    bool consumed_valid[2] = {false, false};
    int next_buf = 0;
    int cur_buf = -1;                      // buffer of the loaded batch (-1: device pointer)
    const uint8_t* frames_cur = nullptr;
    int64_t n_cur = 0;
    bool loaded = false;
    bool expanded = false;                 // the loaded batch is expanded (cpi_correlate_rows)
    bool consumed = false;                 // the loaded batch went through cpi_correlate
    int accumulate = 0;                    // the loaded batch adds to earlier batches' counts
    int64_t gemm_batches = 0;              // batches with frames since the last reset
    bool counts_stale = true;              // kept counts not yet written since the last reset (zero on read)
    void* op_a = nullptr;
    void* op_b = nullptr;
    int32_t* s_a = nullptr;
    int32_t* s_b = nullptr;
    int32_t* counts = nullptr;
    int64_t n_tot = 0;
    int64_t batches = 0;
    float* gamma_current = nullptr;        // Gamma buffer written for the current totals
    float* gamma_ws = nullptr;             // library Gamma for cpi_refocus from counts (lazy)
    CUtensorMap tm_a{}, tm_b{};
    // refocus workspaces
    static constexpr int kS1Planes = cpi::kRefocusMaxFuse;   // planes per KB5 launch
    cpi::AxisTables xs[kS1Planes]{}, ys[kS1Planes]{};
    int n_plane_ws = 0;                    // planes whose xs / ys / T are allocated (grown on demand)
    cpi::GenTables gen_x{}, gen_y{};       // general maps (d != 0): per-axis supports (lazy)
    cpi::AxisTables bxs{}, bys{};          // fractional-B path: B supports per u / v
    float* bws = nullptr;                  // fractional-B path: Gamma resampled onto the B lattice (lazy)
    size_t bws_bytes = 0;
    cpi::TElem* T[kS1Planes]{};
    bool refocus_ready = false;
    int fuse = cpi::kStage1MaxFuse;        // planes per Gamma pass in the TMA stage 1 (CPI_REFOCUS_FUSE)
    uint32_t* xpack = nullptr;             // packed x-tables [kS1Planes][W_b][W_a]
    float* xwpack = nullptr;               // their near-t corner offsets [kS1Planes][W_b][W_a]
    uint2* ypack = nullptr;                // packed y-tables [kRefocusMaxFuse][H_b][H_a]
    uint32_t* xblk = nullptr;              // x-block masks [kS1Planes][W_b / 8]
    bool use_s2_staged = false;
    cpi::Stage1Maps s1maps{};
    bool use_s1_tma = false;
    // v-major refocus (KB5w, refocus_w.cu): per-plane tables of a batch of up to kWBatch planes
    static constexpr int kWBatch = 64;
    bool w_ready = false;
    int w_batch = 0;                       // planes per batch (allocated)
    cpi::AxisTables wxs[kWBatch]{}, wys[kWBatch]{};
    const int32_t** w_i0s = nullptr;       // device arrays of the tables' pointers (pack_w inputs)
    const double** w_ts = nullptr;
    const int32_t** w_ylo = nullptr;
    const int32_t** w_yhi = nullptr;
    uint32_t* w_ent = nullptr;             // [batch][W_b][x_pad] (j0 | t)
    uint4* w_steps = nullptr;              // [batch][W_b][x_pad / 8] walk entries (80 B; 16 B per x allocated)
    int2* w_span = nullptr;                // [groups][x tiles][W_b]
    int2* w_mband = nullptr;               // [groups][v blocks]
    uint2* w_ypack = nullptr;              // [batch][H_b][H_a]
    cpi::TElem* w_T = nullptr;             // [batch][W_a][H_a][H_b]
    // frame-sharded multi-GPU mode (cfg.world >= 2): library-owned NCCL communicator and shard plan
    int world = 1, rank = 0;
    bool sharded = false;                  // multi-GPU mode (shard plan); comm may be null (external mode)
    bool fused = false;                    // CPI_FUSED_REDUCE: GEMM epilogue reduces into the owners' shards
    ncclComm_t comm = nullptr;
    int32_t** d_peers = nullptr;           // [world] device pointers of every rank's shard (own: local)
    std::vector<void*> peer_open;          // IPC-opened peer shard pointers (closed at destroy)
    bool peers_ready = false;
    int sh_block = 0, sh_panels = 1, sh_m_base = 0, sh_m_count = 0, sh_stride = 0;   // A rows
    int32_t* sh_counts = nullptr;          // [m_count * W_a][P_b] reduced pair sums of the owned rows
    int32_t* sh_marg = nullptr;            // [P_a + P_b + 1] all-reduced S_a | S_b | N
    float* sh_gamma_ws = nullptr;          // owned Gamma rows (library workspace)
    float* sh_gamma_cur = nullptr;         // owned Gamma rows written by the last cpi_finalize
    int32_t n_local_i32 = 0;
    double* planes64 = nullptr;            // fp64 plane all-reduce buffer
    size_t planes64_n = 0;
    // accounting
    int64_t launches = 0;
    bool timing = false;
    struct Timed { int cls; cudaEvent_t a, b; };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> event_pool;
    double acc_ms[KC_COUNT] = {};
    int64_t acc_n[KC_COUNT] = {};
    std::string err;
};

namespace {

cpi_status fail(cpi_ctx* c, cpi_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_create_error = buf;
    return s;
}

cpi_status cuda_fail(cpi_ctx* c, cudaError_t e, const char* where) {
    return fail(c, e == cudaErrorMemoryAllocation ? CPI_ERR_OOM : CPI_ERR_CUDA, "%s: %s (%s)", where,
                cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(c, call)                                                   \
    do {                                                              \
        cudaError_t e_ = (call);                                      \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, #call);      \
    } while (0)

cudaEvent_t take_event(cpi_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct TimedScope {
    cpi_ctx* c; int cls; cudaStream_t st; cudaEvent_t a = nullptr;
    TimedScope(cpi_ctx* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
        if (c->timing) { a = take_event(c); cudaEventRecord(a, st); }
    }
    ~TimedScope() {
        if (c->timing) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->timed.push_back({cls, a, b});
        }
    }
};

void drain_timing(cpi_ctx* c) {
    for (auto& t : c->timed) {
        cudaEventSynchronize(t.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.a, t.b);
        c->acc_ms[t.cls] += ms;
        c->acc_n[t.cls] += 1;
        c->event_pool.push_back(t.a);
        c->event_pool.push_back(t.b);
    }
    c->timed.clear();
}

bool roi_ok(const cpi_roi& r, const cpi_layout& l) {
    return r.width >= 1 && r.height >= 1 && r.x0 >= 0 && r.y0 >= 0 &&
           static_cast<int64_t>(r.x0) + r.width <= l.width_px &&
           static_cast<int64_t>(r.y0) + r.height <= l.height_px;
}

}  // namespace

cpi::EncodeTiledFn cpi::encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

namespace {

cpi_status make_tmap(cpi_ctx* c, CUtensorMap* m, void* base, int64_t rows, int64_t cols,
                     uint32_t box_rows) {
    cpi::EncodeTiledFn enc = cpi::encode_tiled_fn();
    if (!enc) return fail(c, CPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};   // bytes between rows
    const cuuint32_t box[2] = {128u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
    return CPI_OK;
}

void free_all(cpi_ctx* c) {
    cudaFree(c->frames_dev[0]);
    cudaFree(c->frames_dev[1]);
    for (int b = 0; b < 2; ++b) {
        if (c->ev_loaded[b]) cudaEventDestroy(c->ev_loaded[b]);
        if (c->ev_consumed[b]) cudaEventDestroy(c->ev_consumed[b]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->op_b != c->op_a) cudaFree(c->op_b);
    cudaFree(c->op_a);
    cudaFree(c->s_a);
    cudaFree(c->s_b);
    cudaFree(c->counts);
    for (int f = 0; f < cpi_ctx::kS1Planes; ++f) {
        cpi::AxisTables* t2[2] = {&c->xs[f], &c->ys[f]};
        for (auto* t : t2) { cudaFree(t->i0); cudaFree(t->t); cudaFree(t->cnt); cudaFree(t->lo); cudaFree(t->hi); }
        if (f == 0)
            for (auto* t : {&c->bxs, &c->bys}) { cudaFree(t->i0); cudaFree(t->t); cudaFree(t->cnt); cudaFree(t->lo); cudaFree(t->hi); }
        cudaFree(c->T[f]);
    }
    for (auto* t : {&c->gen_x, &c->gen_y}) { cudaFree(t->a0); cudaFree(t->at); cudaFree(t->b0); cudaFree(t->bt); cudaFree(t->cnt); }
    cudaFree(c->xpack);
    cudaFree(c->xwpack);
    cudaFree(c->ypack);
    cudaFree(c->xblk);
    cudaFree(c->gamma_ws);
    cudaFree(c->bws);
    for (int f = 0; f < cpi_ctx::kWBatch; ++f)
        for (auto* t : {&c->wxs[f], &c->wys[f]}) { cudaFree(t->i0); cudaFree(t->t); cudaFree(t->cnt); cudaFree(t->lo); cudaFree(t->hi); }
    cudaFree(c->w_i0s); cudaFree(c->w_ts); cudaFree(c->w_ylo); cudaFree(c->w_yhi);
    cudaFree(c->w_ent); cudaFree(c->w_steps); cudaFree(c->w_span); cudaFree(c->w_mband);
    cudaFree(c->w_ypack); cudaFree(c->w_T);
    for (void* p : c->peer_open) cudaIpcCloseMemHandle(p);
    c->peer_open.clear();
    cudaFree(c->d_peers);
    cudaFree(c->sh_counts); cudaFree(c->sh_marg); cudaFree(c->sh_gamma_ws); cudaFree(c->planes64);
    if (c->comm) {
        if (const cpi::NcclApi* api = cpi::nccl_api()) api->comm_destroy(c->comm);
        c->comm = nullptr;
    }
    for (auto& t : c->timed) { c->event_pool.push_back(t.a); c->event_pool.push_back(t.b); }
    for (auto e : c->event_pool) cudaEventDestroy(e);
}

cpi_status alloc_axis(cpi_ctx* c, cpi::AxisTables& t, int W, int Wb) {
    CK(c, cudaMalloc(&t.i0, sizeof(int32_t) * W * Wb));
    CK(c, cudaMalloc(&t.t, sizeof(double) * W * Wb));
    CK(c, cudaMalloc(&t.cnt, sizeof(int32_t) * W));
    CK(c, cudaMalloc(&t.lo, sizeof(int32_t) * Wb));
    CK(c, cudaMalloc(&t.hi, sizeof(int32_t) * Wb));
    return CPI_OK;
}

// Coordinate tables and stage-1 output T of planes [0, n) of a refocus batch (grown on demand:
// T is W_a H_a H_b fp32 per plane).
cpi_status ensure_planes(cpi_ctx* c, int n, int Wa, int Ha, int Wb, int Hb) {
    for (int p = c->n_plane_ws; p < n; ++p) {
        cpi_status s = alloc_axis(c, c->xs[p], Wa, Wb);
        if (s == CPI_OK) s = alloc_axis(c, c->ys[p], Ha, Hb);
        if (s != CPI_OK) return s;
        CK(c, cudaMalloc(&c->T[p], sizeof(cpi::TElem) * size_t(Wa) * Ha * Hb));
        c->n_plane_ws = p + 1;
    }
    return CPI_OK;
}

// Largest union j span (rows, incl. the t -> 1 rounding row) of any (plane group, x tile, u) of
// planes [p0, p0 + n): the A-axis map c(x, u) = ((a (x - c_a)) + (b (u - c_b))) + cc + c_a is affine
// in x, so the union over a tile's outputs and the group's planes is spanned by the endpoint
// values; used samples lie in [0, W_a - 1] (skip) or are clamped into it.
int w_max_span(const double (*maps)[6], int n, int Wa, int Wb) {
    const int xt = cpi::stage1_w_xtile(), gf = cpi::stage1_w_group();
    const double ca = (Wa - 1) / 2.0, cb = (Wb - 1) / 2.0;
    int worst = 0;
    for (int g = 0; g < n; g += gf)
        for (int x0 = 0; x0 < Wa; x0 += xt) {
            const int x1 = std::min(Wa, x0 + xt) - 1;
            for (int u = 0; u < Wb; ++u) {
                double lo = 1e300, hi = -1e300;
                for (int f = g; f < std::min(n, g + gf); ++f)
                    for (int x : {x0, x1}) {
                        const double cc = ((maps[f][0] * (x - ca)) + (maps[f][1] * (u - cb))) + maps[f][2] + ca;
                        lo = std::min(lo, cc);
                        hi = std::max(hi, cc);
                    }
                lo = std::max(lo, 0.0);
                hi = std::min(hi, double(Wa - 1));
                if (hi < lo) continue;
                worst = std::max(worst, int(std::floor(hi) - std::floor(lo)) + 3);
            }
        }
    return worst;
}

// Refocusing for the v-major B order (CPI_GAMMA_VMAJOR): batches of up to kWBatch planes; per
// batch the coordinate tables of every plane, one pack_w, one launch of the window stage 1 (KB5w)
// and the staged stage 2 per group of 4.  Planes of one batch share one Gamma source (the
// caller's Gamma, or one B-resampled Gamma for a fractional B map).
// General maps whose B coordinates depend on the output pixel (dx or dy != 0; refocus_gen.cu):
// per plane, the two axes' support tables, then the two image-sampling stages.
cpi_status refocus_general(cpi_ctx* c, const cpi_refocus_spec* spec, float* planes, cudaStream_t st) {
    const int Wa = c->cfg.roi_a.width, Ha = c->cfg.roi_a.height;
    const int Wb = c->cfg.roi_b.width, Hb = c->cfg.roi_b.height;
    if (c->order != cpi::kOrderRowMajor)
        return fail(c, CPI_ERR_UNSUPPORTED, "maps with output-dependent B coordinates need the row-major B order");
    if (!cpi::refocus_gen_supported(Wa, Ha, Wb, Hb))
        return fail(c, CPI_ERR_UNSUPPORTED, "maps with output-dependent B coordinates need A RoIs of 2..256 px per side "
                                            "and B RoIs of 2..512");
    const int m_count = static_cast<int>(spec->rows / Wa);
    if (spec->row_block > 0 && spec->row_block < m_count)
        return fail(c, CPI_ERR_UNSUPPORTED, "maps with output-dependent B coordinates need contiguous row shards");
    if (!c->gen_x.a0) {
        const int64_t nx = int64_t(Wa) * Wb, ny = int64_t(Ha) * Hb;
        for (auto [t, n, no] : {std::tuple<cpi::GenTables*, int64_t, int>{&c->gen_x, nx, Wa}, {&c->gen_y, ny, Ha}}) {
            CK(c, cudaMalloc(&t->a0, sizeof(int32_t) * n));
            CK(c, cudaMalloc(&t->at, sizeof(float) * n));
            CK(c, cudaMalloc(&t->b0, sizeof(int32_t) * n));
            CK(c, cudaMalloc(&t->bt, sizeof(float) * n));
            CK(c, cudaMalloc(&t->cnt, sizeof(int32_t) * no));
        }
    }
    cpi_status s = ensure_planes(c, 1, Wa, Ha, Wb, Hb);
    if (s != CPI_OK) return s;
    const int m_base = static_cast<int>(spec->row0 / Wa);
    for (int p = 0; p < spec->n_planes; ++p) {
        double mp[12];
        if (spec->affine) {
            for (int i = 0; i < 12; ++i) mp[i] = spec->affine[12 * p + i];
        } else {
            const double al = spec->alphas[p];
            const double d[12] = {al, 1.0 - al, 0.0, 0.0, 1.0, 0.0, al, 1.0 - al, 0.0, 0.0, 1.0, 0.0};
            for (int i = 0; i < 12; ++i) mp[i] = d[i];
        }
        {
            TimedScope ts(c, KC_COORDS, st);
            cudaError_t e = cpi::launch_gen_axis(cpi::GenMap{mp[0], mp[1], mp[2], mp[3], mp[4], mp[5]}, Wa, Wb,
                                                 spec->boundary, c->gen_x, st);
            if (e == cudaSuccess)
                e = cpi::launch_gen_axis(cpi::GenMap{mp[6], mp[7], mp[8], mp[9], mp[10], mp[11]}, Ha, Hb,
                                         spec->boundary, c->gen_y, st);
            c->launches += 2;
            if (e != cudaSuccess) return cuda_fail(c, e, "general-map tables launch");
        }
        {
            TimedScope ts(c, KC_STAGE1, st);
            cudaError_t e = cpi::launch_refocus_gen(spec->gamma_dev, c->p_b, Wa, Ha, Wb, Hb, m_base, m_count, c->gen_x,
                                                    c->gen_y, c->T[0], planes + int64_t(p) * Ha * Wa, st);
            c->launches += 2 + (m_count < Ha ? 1 : 0);
            if (e != cudaSuccess) return cuda_fail(c, e, "general-map refocus launch");
        }
    }
    return CPI_OK;
}

cpi_status refocus_vmajor(cpi_ctx* c, const cpi_refocus_spec* spec, float* planes, cudaStream_t st, bool resample) {
    const int Wa = c->cfg.roi_a.width, Ha = c->cfg.roi_a.height;
    const int Wb = c->cfg.roi_b.width, Hb = c->cfg.roi_b.height;
    const int m_base = static_cast<int>(spec->row0 / Wa), m_count = static_cast<int>(spec->rows / Wa);
    const bool cyclic = spec->row_block > 0 && spec->row_block < m_count;
    const int m_block = cyclic ? spec->row_block : 0, m_stride = cyclic ? spec->row_stride : 0;
    const bool w_ok = cpi::stage1_w_supported(Wa, Hb) && cpi::stage2_staged_supported(Ha) &&
                      (reinterpret_cast<uintptr_t>(spec->gamma_dev) & 15) == 0 && getenv("CPI_STAGE1_SIMPLE") == nullptr;
    if (!w_ok && cyclic)
        return fail(c, CPI_ERR_UNSUPPORTED, "block-cyclic shards in the v-major order need the window stage 1 "
                                            "(W_a <= 256, H_a <= 256, 16-byte aligned Gamma)");
    if (!c->w_ready) {
        const int nb = cpi_ctx::kWBatch;
        for (int f = 0; f < nb; ++f) {
            cpi_status s = alloc_axis(c, c->wxs[f], Wa, Wb);
            if (s == CPI_OK) s = alloc_axis(c, c->wys[f], Ha, Hb);
            if (s != CPI_OK) return s;
        }
        const int64_t xpad = (Wa + cpi::stage1_w_xtile() - 1) / cpi::stage1_w_xtile() * cpi::stage1_w_xtile();
        const int64_t n_xt = xpad / cpi::stage1_w_xtile(), n_vb = (Hb + cpi::stage1_w_vblock() - 1) / cpi::stage1_w_vblock();
        const int64_t n_g = (nb + cpi::stage1_w_group() - 1) / cpi::stage1_w_group();
        CK(c, cudaMalloc(&c->w_i0s, sizeof(void*) * nb));
        CK(c, cudaMalloc(&c->w_ts, sizeof(void*) * nb));
        CK(c, cudaMalloc(&c->w_ylo, sizeof(void*) * nb));
        CK(c, cudaMalloc(&c->w_yhi, sizeof(void*) * nb));
        std::vector<const void*> h(4 * nb);
        for (int f = 0; f < nb; ++f) {
            h[f] = c->wxs[f].i0; h[nb + f] = c->wxs[f].t; h[2 * nb + f] = c->wys[f].lo; h[3 * nb + f] = c->wys[f].hi;
        }
        CK(c, cudaMemcpy(c->w_i0s, h.data(), sizeof(void*) * nb, cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->w_ts, h.data() + nb, sizeof(void*) * nb, cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->w_ylo, h.data() + 2 * nb, sizeof(void*) * nb, cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(c->w_yhi, h.data() + 3 * nb, sizeof(void*) * nb, cudaMemcpyHostToDevice));
        CK(c, cudaMalloc(&c->w_ent, sizeof(uint32_t) * nb * Wb * xpad));
        CK(c, cudaMalloc(&c->w_steps, sizeof(uint4) * nb * Wb * xpad));
        CK(c, cudaMalloc(&c->w_span, sizeof(int2) * n_g * n_xt * Wb));
        CK(c, cudaMalloc(&c->w_mband, sizeof(int2) * n_g * n_vb));
        CK(c, cudaMalloc(&c->w_ypack, sizeof(uint2) * size_t(nb) * Hb * Ha));
        CK(c, cudaMalloc(&c->w_T, sizeof(cpi::TElem) * size_t(nb) * Wa * Ha * Hb));
        c->w_batch = nb;
        c->w_ready = true;
    }
    auto bkey = [&](int p, double* k) {
        const double* mp = spec->affine ? spec->affine + 12 * p : nullptr;
        k[0] = mp ? mp[4] : 1.0; k[1] = mp ? mp[5] : 0.0; k[2] = mp ? mp[10] : 1.0; k[3] = mp ? mp[11] : 0.0;
    };
    auto frac_b = [&](int p) {
        double k[4];
        bkey(p, k);
        return k[0] != 1.0 || k[1] != 0.0 || k[2] != 1.0 || k[3] != 0.0;
    };
    auto same_b = [&](int p, int q) {
        double k[4], l[4];
        bkey(p, k);
        bkey(q, l);
        return k[0] == l[0] && k[1] == l[1] && k[2] == l[2] && k[3] == l[3];
    };
    const int64_t t_plane = int64_t(Wa) * Ha * Hb;
    const int gf = cpi::kRefocusMaxFuse;   // planes per coordinate / stage-2 launch (their argument arrays)
    int resampled = -1;
    for (int p0 = 0; p0 < spec->n_planes;) {
        int nb = 1;   // planes of this batch: one Gamma source
        while (nb < c->w_batch && p0 + nb < spec->n_planes && (!resample || same_b(p0, p0 + nb))) ++nb;
        const bool from_ws = resample && frac_b(p0);
        const float* gsrc = from_ws ? c->bws : spec->gamma_dev;
        double maps[cpi_ctx::kWBatch][6];
        for (int f = 0; f < nb; ++f) {
            if (spec->affine) {
                const double* mp = spec->affine + 12 * (p0 + f);
                const double m6[6] = {mp[0], mp[1], mp[2], mp[6], mp[7], mp[8]};
                for (int i = 0; i < 6; ++i) maps[f][i] = m6[i];
            } else {
                const double alpha = spec->alphas[p0 + f];
                maps[f][0] = maps[f][3] = alpha;
                maps[f][1] = maps[f][4] = 1.0 - alpha;
                maps[f][2] = maps[f][5] = 0.0;
            }
        }
        const bool w_now = w_ok && w_max_span(maps, nb, Wa, Wb) <= cpi::stage1_w_max_span();
        if (!w_now && cyclic)
            return fail(c, CPI_ERR_UNSUPPORTED, "block-cyclic shards in the v-major order need the window stage 1; "
                                                "a plane's span exceeds its stage (A-axis slope above ~2.2)");
        {
            TimedScope ts(c, KC_COORDS, st);
            cudaError_t e = cudaSuccess;
            for (int g0 = 0; g0 < nb && e == cudaSuccess; g0 += gf) {
                const int nf = std::min(gf, nb - g0);
                cpi::CoordsGroupArgs cg{};
                cg.Wa = Wa; cg.Ha = Ha; cg.Wb = Wb; cg.Hb = Hb; cg.boundary = spec->boundary;
                for (int f = 0; f < nf; ++f) {
                    for (int i = 0; i < 6; ++i) cg.map[f][i] = maps[g0 + f][i];
                    cg.xs[f] = c->wxs[g0 + f];
                    cg.ys[f] = c->wys[g0 + f];
                    bkey(p0 + g0 + f, cg.bmap[f]);
                    cg.bx[f] = c->bxs;
                    cg.by[f] = c->bys;
                }
                cg.genb = from_ws ? 1 : 0;
                e = cpi::launch_refocus_coords_group(cg, nf, st);
                c->launches += 2;
                if (e == cudaSuccess) {
                    e = cpi::launch_pack_ytable_group(c->wys + g0, nf, Ha, Hb, c->w_ypack + int64_t(g0) * Hb * Ha, st);
                    c->launches += 1;
                }
            }
            if (e == cudaSuccess && w_now) {
                e = cpi::launch_pack_w(c->w_i0s, c->w_ts, c->w_ylo, c->w_yhi, nb, Wa, Wb, Hb, c->w_ent, c->w_steps,
                                       c->w_span, c->w_mband, st);
                c->launches += 4;
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus coords launch");
        }
        if (from_ws && (resampled < 0 || !same_b(p0, resampled))) {
            TimedScope ts(c, KC_RESAMPLE, st);
            cudaError_t e = cpi::launch_resample_b(spec->gamma_dev, c->bws, spec->rows, Wb, Hb, c->order,
                                                   spec->affine[12 * p0 + 10], c->bxs, c->bys, st);
            c->launches += 1;
            if (e != cudaSuccess) return cuda_fail(c, e, "B resample launch");
            resampled = p0;
        }
        {
            TimedScope ts(c, KC_STAGE1, st);
            cudaError_t e = cudaSuccess;
            if (w_now) {
                cpi::EncodeTiledFn enc = cpi::encode_tiled_fn();
                if (!enc) return fail(c, CPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
                CUtensorMap tg, te;
                // (v % VB, u, v / VB, j, local m) over the blocked v-major columns (kernels.h vmajor_slot)
                const int vbs = cpi::vmajor_block(Hb);
                const cuuint64_t gd[5] = {cuuint64_t(vbs), cuuint64_t(Wb), cuuint64_t(Hb / vbs), cuuint64_t(Wa),
                                          cuuint64_t(m_count)};
                const cuuint64_t gs[4] = {cuuint64_t(vbs) * 4, cuuint64_t(Wb) * vbs * 4, cuuint64_t(c->p_b) * 4,
                                          cuuint64_t(Wa) * c->p_b * 4};
                const cuuint32_t gb[5] = {cuuint32_t(cpi::stage1_w_vblock()), 1u, 1u, cuuint32_t(cpi::stage1_w_jbox()), 1u};
                const cuuint32_t es4[5] = {1u, 1u, 1u, 1u, 1u};
                CUresult r = enc(&tg, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(gsrc), gd, gs, gb, es4,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "Gamma tensor map (v-major) failed (%d)", int(r));
                const int64_t xpad = (Wa + cpi::stage1_w_xtile() - 1) / cpi::stage1_w_xtile() * cpi::stage1_w_xtile();
                // walk entries: 20 words per 8 outputs (refocus_w.cu)
                const cuuint64_t ed[3] = {cuuint64_t(xpad / 8 * 20), cuuint64_t(Wb), cuuint64_t(nb)};
                const cuuint64_t est[2] = {cuuint64_t(xpad / 8 * 20) * 4, cuuint64_t(xpad / 8 * 20) * Wb * 4};
                const cuuint32_t eb[3] = {cuuint32_t(cpi::stage1_w_xtile() / 8 * 20), 1u, cuuint32_t(cpi::stage1_w_group())};
                const cuuint32_t es3[3] = {1u, 1u, 1u};
                r = enc(&te, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, c->w_steps, ed, est, eb, es3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "step-entry tensor map failed (%d)", int(r));
                cpi::S1WArgs a{};
                a.Wa = Wa; a.Ha = Ha; a.Wb = Wb; a.Hb = Hb;
                a.m_base = m_base; a.m_count = m_count; a.m_block = m_block; a.m_stride = m_stride;
                a.n_planes = nb; a.span = c->w_span; a.mband = c->w_mband; a.T = c->w_T; a.t_plane = t_plane;
                if (const char* ev = getenv("CPI_S1W_PROBE")) a.probe = atoi(ev);   // timing probe only
                e = cpi::launch_refocus_stage1_w(&tg, &te, a, c->num_sms, st);
                c->launches += 1;
            } else {
                for (int f = 0; f < nb && e == cudaSuccess; ++f) {
                    e = cpi::launch_refocus_stage1(gsrc, c->p_b, Wa, Ha, Wb, Hb, m_base, m_count, c->wxs[f], c->wys[f],
                                                   c->w_T + f * t_plane, st, 1);
                    c->launches += 1;
                }
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus stage-1 launch");
        }
        {
            TimedScope ts(c, KC_STAGE2, st);
            cudaError_t e = cudaSuccess;
            const int gf2 = cpi::stage2_staged_supported(Ha) ? cpi::kS2MaxPlanes : gf;   // planes per stage-2 launch
            for (int g0 = 0; g0 < nb && e == cudaSuccess; g0 += gf2) {
                const int nf = std::min(gf2, nb - g0);
                if (cpi::stage2_staged_supported(Ha)) {
                    cpi::TElem* Tp[cpi::kS2MaxPlanes];
                    for (int f = 0; f < nf; ++f) Tp[f] = c->w_T + (g0 + f) * t_plane;
                    e = cpi::launch_refocus_stage2_group(Tp, nf, Wa, Ha, Hb, m_base, m_count, m_block, m_stride,
                                                         c->wxs + g0, c->wys + g0, c->w_ypack + int64_t(g0) * Hb * Ha,
                                                         planes + int64_t(p0 + g0) * Ha * Wa, st);
                    c->launches += 1;
                } else {
                    for (int f = 0; f < nf && e == cudaSuccess; ++f) {
                        e = cpi::launch_refocus_stage2(c->w_T + (g0 + f) * t_plane, Wa, Ha, Hb, m_base, m_count,
                                                       c->wxs[g0 + f], c->wys[g0 + f],
                                                       planes + int64_t(p0 + g0 + f) * Ha * Wa, st);
                        c->launches += 1;
                    }
                }
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus stage-2 launch");
        }
        p0 += nb;
    }
    return CPI_OK;
}

}  // namespace

extern "C" {

int32_t cpi_abi_version(void) { return 201; }

const char* cpi_status_string(cpi_status s) {
    switch (s) {
        case CPI_OK: return "CPI_OK";
        case CPI_ERR_INVALID_ARG: return "CPI_ERR_INVALID_ARG";
        case CPI_ERR_LAYOUT: return "CPI_ERR_LAYOUT";
        case CPI_ERR_ROI_OUT_OF_BOUNDS: return "CPI_ERR_ROI_OUT_OF_BOUNDS";
        case CPI_ERR_SIZE_MISMATCH: return "CPI_ERR_SIZE_MISMATCH";
        case CPI_ERR_CAPACITY: return "CPI_ERR_CAPACITY";
        case CPI_ERR_ZERO_FRAMES: return "CPI_ERR_ZERO_FRAMES";
        case CPI_ERR_DEGENERATE_ALPHA: return "CPI_ERR_DEGENERATE_ALPHA";
        case CPI_ERR_EMPTY_ANGULAR_GRID: return "CPI_ERR_EMPTY_ANGULAR_GRID";
        case CPI_ERR_STATE: return "CPI_ERR_STATE";
        case CPI_ERR_CUDA: return "CPI_ERR_CUDA";
        case CPI_ERR_OOM: return "CPI_ERR_OOM";
        case CPI_ERR_UNSUPPORTED: return "CPI_ERR_UNSUPPORTED";
        case CPI_ERR_NCCL: return "CPI_ERR_NCCL";
        default: return "CPI_ERR_UNKNOWN";
    }
}

const char* cpi_last_error(const cpi_ctx* c) {
    return c ? c->err.c_str() : g_create_error.c_str();
}

// ---- dataset files (S:57-64 parse_bin_file) -- host only, no context ----------------
namespace {
cpi_status bin_open(const char* path, const cpi_layout* L, FILE** f, int64_t* frame_bytes, int64_t* n_frames) {
    g_create_error.clear();
    if (!path || !L || !n_frames) return fail(nullptr, CPI_ERR_INVALID_ARG, "path, layout and n_frames must be non-NULL");
    if (L->width_px <= 0 || L->height_px <= 0 || L->width_px % 8 || L->height_px % 8)
        return fail(nullptr, CPI_ERR_LAYOUT, "frame %dx%d: width and height must be positive multiples of 8",
                    L->width_px, L->height_px);
    *frame_bytes = int64_t(L->width_px / 8) * L->height_px;
    FILE* fp = fopen(path, "rb");
    if (!fp) return fail(nullptr, CPI_ERR_INVALID_ARG, "%s: %s", path, strerror(errno));
    if (fseeko(fp, 0, SEEK_END) != 0) {
        fclose(fp);
        return fail(nullptr, CPI_ERR_INVALID_ARG, "%s: %s", path, strerror(errno));
    }
    const int64_t size = ftello(fp);
    if (size < 0) {
        fclose(fp);
        return fail(nullptr, CPI_ERR_INVALID_ARG, "%s: %s", path, strerror(errno));
    }
    if (size % *frame_bytes) {
        fclose(fp);
        return fail(nullptr, CPI_ERR_SIZE_MISMATCH, "%s: %lld bytes is not a whole number of %lld-byte frames", path,
                    static_cast<long long>(size), static_cast<long long>(*frame_bytes));
    }
    *n_frames = size / *frame_bytes;
    if (f) *f = fp; else fclose(fp);
    return CPI_OK;
}
}  // namespace

cpi_status cpi_bin_frames(const char* path, const cpi_layout* layout, int64_t* n_frames) {
    int64_t fb = 0;
    return bin_open(path, layout, nullptr, &fb, n_frames);
}

cpi_status cpi_read_bin(const char* path, const cpi_layout* layout, int64_t frame0, int64_t n_frames, void* dst) {
    if (!dst && n_frames > 0) {
        g_create_error.clear();
        return fail(nullptr, CPI_ERR_INVALID_ARG, "dst must be non-NULL");
    }
    FILE* fp = nullptr;
    int64_t fb = 0, total = 0;
    const cpi_status st = bin_open(path, layout, &fp, &fb, &total);
    if (st != CPI_OK) return st;
    if (frame0 < 0 || n_frames < 0 || frame0 > total || n_frames > total - frame0) {
        fclose(fp);
        return fail(nullptr, CPI_ERR_INVALID_ARG, "%s: frames [%lld, %lld) outside the file's %lld frames", path,
                    static_cast<long long>(frame0), static_cast<long long>(frame0 + n_frames),
                    static_cast<long long>(total));
    }
    const int64_t bytes = n_frames * fb;
    if (bytes > 0) {
        if (fseeko(fp, frame0 * fb, SEEK_SET) != 0 || fread(dst, 1, static_cast<size_t>(bytes), fp) != size_t(bytes)) {
            const int e = errno;
            fclose(fp);
            return fail(nullptr, CPI_ERR_INVALID_ARG, "%s: short read (%s)", path, e ? strerror(e) : "end of file");
        }
    }
    fclose(fp);
    return CPI_OK;
}

cpi_status cpi_create(const cpi_config* cfg, cpi_ctx** out) {
    g_create_error.clear();
    if (!cfg || !out) return fail(nullptr, CPI_ERR_INVALID_ARG, "cfg and out must be non-NULL");
    const cpi_layout& L = cfg->layout;
    if (L.width_px <= 0 || L.height_px <= 0 || L.width_px % 8 || L.height_px % 8)
        return fail(nullptr, CPI_ERR_LAYOUT, "frame %dx%d: width and height must be positive multiples of 8",
                    L.width_px, L.height_px);
    if (L.bit_order != CPI_LSB_FIRST && L.bit_order != CPI_MSB_FIRST)
        return fail(nullptr, CPI_ERR_INVALID_ARG, "bit_order must be CPI_LSB_FIRST or CPI_MSB_FIRST");
    if (!roi_ok(cfg->roi_a, L) || !roi_ok(cfg->roi_b, L))
        return fail(nullptr, CPI_ERR_ROI_OUT_OF_BOUNDS, "RoI outside the %dx%d frame", L.width_px, L.height_px);
    if (cfg->roi_a.width > 512 || cfg->roi_b.width > 512)
        return fail(nullptr, CPI_ERR_UNSUPPORTED, "RoI wider than 512 px");
    if (cfg->max_frames < 1) return fail(nullptr, CPI_ERR_INVALID_ARG, "max_frames must be >= 1");
    if (cfg->max_frames >= (int64_t(1) << 31) - kKAlign)
        return fail(nullptr, CPI_ERR_INVALID_ARG, "max_frames must be < 2^31 (int32 sums)");
    if ((cfg->flags & CPI_GAMMA_UBLOCKED) && cfg->roi_b.width % 8)
        return fail(nullptr, CPI_ERR_UNSUPPORTED, "CPI_GAMMA_UBLOCKED needs roi_b.width %% 8 == 0");
    if ((cfg->flags & CPI_GAMMA_VMAJOR) && (cfg->flags & CPI_GAMMA_UBLOCKED))
        return fail(nullptr, CPI_ERR_INVALID_ARG, "CPI_GAMMA_VMAJOR and CPI_GAMMA_UBLOCKED are exclusive");
    if ((cfg->flags & CPI_GAMMA_VMAJOR) &&
        (cfg->roi_b.height % 4 || (cfg->roi_b.height > cpi::kVMajorBlock && cfg->roi_b.height % cpi::kVMajorBlock)))
        return fail(nullptr, CPI_ERR_UNSUPPORTED, "CPI_GAMMA_VMAJOR needs roi_b.height %% 4 == 0 and, above %d, a "
                                                  "multiple of %d", cpi::kVMajorBlock, cpi::kVMajorBlock);
    if (cfg->flags & ~(CPI_VARIANT_POPC | CPI_KEEP_COUNTS | CPI_VARIANT_FP4 | CPI_GAMMA_UBLOCKED | CPI_GAMMA_VMAJOR |
                       CPI_FUSED_REDUCE | CPI_VARIANT_TC_BITS))
        return fail(nullptr, CPI_ERR_INVALID_ARG, "unknown flags 0x%x", cfg->flags);
    if (__builtin_popcount(cfg->flags & (CPI_VARIANT_POPC | CPI_VARIANT_FP4 | CPI_VARIANT_TC_BITS)) > 1)
        return fail(nullptr, CPI_ERR_INVALID_ARG, "CPI_VARIANT_POPC, CPI_VARIANT_FP4 and CPI_VARIANT_TC_BITS are exclusive");
    if ((cfg->flags & CPI_VARIANT_TC_BITS) && (cfg->flags & CPI_FUSED_REDUCE))
        return fail(nullptr, CPI_ERR_UNSUPPORTED, "CPI_VARIANT_TC_BITS runs the plain GEMM epilogue (no CPI_FUSED_REDUCE)");
    if ((cfg->flags & CPI_VARIANT_FP4) && cfg->max_frames >= (int64_t(1) << 24))
        return fail(nullptr, CPI_ERR_INVALID_ARG, "CPI_VARIANT_FP4 needs max_frames < 2^24 (exact fp32 sums)");

    // multi-GPU mode: world >= 2, or world == 1 with an nccl_id (the same code path as a one-rank group)
    const int world = cfg->world > 1 ? cfg->world : 1;
    const bool sharded = cfg->world > 1 || (cfg->world == 1 && cfg->nccl_id);
    const bool fused = (cfg->flags & CPI_FUSED_REDUCE) != 0;
    if (fused && !sharded) return fail(nullptr, CPI_ERR_INVALID_ARG, "CPI_FUSED_REDUCE needs a multi-GPU config");
    if (fused && ((cfg->flags & CPI_VARIANT_POPC) || getenv("CPI_GEMM_1CTA")))
        return fail(nullptr, CPI_ERR_UNSUPPORTED, "CPI_FUSED_REDUCE runs in the CTA-pair tensor-core GEMM epilogue");
    if (sharded) {
        if (cfg->rank < 0 || cfg->rank >= world)
            return fail(nullptr, CPI_ERR_INVALID_ARG, "rank %d outside [0, world = %d)", cfg->rank, world);
        if (!cfg->nccl_id && !fused)
            return fail(nullptr, CPI_ERR_INVALID_ARG, "multi-GPU config needs nccl_id (or CPI_FUSED_REDUCE)");
        if (!(cfg->flags & CPI_KEEP_COUNTS) && !fused)
            return fail(nullptr, CPI_ERR_INVALID_ARG, "multi-GPU config needs CPI_KEEP_COUNTS (partial pair sums)");
        if (cfg->roi_a.height % world)
            return fail(nullptr, CPI_ERR_INVALID_ARG, "H_a = %d must be divisible by world = %d", cfg->roi_a.height,
                        world);
        if (cfg->nccl_id && !cpi::nccl_api()) return fail(nullptr, CPI_ERR_NCCL, "libnccl.so.2 could not be loaded");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, CPI_ERR_CUDA, "no CUDA device visible");
    if (cfg->device < 0 || cfg->device >= ndev)
        return fail(nullptr, CPI_ERR_INVALID_ARG, "device %d out of range (%d devices)", cfg->device, ndev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess)
        return fail(nullptr, CPI_ERR_CUDA, "cudaGetDeviceProperties failed");
    if (prop.major != 10 || prop.minor != 0)
        return fail(nullptr, CPI_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200)",
                    cfg->device, prop.major, prop.minor);
    if (cudaSetDevice(cfg->device) != cudaSuccess) return fail(nullptr, CPI_ERR_CUDA, "cudaSetDevice failed");

    cpi_ctx* c = new cpi_ctx();
    c->cfg = *cfg;
    c->dev = cfg->device;
    c->num_sms = prop.multiProcessorCount;
    c->popc = (cfg->flags & CPI_VARIANT_POPC) != 0;
    c->fp4 = (cfg->flags & CPI_VARIANT_FP4) != 0;
    c->bits = (cfg->flags & CPI_VARIANT_TC_BITS) != 0;
    c->keep = (cfg->flags & CPI_KEEP_COUNTS) != 0;
    c->p_a = int64_t(cfg->roi_a.width) * cfg->roi_a.height;
    c->p_b = int64_t(cfg->roi_b.width) * cfg->roi_b.height;
    c->k_align = c->fp4 ? 2 * kKAlign : kKAlign;
    c->ublocked = (cfg->flags & CPI_GAMMA_UBLOCKED) != 0;
    c->order = c->ublocked ? cpi::kOrderUBlocked
                           : (cfg->flags & CPI_GAMMA_VMAJOR) ? cpi::kOrderVMajor : cpi::kOrderRowMajor;
    c->k_cap = round_up(cfg->max_frames, c->k_align);
    c->frame_bytes = int64_t(L.width_px / 8) * L.height_px;
    if (c->popc) {
        c->rows_a = round_up(c->p_a, cpi::gemm_popc_block());
        c->rows_b = round_up(c->p_b, cpi::gemm_popc_block());
        c->ld_op = c->k_cap / 32;   // 32-bit words
    } else if (c->bits) {           // bit streams (as popc) padded to the CTA-pair tiles
        c->pair = true;
        c->rows_a = round_up(c->p_a, cpi::gemm_tc2_block_m());
        c->rows_b = round_up(c->p_b, cpi::gemm_tc2_block_n());
        c->ld_op = c->k_cap / 32;   // 32-bit words
    } else if (c->fp4) {
        c->pair = true;
        c->rows_a = round_up(c->p_a, cpi::gemm_tc2_block_m());
        c->rows_b = round_up(c->p_b, cpi::gemm_f4_block_n());
        c->ld_op = c->k_cap / 2;    // bytes (2 frames per byte)
    } else {
        c->pair = getenv("CPI_GEMM_1CTA") == nullptr;
        c->rows_a = round_up(c->p_a, c->pair ? cpi::gemm_tc2_block_m() : cpi::gemm_tc_block_m());
        c->rows_b = round_up(c->p_b, c->pair ? cpi::gemm_tc2_block_n() : cpi::gemm_tc_block_n());
        c->ld_op = c->k_cap;        // bytes
    }
    const size_t op_elem = c->popc || c->bits ? 4 : 1;
    // roi_a == roi_b (e.g. the whole frame as both arms): S_ab is symmetric, so one
    // operand serves both arms and the CTA-pair GEMM computes only tiles touching the upper triangle
    // (SYRK), mirroring them in the epilogue; row-major B order only (the other
    // orders permute the B index), single GPU only.  Opt-in (CPI_SYRK=1): measured on the whole
    // frame (P = 131072, 10^4 frames) the mirrored epilogue stores cost more than the half of the
    // MMAs they save (GEMM 77.5 ms vs 70.8 ms)
    const cpi_roi& ra_ = cfg->roi_a;
    const cpi_roi& rb_ = cfg->roi_b;
    c->symmetric = ra_.x0 == rb_.x0 && ra_.y0 == rb_.y0 && ra_.width == rb_.width && ra_.height == rb_.height &&
                   c->order == cpi::kOrderRowMajor && !c->popc && !c->bits && c->pair && !(cfg->world > 1 || cfg->nccl_id) &&
                   getenv("CPI_SYRK") != nullptr && atoi(getenv("CPI_SYRK")) != 0;
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
    chk(cudaMalloc(&c->frames_dev[0], size_t(c->frame_bytes) * cfg->max_frames));
    chk(cudaMalloc(&c->frames_dev[1], size_t(c->frame_bytes) * cfg->max_frames));
    chk(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        chk(cudaEventCreateWithFlags(&c->ev_loaded[b], cudaEventDisableTiming));
        chk(cudaEventCreateWithFlags(&c->ev_consumed[b], cudaEventDisableTiming));
    }
    chk(cudaMalloc(&c->op_a, size_t(c->rows_a) * c->ld_op * op_elem));
    if (c->symmetric) c->op_b = nullptr;
    else chk(cudaMalloc(&c->op_b, size_t(c->rows_b) * c->ld_op * op_elem));
    chk(cudaMalloc(&c->s_a, sizeof(int32_t) * c->p_a));
    chk(cudaMalloc(&c->s_b, sizeof(int32_t) * c->p_b));
    if (c->keep) chk(cudaMalloc(&c->counts, sizeof(int32_t) * size_t(c->p_a) * c->p_b));
    if (e == cudaSuccess) chk(cudaMemset(c->op_a, 0, size_t(c->rows_a) * c->ld_op * op_elem));
    if (e == cudaSuccess && !c->symmetric) chk(cudaMemset(c->op_b, 0, size_t(c->rows_b) * c->ld_op * op_elem));
    if (c->symmetric) c->op_b = c->op_a;
    if (e == cudaSuccess) chk(cudaMemset(c->s_a, 0, sizeof(int32_t) * c->p_a));
    if (e == cudaSuccess) chk(cudaMemset(c->s_b, 0, sizeof(int32_t) * c->p_b));
    if (e == cudaSuccess && c->keep) chk(cudaMemset(c->counts, 0, sizeof(int32_t) * size_t(c->p_a) * c->p_b));
    if (e == cudaSuccess) chk(cudaDeviceSynchronize());
    if (e != cudaSuccess) {
        cpi_status s = cuda_fail(nullptr, e, "cpi_create allocation");
        free_all(c);
        delete c;
        return s;
    }
    if (sharded) {
        // shard plan: block-cyclic A rows, the smallest block whose panel (world
        // blocks) holds >= 8192 A pixels, so each reduce-scatter call moves >= 32 KB per B pixel row
        c->world = world;
        c->rank = cfg->rank;
        c->sharded = true;
        c->fused = fused;
        const int Wa = cfg->roi_a.width, m_per = cfg->roi_a.height / world;
        int block = m_per;
        for (int b = 1; b <= m_per; ++b)
            if (m_per % b == 0 && int64_t(world) * b * Wa >= std::min<int64_t>(8192, c->p_a)) { block = b; break; }
        c->sh_block = block;
        c->sh_panels = m_per / block;
        c->sh_m_base = c->rank * block;
        c->sh_m_count = m_per;
        c->sh_stride = world * block;
        cudaError_t ea = cudaMalloc(&c->sh_counts, sizeof(int32_t) * size_t(m_per) * Wa * c->p_b);
        if (ea == cudaSuccess) ea = cudaMalloc(&c->sh_marg, sizeof(int32_t) * size_t(c->p_a + c->p_b + 1));
        if (ea == cudaSuccess) ea = cudaMalloc(&c->d_peers, sizeof(int32_t*) * world);
        if (ea == cudaSuccess) ea = cudaMemset(c->sh_counts, 0, sizeof(int32_t) * size_t(m_per) * Wa * c->p_b);
        if (ea != cudaSuccess) {
            cpi_status s = cuda_fail(nullptr, ea, "cpi_create shard workspaces");
            free_all(c);
            delete c;
            return s;
        }
        if (cfg->nccl_id) {
            ncclUniqueId id;
            static_assert(sizeof(id) == CPI_NCCL_ID_BYTES, "NCCL unique id size");
            std::memcpy(&id, cfg->nccl_id, sizeof(id));
            const ncclResult_t r = cpi::nccl_api()->comm_init_rank(&c->comm, world, id, c->rank);
            if (r != ncclSuccess) {
                c->comm = nullptr;
                const cpi_status s = fail(nullptr, CPI_ERR_NCCL, "ncclCommInitRank: %s", cpi::nccl_api()->error_string(r));
                free_all(c);
                delete c;
                return s;
            }
            if (fused) {   // exchange the shard IPC handles over the communicator and map the peers
                std::vector<uint8_t> hs(size_t(world) * CPI_SHARD_HANDLE_BYTES);
                cpi_status s = cpi_shard_ipc_handle(c, hs.data() + size_t(c->rank) * CPI_SHARD_HANDLE_BYTES);
                uint8_t* d_hs = nullptr;
                if (s == CPI_OK && cudaMalloc(&d_hs, hs.size()) != cudaSuccess) s = fail(c, CPI_ERR_OOM, "handle buffer");
                if (s == CPI_OK) {
                    cudaMemcpy(d_hs + size_t(c->rank) * CPI_SHARD_HANDLE_BYTES, hs.data() + size_t(c->rank) * CPI_SHARD_HANDLE_BYTES,
                               CPI_SHARD_HANDLE_BYTES, cudaMemcpyHostToDevice);
                    const ncclResult_t rg = cpi::nccl_api()->all_gather(d_hs + size_t(c->rank) * CPI_SHARD_HANDLE_BYTES, d_hs,
                                                                        CPI_SHARD_HANDLE_BYTES, ncclUint8, c->comm, nullptr);
                    if (rg != ncclSuccess || cudaDeviceSynchronize() != cudaSuccess)
                        s = fail(c, CPI_ERR_NCCL, "shard handle all-gather failed");
                    else if (cudaMemcpy(hs.data(), d_hs, hs.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
                        s = fail(c, CPI_ERR_CUDA, "shard handle copy failed");
                }
                cudaFree(d_hs);
                if (s == CPI_OK) s = cpi_open_peer_shards(c, hs.data());
                if (s != CPI_OK) {
                    g_create_error = c->err;
                    free_all(c);
                    delete c;
                    return s;
                }
            }
        }
    }
    c->cfg.nccl_id = nullptr;   // the caller's buffer is not kept
    if (c->bits) {   // 2D uint32 (words, rows), box 4 words (128 frames) x 128 rows, no swizzle
        cpi_status s = CPI_OK;
        for (int arm = 0; arm < 2 && s == CPI_OK; ++arm) {
            cpi::EncodeTiledFn enc = cpi::encode_tiled_fn();
            if (!enc) { s = fail(c, CPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver"); break; }
            const int64_t rows = arm ? c->rows_b : c->rows_a;
            const cuuint64_t dims[2] = {cuuint64_t(c->ld_op), cuuint64_t(rows)};
            const cuuint64_t strides[1] = {cuuint64_t(c->ld_op) * 4};
            const cuuint32_t box[2] = {4u, cuuint32_t(cpi::gemm_tc2_box_rows())};
            const cuuint32_t estr[2] = {1u, 1u};
            CUresult r = enc(arm ? &c->tm_b : &c->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, arm ? c->op_b : c->op_a, dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) s = fail(c, CPI_ERR_CUDA, "bit-stream tensor map failed (%d)", int(r));
        }
        if (s != CPI_OK) {
            g_create_error = c->err;
            free_all(c);
            delete c;
            return s;
        }
    } else if (!c->popc) {
        const uint32_t box_a = c->pair ? cpi::gemm_tc2_box_rows() : cpi::gemm_tc_block_m();
        const uint32_t box_b = c->fp4 ? cpi::gemm_f4_box_rows_b() : c->pair ? cpi::gemm_tc2_box_rows()
                                                                            : cpi::gemm_tc_block_n();
        cpi_status s = make_tmap(c, &c->tm_a, c->op_a, c->rows_a, c->ld_op, box_a);
        if (s == CPI_OK)   // symmetric: the B map reads the A operand (rows past it are TMA zero fill)
            s = make_tmap(c, &c->tm_b, c->op_b, c->symmetric ? c->rows_a : c->rows_b, c->ld_op, box_b);
        if (s != CPI_OK) {
            g_create_error = c->err;
            free_all(c);
            delete c;
            return s;
        }
    }
    *out = c;
    return CPI_OK;
}

void cpi_destroy(cpi_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    cudaDeviceSynchronize();
    free_all(c);
    delete c;
}

cpi_status cpi_load_frames(cpi_ctx* c, const void* packed, int64_t n, int32_t where, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (n < 0) return fail(c, CPI_ERR_INVALID_ARG, "n_frames < 0");
    if (n > c->cfg.max_frames)
        return fail(c, CPI_ERR_CAPACITY, "%lld frames > max_frames %lld", (long long)n, (long long)c->cfg.max_frames);
    if (n > 0 && !packed) return fail(c, CPI_ERR_INVALID_ARG, "packed is NULL");
    if (where != CPI_HOST && where != CPI_DEVICE) return fail(c, CPI_ERR_INVALID_ARG, "where must be CPI_HOST or CPI_DEVICE");
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    if (where == CPI_HOST) {
        // copy into the staging buffer not used by the previous batch, on the internal copy
        // stream, once the last expand that read this buffer is done; cpi_correlate makes
        // `stream` wait for the copy.  The copy therefore overlaps the previous batch's GEMM and
        // refocusing instead of queueing behind them.
        (void)st;
        const int b = c->next_buf;
        c->next_buf ^= 1;
        if (c->consumed_valid[b]) CK(c, cudaStreamWaitEvent(c->copy_stream, c->ev_consumed[b], 0));
        if (n > 0)
            CK(c, cudaMemcpyAsync(c->frames_dev[b], packed, size_t(n) * c->frame_bytes, cudaMemcpyHostToDevice,
                                  c->copy_stream));
        CK(c, cudaEventRecord(c->ev_loaded[b], c->copy_stream));
        c->frames_cur = c->frames_dev[b];
        c->cur_buf = b;
    } else {
        c->frames_cur = static_cast<const uint8_t*>(packed);
        c->cur_buf = -1;
    }
    c->n_cur = n;
    c->loaded = true;
    c->expanded = false;
    c->consumed = false;
    return CPI_OK;
}

namespace {

// KB1 for the loaded batch: expand both RoIs into the K-major operands and add the batch's
// single-pixel sums and frame count to the totals.
cpi_status expand_batch(cpi_ctx* c, cudaStream_t st) {
    const int64_t n = c->n_cur;
    if (c->n_tot + n >= (int64_t(1) << 31))   // int32 S_a, S_b, S_ab and counts (include/cpi.h)
        return fail(c, CPI_ERR_CAPACITY, "N_TOT would reach %lld >= 2^31 (int32 sums)", (long long)(c->n_tot + n));
    const cpi_layout& L = c->cfg.layout;
    const int64_t k_pad = round_up(n, c->k_align);
    const int mode = c->popc || c->bits ? cpi::kExpandBits : c->fp4 ? cpi::kExpandE2M1 : cpi::kExpandU8;
    TimedScope ts(c, KC_EXPAND, st);
    const cpi::RoiDev ra{c->cfg.roi_a.x0, c->cfg.roi_a.y0, c->cfg.roi_a.width, c->cfg.roi_a.height};
    const cpi::RoiDev rb{c->cfg.roi_b.x0, c->cfg.roi_b.y0, c->cfg.roi_b.width, c->cfg.roi_b.height};
    if (c->cur_buf >= 0) CK(c, cudaStreamWaitEvent(st, c->ev_loaded[c->cur_buf], 0));
    if (n > 0) {
        cpi::launch_expand(c->frames_cur, n, L.width_px / 8, L.height_px, L.bit_order, ra, c->op_a,
                           c->ld_op, k_pad, c->s_a, mode, cpi::kOrderRowMajor, st);
        if (c->symmetric)   // one operand for both arms; S_b = S_a (running totals)
            CK(c, cudaMemcpyAsync(c->s_b, c->s_a, sizeof(int32_t) * c->p_a, cudaMemcpyDeviceToDevice, st));
        else
            cpi::launch_expand(c->frames_cur, n, L.width_px / 8, L.height_px, L.bit_order, rb, c->op_b,
                               c->ld_op, k_pad, c->s_b, mode, c->order, st);
        c->launches += c->symmetric ? 1 : 2;
        CK(c, cudaGetLastError());
    }
    if (c->cur_buf >= 0) {
        CK(c, cudaEventRecord(c->ev_consumed[c->cur_buf], st));
        c->consumed_valid[c->cur_buf] = true;
    }
    // the first batch with frames overwrites the kept counts (no memset after cpi_reset)
    c->accumulate = c->gemm_batches > 0 ? 1 : 0;
    if (n > 0) { c->gemm_batches += 1; c->counts_stale = false; }
    c->n_tot += n;
    c->batches += 1;
    c->expanded = true;
    return CPI_OK;
}

// Kept counts read before any batch wrote them are zero.
cpi_status ensure_counts(cpi_ctx* c, cudaStream_t st) {
    if (c->keep && c->counts_stale) {
        CK(c, cudaMemsetAsync(c->counts, 0, sizeof(int32_t) * size_t(c->p_a) * c->p_b, st));
        c->counts_stale = false;
    }
    return CPI_OK;
}

// Pair-sum GEMM (+ fused Gamma) over A pixel rows [row0, row0 + rows) of the expanded batch.
cpi_status gemm_rows(cpi_ctx* c, int64_t row0, int64_t rows, float* gamma, cudaStream_t st) {
    const int64_t k_pad = round_up(c->n_cur, c->k_align);
    cpi::Epilogue epi{};
    epi.s_a = c->s_a;
    epi.s_b = c->s_b;
    epi.gamma = gamma;
    epi.ldg = c->p_b;
    epi.counts = c->keep && !c->fused ? c->counts : nullptr;
    epi.ldc = c->p_b;
    epi.symmetric = c->symmetric && row0 == 0 && rows == c->p_a ? 1 : 0;   // SYRK on full launches only
    if (c->fused) {
        epi.peers = c->d_peers;
        epi.world = c->world;
        epi.chunk_rows = int64_t(c->sh_block) * c->cfg.roi_a.width;
        epi.panel_rows = epi.chunk_rows * c->world;
    }
    epi.accumulate = c->accumulate;
    epi.p_a = static_cast<int>(std::min(c->p_a, row0 + rows));
    epi.p_b = static_cast<int>(c->p_b);
    epi.vec = (c->p_b % 4) == 0;
    epi.n = static_cast<double>(c->n_tot > 0 ? c->n_tot : 1);
    epi.inv_n2 = 1.0 / (epi.n * epi.n);
    {
        const char* cache_env = getenv("CPI_GEMM_CACHE");   // read per launch (A/B knob)
        epi.cache = cache_env ? atoi(cache_env) : 0;   // L2 policy knob of the CTA-pair GEMM (see kernels.h Epilogue::cache)
    }
    TimedScope ts(c, KC_GEMM, st);
    cudaError_t e;
    if (c->popc) {
        const int64_t T = cpi::gemm_popc_block();
        epi.m_tile0 = static_cast<int>(row0 / T);
        e = cpi::launch_gemm_popc(static_cast<const uint32_t*>(c->op_a), static_cast<const uint32_t*>(c->op_b),
                                  c->ld_op, k_pad / 32, epi, st);
    } else if (c->bits) {
        const int64_t bm = cpi::gemm_tc2_block_m();
        epi.m_tile0 = static_cast<int>(row0 / bm);
        e = cpi::launch_gemm_bits(&c->tm_a, &c->tm_b, static_cast<int>((rows + bm - 1) / bm),
                                  static_cast<int>(c->rows_b / cpi::gemm_tc2_block_n()),
                                  static_cast<int>(k_pad / kKAlign), epi, c->num_sms, st);
    } else if (c->fp4) {
        const int64_t bm = cpi::gemm_tc2_block_m();
        epi.m_tile0 = static_cast<int>(row0 / bm);
        e = cpi::launch_gemm_f4(&c->tm_a, &c->tm_b, static_cast<int>((rows + bm - 1) / bm),
                                static_cast<int>(c->rows_b / cpi::gemm_f4_block_n()),
                                static_cast<int>(k_pad / c->k_align), epi, c->num_sms, st);
    } else if (c->pair) {
        const int64_t bm = cpi::gemm_tc2_block_m();
        epi.m_tile0 = static_cast<int>(row0 / bm);
        e = cpi::launch_gemm_tc2(&c->tm_a, &c->tm_b, static_cast<int>((rows + bm - 1) / bm),
                                 static_cast<int>(c->rows_b / cpi::gemm_tc2_block_n()),
                                 static_cast<int>(k_pad / kKAlign), epi, c->num_sms, st);
    } else {
        const int64_t bm = cpi::gemm_tc_block_m();
        epi.m_tile0 = static_cast<int>(row0 / bm);
        e = cpi::launch_gemm_tc(&c->tm_a, &c->tm_b, static_cast<int>((rows + bm - 1) / bm),
                                static_cast<int>(c->rows_b / cpi::gemm_tc_block_n()),
                                static_cast<int>(k_pad / kKAlign), epi, c->num_sms, st);
    }
    c->launches += 1;
    if (e != cudaSuccess) return cuda_fail(c, e, "pair-sum GEMM launch");
    return CPI_OK;
}

}  // namespace

int64_t cpi_row_align(const cpi_ctx* c) {
    if (!c) return 0;
    if (c->popc) return cpi::gemm_popc_block();
    return c->pair ? cpi::gemm_tc2_block_m() : cpi::gemm_tc_block_m();
}

cpi_status cpi_correlate(cpi_ctx* c, float* gamma, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (!c->loaded || c->consumed || c->expanded)
        return fail(c, CPI_ERR_STATE, "cpi_correlate needs a freshly loaded batch (cpi_load_frames)");
    if (!c->keep && !c->fused && c->batches > 0)
        return fail(c, CPI_ERR_STATE, "second batch needs CPI_KEEP_COUNTS (or cpi_reset)");
    if (!c->keep && !c->fused && !gamma)
        return fail(c, CPI_ERR_STATE, "gamma_dev is NULL and CPI_KEEP_COUNTS is off: pair sums would be lost");
    if (c->sharded && gamma)
        return fail(c, CPI_ERR_STATE, "multi-GPU context: the pair sums are partial; Gamma comes from cpi_finalize");
    if (c->fused && !c->peers_ready)
        return fail(c, CPI_ERR_STATE, "CPI_FUSED_REDUCE: the peer shards are not mapped (cpi_open_peer_shards)");
    const int64_t n = c->n_cur;
    if (gamma && c->n_tot + n == 0) return fail(c, CPI_ERR_ZERO_FRAMES, "Gamma needs N_TOT >= 1");
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    cpi_status s = expand_batch(c, st);
    if (s != CPI_OK) return s;
    if (n > 0) {
        s = gemm_rows(c, 0, c->p_a, gamma, st);
        if (s != CPI_OK) return s;
    } else if (gamma) {
        // empty batch: Gamma of the unchanged totals from the kept counts
        if (!c->keep) return fail(c, CPI_ERR_STATE, "empty batch and no kept counts");
        s = ensure_counts(c, st);
        if (s != CPI_OK) return s;
        TimedScope ts(c, KC_FINALIZE, st);
        cudaError_t e = cpi::launch_finalize(c->counts, c->p_b, c->p_a, c->p_b, c->s_a, c->s_b,
                                             static_cast<double>(c->n_tot), gamma, c->p_b, st);
        c->launches += 1;
        if (e != cudaSuccess) return cuda_fail(c, e, "finalize launch");
    }
    c->consumed = true;
    c->loaded = false;
    c->gamma_current = gamma;
    return CPI_OK;
}

cpi_status cpi_correlate_rows(cpi_ctx* c, int64_t row0, int64_t rows, float* gamma, void* stream);

cpi_status cpi_correlate_rows_to(cpi_ctx* c, int64_t row0, int64_t rows, float* gamma_rows, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (!gamma_rows) return fail(c, CPI_ERR_INVALID_ARG, "gamma_rows_dev is NULL");
    // the kernels address Gamma as base + row * P_b: shift the base so row0 lands on gamma_rows
    float* base = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(gamma_rows) -
                                           static_cast<uintptr_t>(row0) * static_cast<uintptr_t>(c->p_b) * sizeof(float));
    return cpi_correlate_rows(c, row0, rows, base, stream);
}

cpi_status cpi_correlate_rows(cpi_ctx* c, int64_t row0, int64_t rows, float* gamma, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (!c->loaded || c->consumed)
        return fail(c, CPI_ERR_STATE, "cpi_correlate_rows needs a loaded batch not consumed by cpi_correlate");
    if (!c->expanded && !c->keep && !c->fused && c->batches > 0)
        return fail(c, CPI_ERR_STATE, "second batch needs CPI_KEEP_COUNTS (or cpi_reset)");
    if (!c->keep && !c->fused && !gamma)
        return fail(c, CPI_ERR_STATE, "gamma_dev is NULL and CPI_KEEP_COUNTS is off: pair sums would be lost");
    if (c->fused && gamma) return fail(c, CPI_ERR_STATE, "multi-GPU context: Gamma comes from the finalisation");
    const int64_t align = cpi_row_align(c);
    if (row0 < 0 || rows <= 0 || row0 + rows > c->p_a || row0 % align || (rows % align && row0 + rows != c->p_a))
        return fail(c, CPI_ERR_INVALID_ARG, "rows [%lld, +%lld) must lie in [0, P_a) on multiples of %lld",
                    (long long)row0, (long long)rows, (long long)align);
    if (gamma && c->n_tot + (c->expanded ? 0 : c->n_cur) == 0)
        return fail(c, CPI_ERR_ZERO_FRAMES, "Gamma needs N_TOT >= 1");
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    if (!c->expanded) {
        cpi_status s = expand_batch(c, st);
        if (s != CPI_OK) return s;
    }
    if (c->n_cur > 0) {
        cpi_status s = gemm_rows(c, row0, rows, gamma, st);
        if (s != CPI_OK) return s;
    } else if (gamma) {
        if (!c->keep) return fail(c, CPI_ERR_STATE, "empty batch and no kept counts");
        cpi_status s = ensure_counts(c, st);
        if (s != CPI_OK) return s;
        TimedScope ts(c, KC_FINALIZE, st);
        cudaError_t e = cpi::launch_finalize(c->counts + row0 * c->p_b, c->p_b, rows, c->p_b, c->s_a + row0, c->s_b,
                                             static_cast<double>(c->n_tot), gamma + row0 * c->p_b, c->p_b, st);
        c->launches += 1;
        if (e != cudaSuccess) return cuda_fail(c, e, "finalize launch");
    }
    c->gamma_current = nullptr;   // only a panel of Gamma is current
    return CPI_OK;
}

cpi_status cpi_counts_dev(cpi_ctx* c, int32_t** s_ab, int32_t** s_a, int32_t** s_b) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (s_ab && c->keep) {
        CK(c, cudaSetDevice(c->dev));
        cpi_status s = ensure_counts(c, nullptr);   // zeros visible to any later stream work
        if (s != CPI_OK) return s;
        CK(c, cudaDeviceSynchronize());
    }
    if (s_ab) *s_ab = c->fused ? c->sh_counts : c->keep ? c->counts : nullptr;   // fused: this rank's shard rows
    if (s_a) *s_a = c->s_a;
    if (s_b) *s_b = c->s_b;
    return CPI_OK;
}

namespace {
cpi_status nccl_fail(cpi_ctx* c, ncclResult_t r, const char* where) {
    return fail(c, CPI_ERR_NCCL, "%s: %s", where, cpi::nccl_api()->error_string(r));
}
#define NK(c, call)                                                     \
    do {                                                                \
        ncclResult_t r_ = (call);                                       \
        if (r_ != ncclSuccess) return nccl_fail((c), r_, #call);        \
    } while (0)

// Multi-GPU finalize: C2 all-reduce of [S_a | S_b | N], C1 panelised reduce-scatter
// of the int32 partial pair sums (rank r receives block r of every panel), then the owned rows'
// Gamma.  All stream-ordered on st; one host sync to read the global N (the normalisation scale).
cpi_status finalize_sharded(cpi_ctx* c, float* gamma, int64_t* n_tot, cudaStream_t st) {
    const cpi::NcclApi* api = cpi::nccl_api();
    const int Wa = c->cfg.roi_a.width;
    cpi_status s = ensure_counts(c, st);
    if (s != CPI_OK) return s;
    c->n_local_i32 = static_cast<int32_t>(c->n_tot);
    CK(c, cudaMemcpyAsync(c->sh_marg, c->s_a, sizeof(int32_t) * c->p_a, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaMemcpyAsync(c->sh_marg + c->p_a, c->s_b, sizeof(int32_t) * c->p_b, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaMemcpyAsync(c->sh_marg + c->p_a + c->p_b, &c->n_local_i32, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    const int64_t chunk = int64_t(c->sh_block) * Wa, panel = chunk * c->world;
    NK(c, api->group_start());
    NK(c, api->all_reduce(c->sh_marg, c->sh_marg, size_t(c->p_a + c->p_b + 1), ncclInt32, ncclSum, c->comm, st));
    if (!c->fused)   // fused: the GEMM epilogues already reduced into the shards (f2)
        for (int k = 0; k < c->sh_panels; ++k)
            NK(c, api->reduce_scatter(c->counts + k * panel * c->p_b, c->sh_counts + k * chunk * c->p_b,
                                      size_t(chunk * c->p_b), ncclInt32, ncclSum, c->comm, st));
    NK(c, api->group_end());
    int32_t n_glob = 0;
    CK(c, cudaMemcpyAsync(&n_glob, c->sh_marg + c->p_a + c->p_b, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    if (n_glob <= 0) return fail(c, CPI_ERR_ZERO_FRAMES, "global N_TOT = 0");
    float* out = gamma;
    if (!out) {
        if (!c->sh_gamma_ws) CK(c, cudaMalloc(&c->sh_gamma_ws, sizeof(float) * size_t(c->sh_m_count) * Wa * c->p_b));
        out = c->sh_gamma_ws;
    }
    TimedScope ts(c, KC_FINALIZE, st);
    for (int k = 0; k < c->sh_panels; ++k) {
        cudaError_t e = cpi::launch_finalize(c->sh_counts + k * chunk * c->p_b, c->p_b, chunk, c->p_b,
                                             c->sh_marg + k * panel + c->rank * chunk, c->sh_marg + c->p_a,
                                             static_cast<double>(n_glob), out + k * chunk * c->p_b, c->p_b, st);
        c->launches += 1;
        if (e != cudaSuccess) return cuda_fail(c, e, "finalize launch");
    }
    c->sh_gamma_cur = out;
    if (n_tot) *n_tot = n_glob;
    return CPI_OK;
}
}  // namespace

cpi_status cpi_finalize(cpi_ctx* c, float* gamma, int64_t* n_tot, int64_t* row0, int64_t* rows, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    if (c->sharded) {
        if (!c->comm)
            return fail(c, CPI_ERR_STATE, "external multi-GPU mode (no nccl_id): reduce S_a, S_b, N across ranks and "
                                          "finalise the shard (cpi_counts_dev) with cpi_finalize_counts");
        cpi_status s = finalize_sharded(c, gamma, n_tot, st);
        if (s != CPI_OK) return s;
        if (row0) *row0 = int64_t(c->sh_m_base) * c->cfg.roi_a.width;
        if (rows) *rows = int64_t(c->sh_m_count) * c->cfg.roi_a.width;
        return CPI_OK;
    }
    if (c->n_tot == 0) return fail(c, CPI_ERR_ZERO_FRAMES, "N_TOT = 0");
    if (n_tot) *n_tot = c->n_tot;
    if (row0) *row0 = 0;
    if (rows) *rows = c->p_a;
    if (c->gamma_current && (!gamma || gamma == c->gamma_current)) return CPI_OK;
    if (!gamma) return fail(c, CPI_ERR_INVALID_ARG, "gamma_dev is NULL and no fused Gamma exists");
    if (!c->keep) return fail(c, CPI_ERR_STATE, "Gamma from counts needs CPI_KEEP_COUNTS");
    cpi_status s = ensure_counts(c, st);
    if (s != CPI_OK) return s;
    TimedScope ts(c, KC_FINALIZE, st);
    cudaError_t e = cpi::launch_finalize(c->counts, c->p_b, c->p_a, c->p_b, c->s_a, c->s_b,
                                         static_cast<double>(c->n_tot), gamma, c->p_b, st);
    c->launches += 1;
    if (e != cudaSuccess) return cuda_fail(c, e, "finalize launch");
    c->gamma_current = gamma;
    return CPI_OK;
}

cpi_status cpi_shard_layout(const cpi_ctx* c, int32_t* row_block, int32_t* row_stride) {
    if (!c) return CPI_ERR_INVALID_ARG;
    const int ha = c->cfg.roi_a.height;
    if (row_block) *row_block = c->sharded ? c->sh_block : ha;
    if (row_stride) *row_stride = c->sharded ? c->sh_stride : ha;
    return CPI_OK;
}

cpi_status cpi_shard_ipc_handle(cpi_ctx* c, uint8_t* handle) {
    if (!c || !handle) return CPI_ERR_INVALID_ARG;
    if (!c->fused) return fail(c, CPI_ERR_STATE, "CPI_FUSED_REDUCE is off");
    CK(c, cudaSetDevice(c->dev));
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == CPI_SHARD_HANDLE_BYTES, "IPC handle size");
    CK(c, cudaIpcGetMemHandle(&h, c->sh_counts));
    std::memcpy(handle, &h, sizeof(h));
    return CPI_OK;
}

cpi_status cpi_open_peer_shards(cpi_ctx* c, const uint8_t* handles) {
    if (!c || !handles) return CPI_ERR_INVALID_ARG;
    if (!c->fused) return fail(c, CPI_ERR_STATE, "CPI_FUSED_REDUCE is off");
    if (c->peers_ready) return fail(c, CPI_ERR_STATE, "peer shards already mapped");
    CK(c, cudaSetDevice(c->dev));
    std::vector<int32_t*> ptrs(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) { ptrs[r] = c->sh_counts; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + size_t(r) * CPI_SHARD_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcOpenMemHandle (peer shard)");
        c->peer_open.push_back(p);
        ptrs[r] = static_cast<int32_t*>(p);
    }
    CK(c, cudaMemcpy(c->d_peers, ptrs.data(), sizeof(int32_t*) * c->world, cudaMemcpyHostToDevice));
    c->peers_ready = true;
    return CPI_OK;
}

cpi_status cpi_nccl_unique_id(uint8_t* id) {
    if (!id) return CPI_ERR_INVALID_ARG;
    const cpi::NcclApi* api = cpi::nccl_api();
    if (!api) return CPI_ERR_NCCL;
    ncclUniqueId u;
    if (api->get_unique_id(&u) != ncclSuccess) return CPI_ERR_NCCL;
    std::memcpy(id, &u, sizeof(u));
    return CPI_OK;
}

cpi_status cpi_finalize_counts(cpi_ctx* c, const int32_t* s_ab_rows, int64_t row0, int64_t rows,
                               const int32_t* s_a, const int32_t* s_b, int64_t n_tot, float* gamma_rows,
                               void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (n_tot <= 0) return fail(c, CPI_ERR_ZERO_FRAMES, "n_tot must be >= 1");
    if (rows < 0 || row0 < 0 || row0 + rows > c->p_a) return fail(c, CPI_ERR_INVALID_ARG, "row range outside [0, P_a)");
    if (rows > 0 && (!s_ab_rows || !s_a || !s_b || !gamma_rows))
        return fail(c, CPI_ERR_INVALID_ARG, "NULL buffer");
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    TimedScope ts(c, KC_FINALIZE, st);
    cudaError_t e = cpi::launch_finalize(s_ab_rows, c->p_b, rows, c->p_b, s_a + row0, s_b,
                                         static_cast<double>(n_tot), gamma_rows, c->p_b, st);
    c->launches += 1;
    if (e != cudaSuccess) return cuda_fail(c, e, "finalize launch");
    return CPI_OK;
}

cpi_status cpi_get_counts(cpi_ctx* c, int32_t* s_ab, int32_t* s_a, int32_t* s_b, int64_t* n_tot, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (s_ab && !c->keep) return fail(c, CPI_ERR_STATE, "S_ab requested but CPI_KEEP_COUNTS is off");
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    if (s_ab) {
        cpi_status s = ensure_counts(c, st);
        if (s != CPI_OK) return s;
    }
    if (s_ab) CK(c, cudaMemcpyAsync(s_ab, c->counts, sizeof(int32_t) * size_t(c->p_a) * c->p_b, cudaMemcpyDeviceToDevice, st));
    if (s_a) CK(c, cudaMemcpyAsync(s_a, c->s_a, sizeof(int32_t) * c->p_a, cudaMemcpyDeviceToDevice, st));
    if (s_b) CK(c, cudaMemcpyAsync(s_b, c->s_b, sizeof(int32_t) * c->p_b, cudaMemcpyDeviceToDevice, st));
    if (n_tot) *n_tot = c->n_tot;
    return CPI_OK;
}

cpi_status cpi_reset(cpi_ctx* c, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    CK(c, cudaMemsetAsync(c->s_a, 0, sizeof(int32_t) * c->p_a, st));
    CK(c, cudaMemsetAsync(c->s_b, 0, sizeof(int32_t) * c->p_b, st));
    c->counts_stale = true;                  // zeroed lazily: the next batch overwrites them
    if (c->fused) {
        // every rank's GEMM adds into every shard: all shards must be zero before any rank's next GEMM
        // (the NCCL barrier below; in external mode the caller synchronises the ranks)
        CK(c, cudaMemsetAsync(c->sh_counts, 0, sizeof(int32_t) * size_t(c->sh_m_count) * c->cfg.roi_a.width * c->p_b, st));
        if (c->comm) {
            NK(c, cpi::nccl_api()->all_reduce(c->sh_marg, c->sh_marg, 1, ncclInt32, ncclSum, c->comm, st));
        }
    }
    c->n_tot = 0;
    c->batches = 0;
    c->gemm_batches = 0;
    c->gamma_current = nullptr;
    c->loaded = false;
    return CPI_OK;
}

cpi_status cpi_refocus(cpi_ctx* c, const cpi_refocus_spec* spec_in, float* planes, void* stream) {
    if (!c) return CPI_ERR_INVALID_ARG;
    if (!spec_in || !planes) return fail(c, CPI_ERR_INVALID_ARG, "spec and planes_dev must be non-NULL");
    cpi_refocus_spec spec_local = *spec_in;
    const cpi_refocus_spec* spec = &spec_local;
    if (!spec_local.gamma_dev && c->sharded) {
        if (!c->comm) return fail(c, CPI_ERR_STATE, "external multi-GPU mode: refocus the shard rows explicitly");
        // this rank's Gamma rows of the last cpi_finalize, then the fp64 plane all-reduce (C3)
        if (!c->sh_gamma_cur) return fail(c, CPI_ERR_STATE, "multi-GPU refocus from the totals needs cpi_finalize first");
        const int Wa = c->cfg.roi_a.width, Ha = c->cfg.roi_a.height;
        spec_local.gamma_dev = c->sh_gamma_cur;
        spec_local.row0 = int64_t(c->sh_m_base) * Wa;
        spec_local.rows = int64_t(c->sh_m_count) * Wa;
        spec_local.row_block = c->sh_block;
        spec_local.row_stride = c->sh_stride;
        cpi_status s = cpi_refocus(c, &spec_local, planes, stream);
        if (s != CPI_OK) return s;
        auto st = static_cast<cudaStream_t>(stream);
        const size_t n = size_t(spec->n_planes) * Ha * Wa;
        if (c->planes64_n < n) {
            cudaFree(c->planes64);
            c->planes64 = nullptr;
            c->planes64_n = 0;
            CK(c, cudaMalloc(&c->planes64, sizeof(double) * n));
            c->planes64_n = n;
        }
        CK(c, cpi::launch_f32_to_f64(planes, c->planes64, int64_t(n), st));
        NK(c, cpi::nccl_api()->all_reduce(c->planes64, c->planes64, n, ncclFloat64, ncclSum, c->comm, st));
        CK(c, cpi::launch_f64_to_f32(c->planes64, planes, int64_t(n), st));
        c->launches += 2;
        return CPI_OK;
    }
    if (!spec_local.gamma_dev) {
        // the context's current totals (SURVEY §8(b) CPI_FROM_COUNTS): the fused / finalised
        // Gamma of the last call, else Gamma finalised from the kept counts
        if (c->n_tot == 0) return fail(c, CPI_ERR_ZERO_FRAMES, "refocus from counts needs N_TOT >= 1");
        if (!c->gamma_current) {
            if (!c->keep) return fail(c, CPI_ERR_STATE, "gamma_dev is NULL: no current Gamma and no kept counts");
            if (!c->gamma_ws) CK(c, cudaMalloc(&c->gamma_ws, sizeof(float) * size_t(c->p_a) * c->p_b));
            cpi_status s = cpi_finalize(c, c->gamma_ws, nullptr, nullptr, nullptr, stream);
            if (s != CPI_OK) return s;
        }
        spec_local.gamma_dev = c->gamma_current;
        spec_local.row0 = 0;
        spec_local.rows = c->p_a;
        spec_local.row_block = 0;
    }
    if (spec->n_planes < 1 || (!spec->alphas && !spec->affine))
        return fail(c, CPI_ERR_EMPTY_ANGULAR_GRID, "n_planes must be >= 1");
    if (spec->boundary != CPI_SKIP_RENORMALIZE && spec->boundary != CPI_CLAMP)
        return fail(c, CPI_ERR_INVALID_ARG, "unknown boundary policy %d", spec->boundary);
    bool genb = false;   // some plane has fractional B coordinates -> general-B kernels
    bool gen_xy = false; // some plane's B coordinates depend on the output pixel (dx, dy != 0)
    if (spec->affine) {
        for (int p = 0; p < spec->n_planes; ++p) {
            const double* mp = spec->affine + 12 * p;
            for (int i = 0; i < 12; ++i)
                if (!std::isfinite(mp[i])) return fail(c, CPI_ERR_INVALID_ARG, "affine[%d][%d] is not finite", p, i);
            if (mp[3] != 0.0 || mp[9] != 0.0) gen_xy = true;
            if (mp[4] != 1.0 || mp[5] != 0.0 || mp[10] != 1.0 || mp[11] != 0.0) genb = true;
        }
    } else {
        for (int p = 0; p < spec->n_planes; ++p)
            if (!(spec->alphas[p] != 0.0) || !std::isfinite(spec->alphas[p]))
                return fail(c, CPI_ERR_DEGENERATE_ALPHA, "alpha[%d] = %g (must be finite and non-zero)", p,
                            spec->alphas[p]);
    }
    const int Wa = c->cfg.roi_a.width, Ha = c->cfg.roi_a.height;
    const int Wb = c->cfg.roi_b.width, Hb = c->cfg.roi_b.height;
    if (Wa < 2 || Ha < 2) return fail(c, CPI_ERR_UNSUPPORTED, "refocusing needs an A RoI of at least 2x2");
    if (!spec->gamma_dev) return fail(c, CPI_ERR_INVALID_ARG, "gamma_dev is NULL");
    if (spec->row0 < 0 || spec->rows <= 0 || spec->row0 % Wa || spec->rows % Wa || spec->row0 + spec->rows > c->p_a)
        return fail(c, CPI_ERR_INVALID_ARG, "rows [%lld, +%lld) must be whole A rows inside [0, P_a)",
                    (long long)spec->row0, (long long)spec->rows);
    CK(c, cudaSetDevice(c->dev));
    auto st = static_cast<cudaStream_t>(stream);
    if (gen_xy) return refocus_general(c, spec, planes, st);
    if (!c->refocus_ready && c->order != cpi::kOrderVMajor) {
        c->use_s1_tma = cpi::stage1_tma_supported(Wa, Wb, Hb) && getenv("CPI_STAGE1_SIMPLE") == nullptr;
        if (const char* ev = getenv("CPI_REFOCUS_FUSE")) c->fuse = atoi(ev);
        if (c->fuse < 1) c->fuse = 1;
        if (c->fuse > cpi::kStage1MaxFuse) c->fuse = cpi::kStage1MaxFuse;
        c->use_s2_staged = cpi::stage2_staged_supported(Ha) && getenv("CPI_STAGE2_SIMPLE") == nullptr;
        if (c->use_s2_staged)
            CK(c, cudaMalloc(&c->ypack, sizeof(uint2) * size_t(Ha) * Hb * cpi::kRefocusMaxFuse));
        if (c->use_s1_tma) {
            constexpr int kP = cpi_ctx::kS1Planes;
            CK(c, cudaMalloc(&c->xpack, sizeof(uint32_t) * size_t(Wa) * Wb * kP));
            CK(c, cudaMemset(c->xpack, 0, sizeof(uint32_t) * size_t(Wa) * Wb * kP));
            CK(c, cudaMalloc(&c->xwpack, sizeof(float) * size_t(Wa) * Wb * kP));
            CK(c, cudaMemset(c->xwpack, 0, sizeof(float) * size_t(Wa) * Wb * kP));
            CK(c, cudaMalloc(&c->xblk, sizeof(uint32_t) * size_t((Wb + 7) / 8) * kP));
            cpi::EncodeTiledFn enc = cpi::encode_tiled_fn();
            if (!enc) return fail(c, CPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
            const cuuint64_t dims[3] = {cuuint64_t(Wa), cuuint64_t(Wb), cuuint64_t(kP)};
            const cuuint64_t strides[2] = {cuuint64_t(Wa) * 4, cuuint64_t(Wa) * Wb * 4};
            const cuuint32_t box[3] = {cuuint32_t(Wa), 8u, 1u};
            const cuuint32_t es[3] = {1u, 1u, 1u};
            CUresult r = enc(&c->s1maps.xtab, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, c->xpack, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "x-table tensor map failed (%d)", int(r));
            r = enc(&c->s1maps.xwtab, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c->xwpack, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "x-weight tensor map failed (%d)", int(r));
        }
        c->refocus_ready = true;
    }
    // B map of plane p: (ex, fx, ey, fy); identity = integral B lattice
    auto bkey = [&](int p, double* k) {
        const double* mp = spec->affine ? spec->affine + 12 * p : nullptr;
        k[0] = mp ? mp[4] : 1.0; k[1] = mp ? mp[5] : 0.0; k[2] = mp ? mp[10] : 1.0; k[3] = mp ? mp[11] : 0.0;
    };
    auto frac_b = [&](int p) {
        double k[4];
        bkey(p, k);
        return k[0] != 1.0 || k[1] != 0.0 || k[2] != 1.0 || k[3] != 0.0;
    };
    auto same_b = [&](int p, int q) {
        double k[4], l[4];
        bkey(p, k);
        bkey(q, l);
        return k[0] == l[0] && k[1] == l[1] && k[2] == l[2] && k[3] == l[3];
    };
    // Fractional B: resample Gamma onto the B lattice once per distinct B map and run the fast
    // separable path (launch_resample_b); the direct general-B kernels remain for when the
    // workspace (rows x P_b fp32) cannot be allocated, or under CPI_GENB_DIRECT (A/B knob).
    bool resample = false;
    if (genb) {
        if (Wb < 2 || Hb < 2) return fail(c, CPI_ERR_UNSUPPORTED, "fractional B coordinates need a B RoI of 2x2 or more");
        if (!c->bxs.i0) {
            cpi_status s = alloc_axis(c, c->bxs, 1, Wb);
            if (s == CPI_OK) s = alloc_axis(c, c->bys, 1, Hb);
            if (s != CPI_OK) return s;
        }
        resample = getenv("CPI_GENB_DIRECT") == nullptr;
        const size_t need = sizeof(float) * size_t(spec->rows) * size_t(c->p_b);
        if (resample && c->bws_bytes < need) {
            cudaFree(c->bws);
            c->bws = nullptr;
            c->bws_bytes = 0;
            if (cudaMalloc(&c->bws, need) == cudaSuccess) {
                c->bws_bytes = need;
            } else {
                (void)cudaGetLastError();
                resample = false;
            }
        }
    }
    const bool direct = genb && !resample;
    if (c->order == cpi::kOrderVMajor) {
        if (direct)
            return fail(c, CPI_ERR_UNSUPPORTED, "fractional B coordinates without the resample workspace need the "
                                                "row-major B order");
        if (spec->row_block > 0 && spec->row_block < spec->rows / Wa && spec->row_stride < spec->row_block)
            return fail(c, CPI_ERR_INVALID_ARG, "row_stride %d < row_block %d", spec->row_stride, spec->row_block);
        if (spec->row_block > 0 && spec->row_block < spec->rows / Wa) {
            const int mb = static_cast<int>(spec->row0 / Wa), mc = static_cast<int>(spec->rows / Wa);
            const int64_t last = mb + int64_t((mc - 1) / spec->row_block) * spec->row_stride + (mc - 1) % spec->row_block;
            if (last >= Ha) return fail(c, CPI_ERR_INVALID_ARG, "block-cyclic shard reaches A row %lld >= H_a", (long long)last);
        }
        return refocus_vmajor(c, spec, planes, st, resample);
    }
    if (direct && c->ublocked)
        return fail(c, CPI_ERR_UNSUPPORTED, "fractional B coordinates without the resample workspace need the "
                                            "row-major B order");
    bool tma_now = !direct && c->use_s1_tma && (reinterpret_cast<uintptr_t>(spec->gamma_dev) & 15) == 0;
    if (c->ublocked && !tma_now)
        return fail(c, CPI_ERR_UNSUPPORTED, "u-blocked Gamma needs the TMA stage 1 (W_a <= 256, W_b %% 4 == 0, "
                                            "16-byte aligned Gamma)");
    const float* encoded = nullptr;   // Gamma base the stage-1 tensor map currently describes
    auto encode_gamma = [&](const float* g) -> cpi_status {
        if (g == encoded) return CPI_OK;
        cpi::EncodeTiledFn enc = cpi::encode_tiled_fn();
        CUresult r;
        if (c->ublocked) {
            // (u % 8, v, u / 8, j, m): box 8 x 8 x 1 x 32 x 1 lands as [j][v][u] like the 4D map
            const cuuint64_t dims[5] = {8u, cuuint64_t(Hb), cuuint64_t(Wb / 8), cuuint64_t(Wa), cuuint64_t(spec->rows / Wa)};
            const cuuint64_t strides[4] = {32u, cuuint64_t(Hb) * 32, cuuint64_t(c->p_b) * 4, cuuint64_t(Wa) * c->p_b * 4};
            const cuuint32_t box[5] = {8u, cuuint32_t(cpi::stage1_vgroup(Wa)), 1u, 32u, 1u};
            const cuuint32_t es[5] = {1u, 1u, 1u, 1u, 1u};
            r = enc(&c->s1maps.gamma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(g), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            c->s1maps.gamma_5d = 1;
        } else {
            const cuuint64_t dims[4] = {cuuint64_t(Wb), cuuint64_t(Hb), cuuint64_t(Wa), cuuint64_t(spec->rows / Wa)};
            const cuuint64_t strides[3] = {cuuint64_t(Wb) * 4, cuuint64_t(c->p_b) * 4, cuuint64_t(Wa) * c->p_b * 4};
            const cuuint32_t box[4] = {8u, cuuint32_t(cpi::stage1_vgroup(Wa)), 32u, 1u};
            const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
            // L2 sector promotion of the Gamma stream (tuning knob CPI_S1_L2PROMO = 0/64/128/256)
            CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
            if (const char* ev = getenv("CPI_S1_L2PROMO")) {
                const int v = atoi(ev);
                promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                      : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
            }
            r = enc(&c->s1maps.gamma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(g), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            c->s1maps.gamma_5d = 0;
        }
        if (r != CUDA_SUCCESS) return fail(c, CPI_ERR_CUDA, "Gamma tensor map failed (%d)", int(r));
        encoded = g;
        return CPI_OK;
    };
    const int m_base = static_cast<int>(spec->row0 / Wa), m_count = static_cast<int>(spec->rows / Wa);
    const bool cyclic = spec->row_block > 0 && spec->row_block < m_count;
    const int m_block = cyclic ? spec->row_block : 0, m_stride = cyclic ? spec->row_stride : 0;
    if (cyclic) {
        if (m_stride < m_block)
            return fail(c, CPI_ERR_INVALID_ARG, "row_stride %d < row_block %d", m_stride, m_block);
        const int64_t last = m_base + int64_t((m_count - 1) / m_block) * m_stride + (m_count - 1) % m_block;
        if (last >= Ha) return fail(c, CPI_ERR_INVALID_ARG, "block-cyclic shard reaches A row %lld >= H_a", (long long)last);
        if (direct) return fail(c, CPI_ERR_UNSUPPORTED, "fractional B coordinates without the resample workspace "
                                                        "need contiguous row shards");
    }
    const int group = tma_now ? c->fuse : 1;
    // one fused group per KB5 launch (16 groups per launch in slab-major tile order, sharing each
    // Gamma slab through L2, measured 80 vs 76 ms: DESIGN §17)
    const int batch_cap = group;
    const int64_t nch = (Wb + 7) / 8;
    int resampled = -1;   // plane whose B map the workspace currently holds
    for (int p0 = 0; p0 < spec->n_planes;) {
        int nb = 1;
        while (nb < batch_cap && p0 + nb < spec->n_planes && (!resample || same_b(p0, p0 + nb))) ++nb;
        {
            cpi_status s = ensure_planes(c, nb, Wa, Ha, Wb, Hb);
            if (s != CPI_OK) return s;
        }
        const bool from_ws = resample && frac_b(p0);
        const float* gsrc = from_ws ? c->bws : spec->gamma_dev;
        {
            TimedScope ts(c, KC_COORDS, st);
            cudaError_t e = cudaSuccess;
            for (int g0 = 0; g0 < nb && e == cudaSuccess; g0 += group) {
                const int nf = std::min(group, nb - g0);
                cpi::CoordsGroupArgs cg{};
                cg.Wa = Wa; cg.Ha = Ha; cg.Wb = Wb; cg.Hb = Hb; cg.boundary = spec->boundary;
                for (int f = 0; f < nf; ++f) {   // (a, b, c) of the A-axis maps of plane p0 + g0 + f
                    const int p = p0 + g0 + f;
                    if (spec->affine) {
                        const double* mp = spec->affine + 12 * p;
                        const double m6[6] = {mp[0], mp[1], mp[2], mp[6], mp[7], mp[8]};
                        for (int i = 0; i < 6; ++i) cg.map[f][i] = m6[i];
                    } else {
                        const double alpha = spec->alphas[p];
                        cg.map[f][0] = cg.map[f][3] = alpha;
                        cg.map[f][1] = cg.map[f][4] = 1.0 - alpha;
                        cg.map[f][2] = cg.map[f][5] = 0.0;
                    }
                    cg.xs[f] = c->xs[g0 + f];
                    cg.ys[f] = c->ys[g0 + f];
                    bkey(p, cg.bmap[f]);
                    cg.bx[f] = c->bxs;   // one B map per batch: every f writes the same supports
                    cg.by[f] = c->bys;
                }
                cg.genb = direct || from_ws ? 1 : 0;   // B supports for the direct kernels / the resample
                e = cpi::launch_refocus_coords_group(cg, nf, st);
                c->launches += 2;
                if (e == cudaSuccess && tma_now) {
                    e = cpi::launch_pack_xtable_group(c->xs + g0, nf, Wa, Wb, c->xpack + int64_t(g0) * Wa * Wb,
                                                      c->xwpack + int64_t(g0) * Wa * Wb, c->xblk + g0 * nch, st);
                    c->launches += 1;
                }
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus coords launch");
        }
        if (from_ws && (resampled < 0 || !same_b(p0, resampled))) {
            TimedScope ts(c, KC_RESAMPLE, st);
            cudaError_t e = cpi::launch_resample_b(spec->gamma_dev, c->bws, spec->rows, Wb, Hb, c->order,
                                                   spec->affine[12 * p0 + 10], c->bxs, c->bys, st);
            c->launches += 1;
            if (e != cudaSuccess) return cuda_fail(c, e, "B resample launch");
            resampled = p0;
        }
        if (tma_now) {
            cpi_status s = encode_gamma(gsrc);
            if (s != CPI_OK) return s;
        }
        {
            TimedScope ts(c, KC_STAGE1, st);
            cudaError_t e = cudaSuccess;
            if (direct) {
                e = cpi::launch_refocus_stage1_genb(spec->gamma_dev, c->p_b, Wa, Ha, Wb, Hb, m_base, m_count, c->xs[0],
                                                    c->bxs, c->T[0], st);
                c->launches += 1;
            } else if (tma_now) {
                e = cpi::launch_refocus_stage1_tma(&c->s1maps, nb, Wa, Ha, Wb, Hb, m_base, m_count, m_block, m_stride,
                                                   c->xs, c->ys, c->T, c->xblk, c->num_sms, st);
                c->launches += 1;
            } else if (!cyclic) {
                e = cpi::launch_refocus_stage1(gsrc, c->p_b, Wa, Ha, Wb, Hb, m_base, m_count, c->xs[0], c->ys[0],
                                               c->T[0], st);
                c->launches += 1;
            } else {
                return fail(c, CPI_ERR_UNSUPPORTED, "block-cyclic shards need the TMA stage 1 (W_a <= 256, W_b %% 4 == 0, "
                                                    "16-byte aligned Gamma)");
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus stage-1 launch");
        }
        {
            TimedScope ts(c, KC_STAGE2, st);
            cudaError_t e = cudaSuccess;
            for (int g0 = 0; g0 < nb && e == cudaSuccess; g0 += group) {
                const int nf = std::min(group, nb - g0);
                float* pl = planes + int64_t(p0 + g0) * Ha * Wa;
                if (direct) {
                    e = cpi::launch_refocus_stage2_genb(c->T[0], Wa, Ha, Hb, m_base, m_count, c->xs[0], c->ys[0], c->bys,
                                                        pl, st);
                    c->launches += 1;
                } else if (c->use_s2_staged) {
                    e = cpi::launch_pack_ytable_group(c->ys + g0, nf, Ha, Hb, c->ypack, st);
                    if (e == cudaSuccess)
                        e = cpi::launch_refocus_stage2_group(c->T + g0, nf, Wa, Ha, Hb, m_base, m_count, m_block,
                                                             m_stride, c->xs + g0, c->ys + g0, c->ypack, pl, st);
                    c->launches += 2;
                } else if (cyclic) {
                    return fail(c, CPI_ERR_UNSUPPORTED, "block-cyclic shards need H_a <= 256");
                } else {
                    for (int f = 0; f < nf && e == cudaSuccess; ++f) {
                        e = cpi::launch_refocus_stage2(c->T[g0 + f], Wa, Ha, Hb, m_base, m_count, c->xs[g0 + f],
                                                       c->ys[g0 + f], pl + int64_t(f) * Ha * Wa, st);
                        c->launches += 1;
                    }
                }
            }
            if (e != cudaSuccess) return cuda_fail(c, e, "refocus stage-2 launch");
        }
        p0 += nb;
    }
    return CPI_OK;
}

int64_t cpi_launch_count(const cpi_ctx* c) { return c ? c->launches : 0; }


cpi_status cpi_set_timing(cpi_ctx* c, int32_t enable) {
    if (!c) return CPI_ERR_INVALID_ARG;
    drain_timing(c);
    for (int i = 0; i < KC_COUNT; ++i) { c->acc_ms[i] = 0; c->acc_n[i] = 0; }
    c->timing = enable != 0;
    return CPI_OK;
}

cpi_status cpi_kernel_time_ms(cpi_ctx* c, int32_t cls, double* ms, int64_t* launches) {
    if (!c || cls < 0 || cls >= KC_COUNT) return CPI_ERR_INVALID_ARG;
    drain_timing(c);
    if (ms) *ms = c->acc_ms[cls];
    if (launches) *launches = c->acc_n[cls];
    return CPI_OK;
}

}  // extern "C"
