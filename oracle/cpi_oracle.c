/*
 * cpi_oracle.c — CPU ORACLE for the CPI hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant with the
 * CUDA path (paper_2407_20692_b200/csrc); it is plain, slow, obviously-correct C.
 *
 * What it computes (citations: P = /root/reference/PAPER.md line, S = SPEC.md line):
 *   - unpack of SwissSPAD2 1-bpp frames into per-pixel 0/1 values      (§2)
 *   - single-pixel sums S_a, S_b and pair sums S_ab = sum_i A^i_p B^i_q  (Eq. 1)
 *   - Gamma = (N*S_ab - S_a*S_b) / N^2, the exact rational of Eq. (1)
 *   - refocusing: for every output pixel the mean over the angular (B) lattice of the
 *     4D multilinear interpolation of Gamma at plane-dependent coordinates
 *     ("Refocusing", "4D multilinear interpolation", S:274 default map,
 *     S:290-302 interp4/refocus_plane, SURVEY §8(c) Q10-Q14 readings), for the default map
 *     and for a general per-plane affine map of all four coordinates (S:273 RefocusMap,
 *     SURVEY NEXT f3(ii)).
 *
 * Floating point: fp64 throughout; compile with -ffp-contract=off so every
 * a*b+c below is two rounded operations, exactly as written.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t x0, y0, width, height;
} oroi;

/* Pixel (col, row) of frame i: bit (col % 8) of byte col/8 of that row (lsb_first,
 * S:110); msb_first flips the bit index.  Frame-major, row-major, stride W/8 bytes
 * (P:65-66). */
static inline int pixel_bit(const uint8_t *frames, int64_t i, int W, int H, int msb,
                            int col, int row) {
    const int64_t stride = W / 8;
    const uint8_t byte = frames[(i * H + row) * stride + col / 8];
    const int b = msb ? 7 - (col % 8) : (col % 8);
    return (byte >> b) & 1;
}

static int roi_ok(oroi r, int W, int H) {
    return r.width >= 1 && r.height >= 1 && r.x0 >= 0 && r.y0 >= 0 &&
           r.x0 + r.width <= W && r.y0 + r.height <= H;
}

/* A^i_p for every frame i and RoI pixel p = m*width + j (row-major, j horizontal
 * fastest): out[i*P + p] = pixel (x0+j, y0+m) of frame i. */
int oracle_unpack(const uint8_t *frames, int64_t n, int W, int H, int msb, oroi r,
                  uint8_t *out) {
    if (W % 8 || H < 1 || !roi_ok(r, W, H)) return -1;
    const int64_t P = (int64_t)r.width * r.height;
    for (int64_t i = 0; i < n; i++)
        for (int m = 0; m < r.height; m++)
            for (int j = 0; j < r.width; j++)
                out[i * P + (int64_t)m * r.width + j] =
                    (uint8_t)pixel_bit(frames, i, W, H, msb, r.x0 + j, r.y0 + m);
    return 0;
}

/* Single-pixel sums over frames, Eq. (1)'s  sum_i A^i_jm:
 * s[p] = sum_i A^i_p, as a plain loop over frames. */
int oracle_marginals(const uint8_t *frames, int64_t n, int W, int H, int msb, oroi r,
                     int64_t *s) {
    if (W % 8 || H < 1 || !roi_ok(r, W, H)) return -1;
    for (int m = 0; m < r.height; m++)
        for (int j = 0; j < r.width; j++) {
            int64_t acc = 0;
            for (int64_t i = 0; i < n; i++)
                acc += pixel_bit(frames, i, W, H, msb, r.x0 + j, r.y0 + m);
            s[(int64_t)m * r.width + j] = acc;
        }
    return 0;
}

/* Pair sums, Eq. (1)'s  sum_i A^i_jm B^i_kn, for the requested A pixels:
 *   s_ab[r][q] = sum_i A^i_{rows[r]} * B^i_q
 * a plain triple loop in (p_a, i, p_b) order, int64 accumulators, no blocking or
 * packing.  rows == NULL means every A pixel in order.
 * The frames are unpacked first (the prototype's "bit-unpacking is performed").
 * OpenMP splits the outer p_a loop only. */
int oracle_pair_sums(const uint8_t *frames, int64_t n, int W, int H, int msb, oroi ra,
                     oroi rb, const int64_t *rows, int64_t nrows, int64_t *s_ab,
                     int nthreads) {
    if (W % 8 || H < 1 || !roi_ok(ra, W, H) || !roi_ok(rb, W, H)) return -1;
    const int64_t Pa = (int64_t)ra.width * ra.height;
    const int64_t Pb = (int64_t)rb.width * rb.height;
    if (rows == NULL) nrows = Pa;
    for (int64_t r = 0; r < nrows; r++) {
        const int64_t p = rows ? rows[r] : r;
        if (p < 0 || p >= Pa) return -2;
    }
    uint8_t *A = (uint8_t *)malloc((size_t)(n > 0 ? n : 1) * (size_t)(nrows > 0 ? nrows : 1));
    uint8_t *B = (uint8_t *)malloc((size_t)(n > 0 ? n : 1) * (size_t)Pb);
    if (!A || !B) { free(A); free(B); return -3; }
    /* A^i for the selected pixels only; B^i for every B pixel */
    for (int64_t i = 0; i < n; i++) {
        for (int64_t r = 0; r < nrows; r++) {
            const int64_t p = rows ? rows[r] : r;
            const int j = (int)(p % ra.width), m = (int)(p / ra.width);
            A[i * nrows + r] = (uint8_t)pixel_bit(frames, i, W, H, msb, ra.x0 + j, ra.y0 + m);
        }
        for (int k = 0; k < rb.height; k++)
            for (int u = 0; u < rb.width; u++)
                B[i * Pb + (int64_t)k * rb.width + u] =
                    (uint8_t)pixel_bit(frames, i, W, H, msb, rb.x0 + u, rb.y0 + k);
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t r = 0; r < nrows; r++) {
        int64_t *out = s_ab + r * Pb;
        for (int64_t q = 0; q < Pb; q++) out[q] = 0;
        for (int64_t i = 0; i < n; i++) {
            const int64_t a = A[i * nrows + r];
            const uint8_t *b = B + i * Pb;
            for (int64_t q = 0; q < Pb; q++) out[q] += a * (int64_t)b[q];
        }
    }
    free(A);
    free(B);
    (void)nthreads;
    return 0;
}

/* Gamma of Eq. (1) as the exact rational
 *   Gamma = (1/N) S_ab - (S_a/N)(S_b/N) = (N*S_ab - S_a*S_b) / N^2 :
 * the numerator in int64 (|.| <= N^2 < 2^53 for N < 9.4e7), converted to fp64 exactly,
 * divided once by N^2 (exact in fp64) -> correctly rounded fp64 value of the rational.
 * s_a_rows[r] is S_a of the A pixel of row r. */
int oracle_gamma(const int64_t *s_ab, const int64_t *s_a_rows, const int64_t *s_b, int64_t n,
                 int64_t nrows, int64_t Pb, double *out) {
    if (n <= 0) return -1;
    const double n2 = (double)n * (double)n;
    for (int64_t r = 0; r < nrows; r++)
        for (int64_t q = 0; q < Pb; q++) {
            const int64_t num = n * s_ab[r * Pb + q] - s_a_rows[r] * s_b[q];
            out[r * Pb + q] = (double)num / n2;
        }
    return 0;
}

/* SPEC's finalize expression: counts*inv - (ma*inv)*(mb*inv), inv = 1/N once.
 * Kept only so tests can bound its distance from the exact rational. */
int oracle_gamma_spec(const int64_t *s_ab, const int64_t *s_a_rows, const int64_t *s_b,
                      int64_t n, int64_t nrows, int64_t Pb, double *out) {
    if (n <= 0) return -1;
    const double inv = 1.0 / (double)n;
    for (int64_t r = 0; r < nrows; r++)
        for (int64_t q = 0; q < Pb; q++)
            out[r * Pb + q] = (double)s_ab[r * Pb + q] * inv -
                              ((double)s_a_rows[r] * inv) * ((double)s_b[q] * inv);
    return 0;
}

/* ---------------------------------------------------------------- refocusing ---- */

/* Per-axis interpolation support, SURVEY §8(c) c2 / Q14 reading:
 *   i0 = min(floor(c), W-2)  (0 when W == 1),  t = c - i0
 * so integer coordinates give weights exactly 0/1 and the last lattice point uses
 * (i0 = W-2, t = 1). */
static inline void axis_support(double c, int W, int *i0, double *t) {
    int k;
    if (W == 1) {
        k = 0;
    } else {
        k = (int)floor(c);
        if (k > W - 2) k = W - 2;
        if (k < 0) k = 0;
    }
    *i0 = k;
    *t = c - (double)k;
}

/* Gamma value at integer 4D lattice point (j, k, m, n) = (x_a, x_b, y_a, y_b):
 * Gamma[(m*Wa + j)][(n*Wb + k)]  (SURVEY §8(b) "Gamma layout exported", Q1). */
static inline double gamma_at(const void *g, int g_f32, int64_t Pb, int Wa, int Wb, int j,
                              int k, int m, int n) {
    const int64_t idx = ((int64_t)m * Wa + j) * Pb + (int64_t)n * Wb + k;
    return g_f32 ? (double)((const float *)g)[idx] : ((const double *)g)[idx];
}

/* interp4: 4D multilinear interpolation of Gamma at real coordinates
 * (cAx, cBx, cAy, cBy) = 16 lattice corners weighted by the product of per-axis weights
 * (1 - t) or t.  Corners with zero weight are still visited (0 * finite = 0). */
double oracle_interp4(const void *g, int g_f32, int Wa, int Ha, int Wb, int Hb, double cAx,
                      double cBx, double cAy, double cBy) {
    const int64_t Pb = (int64_t)Wb * Hb;
    int j0, k0, m0, n0;
    double tj, tk, tm, tn;
    axis_support(cAx, Wa, &j0, &tj);
    axis_support(cBx, Wb, &k0, &tk);
    axis_support(cAy, Ha, &m0, &tm);
    axis_support(cBy, Hb, &n0, &tn);
    double acc = 0.0;
    for (int dj = 0; dj < 2; dj++) {
        const double wj = dj ? tj : 1.0 - tj;
        const int j = (Wa == 1) ? j0 : j0 + dj;
        for (int dk = 0; dk < 2; dk++) {
            const double wk = dk ? tk : 1.0 - tk;
            const int k = (Wb == 1) ? k0 : k0 + dk;
            for (int dm = 0; dm < 2; dm++) {
                const double wm = dm ? tm : 1.0 - tm;
                const int m = (Ha == 1) ? m0 : m0 + dm;
                for (int dn = 0; dn < 2; dn++) {
                    const double wn = dn ? tn : 1.0 - tn;
                    const int n = (Hb == 1) ? n0 : n0 + dn;
                    const double w = ((wj * wk) * wm) * wn;
                    acc = acc + w * gamma_at(g, g_f32, Pb, Wa, Wb, j, k, m, n);
                }
            }
        }
    }
    return acc;
}

/* One refocused pixel (x, y) of plane alpha:
 *   default map, coordinates relative to the arm centres c = (W-1)/2, (H-1)/2:
 *     c_Ax = alpha*(x - c_ax) + (1 - alpha)*(u - c_bx) + c_ax,   c_Bx = u
 *     c_Ay = alpha*(y - c_ay) + (1 - alpha)*(v - c_by) + c_ay,   c_By = v
 *   boundary 0 (skip_and_renormalize): a sample counts only if 0 <= c_A <= W-1 on both
 *   axes (closed interval); output = sum / count, 0 if count == 0.
 *   boundary 1 (clamp): c_A clamped into [0, W-1]; every sample counts.
 * Summation in (v, u) raster order. */
static double refocus_pixel(const void *g, int g_f32, int Wa, int Ha, int Wb, int Hb,
                            double alpha, int boundary, int x, int y, int64_t *count_out) {
    const double cax = (Wa - 1) / 2.0, cay = (Ha - 1) / 2.0;
    const double cbx = (Wb - 1) / 2.0, cby = (Hb - 1) / 2.0;
    double sum = 0.0;
    int64_t cnt = 0;
    for (int v = 0; v < Hb; v++) {
        double cy = (alpha * ((double)y - cay)) + ((1.0 - alpha) * ((double)v - cby)) + cay;
        for (int u = 0; u < Wb; u++) {
            double cx = (alpha * ((double)x - cax)) + ((1.0 - alpha) * ((double)u - cbx)) + cax;
            double cyy = cy;
            if (boundary == 0) {
                if (!(cx >= 0.0 && cx <= (double)(Wa - 1))) continue;
                if (!(cyy >= 0.0 && cyy <= (double)(Ha - 1))) continue;
            } else {
                cx = fmin(fmax(cx, 0.0), (double)(Wa - 1));
                cyy = fmin(fmax(cyy, 0.0), (double)(Ha - 1));
            }
            sum = sum + oracle_interp4(g, g_f32, Wa, Ha, Wb, Hb, cx, (double)u, cyy, (double)v);
            cnt++;
        }
    }
    if (count_out) *count_out = cnt;
    return cnt ? sum / (double)cnt : 0.0;
}

/* Refocus a stack: out[p][k] = refocused value of plane alphas[p] at output pixel k,
 * where the pixels are pix[k] = (x, y) pairs (pix == NULL: every pixel of the A lattice
 * in row-major order, k = y*Wa + x).  counts (optional) receives the sample counts.
 * Gamma is fp32 (g_f32 = 1, widened exactly) or fp64, layout [Pa][Pb]. */
int oracle_refocus(const void *g, int g_f32, int Wa, int Ha, int Wb, int Hb,
                   const double *alphas, int n_planes, int boundary, const int32_t *pix,
                   int64_t npix, double *out, int64_t *counts, int nthreads) {
    if (Wa < 1 || Ha < 1 || Wb < 1 || Hb < 1 || n_planes < 0) return -1;
    for (int p = 0; p < n_planes; p++)
        if (!(alphas[p] != 0.0) || !isfinite(alphas[p])) return -2;
    if (pix == NULL) npix = (int64_t)Wa * Ha;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
#endif
    for (int p = 0; p < n_planes; p++)
        for (int64_t k = 0; k < npix; k++) {
            const int x = pix ? pix[2 * k] : (int)(k % Wa);
            const int y = pix ? pix[2 * k + 1] : (int)(k / Wa);
            int64_t c = 0;
            out[(int64_t)p * npix + k] =
                refocus_pixel(g, g_f32, Wa, Ha, Wb, Hb, alphas[p], boundary, x, y, &c);
            if (counts) counts[(int64_t)p * npix + k] = c;
        }
    (void)nthreads;
    return 0;
}

/* General RefocusMap: four affine coordinate functions per plane, each of the form
 * a*x + b*u + c on the x axis (a*y + b*v + c on the y axis), with coordinates relative to the
 * arm centres ("coordinates relative to centers"):
 *   c_Ax = ((ax*(x - c_ax)) + (bx*(u - c_bx))) + cx  + c_ax
 *   c_Bx = ((dx*(x - c_ax)) + (ex*(u - c_bx))) + fx  + c_bx
 *   c_Ay = ((ay*(y - c_ay)) + (by*(v - c_by))) + cy  + c_ay
 *   c_By = ((dy*(y - c_ay)) + (ey*(v - c_by))) + fy  + c_by
 * map[12] = {ax, bx, cx, dx, ex, fx, ay, by, cy, dy, ey, fy}.  The default map is
 * {a, 1 - a, 0, 0, 1, 0} on both axes (same values as refocus_pixel: adding +0.0 and
 * c_B = u exactly).  boundary 0: a sample counts only if all four coordinates lie in their
 * closed lattice intervals; boundary 1: each coordinate is clamped.  The sample value is
 * interp4 (16 corners); output = sum / count (0 if no sample). */
static double refocus_pixel_affine(const void *g, int g_f32, int Wa, int Ha, int Wb, int Hb,
                                   const double *mp, int boundary, int x, int y, int64_t *count_out) {
    const double cax = (Wa - 1) / 2.0, cay = (Ha - 1) / 2.0;
    const double cbx = (Wb - 1) / 2.0, cby = (Hb - 1) / 2.0;
    const double xr = (double)x - cax, yr = (double)y - cay;
    double sum = 0.0;
    int64_t cnt = 0;
    for (int v = 0; v < Hb; v++) {
        const double vr = (double)v - cby;
        double cAy = (((mp[6] * yr) + (mp[7] * vr)) + mp[8]) + cay;
        double cBy = (((mp[9] * yr) + (mp[10] * vr)) + mp[11]) + cby;
        for (int u = 0; u < Wb; u++) {
            const double ur = (double)u - cbx;
            double cAx = (((mp[0] * xr) + (mp[1] * ur)) + mp[2]) + cax;
            double cBx = (((mp[3] * xr) + (mp[4] * ur)) + mp[5]) + cbx;
            double ay = cAy, by = cBy;
            if (boundary == 0) {
                if (!(cAx >= 0.0 && cAx <= (double)(Wa - 1))) continue;
                if (!(cBx >= 0.0 && cBx <= (double)(Wb - 1))) continue;
                if (!(ay >= 0.0 && ay <= (double)(Ha - 1))) continue;
                if (!(by >= 0.0 && by <= (double)(Hb - 1))) continue;
            } else {
                cAx = fmin(fmax(cAx, 0.0), (double)(Wa - 1));
                cBx = fmin(fmax(cBx, 0.0), (double)(Wb - 1));
                ay = fmin(fmax(ay, 0.0), (double)(Ha - 1));
                by = fmin(fmax(by, 0.0), (double)(Hb - 1));
            }
            sum = sum + oracle_interp4(g, g_f32, Wa, Ha, Wb, Hb, cAx, cBx, ay, by);
            cnt++;
        }
    }
    if (count_out) *count_out = cnt;
    return cnt ? sum / (double)cnt : 0.0;
}

/* Refocus a stack under general maps: maps[12 * p .. 12 * p + 11] for plane p (layout of
 * refocus_pixel_affine); other arguments as oracle_refocus.  Non-finite coefficient -> -2. */
int oracle_refocus_affine(const void *g, int g_f32, int Wa, int Ha, int Wb, int Hb,
                          const double *maps, int n_planes, int boundary, const int32_t *pix,
                          int64_t npix, double *out, int64_t *counts, int nthreads) {
    if (Wa < 1 || Ha < 1 || Wb < 1 || Hb < 1 || n_planes < 0) return -1;
    for (int i = 0; i < 12 * n_planes; i++)
        if (!isfinite(maps[i])) return -2;
    if (pix == NULL) npix = (int64_t)Wa * Ha;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
#endif
    for (int p = 0; p < n_planes; p++)
        for (int64_t k = 0; k < npix; k++) {
            const int x = pix ? pix[2 * k] : (int)(k % Wa);
            const int y = pix ? pix[2 * k + 1] : (int)(k / Wa);
            int64_t c = 0;
            out[(int64_t)p * npix + k] =
                refocus_pixel_affine(g, g_f32, Wa, Ha, Wb, Hb, maps + 12 * p, boundary, x, y, &c);
            if (counts) counts[(int64_t)p * npix + k] = c;
        }
    (void)nthreads;
    return 0;
}

int oracle_version(void) { return 2; }
