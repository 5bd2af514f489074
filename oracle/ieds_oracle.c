/*
 * ieds_oracle.c -- plain, slow, obviously-correct CPU oracle of the IEDS surface build.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2112_10591_b200/), and the CUDA
 * path never calls it.
 *
 * Source: Brebion, Moreau, Davoine, "Real-Time Optical Flow for Vehicular Perception
 * with Low- and High-Resolution Event Cameras" (arXiv 2112.10591).  Citations "P:N" are
 * /root/reference/PAPER.md line numbers; "S:N" are SPEC.md lines.  The readings of
 * silent / garbled passages are listed in DESIGN.md ("Readings").
 *
 * Images are byte images, row-major [H][W], value 0 or 1; pixel (x, y) = column x, row y.
 * Squared distances are int64; ORACLE_NO_EDGE (-1) marks "no edge pixel in the frame".
 * Floating point is fp64 throughout.
 *
 * Every function is single-threaded and follows the paper's definition step by step.
 * Parity status: all functions pinned by tests/test_oracle_pins.py (none unpinned).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_NO_EDGE (-1LL)
#define ORACLE_OK 0
#define ORACLE_ERANGE (-2)
#define ORACLE_EINVAL (-1)

/* ---- §III-A Accumulation for edge images -------------------------------
 * "These binary matrices indicate whether or not each pixel produced at least one event
 * during the accumulation time"; polarity is not taken into account, so
 * the oracle takes only the (x, y) coordinates.  Events outside the frame are an error
 * (S:42); they are not written. */
int oracle_accumulate(const uint32_t *xy, int64_t n, int W, int H, uint8_t *E)
{
    int status = ORACLE_OK;
    memset(E, 0, (size_t)W * (size_t)H);
    for (int64_t i = 0; i < n; i++) {
        int x = (int)(xy[i] & 0xFFFFu);
        int y = (int)(xy[i] >> 16);
        if (x >= W || y >= H) {
            status = ORACLE_ERANGE;
            continue;
        }
        E[(size_t)y * W + x] = 1;
    }
    return status;
}

/* count of edge pixels among the 4 direct neighbour pixels of p in img
 * (Alg. 1 line "count of edge pixels among the 4 direct neighbour pixels", P:127;
 *  out-of-frame neighbours count as non-edge: DESIGN.md reading R1) */
static int count4(const uint8_t *img, int W, int H, int x, int y)
{
    int n = 0;
    if (x > 0 && img[(size_t)y * W + (x - 1)]) n++;
    if (x + 1 < W && img[(size_t)y * W + (x + 1)]) n++;
    if (y > 0 && img[(size_t)(y - 1) * W + x]) n++;
    if (y + 1 < H && img[(size_t)(y + 1) * W + x]) n++;
    return n;
}

/* ---- Algorithm 1, Denoising -----------------------------------------------
 *   E_d <- E
 *   foreach pixel p in E: if E[p] is an edge pixel:
 *       n_d <- count of edge pixels among the 4 direct neighbours of p in E
 *       if n_d < N_d: E_d[p] <- not an edge pixel anymore */
void oracle_denoise(const uint8_t *E, int W, int H, int N_d, uint8_t *E_d)
{
    memcpy(E_d, E, (size_t)W * (size_t)H);
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            if (E[(size_t)y * W + x]) {
                int n_d = count4(E, W, H, x, y);
                if (n_d < N_d) E_d[(size_t)y * W + x] = 0;
            }
        }
}

/* ---- Algorithm 2, Filling -------------------------------------------------
 *   E_df <- E_d
 *   foreach pixel p in E_d: if E_d[p] is not an edge pixel:
 *       n_f <- count of edge pixels among the 4 direct neighbours of p in E_d
 *       if n_f >= N_f: E_df[p] <- becomes an edge pixel
 * Run strictly after denoising. */
void oracle_fill(const uint8_t *E_d, int W, int H, int N_f, uint8_t *E_df)
{
    memcpy(E_df, E_d, (size_t)W * (size_t)H);
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            if (!E_d[(size_t)y * W + x]) {
                int n_f = count4(E_d, W, H, x, y);
                if (n_f >= N_f) E_df[(size_t)y * W + x] = 1;
            }
        }
}

/* ---- §III-C exact Euclidean distance transform --------------------------
 * d_Euc(p) = Euclidean distance from p to the closest edge pixel of E_df.
 * The paper uses Coeurjolly et al.'s separable exact EDT.  The oracle uses the
 * textbook separable form of that family:
 *   pass 1 (columns): g(x,y) = min |y - y'| over edge pixels (x, y') of column x;
 *   pass 2 (rows):    D2(x,y) = min_q (x - q)^2 + g(q,y)^2, evaluated with the lower
 *                     envelope of parabolas (Felzenszwalb & Huttenlocher 2012, "Distance
 *                     Transforms of Sampled Functions", Algorithm 1 DT(f)), with the
 *                     parabola intersections in fp64 (exact decisions at these sizes, see
 *                     DESIGN.md) and the envelope evaluation in int64.
 * Columns without an edge pixel have g = +inf and contribute no parabola.  If the whole
 * frame has no edge pixel every D2 is ORACLE_NO_EDGE (reading R5). */
void oracle_edt_separable(const uint8_t *E_df, int W, int H, int64_t *D2)
{
    const int64_t INF = INT64_MAX;
    int64_t *g = (int64_t *)malloc(sizeof(int64_t) * (size_t)W * (size_t)H);
    int any = 0;
    /* pass 1: two sweeps per column */
    for (int x = 0; x < W; x++) {
        int64_t last = -1;
        for (int y = 0; y < H; y++) {
            if (E_df[(size_t)y * W + x]) last = y;
            g[(size_t)y * W + x] = (last < 0) ? INF : (int64_t)y - last;
        }
        last = -1;
        for (int y = H - 1; y >= 0; y--) {
            if (E_df[(size_t)y * W + x]) { last = y; any = 1; }
            if (last >= 0) {
                int64_t d = last - (int64_t)y;
                if (d < g[(size_t)y * W + x]) g[(size_t)y * W + x] = d;
            }
        }
    }
    if (!any) {
        for (size_t i = 0; i < (size_t)W * (size_t)H; i++) D2[i] = ORACLE_NO_EDGE;
        free(g);
        return;
    }
    /* pass 2: FH lower envelope per row over f(q) = g(q,y)^2 */
    int *v = (int *)malloc(sizeof(int) * (size_t)W);
    double *z = (double *)malloc(sizeof(double) * (size_t)(W + 1));
    int64_t *f = (int64_t *)malloc(sizeof(int64_t) * (size_t)W);
    for (int y = 0; y < H; y++) {
        for (int q = 0; q < W; q++) {
            int64_t gq = g[(size_t)y * W + q];
            f[q] = (gq == INF) ? INF : gq * gq;
        }
        int k = -1;
        for (int q = 0; q < W; q++) {
            if (f[q] == INF) continue;
            if (k < 0) {
                k = 0; v[0] = q; z[0] = -HUGE_VAL; z[1] = HUGE_VAL;
                continue;
            }
            double s;
            for (;;) {
                int p = v[k];
                s = ((double)(f[q] + (int64_t)q * q) - (double)(f[p] + (int64_t)p * p)) /
                    (2.0 * (double)q - 2.0 * (double)p);
                if (s <= z[k]) {
                    k--;
                    if (k < 0) break;
                } else
                    break;
            }
            if (k < 0) { /* cannot happen: z[0] = -inf */
                k = 0; v[0] = q; z[0] = -HUGE_VAL; z[1] = HUGE_VAL;
                continue;
            }
            k++;
            v[k] = q;
            z[k] = s;
            z[k + 1] = HUGE_VAL;
        }
        /* every row has a finite parabola because some column has an edge pixel */
        k = 0;
        for (int q = 0; q < W; q++) {
            while (z[k + 1] < (double)q) k++;
            int64_t d = (int64_t)q - v[k];
            D2[(size_t)y * W + q] = d * d + f[v[k]];
        }
    }
    free(v); free(z); free(f); free(g);
}

/* Brute force: D2(p) = min over edge pixels q of |p - q|^2 (definition).
 * O(W*H*K); for tiny frames only. */
void oracle_edt_bruteforce(const uint8_t *E_df, int W, int H, int64_t *D2)
{
    int64_t nset = 0;
    for (size_t i = 0; i < (size_t)W * (size_t)H; i++) nset += E_df[i] != 0;
    int *ex = (int *)malloc(sizeof(int) * (size_t)(nset + 1));
    int *ey = (int *)malloc(sizeof(int) * (size_t)(nset + 1));
    int64_t m = 0;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            if (E_df[(size_t)y * W + x]) { ex[m] = x; ey[m] = y; m++; }
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            int64_t best = ORACLE_NO_EDGE;
            for (int64_t i = 0; i < m; i++) {
                int64_t dx = x - ex[i], dy = y - ey[i];
                int64_t d = dx * dx + dy * dy;
                if (best < 0 || d < best) best = d;
            }
            D2[(size_t)y * W + x] = best;
        }
    free(ex); free(ey);
}

/* ---- Eq. (1): d_exp = 1 - exp(-d_Euc / alpha) ------------------------------
 * d_Euc = sqrt(D2) in pixels; a frame with no edge pixel is fully saturated (S = 1,
 * reading R5: the limit d_Euc -> inf). */
void oracle_surface(const int64_t *D2, int64_t n, double alpha, double *S)
{
    for (int64_t i = 0; i < n; i++) {
        if (D2[i] == ORACLE_NO_EDGE) {
            S[i] = 1.0;
        } else {
            double d_euc = sqrt((double)D2[i]);
            S[i] = 1.0 - exp(-d_euc / alpha);
        }
    }
}

/* ---- Windowing of the event stream by Delta T (§III-A; row f2) ---------------
 * Events are time-ordered (t in microseconds).  Window k holds the events with
 * floor((t - t0) / dt) == k, i.e. t in [t0 + k dt, t0 + (k+1) dt) (half-open), where t0 is the
 * first event's timestamp (reading R16; empty interior windows are
 * emitted, trailing empty windows are not).  Writes offsets[0..K] (K = number of windows, i.e.
 * floor((t_last - t0)/dt) + 1) and returns K, 0 for no events, or ORACLE_EINVAL if dt <= 0,
 * -3 (ordering error) if t is not non-decreasing, or -4 if more than max_windows windows. */
int64_t oracle_window_offsets(const int64_t *t, int64_t n, int64_t dt, int64_t *offsets, int64_t max_windows)
{
    if (dt <= 0) return ORACLE_EINVAL;
    if (n == 0) { offsets[0] = 0; return 0; }
    for (int64_t i = 1; i < n; i++)
        if (t[i] < t[i - 1]) return -3;
    const int64_t t0 = t[0];
    const int64_t K = (t[n - 1] - t0) / dt + 1;
    if (K > max_windows) return -4;
    int64_t i = 0;
    for (int64_t k = 0; k <= K; k++) {
        /* first event of window k (or n) */
        while (i < n && (t[i] - t0) / dt < k) i++;
        offsets[k] = i;
    }
    return K;
}

/* ---- Ablation transfers of §IV-D (Fig. 4) --------------------------
 *   kind 0: Eq. (1) inverse exponential  1 - exp(-d/alpha)           (proposed)
 *   kind 1: linear distance transform    Id(d) = d                   (Ours_DS_L,  P:306)
 *   kind 2: upper-bounded                min(d, bound), bound = 6 px (Ours_DS_LB)
 *   kind 3: logarithmic                  ln(d + 1)                   (Ours_DS_Log)
 * d = sqrt(D2) in pixels.  An empty frame (D2 = ORACLE_NO_EDGE) is the limit d -> inf:
 * 1 for kind 0, bound for kind 2, +inf for kinds 1 and 3 (reading R14 in DESIGN.md). */
void oracle_transfer(const int64_t *D2, int64_t n, int kind, double alpha, double bound, double *out)
{
    for (int64_t i = 0; i < n; i++) {
        if (D2[i] == ORACLE_NO_EDGE) {
            out[i] = (kind == 0) ? 1.0 : (kind == 2) ? bound : HUGE_VAL;
            continue;
        }
        double d = sqrt((double)D2[i]);
        switch (kind) {
            case 0: out[i] = 1.0 - exp(-d / alpha); break;
            case 1: out[i] = d; break;
            case 2: out[i] = d < bound ? d : bound; break;
            default: out[i] = log(d + 1.0); break;
        }
    }
}

/* ---- 8-bit coding of the surface ("coded on 8 bits (values ranging from 0 to 1 are
 * represented by values between 0 and 255)"): q = round(255 * d_exp), half away from zero
 * (d_exp >= 0, so floor(255 * d_exp + 0.5)); reading R15. */
void oracle_quantize_u8(const double *S, int64_t n, uint8_t *q)
{
    for (int64_t i = 0; i < n; i++) {
        double v = floor(255.0 * S[i] + 0.5);
        if (v < 0.0) v = 0.0;
        if (v > 255.0) v = 255.0;
        q[i] = (uint8_t)v;
    }
}

/* ---- 8-bit view of an ablation transfer, normalised by its frame maximum (row f1):
 * SPEC S:254 "linear/log variants are first normalized by their frame maximum before
 * quantization" and S:271 (the paper is silent; reading R17).  For one frame of n pixels:
 *     v(p) = transfer(D2(p))  (kind 1 Id, 2 min(d, bound), 3 ln(d + 1); as oracle_transfer)
 *     q(p) = round(255 * v(p) / max_p v(p)), half away from zero, clamped to [0, 255].
 * Empty frame (every D2 is NO_EDGE): q = 255 everywhere (the saturated state).
 * max_p v = 0 (every pixel is an edge pixel): q = 0 everywhere (reading R17).
 * Returns 0, or -1 for kind 0 (Eq. (1) is coded without normalisation, oracle_quantize_u8). */
int oracle_quantize_norm_u8(const int64_t *D2, int64_t n, int kind, double bound, uint8_t *q)
{
    if (kind < 1 || kind > 3) return -1;
    if (n > 0 && D2[0] == ORACLE_NO_EDGE) {
        for (int64_t i = 0; i < n; i++) q[i] = 255;
        return 0;
    }
    double *v = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!v) return -2;
    oracle_transfer(D2, n, kind, 1.0, bound, v);
    double vmax = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (v[i] > vmax) vmax = v[i];
    for (int64_t i = 0; i < n; i++) {
        double t = vmax > 0.0 ? floor(255.0 * (v[i] / vmax) + 0.5) : 0.0;
        if (t < 0.0) t = 0.0;
        if (t > 255.0) t = 255.0;
        q[i] = (uint8_t)t;
    }
    free(v);
    return 0;
}

/* ---- Eq. (2)-(3): alpha = -d_sat / ln(eps), eps = 1/255 --------------------
 * The paper prints alpha ~ d_sat / 5.541, i.e. ln 255 = 5.5413; the oracle keeps
 * the full-precision ln (reading R6).  d_sat <= 0 (or NaN) returns NaN. */
double oracle_alpha_from_dsat(double d_sat)
{
    const double eps = 1.0 / 255.0;
    if (!(d_sat > 0.0)) return NAN;
    return -d_sat / log(eps);
}

/* Composition of the whole path for one window, in the paper's order (Fig. 1):
 * accumulate -> denoise (Alg. 1) -> fill (Alg. 2) -> EDT -> Eq. (1).
 * Any of E, E_d, E_df, D2 may be NULL (scratch is allocated); S may be NULL. */
int oracle_build_window(const uint32_t *xy, int64_t n, int W, int H, int N_d, int N_f,
                        double alpha, uint8_t *E, uint8_t *E_d, uint8_t *E_df, int64_t *D2,
                        double *S)
{
    if (W <= 0 || H <= 0 || N_d < 0 || N_d > 4 || N_f < 1 || N_f > 5 || !(alpha > 0.0))
        return ORACLE_EINVAL;
    size_t npx = (size_t)W * (size_t)H;
    uint8_t *e = E ? E : (uint8_t *)malloc(npx);
    uint8_t *ed = E_d ? E_d : (uint8_t *)malloc(npx);
    uint8_t *edf = E_df ? E_df : (uint8_t *)malloc(npx);
    int64_t *d2 = D2 ? D2 : (int64_t *)malloc(sizeof(int64_t) * npx);
    int st = oracle_accumulate(xy, n, W, H, e);
    oracle_denoise(e, W, H, N_d, ed);
    oracle_fill(ed, W, H, N_f, edf);
    oracle_edt_separable(edf, W, H, d2);
    if (S) oracle_surface(d2, (int64_t)npx, alpha, S);
    if (!E) free(e);
    if (!E_d) free(ed);
    if (!E_df) free(edf);
    if (!D2) free(d2);
    return st;
}

/* ==== Row f3: flow-compensated event image and the Flow Warping Loss ======================
 * PAPER P:293-297 (FWL of Stoffregen et al.): "compensate and accumulate each raw event
 * (considering its polarity and timestamp) by its computed optical flow, in order to recreate
 * an image of compensated events at a reference time t", FWL = sigma^2(I_comp) /
 * sigma^2(I_uncomp), sigma^2 = the image variance.  SPEC S:393-411 fixes the rest:
 *   - event (t, x, y, p) carries signed mass +1 (p > 0) or -1 (reading R19: p <= 0 is -1);
 *   - it is splatted bilinearly at (x, y) + F(x, y) * (t_ref - t) / dt;
 *   - events landing outside the frame are dropped: reading R19, the warped position
 *     must lie in [0, W-1] x [0, H-1], so every bilinear corner that receives a non-zero weight
 *     is a frame pixel;
 *   - I_uncomp is the same accumulation with zero flow (the plain signed event image);
 *   - sigma^2 is the population variance over all W*H pixels, two-pass.
 * F is a dense float32 field [H][W][2] = (dx, dy) in pixels per dt (reading R20).  The warp
 * arithmetic is fp64 in this order: tau = (t_ref - t) / dt; xw = x + Fx * tau; yw = y + Fy * tau;
 * x0 = floor(xw), fx = xw - x0 (same for y); weights (1-fx)(1-fy), fx(1-fy), (1-fx)fy, fx fy.
 * out3 = {var(I_comp), var(I_uncomp), FWL}; FWL is NaN when var(I_uncomp) = 0.
 * I_comp / I_uncomp may be NULL.  Returns ORACLE_OK, or ORACLE_ERANGE if an event lies
 * outside the frame (it is dropped, as in oracle_accumulate) / ORACLE_EINVAL. */
int oracle_fwl(const uint32_t *xy, const int64_t *t, const int8_t *p, int64_t n, int W, int H,
               const float *flow, int64_t t_ref, int64_t dt, double *I_comp, double *I_uncomp,
               double *out3)
{
    if (W <= 0 || H <= 0 || dt <= 0) return ORACLE_EINVAL;
    size_t npx = (size_t)W * (size_t)H;
    double *ic = I_comp ? I_comp : (double *)malloc(sizeof(double) * npx);
    double *iu = I_uncomp ? I_uncomp : (double *)malloc(sizeof(double) * npx);
    if (!ic || !iu) return ORACLE_EINVAL;
    for (size_t i = 0; i < npx; i++) ic[i] = iu[i] = 0.0;
    int st = ORACLE_OK;
    for (int64_t e = 0; e < n; e++) {
        int x = (int)(xy[e] & 0xFFFFu), y = (int)(xy[e] >> 16);
        if (x >= W || y >= H) {
            st = ORACLE_ERANGE;
            continue;
        }
        double s = p[e] > 0 ? 1.0 : -1.0;
        iu[(size_t)y * W + x] += s;
        double tau = (double)(t_ref - t[e]) / (double)dt;
        double fxv = (double)flow[((size_t)y * W + x) * 2 + 0];
        double fyv = (double)flow[((size_t)y * W + x) * 2 + 1];
        double xw = (double)x + fxv * tau;
        double yw = (double)y + fyv * tau;
        if (!(xw >= 0.0 && xw <= (double)(W - 1) && yw >= 0.0 && yw <= (double)(H - 1))) continue;
        double x0 = floor(xw), y0 = floor(yw);
        double fx = xw - x0, fy = yw - y0;
        double ax = 1.0 - fx, ay = 1.0 - fy;
        int ix = (int)x0, iy = (int)y0;
        ic[(size_t)iy * W + ix] += s * (ax * ay);
        if (ix + 1 < W) ic[(size_t)iy * W + ix + 1] += s * (fx * ay);
        if (iy + 1 < H) ic[(size_t)(iy + 1) * W + ix] += s * (ax * fy);
        if (ix + 1 < W && iy + 1 < H) ic[(size_t)(iy + 1) * W + ix + 1] += s * (fx * fy);
    }
    double mc = 0.0, mu = 0.0;
    for (size_t i = 0; i < npx; i++) {
        mc += ic[i];
        mu += iu[i];
    }
    mc /= (double)npx;
    mu /= (double)npx;
    double vc = 0.0, vu = 0.0;
    for (size_t i = 0; i < npx; i++) {
        vc += (ic[i] - mc) * (ic[i] - mc);
        vu += (iu[i] - mu) * (iu[i] - mu);
    }
    vc /= (double)npx;
    vu /= (double)npx;
    out3[0] = vc;
    out3[1] = vu;
    out3[2] = vu > 0.0 ? vc / vu : NAN;
    if (!I_comp) free(ic);
    if (!I_uncomp) free(iu);
    return st;
}

/* ==== Row f4: the flow consumer and the edge masking ===========================
 * The paper feeds the surfaces to a third-party pyramidal update-prediction optical flow
 * (Adarve et al.; it "predicts optical flow using an image warping process, and
 * temporally propagates the optical flow estimations using an incremental framework.
 * Multiple update-prediction loops are stacked as a pyramidal structure") whose equations the
 * paper does not give, then restricts the dense flow "to the edge pixels of the denoised edge
 * image".  The estimator below follows SPEC's declared substitute (pyramid,
 * warping prediction, incremental regularised brightness-constancy update with per-level
 * weights and sweeps, temporal propagation with decay gamma), every open choice fixed as
 * DESIGN reading R21:
 *   images    J = scale * S (scale = 255: the regularisation weights of P:260 are for 8-bit
 *             image values), fp64 here;
 *   pyramid   level l+1 = 2x2 mean of level l, size (W_l / 2, H_l / 2) (floor);
 *   predict   Pt_l(p) = P_l(p - P_l(p)): the previous window's flow at level l transported by
 *             itself (bilinear, border-clamped) -- the "image warping" prediction;
 *   init      coarsest level: Pt_{L-1}; finer levels: upsample(F_{l+1}) -- the bilinear
 *             sample of F_{l+1} at ((x+0.5)/2 - 0.5, (y+0.5)/2 - 0.5), clamped, times 2;
 *   warp      J1(p) = J_prev sampled at p - init(p) (SPEC's warp_image, of -init: a
 *             point at p in the previous window is at p + F in the current one);
 *   gradients central differences of J1, one-sided on the border; It = J_cur - J1;
 *   update    K_l Jacobi sweeps of Horn-Schunck on the total flow w (w^0 = init):
 *             wbar = mean of the 4 neighbours of w (border replicated),
 *             w <- wbar - (Ix, Iy) (Ix (wbar_u - init_u) + Iy (wbar_v - init_v) + It) / (lambda_l + Ix^2 + Iy^2)
 *             (w = wbar where the denominator is 0); F_meas,l = w^K;
 *   filter    F_l = (1 - gamma) F_meas,l + gamma Pt_l  (temporal smoothing);
 *   state     P_l = F_l for every level; the current pyramid becomes the previous one;
 *   output    F_0 (pixels per window); the first window of a sequence gives zero flow.
 *   masking   valid(p) = E_d(p); flow outside the mask is reported as 0. */

static double bl_sample(const double *I, int W, int H, double sx, double sy)
{
    if (sx < 0.0) sx = 0.0;
    if (sx > (double)(W - 1)) sx = (double)(W - 1);
    if (sy < 0.0) sy = 0.0;
    if (sy > (double)(H - 1)) sy = (double)(H - 1);
    int x0 = (int)floor(sx), y0 = (int)floor(sy);
    double fx = sx - x0, fy = sy - y0;
    int x1 = x0 + 1 < W ? x0 + 1 : W - 1, y1 = y0 + 1 < H ? y0 + 1 : H - 1;
    return (1.0 - fx) * (1.0 - fy) * I[(size_t)y0 * W + x0] + fx * (1.0 - fy) * I[(size_t)y0 * W + x1] +
           (1.0 - fx) * fy * I[(size_t)y1 * W + x0] + fx * fy * I[(size_t)y1 * W + x1];
}

/* 2x2 mean: out is (W/2) x (H/2) */
void oracle_downsample(const double *I, int W, int H, double *out)
{
    int w = W / 2, h = H / 2;
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            out[(size_t)y * w + x] = (I[(size_t)(2 * y) * W + 2 * x] + I[(size_t)(2 * y) * W + 2 * x + 1] +
                                      I[(size_t)(2 * y + 1) * W + 2 * x] + I[(size_t)(2 * y + 1) * W + 2 * x + 1]) / 4.0;
}

/* flow (u, v interleaved) from a w x h level up to W x H, vectors x2 */
void oracle_upsample_flow(const double *Fc, int w, int h, int W, int H, double *F)
{
    double *cu = (double *)malloc(sizeof(double) * (size_t)w * h * 2);
    double *cv = cu + (size_t)w * h;
    for (size_t i = 0; i < (size_t)w * h; i++) {
        cu[i] = Fc[2 * i];
        cv[i] = Fc[2 * i + 1];
    }
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            double sx = (x + 0.5) / 2.0 - 0.5, sy = (y + 0.5) / 2.0 - 0.5;
            F[2 * ((size_t)y * W + x)] = 2.0 * bl_sample(cu, w, h, sx, sy);
            F[2 * ((size_t)y * W + x) + 1] = 2.0 * bl_sample(cv, w, h, sx, sy);
        }
    free(cu);
}

/* J1(p) = bilinear sample of I at p + F(p), border-clamped */
void oracle_warp(const double *I, int W, int H, const double *F, double *out)
{
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            size_t i = (size_t)y * W + x;
            out[i] = bl_sample(I, W, H, x + F[2 * i], y + F[2 * i + 1]);
        }
}

/* central differences, one-sided on the border (0 along an axis of length 1) */
void oracle_gradients(const double *J, int W, int H, double *Ix, double *Iy)
{
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            size_t i = (size_t)y * W + x;
            if (W == 1) Ix[i] = 0.0;
            else if (x == 0) Ix[i] = J[i + 1] - J[i];
            else if (x == W - 1) Ix[i] = J[i] - J[i - 1];
            else Ix[i] = (J[i + 1] - J[i - 1]) / 2.0;
            if (H == 1) Iy[i] = 0.0;
            else if (y == 0) Iy[i] = J[i + W] - J[i];
            else if (y == H - 1) Iy[i] = J[i] - J[i - W];
            else Iy[i] = (J[i + W] - J[i - W]) / 2.0;
        }
}

/* K Jacobi sweeps of Horn-Schunck on the total flow w (u, v interleaved) from w^0 = init:
 * w <- wbar - grad (grad . (wbar - init) + It) / (lambda + |grad|^2), wbar = 4-neighbour mean
 * (border replicated); w = wbar where the denominator is 0.  init may be NULL (zero). */
void oracle_hs_jacobi(const double *Ix, const double *Iy, const double *It, const double *init, int W, int H,
                      double lambda, int K, double *w)
{
    size_t n = (size_t)W * H;
    double *a = (double *)malloc(sizeof(double) * 2 * n);
    double *b = (double *)malloc(sizeof(double) * 2 * n);
    for (size_t i = 0; i < 2 * n; i++) a[i] = init ? init[i] : 0.0;
    for (int k = 0; k < K; k++) {
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                size_t i = (size_t)y * W + x;
                size_t l = x > 0 ? i - 1 : i, r = x < W - 1 ? i + 1 : i;
                size_t u = y > 0 ? i - W : i, dn = y < H - 1 ? i + W : i;
                double mu = (a[2 * l] + a[2 * r] + a[2 * u] + a[2 * dn]) / 4.0;
                double mv = (a[2 * l + 1] + a[2 * r + 1] + a[2 * u + 1] + a[2 * dn + 1]) / 4.0;
                double den = lambda + Ix[i] * Ix[i] + Iy[i] * Iy[i];
                if (den > 0.0) {
                    double iu = init ? init[2 * i] : 0.0, iv = init ? init[2 * i + 1] : 0.0;
                    double res = Ix[i] * (mu - iu) + Iy[i] * (mv - iv) + It[i];
                    b[2 * i] = mu - Ix[i] * res / den;
                    b[2 * i + 1] = mv - Iy[i] * res / den;
                } else {
                    b[2 * i] = mu;
                    b[2 * i + 1] = mv;
                }
            }
        double *t = a;
        a = b;
        b = t;
    }
    for (size_t i = 0; i < 2 * n; i++) w[i] = a[i];
    free(a);
    free(b);
}

/* Pt(p) = P(p - P(p)) per component (bilinear, border-clamped): the flow transported by itself */
void oracle_advect_flow(const double *P, int W, int H, double *Pt)
{
    size_t n = (size_t)W * H;
    double *c = (double *)malloc(sizeof(double) * 2 * n);
    double *cu = c, *cv = c + n;
    for (size_t i = 0; i < n; i++) {
        cu[i] = P[2 * i];
        cv[i] = P[2 * i + 1];
    }
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            size_t i = (size_t)y * W + x;
            double sx = x - P[2 * i], sy = y - P[2 * i + 1];
            Pt[2 * i] = bl_sample(cu, W, H, sx, sy);
            Pt[2 * i + 1] = bl_sample(cv, W, H, sx, sy);
        }
    free(c);
}

/* level sizes of the pyramid; returns the total pixel count over levels, or -1 if a level
 * would be smaller than 2 x 2 */
int64_t oracle_flow_levels(int W, int H, int L, int *Ws, int *Hs)
{
    int64_t tot = 0;
    for (int l = 0; l < L; l++) {
        Ws[l] = l == 0 ? W : Ws[l - 1] / 2;
        Hs[l] = l == 0 ? H : Hs[l - 1] / 2;
        if (Ws[l] < 2 || Hs[l] < 2) return -1;
        tot += (int64_t)Ws[l] * Hs[l];
    }
    return tot;
}

/* One window of the estimator.  prev_pyr / P are the caller's state (packed levels: level l
 * at offset sum_{k<l} W_k H_k, flow u,v interleaved); fresh = 1 for the first window.
 * On return prev_pyr holds the current pyramid and P the per-level flow; F0 = the level-0 flow. */
int oracle_flow_step(int W, int H, int L, const double *lambda, const int *iters, double gamma, double scale,
                     int fresh, const double *S, double *prev_pyr, double *P, double *F0)
{
    int Ws[16], Hs[16];
    if (L < 1 || L > 16) return ORACLE_EINVAL;
    int64_t tot = oracle_flow_levels(W, H, L, Ws, Hs);
    if (tot < 0) return ORACLE_EINVAL;
    size_t off[16];
    off[0] = 0;
    for (int l = 1; l < L; l++) off[l] = off[l - 1] + (size_t)Ws[l - 1] * Hs[l - 1];
    double *cur = (double *)malloc(sizeof(double) * (size_t)tot);
    for (size_t i = 0; i < (size_t)W * H; i++) cur[i] = scale * S[i];
    for (int l = 1; l < L; l++) oracle_downsample(cur + off[l - 1], Ws[l - 1], Hs[l - 1], cur + off[l]);
    if (fresh) {
        for (size_t i = 0; i < (size_t)tot; i++) {
            prev_pyr[i] = cur[i];
            P[2 * i] = P[2 * i + 1] = 0.0;
        }
        for (size_t i = 0; i < (size_t)W * H * 2; i++) F0[i] = 0.0;
        free(cur);
        return ORACLE_OK;
    }
    double *Fl = (double *)malloc(sizeof(double) * 2 * (size_t)tot);
    size_t n0 = (size_t)W * H;
    double *init = (double *)malloc(sizeof(double) * 2 * n0);
    double *Pt = (double *)malloc(sizeof(double) * 2 * n0);
    double *neg = (double *)malloc(sizeof(double) * 2 * n0);
    double *J1 = (double *)malloc(sizeof(double) * n0);
    double *Ix = (double *)malloc(sizeof(double) * n0);
    double *Iy = (double *)malloc(sizeof(double) * n0);
    double *It = (double *)malloc(sizeof(double) * n0);
    double *w = (double *)malloc(sizeof(double) * 2 * n0);
    for (int l = L - 1; l >= 0; l--) {
        int wl = Ws[l], hl = Hs[l];
        size_t n = (size_t)wl * hl;
        oracle_advect_flow(P + 2 * off[l], wl, hl, Pt);
        if (l == L - 1) {
            for (size_t i = 0; i < 2 * n; i++) init[i] = Pt[i];
        } else {
            oracle_upsample_flow(Fl + 2 * off[l + 1], Ws[l + 1], Hs[l + 1], wl, hl, init);
        }
        for (size_t i = 0; i < 2 * n; i++) neg[i] = -init[i];
        oracle_warp(prev_pyr + off[l], wl, hl, neg, J1);
        oracle_gradients(J1, wl, hl, Ix, Iy);
        for (size_t i = 0; i < n; i++) It[i] = cur[off[l] + i] - J1[i];
        oracle_hs_jacobi(Ix, Iy, It, init, wl, hl, lambda[l], iters[l], w);
        for (size_t i = 0; i < 2 * n; i++) Fl[2 * off[l] + i] = (1.0 - gamma) * w[i] + gamma * Pt[i];
    }
    for (size_t i = 0; i < (size_t)tot; i++) {
        prev_pyr[i] = cur[i];
        P[2 * i] = Fl[2 * i];
        P[2 * i + 1] = Fl[2 * i + 1];
    }
    for (size_t i = 0; i < 2 * n0; i++) F0[i] = Fl[i];
    free(cur);
    free(Fl);
    free(init);
    free(Pt);
    free(neg);
    free(J1);
    free(Ix);
    free(Iy);
    free(It);
    free(w);
    return ORACLE_OK;
}

/* P:248 edge masking: valid = E_d (0/1 bytes); flow outside the mask is set to 0 */
void oracle_mask_flow(const double *F, const uint8_t *E_d, int64_t n, double *out, uint8_t *valid)
{
    for (int64_t i = 0; i < n; i++) {
        valid[i] = E_d[i] ? 1 : 0;
        out[2 * i] = E_d[i] ? F[2 * i] : 0.0;
        out[2 * i + 1] = E_d[i] ? F[2 * i + 1] : 0.0;
    }
}
