/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, called by, or shipped
 * with the product library (paper_1512_06235_b200/libmsfm_b200.so).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 *
 * Plain-C restatement of the reference's geometry-aware pair matcher,
 * msfm.guided.guided_match_pair(strategy="grid") (pkg/src/msfm/guided.py:393-480)
 * and its helpers, written against the exact IEEE operation order the
 * reference executes under numpy 2.3 / OpenBLAS 0.3.30 / glibc 2.39:
 *
 *   - query epipolar lines  `hom @ F.T`            guided.py:354-355, 443-444
 *       n >= 2 rows (dgemm):  l_i = fl( fma(y, F_i1, fl(x*F_i0)) + F_i2 )
 *       n == 1 row  (dgemv):  l_i = fl( fma(x, F_i0, fl(y*F_i1)) + F_i2 )
 *   - line norm `np.hypot`                           guided.py:356, 445
 *       = glibc's non-FMA Borges kernel (hypot_ref below; verified bit-equal
 *         on 5M random pairs)
 *   - band value `ml[:, :2] @ txy.T + ml[:, 2]`      guided.py:447
 *       m >= 2 members (dgemm):  fl( fma(b, y, fl(a*x)) ) + c
 *       m == 1, or |C'| == 1 with m >= 3 (dgemv):  fl( fma(a, x, fl(b*y)) ) + c
 *   - descriptor distances are exact integers (f32 partials < 2^24),
 *     guided.py:455-457, so they are computed in int32 here
 *   - ratio test in float32 (NEP 50: f32 scalar vs python float),
 *     matching.py:82-103;  target dedupe on (f32 dist, row), matching.py:106-113
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; contraction would change
 * the rounding of the non-fused products above).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* glibc 2.35+ __hypot, non-FMA kernel (sysdeps/ieee754/dbl-64/e_hypot.c),
 * which is what np.hypot resolves to on x86-64. */
static double hyp_kernel(double ax, double ay) {
    double t1, t2;
    double h = sqrt(ax * ax + ay * ay);
    if (h <= 2.0 * ay) {
        double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

double oracle_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return x + y;
    }
    x = fabs(x); y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= ax * 0x1p-54) return ax + ay;
        return hyp_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
    }
    if (ay < 0x1p-511) {
        if (ax >= ay / 0x1p-54) return ax + ay;
        return hyp_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
    }
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hyp_kernel(ax, ay);
}

/* ---------------------------------------------------------------- grid --- */
/* OverlapGrid/build_grid guided.py:46-137: 4 offset grids, cell 2D, offsets
 * (0,0),(D,0),(0,D),(D,D); key = (cx+2^20)*2^21 + (cy+2^20) + g*2^44. */
typedef struct { int64_t key; int32_t fid; } kf_t;

static int cmp_kf(const void* a, const void* b) {
    const kf_t* x = a; const kf_t* y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->fid - y->fid;
}

static const double OFF[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};

static inline int64_t cell_key(double x, double y, int g, double D) {
    int64_t cx = (int64_t)floor((x - OFF[g][0] * D) / (2.0 * D));
    int64_t cy = (int64_t)floor((y - OFF[g][1] * D) / (2.0 * D));
    return (cx + (1LL << 20)) * (1LL << 21) + (cy + (1LL << 20)) + (int64_t)g * (1LL << 44);
}

typedef struct { kf_t* e; int n; } grid_t;

static void grid_build(grid_t* G, const float* txy, int nt, double D) {
    G->n = 4 * nt;
    G->e = (kf_t*)malloc(sizeof(kf_t) * (size_t)(G->n > 0 ? G->n : 1));
    for (int f = 0; f < nt; f++)
        for (int g = 0; g < 4; g++) {
            G->e[4 * f + g].key = cell_key((double)txy[2 * f], (double)txy[2 * f + 1], g, D);
            G->e[4 * f + g].fid = f;
        }
    qsort(G->e, (size_t)G->n, sizeof(kf_t), cmp_kf);
}

static int lower_bound(const kf_t* e, int n, int64_t key) {
    int lo = 0, hi = n;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (e[mid].key < key) lo = mid + 1; else hi = mid; }
    return lo;
}

/* ------------------------------------------------------------ clipping --- */
/* clip_line_to_bounds guided.py:140-170 (scalar, used with pad=d for samples) */
static int clip_scalar(double a, double b, double c, double W, double H, double pad,
                       double pa[2], double pb[2]) {
    double x0 = -pad, x1 = W + pad, y0 = -pad, y1 = H + pad;
    double pts[4][2]; int np_ = 0;
    if (fabs(b) > 1e-15) {
        double xs[2] = {x0, x1};
        for (int k = 0; k < 2; k++) {
            double y = -(a * xs[k] + c) / b;
            if (y0 - 1e-9 <= y && y <= y1 + 1e-9) {
                double yy = y < y0 ? y0 : y;           /* max(y, y0) */
                yy = yy > y1 ? y1 : yy;                /* min(., y1) */
                pts[np_][0] = xs[k]; pts[np_][1] = yy; np_++;
            }
        }
    }
    if (fabs(a) > 1e-15) {
        double ys[2] = {y0, y1};
        for (int k = 0; k < 2; k++) {
            double x = -(b * ys[k] + c) / a;
            if (x0 - 1e-9 <= x && x <= x1 + 1e-9) {
                double xx = x < x0 ? x0 : x;
                xx = xx > x1 ? x1 : xx;
                pts[np_][0] = xx; pts[np_][1] = ys[k]; np_++;
            }
        }
    }
    if (np_ < 2) return 0;
    /* sorted(set(pts)): lexicographic min and max of the distinct points */
    int imin = 0, imax = 0;
    for (int k = 1; k < np_; k++) {
        if (pts[k][0] < pts[imin][0] || (pts[k][0] == pts[imin][0] && pts[k][1] < pts[imin][1])) imin = k;
        if (pts[k][0] > pts[imax][0] || (pts[k][0] == pts[imax][0] && pts[k][1] > pts[imax][1])) imax = k;
    }
    pa[0] = pts[imin][0]; pa[1] = pts[imin][1];
    pb[0] = pts[imax][0]; pb[1] = pts[imax][1];
    if (oracle_hypot(pb[0] - pa[0], pb[1] - pa[1]) < 1e-12) return 0;
    return 1;
}

/* clip_lines_batch guided.py:297-338 (pad 0, argmin/argmax of x*4*span + y) */
static int clip_batch(double a, double b, double c, double W, double H, double pa[2], double pb[2]) {
    const double x0 = -0.0, x1 = W, y0 = -0.0, y1 = H;
    double cand[4][2]; int valid[4] = {0, 0, 0, 0};
    double xs[2] = {x0, x1}, ys[2] = {y0, y1};
    for (int k = 0; k < 2; k++) {
        double y = -(a * xs[k] + c) / b;
        if (fabs(b) > 1e-15 && y >= y0 - 1e-9 && y <= y1 + 1e-9) {
            valid[k] = 1; cand[k][0] = xs[k];
            cand[k][1] = y < y0 ? y0 : (y > y1 ? y1 : y);   /* np.clip */
        }
    }
    for (int k = 0; k < 2; k++) {
        double x = -(b * ys[k] + c) / a;
        if (fabs(a) > 1e-15 && x >= x0 - 1e-9 && x <= x1 + 1e-9) {
            valid[k + 2] = 1; cand[k + 2][0] = x < x0 ? x0 : (x > x1 ? x1 : x);
            cand[k + 2][1] = ys[k];
        }
    }
    double span = x1 - x0; if (y1 - y0 > span) span = y1 - y0; if (span < 1.0) span = 1.0;
    int any = 0, imin = 0, imax = 0; double kmin = INFINITY, kmax = -INFINITY;
    for (int k = 0; k < 4; k++) {
        if (!valid[k]) continue;
        any = 1;
        double key = cand[k][0] * (4.0 * span) + cand[k][1];
        if (key < kmin) { kmin = key; imin = k; }
        if (key > kmax) { kmax = key; imax = k; }
    }
    if (!any) return 0;
    pa[0] = cand[imin][0]; pa[1] = cand[imin][1];
    pb[0] = cand[imax][0]; pb[1] = cand[imax][1];
    return oracle_hypot(pb[0] - pa[0], pb[1] - pa[1]) > 1e-12;
}

static inline void epiline(const double* F, double x, double y, int single_row, double l[3]) {
    for (int i = 0; i < 3; i++) {
        if (single_row) l[i] = fma(x, F[3 * i], y * F[3 * i + 1]) + F[3 * i + 2];
        else            l[i] = fma(y, F[3 * i + 1], x * F[3 * i]) + F[3 * i + 2];
    }
}

typedef struct { int64_t comp; int32_t q; int32_t row; } qk_t;

static int cmp_qk(const void* a, const void* b) {
    const qk_t* x = a; const qk_t* y = b;
    if (x->comp != y->comp) return x->comp < y->comp ? -1 : 1;
    if (x->q != y->q) return x->q < y->q ? -1 : 1;
    return x->row - y->row;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

typedef struct { int32_t row, tgt; float dist, ratio; } acc_t;

static int cmp64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}


/* Returns the number of matches written (sorted by query id), -1 if cap is
 * too small.  stats[0] += queries, stats[1] += comparisons (SearchStats). */
int oracle_guided_match(const float* qxy, const uint8_t* qdesc,
                        const float* txy, const uint8_t* tdesc, int nt,
                        double W, double H, const double* F,
                        const int32_t* qidx, int nqi,
                        double d, double D, float ratio, float single_cap,
                        int32_t* out_q, int32_t* out_t, float* out_dist, float* out_ratio,
                        int cap, int64_t* stats) {
    if (nt == 0 || nqi == 0) return 0;
    grid_t G; grid_build(&G, txy, nt, D);

    /* ---- group_queries guided.py:341-390 ---- */
    double* lines = (double*)malloc(sizeof(double) * 3 * (size_t)nqi);
    qk_t* keys = (qk_t*)malloc(sizeof(qk_t) * (size_t)nqi);
    int nk = 0;
    for (int r = 0; r < nqi; r++) {
        int q = qidx[r];
        double* l = lines + 3 * r;
        epiline(F, (double)qxy[2 * q], (double)qxy[2 * q + 1], nqi == 1, l);
        double nrm = oracle_hypot(l[0], l[1]);
        if (!(nrm > 1e-12)) continue;
        l[0] /= nrm; l[1] /= nrm; l[2] /= nrm;
        double pa[2], pb[2];
        if (!clip_batch(l[0], l[1], l[2], W, H, pa, pb)) continue;
        int64_t c4[4] = {(int64_t)floor(pa[0] / 2.0), (int64_t)floor(pa[1] / 2.0),
                         (int64_t)floor(pb[0] / 2.0), (int64_t)floor(pb[1] / 2.0)};
        int64_t comp = c4[0] + 4096;
        for (int k = 1; k < 4; k++) comp = comp * 8192 + (c4[k] + 4096);
        keys[nk].comp = comp; keys[nk].q = q; keys[nk].row = r; nk++;
    }
    qsort(keys, (size_t)nk, sizeof(qk_t), cmp_qk);

    acc_t* acc = (acc_t*)malloc(sizeof(acc_t) * (size_t)(nk > 0 ? nk : 1));
    int nacc = 0;
    int32_t* stamp = (int32_t*)malloc(sizeof(int32_t) * (size_t)nt);
    for (int i = 0; i < nt; i++) stamp[i] = -1;
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)nt);
    int32_t* members = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nk > 0 ? nk : 1));
    unsigned char* band = NULL; size_t band_cap = 0;
    double* ml = NULL; size_t ml_cap = 0;

    for (int g0 = 0, gid = 0; g0 < nk; gid++) {
        int g1 = g0 + 1;
        while (g1 < nk && keys[g1].comp == keys[g0].comp) g1++;
        const double* rl = lines + 3 * keys[g0].row;     /* representative */
        double a = rl[0], b = rl[1], c = rl[2];
        /* ---- candidates_grid guided.py:238-270 ---- */
        int nc = 0;
        double pa[2], pb[2];
        if (clip_scalar(a, b, c, W, H, d, pa, pb)) {
            double len = oracle_hypot(pb[0] - pa[0], pb[1] - pa[1]);
            long K = (long)ceil(len / d); if (K < 1) K = 1;
            int64_t prev[4] = {INT64_MIN, INT64_MIN, INT64_MIN, INT64_MIN};
            for (long k = 0; k <= K; k++) {
                double kd = (double)k, rk = (double)(K - k);
                double sx = (kd * pa[0] + rk * pb[0]) / (double)K;
                double sy = (kd * pa[1] + rk * pb[1]) / (double)K;
                for (int g = 0; g < 4; g++) {
                    int64_t key = cell_key(sx, sy, g, D);
                    if (key == prev[g]) continue;   /* same cell as the previous sample */
                    prev[g] = key;
                    int p = lower_bound(G.e, G.n, key);
                    for (; p < G.n && G.e[p].key == key; p++) {
                        int f = G.e[p].fid;
                        if (stamp[f] != gid) { stamp[f] = gid; cand[nc++] = f; }
                    }
                }
            }
        }
        if (nc == 0) { g0 = g1; continue; }
        qsort(cand, (size_t)nc, sizeof(int32_t), cmp_i32);
        int m = g1 - g0;
        for (int k = 0; k < m; k++) members[k] = keys[g0 + k].q;   /* sorted by q */
        /* ---- member lines + exact band guided.py:443-452 ---- */
        if ((size_t)m * nc > band_cap) { band_cap = (size_t)m * nc * 2; band = realloc(band, band_cap); }
        if ((size_t)m * 3 > ml_cap) { ml_cap = (size_t)m * 6; ml = realloc(ml, sizeof(double) * ml_cap); }
        int gemv_band = (m == 1) || (nc == 1 && m >= 3);
        for (int k = 0; k < m; k++) {
            int q = members[k];
            double* l = ml + 3 * k;
            epiline(F, (double)qxy[2 * q], (double)qxy[2 * q + 1], m == 1, l);
            double nrm = oracle_hypot(l[0], l[1]);
            if (nrm < 1e-15) nrm = 1e-15;
            l[0] /= nrm; l[1] /= nrm; l[2] /= nrm;
            for (int j = 0; j < nc; j++) {
                double x = (double)txy[2 * cand[j]], y = (double)txy[2 * cand[j] + 1];
                double v = gemv_band ? fma(l[0], x, l[1] * y) : fma(l[1], y, l[0] * x);
                v = v + l[2];
                band[(size_t)k * nc + j] = fabs(v) <= d;
            }
        }
        int ncols = 0;
        for (int j = 0; j < nc; j++) {
            int any = 0;
            for (int k = 0; k < m && !any; k++) any = band[(size_t)k * nc + j];
            ncols += any;
        }
        if (ncols == 0) { g0 = g1; continue; }
        if (stats) { stats[0] += m; stats[1] += (int64_t)m * ncols; }
        /* ---- exact distances, top-2, ratio_filter ---- */
        for (int k = 0; k < m; k++) {
            const uint8_t* qd = qdesc + (size_t)members[k] * 128;
            int32_t b1 = INT32_MAX, b2 = INT32_MAX; int i1 = -1, i2 = -1;
            for (int j = 0; j < nc; j++) {
                if (!band[(size_t)k * nc + j]) continue;
                const uint8_t* td = tdesc + (size_t)cand[j] * 128;
                int32_t s = 0;
                for (int e = 0; e < 128; e++) { int32_t df = (int32_t)qd[e] - (int32_t)td[e]; s += df * df; }
                if (s < b1) { b2 = b1; i2 = i1; b1 = s; i1 = j; }
                else if (s < b2) { b2 = s; i2 = j; }
            }
            if (i1 < 0) continue;
            float best = sqrtf((float)b1);
            if (i2 < 0) {
                if (best < single_cap) { acc[nacc].row = members[k]; acc[nacc].tgt = cand[i1];
                                         acc[nacc].dist = best; acc[nacc].ratio = 0.0f; nacc++; }
                continue;
            }
            float second = sqrtf((float)b2);
            float r = second > 0.0f ? best / second : 1.0f;
            if (r < ratio) { acc[nacc].row = members[k]; acc[nacc].tgt = cand[i1];
                             acc[nacc].dist = best; acc[nacc].ratio = r; nacc++; }
        }
        g0 = g1;
    }
    /* ---- _dedupe_targets matching.py:106-113 ---- */
    int32_t* win = stamp;  /* reuse: per-target winning acc index */
    for (int i = 0; i < nt; i++) win[i] = -1;
    for (int i = 0; i < nacc; i++) {
        int t = acc[i].tgt; int w = win[t];
        if (w < 0 || acc[i].dist < acc[w].dist || (acc[i].dist == acc[w].dist && acc[i].row < acc[w].row))
            win[t] = i;
    }
    /* collect winners sorted by row (rows are unique per accepted match) */
    int nout = 0;
    int32_t* order = members;  /* reuse */
    for (int t = 0; t < nt; t++) if (win[t] >= 0) order[nout++] = win[t];
    /* sort winner indices by row (one accepted match per row) */
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nout > 0 ? nout : 1));
    for (int i = 0; i < nout; i++) tmp[i] = ((int64_t)acc[order[i]].row << 32) | (uint32_t)order[i];
    qsort(tmp, (size_t)nout, sizeof(int64_t), cmp64);
    for (int i = 0; i < nout; i++) order[i] = (int32_t)(tmp[i] & 0xffffffff);
    free(tmp);
    int ret = nout;
    if (nout > cap) ret = -1;
    else for (int i = 0; i < nout; i++) {
        const acc_t* e = &acc[order[i]];
        out_q[i] = e->row; out_t[i] = e->tgt; out_dist[i] = e->dist; out_ratio[i] = e->ratio;
    }
    free(G.e); free(lines); free(keys); free(acc); free(stamp); free(cand); free(members);
    free(band); free(ml);
    return ret;
}

