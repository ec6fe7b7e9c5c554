// Two-view geometry of the coarse match graph: estimate_fundamental_ransac
// (geometry.py:153-198) batched over image pairs.
//
// Hypotheses come from host-supplied 8-point samples (the reference's own numpy
// choice stream, msfm_ransac_samples with sample_size 8); each is the normalized
// 8-point fit (geometry.py:117-138): Hartley normalization, the null vector of
// the 8x9 design matrix (smallest eigenvector of its 9x9 normal matrix, cyclic
// Jacobi), rank-2 projection (F0 - (F0 v3) v3^T with v3 the smallest right
// singular vector), denormalization and the canonical scaling of _normalize_f.
// Scoring counts Sampson distances below the threshold (geometry.py:141-150),
// one warp per hypothesis.  The caller replays the adaptive stop on the counts
// and msfm_fundamental_refit refits the winner on its inliers (one CTA per pair).
#include <stdint.h>

#include "common.cuh"

namespace msfm {
namespace {

struct FArgs {
    const double* q; const double* c; const int64_t* off;   // [..][2] per pair
    const int32_t* samples; int H;                            // [pair][H][8]
    double thr;
    double* F; int32_t* count;                                // [pair][H][9], [pair][H]
    int n_pairs;
};

// cyclic Jacobi eigen-decomposition of a symmetric N x N matrix (row-major);
// eigenvalues in w (unsorted), eigenvectors in the columns of V
template <int N>
__device__ void sym_eig(double* a, double* w, double* V) {
    for (int i = 0; i < N * N; i++) V[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 40; sweep++) {
        double off = 0.0, diag = 0.0;
        for (int p = 0; p < N; p++) {
            diag += fabs(a[p * N + p]);
            for (int q = p + 1; q < N; q++) off += fabs(a[p * N + q]);
        }
        if (off <= 1e-300 || off < 1e-22 * diag) break;
        for (int p = 0; p < N - 1; p++)
            for (int q = p + 1; q < N; q++) {
                const double apq = a[p * N + q];
                if (fabs(apq) < 1e-300) continue;
                const double app = a[p * N + p], aqq = a[q * N + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < N; k++) {
                    const double akp = a[k * N + p], akq = a[k * N + q];
                    a[k * N + p] = cs * akp - sn * akq;
                    a[k * N + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < N; k++) {
                    const double apk = a[p * N + k], aqk = a[q * N + k];
                    a[p * N + k] = cs * apk - sn * aqk;
                    a[q * N + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < N; k++) {
                    const double vkp = V[k * N + p], vkq = V[k * N + q];
                    V[k * N + p] = cs * vkp - sn * vkq;
                    V[k * N + q] = sn * vkp + cs * vkq;
                }
            }
    }
    for (int i = 0; i < N; i++) w[i] = a[i * N + i];
}

struct Hartley { double cx, cy, s; };

// the 9-vector of one correspondence in normalized coordinates (geometry.py:131)
__device__ __forceinline__ void design_row(double x, double y, double xp, double yp, double r[9]) {
    r[0] = xp * x; r[1] = xp * y; r[2] = xp;
    r[3] = yp * x; r[4] = yp * y; r[5] = yp;
    r[6] = x; r[7] = y; r[8] = 1.0;
}

// F from the normal matrix M (destroyed): null vector, rank 2, denormalize,
// _normalize_f (geometry.py:60-66).  w_sorted (optional) receives the eigenvalues
// in descending order.
__device__ void f_from_normal(double M[81], const Hartley& hq, const Hartley& hc, double F[9],
                              double* w_sorted) {
    double w[9], V[81];
    sym_eig<9>(M, w, V);
    int imin = 0;
    for (int i = 1; i < 9; i++) if (w[i] < w[imin]) imin = i;
    double F0[9];
    for (int i = 0; i < 9; i++) F0[i] = V[i * 9 + imin];
    if (w_sorted) {
        for (int i = 0; i < 9; i++) w_sorted[i] = w[i];
        for (int i = 1; i < 9; i++) {
            const double x = w_sorted[i];
            int j = i - 1;
            while (j >= 0 && w_sorted[j] < x) { w_sorted[j + 1] = w_sorted[j]; j--; }
            w_sorted[j + 1] = x;
        }
    }
    // rank 2: remove the smallest singular direction of F0
    double G[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0.0;
            for (int k = 0; k < 3; k++) s += F0[k * 3 + i] * F0[k * 3 + j];
            G[i * 3 + j] = s;
        }
    double g[3], W[9];
    sym_eig<3>(G, g, W);
    int jm = 0;
    for (int i = 1; i < 3; i++) if (g[i] < g[jm]) jm = i;
    const double v[3] = {W[0 * 3 + jm], W[1 * 3 + jm], W[2 * 3 + jm]};
    double Fv[3];
    for (int i = 0; i < 3; i++) Fv[i] = F0[i * 3 + 0] * v[0] + F0[i * 3 + 1] * v[1] + F0[i * 3 + 2] * v[2];
    double R2[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) R2[i * 3 + j] = F0[i * 3 + j] - Fv[i] * v[j];
    // F = Tc^T R2 Tq, T = [[s, 0, -s cx], [0, s, -s cy], [0, 0, 1]]
    double Tq[9] = {hq.s, 0.0, -hq.s * hq.cx, 0.0, hq.s, -hq.s * hq.cy, 0.0, 0.0, 1.0};
    double Tc[9] = {hc.s, 0.0, -hc.s * hc.cx, 0.0, hc.s, -hc.s * hc.cy, 0.0, 0.0, 1.0};
    double tmp[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0.0;
            for (int k = 0; k < 3; k++) s += R2[i * 3 + k] * Tq[k * 3 + j];
            tmp[i * 3 + j] = s;
        }
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0.0;
            for (int k = 0; k < 3; k++) s += Tc[k * 3 + i] * tmp[k * 3 + j];
            F[i * 3 + j] = s;
        }
    double nrm = 0.0;
    for (int i = 0; i < 9; i++) nrm += F[i] * F[i];
    nrm = sqrt(nrm);
    int am = 0;
    for (int i = 1; i < 9; i++) if (fabs(F[i]) > fabs(F[am])) am = i;
    const double sg = F[am] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < 9; i++) F[i] = sg * F[i] / nrm;
}

// Sampson distance below the threshold (geometry.py:141-150)
__device__ __forceinline__ bool sampson_in(const double F[9], double xq, double yq, double xc,
                                           double yc, double thr) {
    const double l0 = F[0] * xq + F[1] * yq + F[2];
    const double l1 = F[3] * xq + F[4] * yq + F[5];
    const double l2 = F[6] * xq + F[7] * yq + F[8];
    const double m0 = F[0] * xc + F[3] * yc + F[6];
    const double m1 = F[1] * xc + F[4] * yc + F[7];
    const double num = xc * l0 + yc * l1 + l2;
    const double den = l0 * l0 + l1 * l1 + m0 * m0 + m1 * m1;
    return fabs(num) / sqrt(fmax(den, 1e-30)) < thr;
}

__global__ void __launch_bounds__(128) f_hyp_kernel(FArgs a) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= a.n_pairs * a.H) return;
    const int p = gid / a.H;
    const int64_t o = a.off[p];
    const int32_t* smp = a.samples + (int64_t)gid * 8;
    double xq[8], yq[8], xc[8], yc[8];
    for (int k = 0; k < 8; k++) {
        const int64_t i = o + smp[k];
        xq[k] = a.q[2 * i]; yq[k] = a.q[2 * i + 1];
        xc[k] = a.c[2 * i]; yc[k] = a.c[2 * i + 1];
    }
    Hartley hq, hc;
    {
        double sx = 0, sy = 0, tx = 0, ty = 0;
        for (int k = 0; k < 8; k++) { sx += xq[k]; sy += yq[k]; tx += xc[k]; ty += yc[k]; }
        hq.cx = sx / 8.0; hq.cy = sy / 8.0; hc.cx = tx / 8.0; hc.cy = ty / 8.0;
        double rq = 0, rc = 0;
        for (int k = 0; k < 8; k++) {
            const double ax = xq[k] - hq.cx, ay = yq[k] - hq.cy;
            const double bx = xc[k] - hc.cx, by = yc[k] - hc.cy;
            rq += ax * ax + ay * ay;
            rc += bx * bx + by * by;
        }
        hq.s = sqrt(2.0) / fmax(sqrt(rq / 8.0), 1e-12);
        hc.s = sqrt(2.0) / fmax(sqrt(rc / 8.0), 1e-12);
    }
    double M[81];
    for (int i = 0; i < 81; i++) M[i] = 0.0;
    for (int k = 0; k < 8; k++) {
        double r[9];
        design_row((xq[k] - hq.cx) * hq.s, (yq[k] - hq.cy) * hq.s, (xc[k] - hc.cx) * hc.s,
                   (yc[k] - hc.cy) * hc.s, r);
        for (int i = 0; i < 9; i++)
            for (int j = i; j < 9; j++) M[i * 9 + j] += r[i] * r[j];
    }
    for (int i = 0; i < 9; i++)
        for (int j = 0; j < i; j++) M[i * 9 + j] = M[j * 9 + i];
    double F[9];
    f_from_normal(M, hq, hc, F, nullptr);
    bool ok = true;
    for (int i = 0; i < 9; i++) ok = ok && isfinite(F[i]);
    double* out = a.F + (int64_t)gid * 9;
    for (int i = 0; i < 9; i++) out[i] = F[i];
    a.count[gid] = ok ? 0 : -1;
}

__global__ void __launch_bounds__(256) f_score_kernel(FArgs a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.n_pairs * a.H) return;
    if (a.count[warp] < 0) return;
    const int p = warp / a.H;
    const int64_t o = a.off[p];
    const int n = (int)(a.off[p + 1] - o);
    double F[9];
    for (int i = 0; i < 9; i++) F[i] = a.F[(int64_t)warp * 9 + i];
    int c = 0;
    for (int i = lane; i < n; i += 32)
        c += sampson_in(F, a.q[2 * (o + i)], a.q[2 * (o + i) + 1], a.c[2 * (o + i)],
                        a.c[2 * (o + i) + 1], a.thr);
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if (lane == 0) a.count[warp] = c;
}

// ---------------------------------------------------------------- refit ----
struct FRefitArgs {
    const double* q; const double* c; const int64_t* off;
    const double* F_best; const int32_t* status; double thr;
    double* F_out; uint8_t* mask_out; int32_t* count_out; double* gap_out;
    int n_pairs;
};

constexpr int FT = 256;

template <int NV>
__device__ void fblock_sum(double (&v)[NV], double* sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = 0; k < NV; k++) {
        double x = v[k];
        for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        if (lane == 0) sm[w * NV + k] = x;
    }
    __syncthreads();
    for (int k = 0; k < NV; k++) {
        double s = 0.0;
        for (int j = 0; j < FT / 32; j++) s += sm[j * NV + k];
        v[k] = s;
    }
    __syncthreads();
}

// Fold one row (nonzero from column c0) into the upper-triangular 9x9 R (packed
// by rows) with Givens rotations: the R of a stacked QR, so the design matrix's
// singular values come out accurate down to ~1e-16 of the largest (the normal
// matrix squares them and loses the small ones; geometry.py:132's planar gap
// s[-2]/s[0] < 1e-9 needs them).
__device__ __forceinline__ int rix(int i, int j) { return i * 9 - (i * (i - 1)) / 2 + (j - i); }

__device__ void qr_fold(double R[45], double r[9], int c0) {
    for (int j = c0; j < 9; j++) {
        const double b = r[j];
        if (b == 0.0) continue;
        const double a = R[rix(j, j)];
        const double rad = hypot(a, b);
        const double c = a / rad, sn = b / rad;
        R[rix(j, j)] = rad;
        for (int k = j + 1; k < 9; k++) {
            const double t1 = R[rix(j, k)], t2 = r[k];
            R[rix(j, k)] = c * t1 + sn * t2;
            r[k] = c * t2 - sn * t1;
        }
    }
}

__device__ void qr_merge(double Ra[45], const double Rb[45]) {
    for (int i = 0; i < 9; i++) {
        double r[9];
        for (int k = 0; k < 9; k++) r[k] = k < i ? 0.0 : Rb[rix(i, k)];
        qr_fold(Ra, r, i);
    }
}

// singular values of the 9x9 upper-triangular R (one-sided Jacobi), descending
__device__ void sv_of_r(const double R[45], double s[9]) {
    double A[81];
    for (int i = 0; i < 9; i++)
        for (int j = 0; j < 9; j++) A[i * 9 + j] = j < i ? 0.0 : R[rix(i, j)];
    for (int sweep = 0; sweep < 60; sweep++) {
        double off = 0.0;
        for (int p = 0; p < 8; p++)
            for (int q = p + 1; q < 9; q++) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = 0; i < 9; i++) {
                    al += A[i * 9 + p] * A[i * 9 + p];
                    be += A[i * 9 + q] * A[i * 9 + q];
                    ga += A[i * 9 + p] * A[i * 9 + q];
                }
                if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
                off = fmax(off, fabs(ga) / sqrt(al * be));
                const double z = (be - al) / (2.0 * ga);
                const double t = (z >= 0 ? 1.0 : -1.0) / (fabs(z) + sqrt(1.0 + z * z));
                const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
                for (int i = 0; i < 9; i++) {
                    const double x = A[i * 9 + p], y = A[i * 9 + q];
                    A[i * 9 + p] = c * x - sn * y;
                    A[i * 9 + q] = sn * x + c * y;
                }
            }
        if (off < 1e-15) break;
    }
    for (int j = 0; j < 9; j++) {
        double n2 = 0.0;
        for (int i = 0; i < 9; i++) n2 += A[i * 9 + j] * A[i * 9 + j];
        s[j] = sqrt(n2);
    }
    for (int i = 1; i < 9; i++)       // insertion sort, descending
        for (int j = i; j > 0 && s[j] > s[j - 1]; j--) { const double t = s[j]; s[j] = s[j - 1]; s[j - 1] = t; }
}

__global__ void __launch_bounds__(FT) f_refit_kernel(FRefitArgs a) {
    const int p = blockIdx.x;
    if (!a.status[p]) return;
    __shared__ double sm[FT / 32 * 45];
    __shared__ double Fs[9];
    const int64_t o = a.off[p];
    const int n = (int)(a.off[p + 1] - o);
    double Fb[9];
    for (int i = 0; i < 9; i++) Fb[i] = a.F_best[9 * (int64_t)p + i];
    // inliers of the winning hypothesis: centroids and counts
    double s5[5] = {0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += FT) {
        const double xq = a.q[2 * (o + i)], yq = a.q[2 * (o + i) + 1];
        const double xc = a.c[2 * (o + i)], yc = a.c[2 * (o + i) + 1];
        if (sampson_in(Fb, xq, yq, xc, yc, a.thr)) {
            s5[0] += xq; s5[1] += yq; s5[2] += xc; s5[3] += yc; s5[4] += 1.0;
        }
    }
    fblock_sum<5>(s5, sm);
    const double m = s5[4];
    Hartley hq, hc;
    hq.cx = s5[0] / m; hq.cy = s5[1] / m; hc.cx = s5[2] / m; hc.cy = s5[3] / m;
    double r2[2] = {0, 0};
    for (int i = threadIdx.x; i < n; i += FT) {
        const double xq = a.q[2 * (o + i)], yq = a.q[2 * (o + i) + 1];
        const double xc = a.c[2 * (o + i)], yc = a.c[2 * (o + i) + 1];
        if (sampson_in(Fb, xq, yq, xc, yc, a.thr)) {
            const double ax = xq - hq.cx, ay = yq - hq.cy, bx = xc - hc.cx, by = yc - hc.cy;
            r2[0] += ax * ax + ay * ay;
            r2[1] += bx * bx + by * by;
        }
    }
    fblock_sum<2>(r2, sm);
    hq.s = sqrt(2.0) / fmax(sqrt(r2[0] / m), 1e-12);
    hc.s = sqrt(2.0) / fmax(sqrt(r2[1] / m), 1e-12);
    // normal matrix of the inlier design matrix (-> F), and the R factor of its QR
    // (-> the singular values for the planar gap)
    double acc[45], Rq[45];
    for (int k = 0; k < 45; k++) { acc[k] = 0.0; Rq[k] = 0.0; }
    for (int i = threadIdx.x; i < n; i += FT) {
        const double xq = a.q[2 * (o + i)], yq = a.q[2 * (o + i) + 1];
        const double xc = a.c[2 * (o + i)], yc = a.c[2 * (o + i) + 1];
        if (!sampson_in(Fb, xq, yq, xc, yc, a.thr)) continue;
        double r[9];
        design_row((xq - hq.cx) * hq.s, (yq - hq.cy) * hq.s, (xc - hc.cx) * hc.s,
                   (yc - hc.cy) * hc.s, r);
        int k = 0;
        for (int u = 0; u < 9; u++)
            for (int v = u; v < 9; v++) acc[k++] += r[u] * r[v];
        qr_fold(Rq, r, 0);
    }
    // tree-merge the per-thread R factors: warps by shuffles, then the warp results
    {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            double other[45];
            for (int k = 0; k < 45; k++) other[k] = __shfl_xor_sync(0xffffffffu, Rq[k], o);
            if ((lane & o) == 0) qr_merge(Rq, other);
        }
        __shared__ double rsm[FT / 32][45];
        if (lane == 0)
            for (int k = 0; k < 45; k++) rsm[w][k] = Rq[k];
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int v = 1; v < FT / 32; v++) qr_merge(Rq, rsm[v]);
            double sv[9];
            sv_of_r(Rq, sv);
            rsm[0][0] = sv[0] > 0.0 ? sv[7] / sv[0] : 0.0;
        }
        __syncthreads();
        Rq[0] = rsm[0][0];
        __syncthreads();
    }
    fblock_sum<45>(acc, sm);
    if (threadIdx.x == 0) {
        double M[81];
        int k = 0;
        for (int u = 0; u < 9; u++)
            for (int v = u; v < 9; v++) { M[u * 9 + v] = acc[k]; M[v * 9 + u] = acc[k]; k++; }
        double F[9], w[9];
        f_from_normal(M, hq, hc, F, w);
        for (int i = 0; i < 9; i++) Fs[i] = F[i];
        // s[-2] / s[0] of the design matrix (0 for fewer than 9 rows, geometry.py:132),
        // from the singular values of its R factor
        a.gap_out[p] = m >= 9.0 ? Rq[0] : 0.0;
        for (int i = 0; i < 9; i++) a.F_out[9 * (int64_t)p + i] = F[i];
    }
    __syncthreads();
    double F[9];
    for (int i = 0; i < 9; i++) F[i] = Fs[i];
    double cnt[1] = {0.0};
    for (int i = threadIdx.x; i < n; i += FT) {
        const bool in = sampson_in(F, a.q[2 * (o + i)], a.q[2 * (o + i) + 1], a.c[2 * (o + i)],
                                   a.c[2 * (o + i) + 1], a.thr);
        a.mask_out[o + i] = in ? 1 : 0;
        cnt[0] += in ? 1.0 : 0.0;
    }
    fblock_sum<1>(cnt, sm);
    if (threadIdx.x == 0) a.count_out[p] = (int32_t)cnt[0];
}

}  // namespace
}  // namespace msfm

using namespace msfm;

extern "C" int msfm_fundamental_hypotheses(const double* d_q, const double* d_c,
                                           const int64_t* d_off, int32_t n_pairs,
                                           const int32_t* d_samples, int32_t n_hyp,
                                           double threshold, double* d_F, int32_t* d_count,
                                           void* stream) {
    if (n_pairs < 0 || n_hyp < 0 || !(threshold > 0)) {
        set_error("msfm_fundamental_hypotheses: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_pairs == 0 || n_hyp == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    FArgs a{d_q, d_c, d_off, d_samples, n_hyp, threshold, d_F, d_count, n_pairs};
    const int total = n_pairs * n_hyp;
    {
        ProfScope ps("f_hyp_kernel", st);
        f_hyp_kernel<<<(total + 127) / 128, 128, 0, st>>>(a);
    }
    {
        ProfScope ps("f_score_kernel", st);
        f_score_kernel<<<(total + 7) / 8, 256, 0, st>>>(a);
    }
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    return MSFM_OK;
}

extern "C" int msfm_fundamental_refit(const double* d_q, const double* d_c, const int64_t* d_off,
                                      int32_t n_pairs, const double* d_F_best,
                                      const int32_t* d_status, double threshold, double* d_F,
                                      uint8_t* d_mask, int32_t* d_count, double* d_gap,
                                      void* stream) {
    if (n_pairs < 0 || !(threshold > 0)) {
        set_error("msfm_fundamental_refit: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_pairs == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    FRefitArgs a{d_q, d_c, d_off, d_F_best, d_status, threshold, d_F, d_mask, d_count, d_gap,
                 n_pairs};
    {
        ProfScope ps("f_refit_kernel", st);
        f_refit_kernel<<<n_pairs, FT, 0, st>>>(a);
    }
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}
