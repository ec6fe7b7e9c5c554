// PnP-RANSAC on sm_100a (K9 hypotheses + scoring, K10 refit + LM).
//
// Native body of msfm.reconstruct.pnp_ransac (reconstruct.py:168-226) with
// dlt_pose (:53-103) and refine_pose_lm (:106-165), batched over images.  The
// hypothesis stream is host-supplied (the numpy choice sequence, sampler.cpp),
// so every hypothesis can be scored independently; the adaptive stop and the
// OverflowError quirk are replayed on the host in numpy.  DLT null vectors come
// from the normal matrix AᵀA (assembled from four 4x4 moment matrices) by
// shifted-Cholesky inverse iteration; R = polar factor of K⁻¹P via a 3x3 Jacobi
// eigen-decomposition.  Poses agree with LAPACK's SVD to ~1e-12; inlier sets are
// identical except for residuals within that distance of the threshold.
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "rng.cuh"

namespace msfm {
namespace {

struct PnpArgs {
    const double* X;       // [n_corr_total][3]
    const double* uv;      // [n_corr_total][2]
    const int64_t* off;    // [n_img+1] correspondence offsets
    const double* K;       // [n_img][9]
    const int32_t* samples;   // [n_img][H][6] (image-local correspondence indices)
    int H;                 // hypotheses per image in this launch
    int h0;                // global index of the first hypothesis
    double thr;
    double* hyp;           // [n_img][H][12] R (9) t (3)
    int32_t* count;        // [n_img][H]  -1: DLT failed
    int n_img;
};

// ---- small dense helpers (fp64) ------------------------------------------
__device__ void sym3_eig(const double A[9], double w[3], double V[9]) {
    double a[9];
    for (int i = 0; i < 9; i++) a[i] = A[i];
    for (int i = 0; i < 9; i++) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 30; sweep++) {
        double off = fabs(a[1]) + fabs(a[2]) + fabs(a[5]);
        if (off < 1e-300) break;
        for (int p = 0; p < 2; p++)
            for (int q = p + 1; q < 3; q++) {
                double apq = a[3 * p + q];
                if (fabs(apq) < 1e-300) continue;
                double app = a[3 * p + p], aqq = a[3 * q + q];
                double theta = (aqq - app) / (2.0 * apq);
                double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
                for (int k = 0; k < 3; k++) {
                    double akp = a[3 * k + p], akq = a[3 * k + q];
                    a[3 * k + p] = c * akp - s * akq;
                    a[3 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; k++) {
                    double apk = a[3 * p + k], aqk = a[3 * q + k];
                    a[3 * p + k] = c * apk - s * aqk;
                    a[3 * q + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; k++) {
                    double vkp = V[3 * k + p], vkq = V[3 * k + q];
                    V[3 * k + p] = c * vkp - s * vkq;
                    V[3 * k + q] = s * vkp + c * vkq;
                }
            }
    }
    w[0] = a[0]; w[1] = a[4]; w[2] = a[8];
}

__device__ double det3(const double* m) {
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

__device__ bool inv3(const double* m, double* o) {
    double d = det3(m);
    if (d == 0.0) return false;
    double id = 1.0 / d;
    o[0] = (m[4] * m[8] - m[5] * m[7]) * id;
    o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    o[3] = (m[5] * m[6] - m[3] * m[8]) * id;
    o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    o[6] = (m[3] * m[7] - m[4] * m[6]) * id;
    o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
    return true;
}

// Moments of the normalised DLT rows: W[k] = sum w_k * Xh Xh^T, w = {1, u, v, u²+v²}
struct Moments {
    double m[4][10];  // packed upper triangle of 4x4 (00,01,02,03,11,12,13,22,23,33)
};

__device__ __forceinline__ void moments_add(Moments& M, const double xh[4], double u, double v) {
    const double w[4] = {1.0, u, v, u * u + v * v};
    int k = 0;
    for (int i = 0; i < 4; i++)
        for (int j = i; j < 4; j++, k++) {
            const double p = xh[i] * xh[j];
            for (int c = 0; c < 4; c++) M.m[c][k] += w[c] * p;
        }
}

__device__ __forceinline__ double mget(const double* p, int i, int j) {
    if (i > j) { int t = i; i = j; j = t; }
    const int base[4] = {0, 4, 7, 9};
    return p[base[i] + (j - i)];
}

// 12x12 normal matrix AᵀA of dlt_pose's A (reconstruct.py:71-76)
__device__ void normal_matrix(const Moments& M, double N[144]) {
    for (int i = 0; i < 144; i++) N[i] = 0.0;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            const double s0 = mget(M.m[0], i, j), su = mget(M.m[1], i, j), sv = mget(M.m[2], i, j),
                         sw = mget(M.m[3], i, j);
            N[i * 12 + j] = s0;
            N[(4 + i) * 12 + 4 + j] = s0;
            N[i * 12 + 8 + j] = -su;
            N[(8 + i) * 12 + j] = -su;
            N[(4 + i) * 12 + 8 + j] = -sv;
            N[(8 + i) * 12 + 4 + j] = -sv;
            N[(8 + i) * 12 + 8 + j] = sw;
        }
}

// smallest-eigenvalue eigenvector of a 12x12 SPD(-ish) matrix: inverse iteration
// on N + delta I with a Cholesky factor.
__device__ bool smallest_eigvec(double N[144], double x[12]) {
    double tr = 0.0;
    for (int i = 0; i < 12; i++) tr += N[i * 13];
    if (!(tr > 0.0) || !isfinite(tr)) return false;
    const double delta = tr * 1e-15;
    for (int i = 0; i < 12; i++) N[i * 13] += delta;
    // in-place Cholesky (lower)
    for (int j = 0; j < 12; j++) {
        double d = N[j * 13];
        for (int k = 0; k < j; k++) d -= N[j * 12 + k] * N[j * 12 + k];
        if (!(d > 0.0)) return false;
        d = sqrt(d);
        N[j * 13] = d;
        for (int i = j + 1; i < 12; i++) {
            double s = N[i * 12 + j];
            for (int k = 0; k < j; k++) s -= N[i * 12 + k] * N[j * 12 + k];
            N[i * 12 + j] = s / d;
        }
    }
    for (int i = 0; i < 12; i++) x[i] = 1.0 / sqrt(12.0) * (1.0 + 0.01 * i);
    for (int it = 0; it < 8; it++) {
        double y[12];
        for (int i = 0; i < 12; i++) {
            double s = x[i];
            for (int k = 0; k < i; k++) s -= N[i * 12 + k] * y[k];
            y[i] = s / N[i * 13];
        }
        for (int i = 11; i >= 0; i--) {
            double s = y[i];
            for (int k = i + 1; k < 12; k++) s -= N[k * 12 + i] * x[k];
            x[i] = s / N[i * 13];
        }
        double nrm = 0.0;
        for (int i = 0; i < 12; i++) nrm += x[i] * x[i];
        nrm = sqrt(nrm);
        if (!(nrm > 0.0) || !isfinite(nrm)) return false;
        for (int i = 0; i < 12; i++) x[i] /= nrm;
    }
    return true;
}

// dlt_pose tail (reconstruct.py:77-103): pose from the normalised null vector.
// depth_front(R, t) counts points in front; returns false when no orientation is valid.
struct Norm {
    double cx[3], sx, cu[2], su;
};

__device__ bool pose_from_nullvec(const double x[12], const Norm& nm, const double* K, double R[9],
                                  double t[3], double Gout[12]) {
    // P = Tu^-1 Pn Tx ; G = K^-1 P
    double Tui[9] = {1.0 / nm.su, 0, nm.cu[0], 0, 1.0 / nm.su, nm.cu[1], 0, 0, 1.0};
    double Pn[12];
    for (int i = 0; i < 12; i++) Pn[i] = x[i];
    double Tx[16] = {nm.sx, 0, 0, -nm.sx * nm.cx[0], 0, nm.sx, 0, -nm.sx * nm.cx[1],
                     0, 0, nm.sx, -nm.sx * nm.cx[2], 0, 0, 0, 1.0};
    double A[12], P[12];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 4; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += Tui[3 * i + k] * Pn[4 * k + j];
            A[4 * i + j] = s;
        }
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 4; j++) {
            double s = 0;
            for (int k = 0; k < 4; k++) s += A[4 * i + k] * Tx[4 * k + j];
            P[4 * i + j] = s;
        }
    double Ki[9];
    if (!inv3(K, Ki)) return false;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 4; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += Ki[3 * i + k] * P[4 * k + j];
            Gout[4 * i + j] = s;
        }
    return true;
}

__device__ bool polar_pose(const double G[12], double sign, double R[9], double t[3]) {
    double M[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = sign * G[4 * i + j];
    if (det3(M) <= 0.0) return false;       // det(U Vt) = sign(det M): skipped by the reference
    double MtM[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += M[3 * k + i] * M[3 * k + j];
            MtM[3 * i + j] = s;
        }
    double w[3], V[9];
    sym3_eig(MtM, w, V);
    double sg[3];
    for (int i = 0; i < 3; i++) {
        if (!(w[i] > 0.0)) return false;
        sg[i] = sqrt(w[i]);
    }
    const double scale = (sg[0] + sg[1] + sg[2]) / 3.0;
    if (scale < 1e-12) return false;
    // R = M V diag(1/s) V^T
    double MV[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += M[3 * i + k] * V[3 * k + j];
            MV[3 * i + j] = s / sg[j];
        }
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += MV[3 * i + k] * V[3 * j + k];
            R[3 * i + j] = s;
        }
    for (int i = 0; i < 3; i++) t[i] = sign * G[4 * i + 3] / scale;
    return true;
}

__device__ __forceinline__ void transform(const double R[9], const double t[3], const double* X,
                                          double xc[3]) {
    // X @ R.T + t as numpy/OpenBLAS rounds a (n,3)@(3,3) dgemm
    for (int j = 0; j < 3; j++)
        xc[j] = fma(X[2], R[3 * j + 2], fma(X[1], R[3 * j + 1], X[0] * R[3 * j])) + t[j];
}

__device__ __forceinline__ bool is_inlier(const double R[9], const double t[3], const double* X,
                                          const double* uv, const double* K, double thr,
                                          double* err_out = nullptr) {
    double xc[3];
    transform(R, t, X, xc);
    const double f = K[0];
    const double px = f * xc[0] / xc[2] + K[2];
    const double py = f * xc[1] / xc[2] + K[5];
    const double dx = px - uv[0], dy = py - uv[1];
    const double err = sqrt(dx * dx + dy * dy);
    if (err_out) *err_out = err;
    return xc[2] > 0.0 && isfinite(err) && err < thr;
}

// ---------------------------------------------------------------- kernels --
__global__ void __launch_bounds__(128) pnp_hyp_kernel(PnpArgs a) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= a.n_img * a.H) return;
    const int s = gid / a.H, h = gid - s * a.H;
    const int64_t o = a.off[s];
    const int n = (int)(a.off[s + 1] - o);
    double* out = a.hyp + (int64_t)gid * 12;
    a.count[gid] = -1;
    if (n < 6) return;
    const int32_t* smp = a.samples + ((int64_t)s * a.H + h) * 6;
    double X[6][3], U[6][2];
    for (int k = 0; k < 6; k++) {
        const int i = smp[k];
        for (int c = 0; c < 3; c++) X[k][c] = a.X[(o + i) * 3 + c];
        U[k][0] = a.uv[(o + i) * 2];
        U[k][1] = a.uv[(o + i) * 2 + 1];
    }
    // normalisation (reconstruct.py:64-70)
    Norm nm;
    for (int c = 0; c < 3; c++) {
        double m = 0;
        for (int k = 0; k < 6; k++) m += X[k][c];
        nm.cx[c] = m / 6.0;
    }
    for (int c = 0; c < 2; c++) {
        double m = 0;
        for (int k = 0; k < 6; k++) m += U[k][c];
        nm.cu[c] = m / 6.0;
    }
    double dx = 0, du = 0;
    for (int k = 0; k < 6; k++) {
        const double a0 = X[k][0] - nm.cx[0], a1 = X[k][1] - nm.cx[1], a2 = X[k][2] - nm.cx[2];
        dx += sqrt(a0 * a0 + a1 * a1 + a2 * a2);
        const double b0 = U[k][0] - nm.cu[0], b1 = U[k][1] - nm.cu[1];
        du += sqrt(b0 * b0 + b1 * b1);
    }
    nm.sx = sqrt(3.0) / fmax(dx / 6.0, 1e-12);
    nm.su = sqrt(2.0) / fmax(du / 6.0, 1e-12);
    Moments M;
    for (int c = 0; c < 4; c++)
        for (int k = 0; k < 10; k++) M.m[c][k] = 0.0;
    for (int k = 0; k < 6; k++) {
        const double xh[4] = {(X[k][0] - nm.cx[0]) * nm.sx, (X[k][1] - nm.cx[1]) * nm.sx,
                              (X[k][2] - nm.cx[2]) * nm.sx, 1.0};
        moments_add(M, xh, (U[k][0] - nm.cu[0]) * nm.su, (U[k][1] - nm.cu[1]) * nm.su);
    }
    double N[144], x[12], G[12];
    normal_matrix(M, N);
    if (!smallest_eigvec(N, x)) return;
    const double* K = a.K + 9 * (int64_t)s;
    if (!pose_from_nullvec(x, nm, K, nullptr, nullptr, G)) return;
    int best_front = -1;
    double bR[9], bt[3];
    for (int si = 0; si < 2; si++) {
        const double sign = si == 0 ? 1.0 : -1.0;
        double R[9], t[3];
        if (!polar_pose(G, sign, R, t)) continue;
        int front = 0;
        for (int k = 0; k < 6; k++) {
            double xc[3];
            transform(R, t, X[k], xc);
            front += xc[2] > 0.0;
        }
        if (best_front < 0 || front > best_front) {
            best_front = front;
            for (int i = 0; i < 9; i++) bR[i] = R[i];
            for (int i = 0; i < 3; i++) bt[i] = t[i];
        }
    }
    if (best_front <= 0) return;       // "resection produced no valid orientation"
    for (int i = 0; i < 9; i++) out[i] = bR[i];
    for (int i = 0; i < 3; i++) out[9 + i] = bt[i];
    a.count[gid] = 0;                  // valid; scored next
}

__global__ void __launch_bounds__(256) pnp_score_kernel(PnpArgs a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.n_img * a.H) return;
    if (a.count[warp] < 0) return;
    const int s = warp / a.H;
    const int64_t o = a.off[s];
    const int n = (int)(a.off[s + 1] - o);
    const double* hp = a.hyp + (int64_t)warp * 12;
    double R[9], t[3];
    for (int i = 0; i < 9; i++) R[i] = hp[i];
    for (int i = 0; i < 3; i++) t[i] = hp[9 + i];
    const double* K = a.K + 9 * (int64_t)s;
    int c = 0;
    for (int i = lane; i < n; i += 32) c += is_inlier(R, t, a.X + (o + i) * 3, a.uv + (o + i) * 2, K, a.thr);
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if (lane == 0) a.count[warp] = c;
}

// ---------------------------------------------------------------- refit ----
struct RefitArgs {
    const double* X; const double* uv; const int64_t* off; const double* K;
    const double* hyp_best;   // [n_img][12] winning hypothesis pose (host-selected)
    const int32_t* status;    // [n_img] 1: refit this image
    double thr; int min_inliers; int iters;
    double* R_out; double* t_out; uint8_t* mask_out; int32_t* n_inl; int32_t* ok;
    int n_img;
};

constexpr int RT = 256;

template <int NV>
__device__ void block_sum(double (&v)[NV], double* sm /* RT/32*NV */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = 0; k < NV; k++) {
        double x = v[k];
        for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        v[k] = x;
    }
    __syncthreads();
    if (lane == 0)
        for (int k = 0; k < NV; k++) sm[w * NV + k] = v[k];
    __syncthreads();
    for (int k = 0; k < NV; k++) {
        double x = 0;
        for (int ww = 0; ww < RT / 32; ww++) x += sm[ww * NV + k];
        v[k] = x;
    }
    __syncthreads();
}

__device__ void rodrigues(const double w[3], double R[9]) {
    const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    if (th < 1e-12) {
        const double Rm[9] = {1, -w[2], w[1], w[2], 1, -w[0], -w[1], w[0], 1};
        for (int i = 0; i < 9; i++) R[i] = Rm[i];
        return;
    }
    const double k[3] = {w[0] / th, w[1] / th, w[2] / th};
    const double Km[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
    double K2[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int q = 0; q < 3; q++) s += Km[3 * i + q] * Km[3 * q + j];
            K2[3 * i + j] = s;
        }
    const double sn = sin(th), cs = 1.0 - cos(th);
    for (int i = 0; i < 9; i++) R[i] = (i % 4 == 0 ? 1.0 : 0.0) + sn * Km[i] + cs * K2[i];
}

// np.linalg.solve (LU with partial pivoting) of a 6x6 system
__device__ bool solve6(double A[36], double b[6]) {
    for (int c = 0; c < 6; c++) {
        int p = c;
        for (int r = c + 1; r < 6; r++)
            if (fabs(A[6 * r + c]) > fabs(A[6 * p + c])) p = r;
        if (A[6 * p + c] == 0.0) return false;
        if (p != c) {
            for (int k = 0; k < 6; k++) { double tmp = A[6 * c + k]; A[6 * c + k] = A[6 * p + k]; A[6 * p + k] = tmp; }
            double tmp = b[c]; b[c] = b[p]; b[p] = tmp;
        }
        for (int r = c + 1; r < 6; r++) {
            const double f = A[6 * r + c] / A[6 * c + c];
            for (int k = c; k < 6; k++) A[6 * r + k] -= f * A[6 * c + k];
            b[r] -= f * b[c];
        }
    }
    for (int r = 5; r >= 0; r--) {
        double s = b[r];
        for (int k = r + 1; k < 6; k++) s -= A[6 * r + k] * b[k];
        b[r] = s / A[6 * r + r];
    }
    return true;
}

__global__ void __launch_bounds__(RT) pnp_refit_kernel(RefitArgs a) {
    __shared__ double sm[RT / 32 * 40];
    __shared__ double shR[9], sht[3], shG[12];
    __shared__ int shflag;
    const int s = blockIdx.x;
    if (!a.status[s]) return;
    const int64_t o = a.off[s];
    const int n = (int)(a.off[s + 1] - o);
    const double* K = a.K + 9 * (int64_t)s;
    const double* hp = a.hyp_best + 12 * (int64_t)s;
    double R[9], t[3];
    for (int i = 0; i < 9; i++) R[i] = hp[i];
    for (int i = 0; i < 3; i++) t[i] = hp[9 + i];
    uint8_t* mask = a.mask_out + o;
    // best_mask of the winning hypothesis
    for (int i = threadIdx.x; i < n; i += RT)
        mask[i] = is_inlier(R, t, a.X + (o + i) * 3, a.uv + (o + i) * 2, K, a.thr);
    __syncthreads();
    // ---- dlt_pose on the inliers (reconstruct.py:215): normalisation
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += RT) {
        if (!mask[i]) continue;
        const double* X = a.X + (o + i) * 3;
        const double* U = a.uv + (o + i) * 2;
        v[0] += X[0]; v[1] += X[1]; v[2] += X[2]; v[3] += U[0]; v[4] += U[1]; v[5] += 1.0;
    }
    block_sum<6>(v, sm);
    const double cnt = v[5];
    Norm nm;
    nm.cx[0] = v[0] / cnt; nm.cx[1] = v[1] / cnt; nm.cx[2] = v[2] / cnt;
    nm.cu[0] = v[3] / cnt; nm.cu[1] = v[4] / cnt;
    double w2[2] = {0, 0};
    for (int i = threadIdx.x; i < n; i += RT) {
        if (!mask[i]) continue;
        const double* X = a.X + (o + i) * 3;
        const double* U = a.uv + (o + i) * 2;
        const double a0 = X[0] - nm.cx[0], a1 = X[1] - nm.cx[1], a2 = X[2] - nm.cx[2];
        w2[0] += sqrt(a0 * a0 + a1 * a1 + a2 * a2);
        const double b0 = U[0] - nm.cu[0], b1 = U[1] - nm.cu[1];
        w2[1] += sqrt(b0 * b0 + b1 * b1);
    }
    block_sum<2>(w2, sm);
    nm.sx = sqrt(3.0) / fmax(w2[0] / cnt, 1e-12);
    nm.su = sqrt(2.0) / fmax(w2[1] / cnt, 1e-12);
    double mom[40];
    for (int k = 0; k < 40; k++) mom[k] = 0.0;
    for (int i = threadIdx.x; i < n; i += RT) {
        if (!mask[i]) continue;
        const double* X = a.X + (o + i) * 3;
        const double* U = a.uv + (o + i) * 2;
        const double xh[4] = {(X[0] - nm.cx[0]) * nm.sx, (X[1] - nm.cx[1]) * nm.sx,
                              (X[2] - nm.cx[2]) * nm.sx, 1.0};
        const double u = (U[0] - nm.cu[0]) * nm.su, vv = (U[1] - nm.cu[1]) * nm.su;
        const double w[4] = {1.0, u, vv, u * u + vv * vv};
        int k = 0;
        for (int p = 0; p < 4; p++)
            for (int q = p; q < 4; q++, k++) {
                const double pr = xh[p] * xh[q];
                for (int c = 0; c < 4; c++) mom[c * 10 + k] += w[c] * pr;
            }
    }
    block_sum<40>(mom, sm);
    if (threadIdx.x == 0) {
        Moments M;
        for (int c = 0; c < 4; c++)
            for (int k = 0; k < 10; k++) M.m[c][k] = mom[c * 10 + k];
        double N[144], x[12], G[12];
        normal_matrix(M, N);
        shflag = 0;
        if (smallest_eigvec(N, x) && pose_from_nullvec(x, nm, K, nullptr, nullptr, G)) {
            shflag = 1;
            for (int i = 0; i < 12; i++) shG[i] = G[i];
        }
    }
    __syncthreads();
    if (!shflag) { if (threadIdx.x == 0) a.ok[s] = 0; return; }
    // pick the sign (most inliers in front), reconstruct.py:87-103
    int bestf = -1;
    double bR[9], bt[3];
    for (int si = 0; si < 2; si++) {
        const double sign = si == 0 ? 1.0 : -1.0;
        double Rc[9], tc[3];
        double G[12];
        for (int i = 0; i < 12; i++) G[i] = shG[i];
        const bool valid = polar_pose(G, sign, Rc, tc);
        double f1[1] = {0.0};
        if (valid)
            for (int i = threadIdx.x; i < n; i += RT) {
                if (!mask[i]) continue;
                double xc[3];
                transform(Rc, tc, a.X + (o + i) * 3, xc);
                f1[0] += xc[2] > 0.0 ? 1.0 : 0.0;
            }
        block_sum<1>(f1, sm);
        if (valid && (bestf < 0 || (int)f1[0] > bestf)) {
            bestf = (int)f1[0];
            for (int i = 0; i < 9; i++) bR[i] = Rc[i];
            for (int i = 0; i < 3; i++) bt[i] = tc[i];
        }
    }
    if (bestf <= 0) { if (threadIdx.x == 0) a.ok[s] = 0; return; }
    for (int i = 0; i < 9; i++) R[i] = bR[i];
    for (int i = 0; i < 3; i++) t[i] = bt[i];
    // ---- refine_pose_lm (reconstruct.py:106-165) over the inliers
    const double f = K[0], ppx = K[2], ppy = K[5];
    auto cost_of = [&](const double* Rc, const double* tc) {
        double c1[1] = {0.0};
        for (int i = threadIdx.x; i < n; i += RT) {
            if (!mask[i]) continue;
            double xc[3];
            transform(Rc, tc, a.X + (o + i) * 3, xc);
            const double* U = a.uv + (o + i) * 2;
            const double rx = f * xc[0] / xc[2] + ppx - U[0];
            const double ry = f * xc[1] / xc[2] + ppy - U[1];
            c1[0] += rx * rx + ry * ry;
        }
        block_sum<1>(c1, sm);
        return c1[0];
    };
    double cost = cost_of(R, t);
    double lam = 1e-6;
    bool done = false;
    for (int it = 0; it < a.iters && !done; it++) {
        double hg[28];
        for (int k = 0; k < 28; k++) hg[k] = 0.0;
        for (int i = threadIdx.x; i < n; i += RT) {
            if (!mask[i]) continue;
            double xc[3];
            transform(R, t, a.X + (o + i) * 3, xc);
            const double* U = a.uv + (o + i) * 2;
            const double x = xc[0], y = xc[1], z = xc[2];
            const double r2[2] = {f * x / z + ppx - U[0], f * y / z + ppy - U[1]};
            const double du[2][3] = {{f / z, 0.0, -f * x / (z * z)}, {0.0, f / z, -f * y / (z * z)}};
            const double RX[3] = {xc[0] - t[0], xc[1] - t[1], xc[2] - t[2]};
            const double dr[3][3] = {{0.0, RX[2], -RX[1]}, {-RX[2], 0.0, RX[0]}, {RX[1], -RX[0], 0.0}};
            double J[2][6];
            for (int rr = 0; rr < 2; rr++) {
                for (int c = 0; c < 3; c++) {
                    double sacc = 0;
                    for (int q = 0; q < 3; q++) sacc += du[rr][q] * dr[q][c];
                    J[rr][c] = sacc;
                    J[rr][3 + c] = du[rr][c];
                }
            }
            int k = 0;
            for (int p = 0; p < 6; p++)
                for (int q = p; q < 6; q++, k++) hg[k] += J[0][p] * J[0][q] + J[1][p] * J[1][q];
            for (int p = 0; p < 6; p++) hg[21 + p] += J[0][p] * r2[0] + J[1][p] * r2[1];
            hg[27] += 0.0;
        }
        block_sum<28>(hg, sm);
        double H[36], g[6];
        {
            int k = 0;
            for (int p = 0; p < 6; p++)
                for (int q = p; q < 6; q++, k++) { H[6 * p + q] = hg[k]; H[6 * q + p] = hg[k]; }
            for (int p = 0; p < 6; p++) g[p] = hg[21 + p];
        }
        bool stepped = false;
        for (int tr = 0; tr < 8; tr++) {
            double Hd[36], delta[6];
            for (int i = 0; i < 36; i++) Hd[i] = H[i];
            for (int p = 0; p < 6; p++) Hd[7 * p] += lam * fmax(H[7 * p], 1e-12);
            for (int p = 0; p < 6; p++) delta[p] = -g[p];
            if (!solve6(Hd, delta)) { lam *= 10.0; continue; }
            double Rd[9], Rn[9], tn[3];
            rodrigues(delta, Rd);
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double sacc = 0;
                    for (int q = 0; q < 3; q++) sacc += Rd[3 * i + q] * R[3 * q + j];
                    Rn[3 * i + j] = sacc;
                }
            for (int i = 0; i < 3; i++) tn[i] = t[i] + delta[3 + i];
            const double cn = cost_of(Rn, tn);
            if (isfinite(cn) && cn < cost) {
                const double rel = (cost - cn) / fmax(cost, 1e-30);
                for (int i = 0; i < 9; i++) R[i] = Rn[i];
                for (int i = 0; i < 3; i++) t[i] = tn[i];
                cost = cn;
                lam = fmax(lam / 10.0, 1e-15);
                stepped = true;
                if (rel < 1e-10) done = true;
                break;
            }
            lam *= 10.0;
        }
        if (!stepped) break;
    }
    // final mask (reconstruct.py:219-226)
    double c1[1] = {0.0};
    for (int i = threadIdx.x; i < n; i += RT) {
        const bool in = is_inlier(R, t, a.X + (o + i) * 3, a.uv + (o + i) * 2, K, a.thr);
        mask[i] = in;
        c1[0] += in ? 1.0 : 0.0;
    }
    block_sum<1>(c1, sm);
    if (threadIdx.x == 0) {
        const int ni = (int)c1[0];
        a.n_inl[s] = ni;
        a.ok[s] = ni >= a.min_inliers;
        for (int i = 0; i < 9; i++) a.R_out[9 * (int64_t)s + i] = R[i];
        for (int i = 0; i < 3; i++) a.t_out[3 * (int64_t)s + i] = t[i];
    }
    (void)shR; (void)sht;
}

}  // namespace
}  // namespace msfm

using namespace msfm;

// np.random.default_rng(seed_k).choice(n_k, size, replace=False) x count.
// Every choice consumes a fixed number of 32-bit draws unless Lemire's bounded
// draw rejects (probability ~ n / 2^32 per draw), so thread (k, h) jumps stream k
// to draw h * (2 size - 1) with PCG64's O(log) advance and makes choice h alone;
// a stream where any draw would have been rejected is flagged and redone
// sequentially (one thread) by ransac_samples_fixup_kernel.
__global__ void ransac_samples_kernel(int32_t n_items, const uint64_t* __restrict__ seeds,
                                      const int64_t* __restrict__ n, int32_t sample_size,
                                      int32_t count, int32_t* __restrict__ out,
                                      uint64_t* __restrict__ state_out, int32_t* __restrict__ redo,
                                      int32_t* __restrict__ bad) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)count + 1;          // count choices + the end state
    if (tid >= (int64_t)n_items * per) return;
    const int it = (int)(tid / per), h = (int)(tid - (int64_t)it * per);
    const int64_t pop = n[it];
    if (pop > 10000 && sample_size > pop / 50) { atomicExch(bad, 1); return; }
    msfm_rng::Pcg64 g0;
    msfm_rng::seed_pcg64(seeds[it], g0);
    // draws per choice: one per bounded call with a non-zero range (Floyd's j = 0,
    // reached when pop == size, returns 0 without drawing)
    const uint64_t draws = 2 * (uint64_t)sample_size - 1 - (pop == sample_size ? 1 : 0);
    msfm_rng::Pcg64 g;
    msfm_rng::pcg_at_draw(g0.state, g0.inc, draws * (uint64_t)h, g);
    if (h == count) {
        // numpy keeps the last buffered half in `uinteger` after using it: after an
        // even number of draws that is the high half of the last 64-bit output
        if (!g.has32 && count > 0 && draws > 0) {
            const uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
            const unsigned rot = (unsigned)(hi >> 58);
            const uint64_t x = hi ^ lo;
            g.u32 = (uint32_t)(((x >> rot) | (x << ((64 - rot) & 63))) >> 32);
        }
        if (state_out) {
            uint64_t* so = state_out + 6 * (int64_t)it;
            so[0] = (uint64_t)(g.state >> 64);
            so[1] = (uint64_t)g.state;
            so[2] = (uint64_t)(g.inc >> 64);
            so[3] = (uint64_t)g.inc;
            so[4] = (uint64_t)g.has32;
            so[5] = (uint64_t)g.u32;
        }
        return;
    }
    int64_t tmp[48];
    bool rej = false;
    msfm_rng::choice_floyd_once(g, pop, sample_size, tmp, rej);
    if (rej) atomicExch(redo + it, 1);
    int32_t* o = out + ((int64_t)it * count + h) * sample_size;
    for (int k = 0; k < sample_size; k++) o[k] = (int32_t)tmp[k];
}

// the sequential stream, for the flagged items only
__global__ void ransac_samples_fixup_kernel(int32_t n_items, const uint64_t* __restrict__ seeds,
                                            const int64_t* __restrict__ n, int32_t sample_size,
                                            int32_t count, int32_t* __restrict__ out,
                                            uint64_t* __restrict__ state_out,
                                            const int32_t* __restrict__ redo,
                                            int32_t* __restrict__ bad) {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= n_items || !redo[it]) return;
    msfm_rng::Pcg64 g;
    msfm_rng::seed_pcg64(seeds[it], g);
    int64_t tmp[48];
    int32_t* o = out + (int64_t)it * count * sample_size;
    for (int32_t h = 0; h < count; h++) {
        if (!msfm_rng::choice_floyd(g, n[it], sample_size, tmp)) {
            atomicExch(bad, 1);
            return;
        }
        for (int k = 0; k < sample_size; k++) o[(int64_t)h * sample_size + k] = (int32_t)tmp[k];
    }
    if (state_out) {
        uint64_t* so = state_out + 6 * (int64_t)it;
        so[0] = (uint64_t)(g.state >> 64);
        so[1] = (uint64_t)g.state;
        so[2] = (uint64_t)(g.inc >> 64);
        so[3] = (uint64_t)g.inc;
        so[4] = (uint64_t)g.has32;
        so[5] = (uint64_t)g.u32;
    }
}

extern "C" int msfm_pnp_hypotheses(const double* d_X, const double* d_uv, const int64_t* d_off,
                                   const double* d_K, int32_t n_images, const int32_t* d_samples,
                                   int32_t n_hyp, double threshold, double* d_hyp,
                                   int32_t* d_count, void* stream) {
    if (n_images < 0 || n_hyp < 0 || !(threshold > 0)) {
        set_error("msfm_pnp_hypotheses: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_images == 0 || n_hyp == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    PnpArgs a{d_X, d_uv, d_off, d_K, d_samples, n_hyp, 0, threshold, d_hyp, d_count, n_images};
    const int total = n_images * n_hyp;
    {
        ProfScope ps("pnp_hyp_kernel", st);
        pnp_hyp_kernel<<<(total + 127) / 128, 128, 0, st>>>(a);
    }
    {
        ProfScope ps("pnp_score_kernel", st);
        pnp_score_kernel<<<(total + 7) / 8, 256, 0, st>>>(a);
    }
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    return MSFM_OK;
}

extern "C" int msfm_pnp_refit(const double* d_X, const double* d_uv, const int64_t* d_off,
                              const double* d_K, int32_t n_images, const double* d_hyp_best,
                              const int32_t* d_status, double threshold, int32_t min_inliers,
                              int32_t lm_iters, double* d_R, double* d_t, uint8_t* d_mask,
                              int32_t* d_n_inliers, int32_t* d_ok, void* stream) {
    if (n_images < 0 || !(threshold > 0)) {
        set_error("msfm_pnp_refit: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_images == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    MSFM_CUDA_TRY(cudaMemsetAsync(d_ok, 0, sizeof(int32_t) * n_images, st));
    RefitArgs a{d_X, d_uv, d_off, d_K, d_hyp_best, d_status, threshold, min_inliers, lm_iters,
                d_R, d_t, d_mask, d_n_inliers, d_ok, n_images};
    {
        ProfScope ps("pnp_refit_kernel", st);
        pnp_refit_kernel<<<n_images, RT, 0, st>>>(a);
    }
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

extern "C" int msfm_ransac_samples_seeded_device(int32_t n_items, const uint64_t* d_seeds,
                                                 const int64_t* d_n, int32_t sample_size,
                                                 int32_t count, int32_t* d_out,
                                                 uint64_t* d_state_out, int32_t* d_bad,
                                                 void* stream) {
    if (n_items < 0 || sample_size < 1 || sample_size > 48 || count < 0 || !d_bad) {
        set_error("msfm_ransac_samples_seeded_device: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_items == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // per-item redo flags live after the bad flag's int: the caller's d_bad must
    // hold 1 + n_items int32
    int32_t* redo = d_bad + 1;
    MSFM_CUDA_TRY(cudaMemsetAsync(redo, 0, sizeof(int32_t) * n_items, st));
    const int64_t threads = (int64_t)n_items * ((int64_t)count + 1);
    ransac_samples_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(
        n_items, d_seeds, d_n, sample_size, count, d_out, d_state_out, redo, d_bad);
    ransac_samples_fixup_kernel<<<(n_items + 63) / 64, 64, 0, st>>>(
        n_items, d_seeds, d_n, sample_size, count, d_out, d_state_out, redo, d_bad);
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    return MSFM_OK;
}
