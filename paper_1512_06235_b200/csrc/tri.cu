// Batched multi-view DLT triangulation (K11) on sm_100a.
//
// Native body of msfm.geometry.triangulate_track (geometry.py:276-357) for many
// tracks at once (densify.py:244-276): 2n x 4 DLT via its 4x4 normal matrix
// (smallest eigenvector, cyclic Jacobi), reprojection, one Gauss-Newton step
// kept only if it does not increase the mean error, then the depth /
// reprojection / triangulation-angle gates.  One thread per track.
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace msfm {
namespace {

struct TriArgs {
    const double* K; const double* R; const double* t;   // per camera [9],[9],[3]
    const int64_t* ptr; const int32_t* cam; const double* pix;
    int n_tracks;
    double max_error, min_angle_deg;
    double* X; double* err; int32_t* status;
};

__device__ void jacobi4(double a[16], double V[16]) {
    for (int i = 0; i < 16; i++) V[i] = (i % 5 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 40; sweep++) {
        double off = 0.0;
        for (int p = 0; p < 4; p++)
            for (int q = p + 1; q < 4; q++) off += fabs(a[4 * p + q]);
        if (off < 1e-300) break;
        for (int p = 0; p < 3; p++)
            for (int q = p + 1; q < 4; q++) {
                const double apq = a[4 * p + q];
                if (apq == 0.0) continue;
                const double th = (a[4 * q + q] - a[4 * p + p]) / (2.0 * apq);
                const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
                for (int k = 0; k < 4; k++) {
                    const double akp = a[4 * k + p], akq = a[4 * k + q];
                    a[4 * k + p] = c * akp - s * akq;
                    a[4 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 4; k++) {
                    const double apk = a[4 * p + k], aqk = a[4 * q + k];
                    a[4 * p + k] = c * apk - s * aqk;
                    a[4 * q + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 4; k++) {
                    const double vkp = V[4 * k + p], vkq = V[4 * k + q];
                    V[4 * k + p] = c * vkp - s * vkq;
                    V[4 * k + q] = s * vkp + c * vkq;
                }
            }
    }
}

// residuals of all observations at X; returns mean error (inf if any non-finite)
__device__ double reproject(const TriArgs& a, int64_t o, int n, const double X[3], bool* depth_ok) {
    double sum = 0.0;
    bool finite = true;
    *depth_ok = true;
    for (int i = 0; i < n; i++) {
        const int c = a.cam[o + i];
        const double* R = a.R + 9 * c;
        const double* t = a.t + 3 * c;
        const double* K = a.K + 9 * c;
        double xc[3];
        for (int j = 0; j < 3; j++) xc[j] = R[3 * j] * X[0] + R[3 * j + 1] * X[1] + R[3 * j + 2] * X[2] + t[j];
        if (xc[2] <= 0.0) *depth_ok = false;
        if (xc[2] <= 1e-12) { finite = false; continue; }
        double uv[3];
        for (int j = 0; j < 3; j++) uv[j] = K[3 * j] * xc[0] + K[3 * j + 1] * xc[1] + K[3 * j + 2] * xc[2];
        const double rx = uv[0] / uv[2] - a.pix[2 * (o + i)];
        const double ry = uv[1] / uv[2] - a.pix[2 * (o + i) + 1];
        const double e = sqrt(rx * rx + ry * ry);
        if (!isfinite(e)) finite = false;
        sum += e;
    }
    return finite ? sum / n : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ bool solve3(double A[9], double b[3]) {
    for (int c = 0; c < 3; c++) {
        int p = c;
        for (int r = c + 1; r < 3; r++)
            if (fabs(A[3 * r + c]) > fabs(A[3 * p + c])) p = r;
        if (A[3 * p + c] == 0.0) return false;
        if (p != c) {
            for (int k = 0; k < 3; k++) { double tmp = A[3 * c + k]; A[3 * c + k] = A[3 * p + k]; A[3 * p + k] = tmp; }
            double tmp = b[c]; b[c] = b[p]; b[p] = tmp;
        }
        for (int r = c + 1; r < 3; r++) {
            const double f = A[3 * r + c] / A[3 * c + c];
            for (int k = c; k < 3; k++) A[3 * r + k] -= f * A[3 * c + k];
            b[r] -= f * b[c];
        }
    }
    for (int r = 2; r >= 0; r--) {
        double s = b[r];
        for (int k = r + 1; k < 3; k++) s -= A[3 * r + k] * b[k];
        b[r] = s / A[3 * r + r];
    }
    return true;
}

__global__ void __launch_bounds__(128) tri_kernel(TriArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n_tracks) return;
    const int64_t o = a.ptr[k];
    const int n = (int)(a.ptr[k + 1] - o);
    double* Xo = a.X + 3 * (int64_t)k;
    Xo[0] = Xo[1] = Xo[2] = __longlong_as_double(0x7ff8000000000000LL);
    a.err[k] = __longlong_as_double(0x7ff8000000000000LL);
    if (n < 2) { a.status[k] = -2; return; }       // InsufficientDataError
    double C0[3];
    bool all_same = true;
    for (int i = 0; i < n; i++) {
        const int c = a.cam[o + i];
        const double* R = a.R + 9 * c;
        const double* t = a.t + 3 * c;
        double C[3];
        for (int j = 0; j < 3; j++) C[j] = -(R[j] * t[0] + R[3 + j] * t[1] + R[6 + j] * t[2]);
        if (i == 0) { C0[0] = C[0]; C0[1] = C[1]; C0[2] = C[2]; }
        const double d0 = C[0] - C0[0], d1 = C[1] - C0[1], d2 = C[2] - C0[2];
        if (!(sqrt(d0 * d0 + d1 * d1 + d2 * d2) < 1e-12)) all_same = false;
    }
    if (all_same) { a.status[k] = -1; return; }     // DegenerateGeometryError
    // normal matrix of the DLT rows u*P3 - P1, v*P3 - P2 (P = K [R|t])
    double N[16];
    for (int i = 0; i < 16; i++) N[i] = 0.0;
    for (int i = 0; i < n; i++) {
        const int c = a.cam[o + i];
        const double* R = a.R + 9 * c;
        const double* t = a.t + 3 * c;
        const double* K = a.K + 9 * c;
        double P[12];
        for (int r = 0; r < 3; r++)
            for (int cc = 0; cc < 4; cc++) {
                double s = 0.0;
                for (int q = 0; q < 3; q++) s += K[3 * r + q] * (cc < 3 ? R[3 * q + cc] : t[q]);
                P[4 * r + cc] = s;
            }
        const double u = a.pix[2 * (o + i)], v = a.pix[2 * (o + i) + 1];
        double r1[4], r2[4];
        for (int cc = 0; cc < 4; cc++) {
            r1[cc] = u * P[8 + cc] - P[cc];
            r2[cc] = v * P[8 + cc] - P[4 + cc];
        }
        for (int p = 0; p < 4; p++)
            for (int q = 0; q < 4; q++) N[4 * p + q] += r1[p] * r1[q] + r2[p] * r2[q];
    }
    double V[16];
    jacobi4(N, V);
    int m = 0;
    for (int i = 1; i < 4; i++)
        if (N[5 * i] < N[5 * m]) m = i;
    const double Xh[4] = {V[m], V[4 + m], V[8 + m], V[12 + m]};
    const double n3 = sqrt(Xh[0] * Xh[0] + Xh[1] * Xh[1] + Xh[2] * Xh[2]);
    if (fabs(Xh[3]) < 1e-12 * n3) { a.status[k] = -1; return; }   // parallel rays
    double X[3] = {Xh[0] / Xh[3], Xh[1] / Xh[3], Xh[2] / Xh[3]};
    bool depth_ok;
    double err = reproject(a, o, n, X, &depth_ok);
    if (isfinite(err)) {
        // one Gauss-Newton pass (geometry.py:322-344), f = K[0,0]
        double H[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, g[3] = {0, 0, 0};
        for (int i = 0; i < n; i++) {
            const int c = a.cam[o + i];
            const double* R = a.R + 9 * c;
            const double* t = a.t + 3 * c;
            const double* K = a.K + 9 * c;
            double xc[3];
            for (int j = 0; j < 3; j++) xc[j] = R[3 * j] * X[0] + R[3 * j + 1] * X[1] + R[3 * j + 2] * X[2] + t[j];
            double uv[3];
            for (int j = 0; j < 3; j++) uv[j] = K[3 * j] * xc[0] + K[3 * j + 1] * xc[1] + K[3 * j + 2] * xc[2];
            const double rr[2] = {uv[0] / uv[2] - a.pix[2 * (o + i)], uv[1] / uv[2] - a.pix[2 * (o + i) + 1]};
            const double f = K[0], z = xc[2];
            const double du[2][3] = {{f / z, 0.0, -f * xc[0] / (z * z)}, {0.0, f / z, -f * xc[1] / (z * z)}};
            double J[2][3];
            for (int r = 0; r < 2; r++)
                for (int cc = 0; cc < 3; cc++)
                    J[r][cc] = du[r][0] * R[cc] + du[r][1] * R[3 + cc] + du[r][2] * R[6 + cc];
            for (int p = 0; p < 3; p++) {
                for (int q = 0; q < 3; q++) H[3 * p + q] += J[0][p] * J[0][q] + J[1][p] * J[1][q];
                g[p] += J[0][p] * rr[0] + J[1][p] * rr[1];
            }
        }
        for (int p = 0; p < 3; p++) H[4 * p] += 1e-12;
        double step[3] = {-g[0], -g[1], -g[2]};
        if (solve3(H, step)) {
            const double Xn[3] = {X[0] + step[0], X[1] + step[1], X[2] + step[2]};
            bool dn;
            const double en = reproject(a, o, n, Xn, &dn);
            if (isfinite(en) && en <= err) {
                X[0] = Xn[0]; X[1] = Xn[1]; X[2] = Xn[2];
                err = en;
                depth_ok = dn;
            }
        }
    }
    Xo[0] = X[0]; Xo[1] = X[1]; Xo[2] = X[2];
    a.err[k] = err;
    if (!isfinite(err) || !depth_ok || err > a.max_error) { a.status[k] = 0; return; }
    // widest pairwise ray angle >= min_angle (geometry.py:350-356).  The gate only
    // asks whether the widest angle reaches min_angle: the first pair whose own
    // angle (the same acos formula, monotone in the cosine) reaches it settles the
    // status, so well-spread tracks stop after a few pairs instead of n^2/2
    const double deg = 180.0 / 3.141592653589793;
    double minc = 1.0;
    for (int i = 0; i < n; i++) {
        double ri[3];
        {
            const int c = a.cam[o + i];
            const double* R = a.R + 9 * c;
            const double* t = a.t + 3 * c;
            for (int j = 0; j < 3; j++) ri[j] = X[j] + (R[j] * t[0] + R[3 + j] * t[1] + R[6 + j] * t[2]);
            const double nr = fmax(sqrt(ri[0] * ri[0] + ri[1] * ri[1] + ri[2] * ri[2]), 1e-15);
            for (int j = 0; j < 3; j++) ri[j] /= nr;
        }
        for (int jj = i + 1; jj < n; jj++) {
            const int c = a.cam[o + jj];
            const double* R = a.R + 9 * c;
            const double* t = a.t + 3 * c;
            double rj[3];
            for (int j = 0; j < 3; j++) rj[j] = X[j] + (R[j] * t[0] + R[3 + j] * t[1] + R[6 + j] * t[2]);
            const double nr = fmax(sqrt(rj[0] * rj[0] + rj[1] * rj[1] + rj[2] * rj[2]), 1e-15);
            const double cs = (ri[0] * rj[0] + ri[1] * rj[1] + ri[2] * rj[2]) / nr;
            if (cs < minc) {
                minc = cs;
                if (!(acos(fmin(fmax(minc, -1.0), 1.0)) * deg < a.min_angle_deg)) {
                    a.status[k] = 1;
                    return;
                }
            }
        }
    }
    const double ang = acos(fmin(fmax(minc, -1.0), 1.0)) * deg;
    a.status[k] = ang < a.min_angle_deg ? 0 : 1;
}

}  // namespace
}  // namespace msfm

using namespace msfm;

extern "C" int msfm_triangulate_batch(const double* d_K, const double* d_R, const double* d_t,
                                      int32_t n_tracks, const int64_t* d_ptr,
                                      const int32_t* d_cam, const double* d_pix, double max_error,
                                      double min_angle_deg, double* d_X, double* d_err,
                                      int32_t* d_status, void* stream) {
    if (n_tracks < 0) {
        set_error("msfm_triangulate_batch: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_tracks == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    TriArgs a{d_K, d_R, d_t, d_ptr, d_cam, d_pix, n_tracks, max_error, min_angle_deg, d_X, d_err,
              d_status};
    {
        ProfScope ps("tri_kernel", st);
        tri_kernel<<<(n_tracks + 127) / 128, 128, 0, st>>>(a);
    }
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}
