// Shared device helpers for libmsfm_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "msfm_b200.h"

namespace msfm {

void set_error(const char* fmt, ...);
void count_launches(int n);
bool profiling();
void prof_begin(const char* name, cudaStream_t st, void** token);
void prof_end(void* token, cudaStream_t st);

// RAII: CUDA events around the kernels launched in scope (when profiling is on)
struct ProfScope {
    void* tok;
    cudaStream_t st;
    ProfScope(const char* name, cudaStream_t s) : tok(nullptr), st(s) { prof_begin(name, s, &tok); }
    ~ProfScope() { prof_end(tok, st); }
};

#define MSFM_CUDA_TRY(expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            ::msfm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                              cudaGetErrorString(_e));                               \
            return MSFM_ECUDA;                                                       \
        }                                                                            \
    } while (0)

#define MSFM_LAUNCH_CHECK()                                                          \
    do {                                                                             \
        cudaError_t _e = cudaGetLastError();                                         \
        if (_e != cudaSuccess) {                                                     \
            ::msfm::set_error("%s:%d launch: %s", __FILE__, __LINE__,                \
                              cudaGetErrorString(_e));                               \
            return MSFM_ECUDA;                                                       \
        }                                                                            \
    } while (0)

// Bump allocator over a caller-provided workspace.
struct Arena {
    char* base;
    size_t cap, used;
    __host__ Arena(void* p, size_t n) : base((char*)p), cap(n), used(0) {}
    template <class T>
    __host__ T* take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        used = off + count * sizeof(T);
        return (T*)(base + off);
    }
    __host__ bool ok() const { return used <= cap; }
};

template <class T>
__host__ __device__ inline size_t aligned_bytes(size_t count) {
    return ((count * sizeof(T) + 255) & ~size_t(255));
}

// ---------------------------------------------------------------------------
// np.hypot on x86-64 glibc 2.39 = the non-FMA Borges kernel of
// sysdeps/ieee754/dbl-64/e_hypot.c.  Every product/sum is rounded separately
// (this translation unit is compiled with -fmad=false), which is what makes
// the line normalisation bit-identical to the reference's guided.py:356,445.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double hyp_kernel(double ax, double ay) {
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

__device__ __forceinline__ double np_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000LL);
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
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

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdULL;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ULL;
    z ^= z >> 33;
    return z;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace msfm
