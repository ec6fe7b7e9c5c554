// Block / device exclusive scans shared by the matcher and the track merge.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace msfm {
namespace {

template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* total, int* smem /*NT/32+1*/) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < NT / 32 ? smem[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NT / 32) smem[lane] = s;
        if (lane == NT / 32 - 1) smem[NT / 32] = s;
    }
    __syncthreads();
    int base = wid > 0 ? smem[wid - 1] : 0;
    *total = smem[NT / 32];
    __syncthreads();
    return base + x - v;
}

// exclusive scan of int32 (in place) over n elements: tiles of 4096
constexpr int SCAN_T = 1024, SCAN_PER = 4;
__global__ void scan_tiles_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* bsum) {
    __shared__ int sm[SCAN_T / 32 + 1];
    int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_PER;
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        if (i < n) s += in[i];
    }
    int total;
    block_exclusive_scan<SCAN_T>(s, &total, sm);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void scan_bsum_kernel(int32_t* bsum, int64_t nb) {
    __shared__ int sm[SCAN_T / 32 + 1];
    int carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
        int64_t i = b0 + threadIdx.x;
        int v = i < nb ? bsum[i] : 0;
        int total;
        int ex = block_exclusive_scan<SCAN_T>(v, &total, sm);
        if (i < nb) bsum[i] = carry + ex;
        carry += total;
    }
}

__global__ void scan_apply_kernel(int32_t* data, int64_t n, const int32_t* bsum, int32_t* copy,
                                  int32_t base0) {
    __shared__ int sm[SCAN_T / 32 + 1];
    int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_PER;
    int v[SCAN_PER];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        v[k] = i < n ? data[i] : 0;
        s += v[k];
    }
    int total;
    int ex = block_exclusive_scan<SCAN_T>(s, &total, sm) + bsum[blockIdx.x] + base0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        if (i < n) {
            data[i] = ex;
            if (copy) copy[i] = ex;
        }
        ex += v[k];
    }
}

// two independent exclusive scans of the same length in one launch set
// (blockIdx.y selects the array): the row and column bucket tables of a grid build
struct Scan2 {
    int32_t* data[2]; int32_t* copy[2]; int32_t* bsum[2];
    int64_t n; int32_t base0;
};

__global__ void scan2_tiles_kernel(Scan2 s) {
    __shared__ int sm[SCAN_T / 32 + 1];
    const int y = blockIdx.y;
    const int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_PER;
    int v = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        const int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        if (i < s.n) v += s.data[y][i];
    }
    int total;
    block_exclusive_scan<SCAN_T>(v, &total, sm);
    if (threadIdx.x == 0) s.bsum[y][blockIdx.x] = total;
}

__global__ void scan2_bsum_kernel(Scan2 s, int64_t nb) {
    __shared__ int sm[SCAN_T / 32 + 1];
    int32_t* bsum = s.bsum[blockIdx.y];
    int carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_T) {
        const int64_t i = b0 + threadIdx.x;
        const int v = i < nb ? bsum[i] : 0;
        int total;
        const int ex = block_exclusive_scan<SCAN_T>(v, &total, sm);
        if (i < nb) bsum[i] = carry + ex;
        carry += total;
    }
}

__global__ void scan2_apply_kernel(Scan2 s) {
    __shared__ int sm[SCAN_T / 32 + 1];
    const int y = blockIdx.y;
    int32_t* data = s.data[y];
    int32_t* copy = s.copy[y];
    const int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_PER;
    int v[SCAN_PER];
    int t = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        const int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        v[k] = i < s.n ? data[i] : 0;
        t += v[k];
    }
    int total;
    int ex = block_exclusive_scan<SCAN_T>(t, &total, sm) + s.bsum[y][blockIdx.x] + s.base0;
#pragma unroll
    for (int k = 0; k < SCAN_PER; k++) {
        const int64_t i = base + (int64_t)threadIdx.x * SCAN_PER + k;
        if (i < s.n) {
            data[i] = ex;
            if (copy) copy[i] = ex;
        }
        ex += v[k];
    }
}

int exclusive_scan2(const Scan2& s, cudaStream_t st) {
    const int64_t nb = (s.n + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER);
    if (nb == 0) return MSFM_OK;
    scan2_tiles_kernel<<<dim3((unsigned)nb, 2), SCAN_T, 0, st>>>(s);
    scan2_bsum_kernel<<<dim3(1, 2), SCAN_T, 0, st>>>(s, nb);
    scan2_apply_kernel<<<dim3((unsigned)nb, 2), SCAN_T, 0, st>>>(s);
    MSFM_LAUNCH_CHECK();
    count_launches(3);
    return MSFM_OK;
}

// exclusive prefix sums of data[0, n) in place (+ base0), mirrored into copy if given
int exclusive_scan(int32_t* data, int64_t n, int32_t* copy, int32_t* bsum, cudaStream_t st,
                   int32_t base0 = 0) {
    int64_t nb = (n + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER);
    if (nb == 0) return MSFM_OK;
    scan_tiles_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(data, n, bsum);
    scan_bsum_kernel<<<1, SCAN_T, 0, st>>>(bsum, nb);
    scan_apply_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(data, n, bsum, copy, base0);
    MSFM_LAUNCH_CHECK();
    count_launches(3);
    return MSFM_OK;
}

}  // namespace
}  // namespace msfm
