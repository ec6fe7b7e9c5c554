// 3D-2D localization kNN on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// Native body of DescriptorIndex.knn2's exact path (descriptors.py:35-72) for the
// queries of direct_3d2d_search (localize.py:99-122), batched over points x
// images.  A point is its track-descriptor sum S (<= 255 n) and track length n
// (mean = S/n, localize.py:51-59); against feature f the exact rank key is
//     key = n |f|^2 - 2 S.f            (N = |S - n f|^2 = n*key + |S|^2)
// 2 S.f is computed exactly as two u8 x u8 -> s32 GEMMs over the digit planes
// 2S = lo + 256 hi (lo = 2 (S mod 128), hi = S >> 7).  Per (point, image) the epilogue keeps the running top-2
// (lowest feature index wins ties), so no distance matrix is ever stored.
//
// CTA (persistent, 1 per SM, 384 threads):
//   warp 0      TMA producer: A planes (128 points x 128 B, once per unit) and
//               B tiles (128 features x 128 B, 4-stage ring), SWIZZLE_128B
//   warp 1      MMA issuer: tcgen05.mma M=128 N=128 K=32 x 4 per plane,
//               accumulators in TMEM (2 stages x 2 planes x 128 columns)
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: tcgen05.ld -> key -> top-2, 2 warps per lane quadrant
// unit = (image, 128-point tile), image-major; tile = 128 features of that image.
#include <cuda.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace msfm {
namespace {

#ifndef MSFM_KNN_EPI_WARPS
#define MSFM_KNN_EPI_WARPS 16
#endif
constexpr int KN_STAGES = 4;
constexpr int TILE_M = 128, TILE_N = 128, KB = 128;   // K = 128 bytes per plane
constexpr int EPI_WARP0 = 4, EPI_WARPS = MSFM_KNN_EPI_WARPS;
constexpr int KN_THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int EPI_COLS = TILE_N / (EPI_WARPS / 4);   // columns per epilogue warp per tile
constexpr uint32_t B_TILE_BYTES = TILE_N * KB;          // 16 KB
constexpr uint32_t A_PLANE_BYTES = TILE_M * KB;         // 16 KB
constexpr int INT_BIG = 0x7fffffff;

constexpr long long KEY_BIG64 = 0x7fffffffffffffffLL;   // "no second neighbour"

struct KnnSmem {
    uint8_t a[3][A_PLANE_BYTES];            // digit planes of 2S (1024-B aligned)
    uint8_t b[KN_STAGES][B_TILE_BYTES];
    uint64_t full[KN_STAGES], empty[KN_STAGES];
    uint64_t a_full, a_empty;
    uint64_t t_full[2], t_empty[2];
    uint32_t tmem_base;
    long long merge_k1[EPI_WARPS / 4][TILE_M], merge_k2[EPI_WARPS / 4][TILE_M];
    int merge_i1[EPI_WARPS / 4][TILE_M];
    // fvs[fn_stride]: |f|^2 of the current unit's image; with SAVEK it is followed by
    // savek[EPI_WARPS * 32][16]: per epilogue thread, the 16 keys of the chunk that
    // holds its running best (the column is looked up once per unit)
    alignas(16) int fvs[];   // |f|^2 of the current unit's image (fn_stride ints)
};

struct KnnArgs {
    const int32_t* count;      // rows of this launch's point subset (device)
    const int32_t* rowmap;     // subset row -> output row
    const int32_t* n;          // [M_pad] track length of each subset row
    const int32_t* fnorm;      // bank |f|^2
    const int32_t* fn_pad;     // [n_img][fn_stride] |f|^2 per query image, 16-B aligned tiles
    int fn_stride;
    const int64_t* img_off;    // bank image offsets
    const int32_t* img_n;      // bank image sizes
    const int32_t* images;     // [n_img] bank image index of each query image
    int n_img;
    int M;                     // real points
    long long* out_k1;         // [n_img][M_pad] (output rows)
    int32_t* out_i1;
    long long* out_k2;
    int M_pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Bounded wait with back-off (epilogue warps waiting for the next accumulator
// should not steal issue slots from the warps still draining the current one).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity) {
    const uint32_t addr = smem_u32(b);
    uint32_t done = 0;
    for (long long it = 0; it < (1LL << 28); it++) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
#ifndef MSFM_KNN_NO_BACKOFF
        __nanosleep(64);
#endif
    }
    __trap();
}

// Bounded wait: a protocol bug traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t addr = smem_u32(b);
    uint32_t done = 0;
    for (long long it = 0; it < (1LL << 31); it++) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// K-major, 128-byte swizzle UMMA shared-memory descriptor (8 rows x 128 B atoms)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8-row group stride
    d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}

// instruction descriptor: kind::i8, D = s32, A/B unsigned 8-bit, K-major, M=128, N=128
constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TILE_N >> 3) << 17) |
                           ((uint32_t)(TILE_M >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
        " [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ uint4 lds_u4(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
    return v;
}

__device__ __forceinline__ void sts_u4(void* p, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ int unit_tiles(const KnnArgs& a, int m_tiles, int u, int& img, int& mt,
                                          int64_t& off, int& n) {
    // image-major: the CTAs running at one time share a few images' feature tiles
    // (L2 hits) instead of streaming every image once per point tile
    const int s = u / m_tiles;
    mt = u - s * m_tiles;
    img = a.images[s];
    off = a.img_off[img];
    n = a.img_n[img];
    return (n + TILE_N - 1) / TILE_N;
}

// PLANES = 2: track length <= 100 (2S = lo + 256 hi, int32 keys, two accumulator
// stages of 2 x 128 TMEM columns).  PLANES = 3: any track length up to 32767 (2S
// in base-256 digits, int64 keys, one stage of 3 x 128 columns).
constexpr size_t SAVEK_BYTES = (size_t)EPI_WARPS * 32 * 16 * sizeof(int);

template <int PLANES, bool SAVEK>
__global__ void __launch_bounds__(KN_THREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap map_p0, const __grid_constant__ CUtensorMap map_p1,
              const __grid_constant__ CUtensorMap map_p2, const __grid_constant__ CUtensorMap map_b,
              KnnArgs a) {
    using Key = typename std::conditional<PLANES == 2, int, long long>::type;
    constexpr Key KBIG = PLANES == 2 ? (Key)INT_BIG : (Key)KEY_BIG64;
    constexpr int ACC_STAGES = PLANES == 2 ? 2 : 1;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    KnnSmem& S = *reinterpret_cast<KnnSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int count = *a.count;
    const int m_tiles = (count + TILE_M - 1) / TILE_M;
    const int n_units = m_tiles * a.n_img;
    if (n_units == 0) return;
    const CUtensorMap* maps[3] = {&map_p0, &map_p1, &map_p2};

    if (threadIdx.x == 0) {
        for (int s = 0; s < KN_STAGES; s++) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        mbar_init(&S.a_full, 1);
        mbar_init(&S.a_empty, 1);
        for (int s = 0; s < 2; s++) {
            mbar_init(&S.t_full[s], 1);
            mbar_init(&S.t_empty[s], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = S.tmem_base;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            int first = 1;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                int img, mt, n;
                int64_t off;
                const int nt = unit_tiles(a, m_tiles, u, img, mt, off, n);
                if (nt == 0) continue;
                if (!first) {
                    mbar_wait(&S.a_empty, a_phase);
                    a_phase ^= 1;
                }
                first = 0;
                mbar_expect_tx(&S.a_full, PLANES * A_PLANE_BYTES);
#pragma unroll
                for (int p = 0; p < PLANES; p++) tma_load_2d(S.a[p], maps[p], &S.a_full, 0, mt * TILE_M);
                for (int j = 0; j < nt; j++) {
                    mbar_wait(&S.empty[stage], phase ^ 1);
                    mbar_expect_tx(&S.full[stage], B_TILE_BYTES);
                    tma_load_2d(S.b[stage], &map_b, &S.full[stage], 0, (int)(off + (int64_t)j * TILE_N));
                    if (++stage == KN_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            int stage = 0, acc = 0;
            uint32_t phase = 0, a_phase = 0, acc_phase = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                int img, mt, n;
                int64_t off;
                const int nt = unit_tiles(a, m_tiles, u, img, mt, off, n);
                if (nt == 0) continue;
                mbar_wait(&S.a_full, a_phase);
                a_phase ^= 1;
                tc_fence_after();
                for (int j = 0; j < nt; j++) {
                    mbar_wait(&S.t_empty[acc], acc_phase ^ 1);
                    mbar_wait(&S.full[stage], phase);
                    tc_fence_after();
                    const uint32_t b_addr = smem_u32(S.b[stage]);
#pragma unroll
                    for (int p = 0; p < PLANES; p++) {
                        const uint32_t d = tbase + (uint32_t)(acc * 256 + p * 128);
                        const uint32_t ap = smem_u32(S.a[p]);
#pragma unroll
                        for (int k = 0; k < KB / 32; k++)
                            umma_i8(d, umma_desc_sw128(ap + 32 * k), umma_desc_sw128(b_addr + 32 * k), k > 0);
                    }
                    umma_commit(&S.empty[stage]);     // B stage reusable once these MMAs retire
                    umma_commit(&S.t_full[acc]);      // accumulator ready for the epilogue
                    if (++stage == KN_STAGES) { stage = 0; phase ^= 1; }
                    if (++acc == ACC_STAGES) { acc = 0; acc_phase ^= 1; }
                }
                umma_commit(&S.a_empty);              // A planes reusable after this unit
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------- epilogue
        const int ew = warp - EPI_WARP0;          // 0..EPI_WARPS-1
        const int quad = warp & 3;                // TMEM lane quadrant this warp may access
        const int half = ew >> 2;                 // column slice
        const int row = quad * 32 + lane;         // point row within the tile
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            int img, mt, n;
            int64_t off;
            const int nt = unit_tiles(a, m_tiles, u, img, mt, off, n);
            const int grow = mt * TILE_M + row;
            const int np = grow < count ? a.n[grow] : 0;
            {
                // stage the image's |f|^2 row in shared memory (broadcast reads per chunk)
                const int slot = u / m_tiles;       // image slot of the unit (unit_tiles)
                const int4* src = reinterpret_cast<const int4*>(a.fn_pad + (int64_t)slot * a.fn_stride);
                int4* dst = reinterpret_cast<int4*>(S.fvs);
                for (int i = ew * 32 + lane; i < a.fn_stride / 4; i += EPI_WARPS * 32) dst[i] = __ldg(src + i);
                asm volatile("bar.sync 1, %0;" ::"r"(EPI_WARPS * 32));
            }
            // running top-2 of this row over its column slice: k1 (best key), k2 (second
            // smallest key value), best column = ibase + il.
            Key k1 = KBIG, k2 = KBIG;
            int il = 0, ibase = 0;
            for (int j = 0; j < nt; j++) {
                mbar_wait_backoff(&S.t_full[acc], acc_phase);
                tc_fence_after();
                const uint32_t t0 = tbase + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 256 + half * EPI_COLS);
                const int cbase = j * TILE_N + half * EPI_COLS;
                const uint4* fp = reinterpret_cast<const uint4*>(S.fvs + cbase);
                const bool full = cbase + EPI_COLS <= n;
                // scores of one 16-column chunk -> running top-2 (FULLC: every column is
                // a feature of the image, no per-column bound tests)
                auto scores = [&](int c0, const uint32_t (&pl)[PLANES][16], auto full_tag) {
                    constexpr bool FULLC = decltype(full_tag)::value;
                    int fv[16];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint4 f4 = lds_u4(fp + (c0 >> 2) + q);
                        fv[4 * q] = (int)f4.x; fv[4 * q + 1] = (int)f4.y;
                        fv[4 * q + 2] = (int)f4.z; fv[4 * q + 3] = (int)f4.w;
                    }
                    const Key k1_in = k1;
                    const int lim = FULLC ? 16 : n - (cbase + c0);
                    Key key[16];
#pragma unroll
                    for (int c = 0; c < 16; c++) {
                        if (PLANES == 2) {
                            key[c] = (Key)(np * fv[c] - ((int)pl[0][c] + ((int)pl[1][c] << 8)));
                        } else {
                            key[c] = (Key)((long long)np * fv[c] -
                                           ((long long)pl[0][c] + ((long long)pl[1][c] << 8) +
                                            ((long long)pl[PLANES - 1][c] << 16)));
                        }
                        if (!FULLC && c >= lim) key[c] = KBIG;
                    }
                    // values only in the loop (three min/max per score); the column of a
                    // new best is found afterwards, rarely
#pragma unroll
                    for (int c = 0; c < 16; c++) {
                        k2 = min(k2, max(k1, key[c]));
                        k1 = min(k1, key[c]);
                    }
                    if (SAVEK) {
                        // a new best: keep the chunk's keys (predicated stores, no
                        // divergent search); its column is found once per unit
                        if (k1 != k1_in) {
                            uint4* sk = reinterpret_cast<uint4*>(S.fvs + a.fn_stride) + (ew * 32 + lane) * 4;
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                sts_u4(sk + q, make_uint4((unsigned)key[4 * q], (unsigned)key[4 * q + 1],
                                                          (unsigned)key[4 * q + 2], (unsigned)key[4 * q + 3]));
                            ibase = cbase + c0;
                        }
                    } else if (k1 != k1_in) {
#pragma unroll
                        for (int c = 15; c >= 0; c--)
                            if (key[c] == k1) il = c;     // lowest column at the best
                        ibase = cbase + c0;
                    }
                };
                auto release = [&]() {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&S.t_empty[acc]);
                };
#pragma unroll
                for (int c0 = 0; c0 < EPI_COLS; c0 += 16) {
                    uint32_t pl[PLANES][16];
#pragma unroll
                    for (int p = 0; p < PLANES; p++) tmem_ld16(t0 + p * 128 + c0, pl[p]);
                    tmem_wait_ld();
                    if (full) scores(c0, pl, std::true_type{});
                    else      scores(c0, pl, std::false_type{});
                }
                release();
                if (++acc == ACC_STAGES) { acc = 0; acc_phase ^= 1; }
            }
            if (SAVEK && k1 != KBIG) {
                const int* sk = S.fvs + a.fn_stride + (ew * 32 + lane) * 16;
                il = 15;
                for (int c = 15; c >= 0; c--)
                    if ((Key)sk[c] == k1) il = c;         // lowest column at the best
            }
            int i1 = k1 == KBIG ? -1 : ibase + il;
            // merge the column slices of each row
            S.merge_k1[half][row] = k1 == KBIG ? KEY_BIG64 : (long long)k1;
            S.merge_i1[half][row] = i1;
            S.merge_k2[half][row] = k2 == KBIG ? KEY_BIG64 : (long long)k2;
            asm volatile("bar.sync 1, %0;" ::"r"(EPI_WARPS * 32));
            if (half == 0) {
                long long b1 = S.merge_k1[0][row], b2 = S.merge_k2[0][row];
                for (int h = 1; h < EPI_WARPS / 4; h++) {
                    const long long ok1 = S.merge_k1[h][row], ok2 = S.merge_k2[h][row];
                    const int oi1 = S.merge_i1[h][row];
                    // best = min by (key, index); second = 2nd smallest key value
                    const bool other_first = (ok1 < b1) || (ok1 == b1 && oi1 >= 0 && (i1 < 0 || oi1 < i1));
                    const long long hi_k = other_first ? b1 : ok1;
                    if (other_first) { b1 = ok1; i1 = oi1; }
                    b2 = min(hi_k, min(b2, ok2));
                }
                const int slot = u / m_tiles;       // image slot of the unit (unit_tiles)
                if (grow < count) {
                    const int64_t o = (int64_t)slot * a.M_pad + a.rowmap[grow];
                    a.out_k1[o] = b1; a.out_i1[o] = i1; a.out_k2[o] = b2;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(EPI_WARPS * 32));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
}

// ------------------------------------------------------------------ helpers
__global__ void fn_pad_kernel(const int32_t* __restrict__ fnorm, const int64_t* __restrict__ img_off,
                              const int32_t* __restrict__ img_n, const int32_t* __restrict__ images,
                              int stride, int32_t* __restrict__ out) {
    const int s = blockIdx.y;
    const int img = images[s];
    const int64_t off = img_off[img];
    const int n = img_n[img];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < stride; j += gridDim.x * blockDim.x)
        out[(int64_t)s * stride + j] = j < n ? fnorm[off + j] : 0;
}

// Split the points into the short-track (n <= SHORT_N, two planes) and long-track
// (three planes) subsets: a warp per point row claims a slot in its subset, writes
// the row's digit planes there and the subset -> point row map.  Slot order inside
// a subset is arbitrary (every row's top-2 is independent of its tile mates).
constexpr int SHORT_N = 100;
__global__ void digit_planes_kernel(const int32_t* __restrict__ S, const int32_t* __restrict__ n,
                                    int64_t M, int32_t* __restrict__ cnt,
                                    uint8_t* __restrict__ s_lo, uint8_t* __restrict__ s_hi,
                                    int32_t* __restrict__ s_n, int32_t* __restrict__ s_map,
                                    uint8_t* __restrict__ l_p0, uint8_t* __restrict__ l_p1,
                                    uint8_t* __restrict__ l_p2, int32_t* __restrict__ l_n,
                                    int32_t* __restrict__ l_map) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= M) return;
    const int nr = n[r];
    const bool lng = nr > SHORT_N;
    int pos = 0;
    if (lane == 0) pos = atomicAdd(cnt + (lng ? 1 : 0), 1);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (lane == 0) {
        if (lng) { l_n[pos] = nr; l_map[pos] = (int32_t)r; }
        else     { s_n[pos] = nr; s_map[pos] = (int32_t)r; }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int k = lane + 32 * q;
        const int v = S[r * 128 + k];
        const int64_t o = (int64_t)pos * 128 + k;
        if (!lng) {
            // 2S = lo + 256 hi, lo = 2 (S mod 128), hi = S >> 7 (S <= 255 * 100)
            s_lo[o] = (uint8_t)((v & 127) << 1);
            s_hi[o] = (uint8_t)(v >> 7);
        } else {
            // 2S in base-256 digits (S <= 255 * 32767 < 2^23)
            const int w = 2 * v;
            l_p0[o] = (uint8_t)(w & 255);
            l_p1[o] = (uint8_t)((w >> 8) & 255);
            l_p2[o] = (uint8_t)(w >> 16);
        }
    }
}

// ratio test + one point per feature (localize.py:108-122, matching.py:82-103)
struct DirectArgs {
    const int32_t* n; const int64_t* SS; const long long* k1; const int32_t* i1; const long long* k2;
    const int32_t* images; const int32_t* img_n;
    int32_t* win; const int64_t* win_off; int32_t* row_out; int32_t* fid_out; int32_t* cnt_out;
    int M, M_pad, n_img;
    long long p, q;
    double cap;
};

__device__ __forceinline__ long long exact_N(const DirectArgs& a, int s, int r, long long k) {
    return (long long)a.n[r] * k + a.SS[r];
}

__device__ __forceinline__ bool accepted(const DirectArgs& a, int s, int r, long long& Nb) {
    const int64_t o = (int64_t)s * a.M_pad + r;
    const int i1 = a.i1[o];
    if (i1 < 0) return false;
    Nb = exact_N(a, s, r, a.k1[o]);
    const long long k2 = a.k2[o];
    if (k2 == KEY_BIG64) return sqrt((double)Nb) / (double)a.n[r] < a.cap;
    const long long Ns = exact_N(a, s, r, k2);
    return (__int128)a.q * a.q * Nb < (__int128)a.p * a.p * Ns;
}

// total order on (N/n^2, row): true if row r beats row c
__device__ __forceinline__ bool closer(const DirectArgs& a, int s, int r, long long Nr, int c) {
    const int64_t oc = (int64_t)s * a.M_pad + c;
    const long long Nc = exact_N(a, s, c, a.k1[oc]);
    const __int128 lhs = (__int128)Nr * a.n[c] * a.n[c];
    const __int128 rhs = (__int128)Nc * a.n[r] * a.n[r];
    return lhs < rhs || (lhs == rhs && r < c);
}

__global__ void direct_claim_kernel(DirectArgs a) {
    const int s = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.M) return;
    long long Nb;
    if (!accepted(a, s, r, Nb)) return;
    const int f = a.i1[(int64_t)s * a.M_pad + r];
    int* w = a.win + a.win_off[s] + f;
    int cur = *w;
    while (cur < 0 || closer(a, s, r, Nb, cur)) {
        const int prev = atomicCAS(w, cur, r);
        if (prev == cur) break;
        cur = prev;
    }
}

__global__ void direct_init_kernel(DirectArgs a) {
    const int s = blockIdx.y;
    const int n = a.img_n[a.images[s]];
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x)
        a.win[a.win_off[s] + f] = -1;
}

__global__ void __launch_bounds__(1024) direct_compact_kernel(DirectArgs a) {
    __shared__ int wsum[33];
    const int s = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int carry = 0;
    for (int r0 = 0; r0 < a.M; r0 += 1024) {
        const int r = r0 + threadIdx.x;
        bool keep = false;
        int f = -1;
        if (r < a.M) {
            long long Nb;
            if (accepted(a, s, r, Nb)) {
                f = a.i1[(int64_t)s * a.M_pad + r];
                keep = a.win[a.win_off[s] + f] == r;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        if (wid == 0) {
            int v = wsum[lane], x = v;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            wsum[lane] = x - v;
            if (lane == 31) wsum[32] = x;
        }
        __syncthreads();
        if (keep) {
            const int pos = carry + wsum[wid] + __popc(bal & ((1u << lane) - 1u));
            a.row_out[(int64_t)s * a.M_pad + pos] = r;
            a.fid_out[(int64_t)s * a.M_pad + pos] = f;
        }
        carry += wsum[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.cnt_out[s] = carry;
}

// index of the second neighbour (lowest feature index with key == k2, other than
// i1): one warp per (query image slot, point), lanes over features, early exit
__global__ void knn_second_kernel(const uint8_t* __restrict__ desc, const int32_t* __restrict__ fnorm,
                                  const int64_t* __restrict__ img_off, const int32_t* __restrict__ img_n,
                                  const int32_t* __restrict__ images, int n_img, int M, int M_pad,
                                  const int32_t* __restrict__ S, const int32_t* __restrict__ n,
                                  const long long* __restrict__ k1, const int32_t* __restrict__ i1,
                                  const long long* __restrict__ k2, int32_t* __restrict__ i2) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n_img * M) return;
    const int s = warp / M, r = warp - s * M;
    const int64_t o = (int64_t)s * M_pad + r;
    const long long want = k2[o];
    const int best = i1[o];
    if (lane == 0) i2[o] = -1;
    if (best < 0 || want == KEY_BIG64) return;
    const int img = images[s];
    const int64_t off = img_off[img];
    const int nf = img_n[img];
    const int np = n[r];
    const int32_t* Sr = S + (int64_t)r * 128;
    for (int f0 = 0; f0 < nf; f0 += 32) {
        const int f = f0 + lane;
        bool hit = false;
        if (f < nf && f != best) {
            const uint8_t* d = desc + (off + f) * 128;
            long long dot = 0;
            for (int k = 0; k < 128; k++) dot += (long long)Sr[k] * d[k];
            const long long key = (long long)np * fnorm[off + f] - 2 * dot;
            hit = key == want;
        }
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) {
            if (lane == 0) i2[o] = f0 + __ffs(b) - 1;
            return;
        }
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_rows128_map(CUtensorMap* map, const void* base, int64_t rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return MSFM_ECUDA;
        }
        fn = (EncodeTiledFn)p;
    }
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return MSFM_ECUDA;
    }
    return MSFM_OK;
}

}  // namespace
}  // namespace msfm

using namespace msfm;

static int64_t fn_stride_of(int32_t max_n) {
    return ((int64_t)(max_n > 0 ? max_n : 1) + TILE_N - 1) / TILE_N * TILE_N;
}

extern "C" size_t msfm_knn_workspace_bytes(int32_t n_points, int32_t n_images, int32_t max_n) {
    const int64_t M_pad = ((int64_t)n_points + TILE_M - 1) / TILE_M * TILE_M;
    // short subset: 2 planes, long subset: 3 planes (each sized for every point),
    // per-subset track lengths and row maps, 2 counters, the images' |f|^2 rows
    return aligned_bytes<uint8_t>(M_pad * 128) * 5 + aligned_bytes<int32_t>(M_pad) * 4 +
           aligned_bytes<int32_t>(2) +
           aligned_bytes<int32_t>((int64_t)(n_images > 0 ? n_images : 1) * fn_stride_of(max_n)) + 4096;
}

extern "C" int msfm_knn2_second_index(const msfm_bank* bank, int32_t n_points, const int32_t* d_S,
                                      const int32_t* d_n, int32_t n_images, const int32_t* d_images,
                                      const int64_t* d_k1, const int32_t* d_i1, const int64_t* d_k2,
                                      int32_t* d_i2, void* stream) {
    if (!bank || n_points < 0 || n_images < 0) {
        set_error("msfm_knn2_second_index: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_points == 0 || n_images == 0) return MSFM_OK;
    const int M_pad = (int)(((int64_t)n_points + TILE_M - 1) / TILE_M * TILE_M);
    const int64_t warps = (int64_t)n_images * n_points;
    knn_second_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        bank->d_desc, bank->d_norm2, bank->d_img_off, bank->d_img_n, d_images, n_images, n_points,
        M_pad, d_S, d_n, reinterpret_cast<const long long*>(d_k1), d_i1,
        reinterpret_cast<const long long*>(d_k2), d_i2);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

// one CTA per selected image, threads over its correspondences
__global__ void gather_3d2d_kernel(const int32_t* __restrict__ crow, const int32_t* __restrict__ cfid,
                                   int m_pad, const int64_t* __restrict__ sel,
                                   const int64_t* __restrict__ row0, const int64_t* __restrict__ out_off,
                                   const double* __restrict__ xyz, const float2* __restrict__ bxy,
                                   double* __restrict__ X, double* __restrict__ uv) {
    const int k = blockIdx.x;
    const int64_t src = (int64_t)sel[k] * m_pad, o = out_off[k], n = out_off[k + 1] - o;
    const int64_t r0 = row0[k];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t p = crow[src + i];
        const float2 q = bxy[r0 + cfid[src + i]];
        double* x = X + 3 * (o + i);
        x[0] = xyz[3 * p]; x[1] = xyz[3 * p + 1]; x[2] = xyz[3 * p + 2];
        uv[2 * (o + i)] = (double)q.x;
        uv[2 * (o + i) + 1] = (double)q.y;
    }
}

extern "C" int msfm_gather_3d2d(const int32_t* d_corr_row, const int32_t* d_corr_fid, int32_t m_pad,
                                int32_t n_sel, const int64_t* d_sel, const int64_t* d_row0,
                                const int64_t* d_out_off, const double* d_xyz,
                                const float* d_bank_xy, double* d_X, double* d_uv, void* stream) {
    if (n_sel < 0 || m_pad < 0) {
        set_error("msfm_gather_3d2d: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_sel == 0) return MSFM_OK;
    gather_3d2d_kernel<<<n_sel, 256, 0, (cudaStream_t)stream>>>(
        d_corr_row, d_corr_fid, m_pad, d_sel, d_row0, d_out_off, d_xyz,
        reinterpret_cast<const float2*>(d_bank_xy), d_X, d_uv);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

extern "C" int msfm_direct_3d2d(const msfm_bank* bank, int32_t n_points, const int32_t* d_n,
                                const int64_t* d_SS, int32_t n_images, const int32_t* d_images,
                                const int64_t* d_k1, const int32_t* d_i1, const int64_t* d_k2,
                                int64_t ratio_p, int64_t ratio_q, double single_cap,
                                int32_t* d_win, const int64_t* d_win_off, int32_t* d_corr_row,
                                int32_t* d_corr_fid, int32_t* d_corr_n, void* stream) {
    if (!bank || n_points < 0 || n_images < 0 || ratio_p <= 0 || ratio_q <= 0 ||
        ratio_p > (1 << 20) || ratio_q > (1 << 20)) {
        set_error("msfm_direct_3d2d: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_images == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DirectArgs a;
    a.n = d_n; a.SS = d_SS; a.k1 = reinterpret_cast<const long long*>(d_k1); a.i1 = d_i1;
    a.k2 = reinterpret_cast<const long long*>(d_k2);
    a.images = d_images; a.img_n = bank->d_img_n;
    a.win = d_win; a.win_off = d_win_off; a.row_out = d_corr_row; a.fid_out = d_corr_fid;
    a.cnt_out = d_corr_n;
    a.M = n_points;
    a.M_pad = (int)(((int64_t)n_points + TILE_M - 1) / TILE_M * TILE_M);
    a.n_img = n_images;
    a.p = ratio_p; a.q = ratio_q; a.cap = single_cap;
    if (n_points == 0) {
        MSFM_CUDA_TRY(cudaMemsetAsync(d_corr_n, 0, sizeof(int32_t) * n_images, st));
        return MSFM_OK;
    }
    direct_init_kernel<<<dim3(16, n_images), 256, 0, st>>>(a);
    direct_claim_kernel<<<dim3((n_points + 255) / 256, n_images), 256, 0, st>>>(a);
    direct_compact_kernel<<<n_images, 1024, 0, st>>>(a);
    MSFM_LAUNCH_CHECK();
    count_launches(3);
    return MSFM_OK;
}

extern "C" int msfm_knn2_tracks(const msfm_bank* bank, int32_t n_points, const int32_t* d_S,
                                const int32_t* d_n, int32_t n_images, const int32_t* d_images,
                                int32_t max_track, int32_t max_n, int64_t* d_k1, int32_t* d_i1,
                                int64_t* d_k2, void* d_workspace, size_t workspace_bytes,
                                void* stream) {
    if (!bank || n_points < 0 || n_images < 0 || (n_points > 0 && (!d_S || !d_n))) {
        set_error("msfm_knn2_tracks: bad arguments");
        return MSFM_EINVAL;
    }
    if (max_track > 32767) {
        set_error("msfm_knn2_tracks: track length %d > 32767 (2S must fit three digit planes)",
                  max_track);
        return MSFM_EINVAL;
    }
    if (n_points == 0 || n_images == 0) return MSFM_OK;
    if (workspace_bytes < msfm_knn_workspace_bytes(n_points, n_images, max_n)) {
        set_error("msfm_knn2_tracks: workspace too small");
        return MSFM_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t M_pad = ((int64_t)n_points + TILE_M - 1) / TILE_M * TILE_M;
    Arena ar(d_workspace, workspace_bytes);
    uint8_t* s_lo = ar.take<uint8_t>(M_pad * 128);
    uint8_t* s_hi = ar.take<uint8_t>(M_pad * 128);
    uint8_t* l_p0 = ar.take<uint8_t>(M_pad * 128);
    uint8_t* l_p1 = ar.take<uint8_t>(M_pad * 128);
    uint8_t* l_p2 = ar.take<uint8_t>(M_pad * 128);
    int32_t* s_n = ar.take<int32_t>(M_pad);
    int32_t* s_map = ar.take<int32_t>(M_pad);
    int32_t* l_n = ar.take<int32_t>(M_pad);
    int32_t* l_map = ar.take<int32_t>(M_pad);
    int32_t* cnt = ar.take<int32_t>(2);
    const int64_t fstride = fn_stride_of(max_n);
    int32_t* fpad = ar.take<int32_t>((int64_t)n_images * fstride);
    fn_pad_kernel<<<dim3(8, n_images), 256, 0, st>>>(bank->d_norm2, bank->d_img_off, bank->d_img_n,
                                                    d_images, (int)fstride, fpad);
    MSFM_LAUNCH_CHECK();
    MSFM_CUDA_TRY(cudaMemsetAsync(cnt, 0, 2 * sizeof(int32_t), st));
    digit_planes_kernel<<<(unsigned)(((int64_t)n_points * 32 + 255) / 256), 256, 0, st>>>(
        d_S, d_n, n_points, cnt, s_lo, s_hi, s_n, s_map, l_p0, l_p1, l_p2, l_n, l_map);
    MSFM_LAUNCH_CHECK();
    const int64_t n_total = bank->n_total;
    if (n_total <= 0) {
        set_error("msfm_knn2_tracks: empty feature bank");
        return MSFM_EINVAL;
    }
    CUtensorMap ms0, ms1, ml0, ml1, ml2, mb;
    int rc;
    if ((rc = make_rows128_map(&ms0, s_lo, M_pad))) return rc;
    if ((rc = make_rows128_map(&ms1, s_hi, M_pad))) return rc;
    if ((rc = make_rows128_map(&ml0, l_p0, M_pad))) return rc;
    if ((rc = make_rows128_map(&ml1, l_p1, M_pad))) return rc;
    if ((rc = make_rows128_map(&ml2, l_p2, M_pad))) return rc;
    if ((rc = make_rows128_map(&mb, bank->d_desc, n_total))) return rc;
    KnnArgs a;
    a.fnorm = bank->d_norm2;
    a.fn_pad = fpad;
    a.fn_stride = (int)fstride;
    a.img_off = bank->d_img_off;
    a.img_n = bank->d_img_n;
    a.images = d_images;
    a.n_img = n_images;
    a.M = n_points;
    a.M_pad = (int)M_pad;
    a.out_k1 = reinterpret_cast<long long*>(d_k1);
    a.out_i1 = d_i1;
    a.out_k2 = reinterpret_cast<long long*>(d_k2);
    const size_t smem = sizeof(KnnSmem) + (size_t)fstride * sizeof(int32_t) + 1024;
    if (smem > 227 * 1024) {
        set_error("msfm_knn2_tracks: %d features per image exceed the shared-memory |f|^2 row",
                  max_n);
        return MSFM_EINVAL;
    }
    // the saved-chunk epilogue when its 32 KB fit next to the |f|^2 row
    const bool savek = smem + SAVEK_BYTES <= 227 * 1024;
    const size_t smem2 = savek ? smem + SAVEK_BYTES : smem;
    MSFM_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::min<size_t>(smem + SAVEK_BYTES, 227 * 1024)));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // the subsets' sizes stay on the device: each launch reads its count, grids are
    // sized for the worst case (persistent CTAs, surplus CTAs exit at once)
    const int64_t units = (M_pad / TILE_M) * n_images;
    const int grid = (int)(units < nsm ? units : nsm);
    {
        ProfScope ps("knn_tc_kernel", st);
        a.count = cnt; a.rowmap = s_map; a.n = s_n;
        if (savek) knn_tc_kernel<2, true><<<grid, KN_THREADS, smem2, st>>>(ms0, ms1, ms1, mb, a);
        else       knn_tc_kernel<2, false><<<grid, KN_THREADS, smem, st>>>(ms0, ms1, ms1, mb, a);
    }
    MSFM_LAUNCH_CHECK();
    if (max_track > SHORT_N) {
        ProfScope ps("knn_tc_kernel_long", st);
        a.count = cnt + 1; a.rowmap = l_map; a.n = l_n;
        knn_tc_kernel<3, false><<<grid, KN_THREADS, smem, st>>>(ml0, ml1, ml2, mb, a);
        MSFM_LAUNCH_CHECK();
        count_launches(1);
    }
    count_launches(4);
    return MSFM_OK;
}

// ---------------------------------------------------------------------------
// Real-valued 2-NN (two_nearest_bruteforce, descriptors.py:35-72, for float rows
// that are not integer-valued): one warp per query, lanes stride over the
// targets, squared distance as sum((q_i - t_i)^2) in f64 (each difference and
// square exact for f32 inputs), top-2 with the lowest target index winning ties.
namespace msfm {
namespace knnf {
__device__ __forceinline__ bool dless(double a, int64_t ia, double b, int64_t ib) {
    return a < b || (a == b && ia < ib);
}

__global__ void __launch_bounds__(256) knn_float_kernel(const float* __restrict__ q,
                                                        const float* __restrict__ t, int64_t nq,
                                                        int64_t nt, int dim, double* __restrict__ d2,
                                                        int64_t* __restrict__ idx) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nq) return;
    const float* qr = q + w * dim;
    double b1 = INFINITY, b2 = INFINITY;
    int64_t i1 = -1, i2 = -1;
    for (int64_t j = lane; j < nt; j += 32) {
        const float* tr = t + j * dim;
        double s = 0.0;
        for (int k = 0; k < dim; k++) {
            const double e = (double)__ldg(qr + k) - (double)__ldg(tr + k);
            s = fma(e, e, s);
        }
        if (dless(s, j, b1, i1)) { b2 = b1; i2 = i1; b1 = s; i1 = j; }
        else if (dless(s, j, b2, i2)) { b2 = s; i2 = j; }
    }
    for (int o = 16; o; o >>= 1) {
        const double c1 = __shfl_xor_sync(0xffffffffu, b1, o), c2 = __shfl_xor_sync(0xffffffffu, b2, o);
        const int64_t j1 = __shfl_xor_sync(0xffffffffu, i1, o), j2 = __shfl_xor_sync(0xffffffffu, i2, o);
        // merge two sorted pairs (b1 <= b2, c1 <= c2) into the smallest two
        if (dless(c1, j1, b1, i1)) {
            const double nb2 = dless(b1, i1, c2, j2) ? b1 : c2;
            const int64_t ni2 = dless(b1, i1, c2, j2) ? i1 : j2;
            b1 = c1; i1 = j1; b2 = nb2; i2 = ni2;
        } else if (dless(c1, j1, b2, i2)) {
            b2 = c1; i2 = j1;
        }
    }
    if (lane == 0) {
        d2[2 * w] = b1; d2[2 * w + 1] = b2;
        idx[2 * w] = i1; idx[2 * w + 1] = i2;
    }
}
}  // namespace knnf
}  // namespace msfm

extern "C" int msfm_knn2_float(const float* d_q, int64_t n_queries, const float* d_t,
                               int64_t n_targets, int32_t dim, double* d_d2, int64_t* d_idx,
                               void* stream) {
    if (n_queries < 0 || n_targets < 0 || dim <= 0) {
        set_error("msfm_knn2_float: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_queries == 0) return MSFM_OK;
    const int64_t threads = n_queries * 32;
    msfm::knnf::knn_float_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        d_q, d_t, n_queries, n_targets, dim, d_d2, d_idx);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

// ---------------------------------------------------------------------------
// K7 track sums (mean_descriptor, localize.py:51-59, in its exact integer form):
// one warp per point, lane l owns descriptor bytes [4l, 4l+4); S[p] = sum over the
// point's track (CSR rows of bank features) of the u8 rows, n[p] = track length,
// SS[p] = |S[p]|^2 in int64.  Coalesced 128-B row reads, no atomics.
namespace msfm {
namespace k7 {
__global__ void __launch_bounds__(256) track_sum_kernel(const uint8_t* __restrict__ desc,
                                                        const int64_t* __restrict__ ptr,
                                                        const int64_t* __restrict__ row, int64_t M,
                                                        int32_t* __restrict__ S, int32_t* __restrict__ n,
                                                        int64_t* __restrict__ SS) {
    const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= M) return;
    const int64_t a = ptr[p], b = ptr[p + 1];
    int s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int64_t o = a; o < b; o++) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(desc + row[o] * 128) + lane);
        s0 += w & 255; s1 += (w >> 8) & 255; s2 += (w >> 16) & 255; s3 += w >> 24;
    }
    reinterpret_cast<int4*>(S + p * 128)[lane] = make_int4(s0, s1, s2, s3);
    long long q = (long long)s0 * s0 + (long long)s1 * s1 + (long long)s2 * s2 + (long long)s3 * s3;
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) {
        n[p] = (int32_t)(b - a);
        SS[p] = q;
    }
}
}  // namespace k7
}  // namespace msfm

extern "C" int msfm_track_sums(const msfm_bank* bank, int64_t n_points, const int64_t* d_track_ptr,
                               const int64_t* d_track_row, int32_t* d_S, int32_t* d_n,
                               int64_t* d_SS, void* stream) {
    if (!bank || n_points < 0 || (n_points > 0 && (!d_track_ptr || !d_track_row || !d_S || !d_n ||
                                                   !d_SS))) {
        set_error("msfm_track_sums: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_points == 0) return MSFM_OK;
    const int64_t threads = n_points * 32;
    msfm::k7::track_sum_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        bank->d_desc, d_track_ptr, d_track_row, n_points, d_S, d_n, d_SS);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}
