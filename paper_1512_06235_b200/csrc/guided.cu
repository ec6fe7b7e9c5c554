// Geometry-aware (epipolar-guided) pair matching on sm_100a.
//
// Native body of msfm.guided.guided_match_pair (pkg/src/msfm/guided.py:393-480)
// batched over densify_stage's pair loop (densify.py:220-240), bit-exact with the
// reference.  Compiled with -fmad=false: every fp64
// product/sum that the reference rounds separately is rounded separately here,
// and the fused ones are written as explicit fma().
//
// Pipeline per chunk of pairs (all device-side, no host round trips):
//   plan     1 CTA      per-pair table / dedupe offsets (scan)
//   lines    CTA/pair   epipolar line, clip, bucket key, hash-group insert
//   groups   CTA/pair   compact occupied hash slots into group records
//   gscan    1 CTA      group prefix over pairs
//   scatter  CTA/pair   member lists
//   prep     thr/group  padded clip + sample count, member-band deviation -> strip R
//   match    warp/group strip gather, exact C' test, mma.sync u8 distance tiles,
//                      fp32 band prefilter (+exact fp64 fallback), top-2, ratio, dedupe
//   compact  CTA/pair   ordered compaction of dedupe winners
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace msfm {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long EMPTY = 0xffffffffffffffffull;
constexpr int CAP = 512;       // candidates per round (9-bit local index in keys)
constexpr int WARPS = 4;       // match kernel warps per CTA
constexpr unsigned NONE = 0xffffffffu;

// ------------------------------------------------------------------ geometry
// `hom @ F.T` as numpy/OpenBLAS rounds it: dgemm for >= 2 rows, dgemv for 1.
__device__ __forceinline__ void epiline(const double* F, double x, double y, bool single_row,
                                        double l[3]) {
#pragma unroll
    for (int i = 0; i < 3; i++) {
        if (single_row) l[i] = fma(x, F[3 * i], y * F[3 * i + 1]) + F[3 * i + 2];
        else            l[i] = fma(y, F[3 * i + 1], x * F[3 * i]) + F[3 * i + 2];
    }
}

// The segment-length tests of the clips (hypot(dx, dy) > tol, >= tol): glibc's hypot is
// within an ulp of the exact value, which is >= max(|dx|, |dy|), so a segment with a
// coordinate difference above 2 tol passes without evaluating the hypot.
__device__ __forceinline__ bool seg_gt(double dx, double dy, double tol) {
    if (fmax(fabs(dx), fabs(dy)) > 2.0 * tol) return true;
    return np_hypot(dx, dy) > tol;
}
__device__ __forceinline__ bool seg_not_lt(double dx, double dy, double tol) {
    if (fmax(fabs(dx), fabs(dy)) > 2.0 * tol) return true;
    return !(np_hypot(dx, dy) < tol);
}

// clip_lines_batch (guided.py:297-338) with pad 0.
__device__ bool clip_batch(const double l[3], double W, double H, double pa[2], double pb[2]) {
    const double a = l[0], b = l[1], c = l[2];
    const double x0 = -0.0, x1 = W, y0 = -0.0, y1 = H;
    double cx[4], cy[4];
    bool valid[4];
    const double xs[2] = {x0, x1}, ys[2] = {y0, y1};
#pragma unroll
    for (int k = 0; k < 2; k++) {
        double y = -(a * xs[k] + c) / b;
        valid[k] = fabs(b) > 1e-15 && y >= y0 - 1e-9 && y <= y1 + 1e-9;
        cx[k] = xs[k];
        cy[k] = y < y0 ? y0 : (y > y1 ? y1 : y);
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
        double x = -(b * ys[k] + c) / a;
        valid[k + 2] = fabs(a) > 1e-15 && x >= x0 - 1e-9 && x <= x1 + 1e-9;
        cx[k + 2] = x < x0 ? x0 : (x > x1 ? x1 : x);
        cy[k + 2] = ys[k];
    }
    double span = x1 - x0;
    if (y1 - y0 > span) span = y1 - y0;
    if (span < 1.0) span = 1.0;
    int imin = -1, imax = -1;
    double kmin = 0, kmax = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (!valid[k]) continue;
        double key = cx[k] * (4.0 * span) + cy[k];
        if (imin < 0 || key < kmin) { kmin = key; imin = k; }
        if (imax < 0 || key > kmax) { kmax = key; imax = k; }
    }
    if (imin < 0) return false;
    pa[0] = cx[imin]; pa[1] = cy[imin];
    pb[0] = cx[imax]; pb[1] = cy[imax];
    return seg_gt(pb[0] - pa[0], pb[1] - pa[1], 1e-12);
}

// clip_line_to_bounds (guided.py:140-170), scalar path, used with pad = d.
__device__ bool clip_scalar(double a, double b, double c, double W, double H, double pad,
                            double pa[2], double pb[2]) {
    const double x0 = -pad, x1 = W + pad, y0 = -pad, y1 = H + pad;
    double px[4], py[4];
    int n = 0;
    if (fabs(b) > 1e-15) {
        const double xs[2] = {x0, x1};
        for (int k = 0; k < 2; k++) {
            double y = -(a * xs[k] + c) / b;
            if (y0 - 1e-9 <= y && y <= y1 + 1e-9) {
                double yy = y < y0 ? y0 : y;
                yy = yy > y1 ? y1 : yy;
                px[n] = xs[k]; py[n] = yy; n++;
            }
        }
    }
    if (fabs(a) > 1e-15) {
        const double ys[2] = {y0, y1};
        for (int k = 0; k < 2; k++) {
            double x = -(b * ys[k] + c) / a;
            if (x0 - 1e-9 <= x && x <= x1 + 1e-9) {
                double xx = x < x0 ? x0 : x;
                xx = xx > x1 ? x1 : xx;
                px[n] = xx; py[n] = ys[k]; n++;
            }
        }
    }
    if (n < 2) return false;
    int imin = 0, imax = 0;
    for (int k = 1; k < n; k++) {
        if (px[k] < px[imin] || (px[k] == px[imin] && py[k] < py[imin])) imin = k;
        if (px[k] > px[imax] || (px[k] == px[imax] && py[k] > py[imax])) imax = k;
    }
    pa[0] = px[imin]; pa[1] = py[imin];
    pb[0] = px[imax]; pb[1] = py[imax];
    return seg_not_lt(pb[0] - pa[0], pb[1] - pa[1], 1e-12);
}

// group_queries composite key (guided.py:363-373), int64 wrap semantics.
__device__ __forceinline__ unsigned long long composite_key(const double pa[2], const double pb[2]) {
    long long c[4] = {(long long)floor(pa[0] / 2.0), (long long)floor(pa[1] / 2.0),
                      (long long)floor(pb[0] / 2.0), (long long)floor(pb[1] / 2.0)};
    unsigned long long k = (unsigned long long)(c[0] + 4096);
#pragma unroll
    for (int i = 1; i < 4; i++) k = k * 8192ull + (unsigned long long)(c[i] + 4096);
    return k;
}

// Reference subcell index of a coordinate (see msfm_grids in the header):
// u = 2*floor(fl(x/2D)) + [floor(fl((x-D)/2D)) == floor(fl(x/2D))]   (guided.py:64-68)
__device__ __forceinline__ int exact_subcell(double x, double D) {
    double c0 = floor(x / (2.0 * D));
    double c1 = floor((x - D) / (2.0 * D));
    return 2 * (int)c0 + (c1 == c0 ? 1 : 0);
}

// ------------------------------------------------------------------ block scan

// ------------------------------------------------------------------ features
__global__ void norms_kernel(const uint8_t* __restrict__ desc, int64_t n, int32_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4* row = reinterpret_cast<const uint4*>(desc + i * 128);
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        uint4 v = row[k];
        s = __dp4a(v.x, v.x, s); s = __dp4a(v.y, v.y, s);
        s = __dp4a(v.z, v.z, s); s = __dp4a(v.w, v.w, s);
    }
    out[i] = (int32_t)s;
}

// ------------------------------------------------------------------ grid build
constexpr int GRID_SPLIT = 8;   // CTAs per image in the grid build

struct GridBuildArgs {
    const float2* xy; const int64_t* img_off; const int32_t* img_n; const int32_t* img_wh;
    const int32_t* dims; const int64_t* roff; const int64_t* coff;
    int32_t* sub; int32_t* rcount; int32_t* ccount; int32_t* rcur; int32_t* ccur;
    int32_t* rmem; int32_t* cmem; int4* rrec; int4* crec; const int32_t* norm2; double D;
    int img0;             // first image of the range this launch builds (blockIdx.x + img0)
    const uint8_t* desc;  // when norm_out is set, grid_count also writes |desc|^2 there
    int32_t* norm_out;
};

__device__ __forceinline__ int bucket_of(float v, double D, int nb) {
    int b = (int)floor((double)v / D);
    return b < 0 ? 0 : (b >= nb ? nb - 1 : b);
}

__global__ void grid_count_kernel(GridBuildArgs a) {
    // GRID_SPLIT CTAs per image (a range of 8 images would otherwise run on 8 SMs)
    const int img = a.img0 + blockIdx.x / GRID_SPLIT;
    const int part = blockIdx.x % GRID_SPLIT;
    const int64_t off = a.img_off[img];
    const int n = a.img_n[img];
    const int nbx = a.dims[2 * img], nby = a.dims[2 * img + 1];
    for (int f = part * blockDim.x + threadIdx.x; f < n; f += GRID_SPLIT * blockDim.x) {
        if (a.norm_out) {
            const uint4* row = reinterpret_cast<const uint4*>(a.desc + (off + f) * 128);
            unsigned s = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint4 v = __ldg(row + k);
                const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; j++) s = __dp4a(w[j], w[j], s);   // u8 x u8, exact
            }
            a.norm_out[off + f] = (int32_t)s;
        }
        float2 p = a.xy[off + f];
        int u = exact_subcell((double)p.x, a.D), v = exact_subcell((double)p.y, a.D);
        a.sub[off + f] = (u & 0xffff) | (v << 16);
        int bx = bucket_of(p.x, a.D, nbx), by = bucket_of(p.y, a.D, nby);
        atomicAdd(&a.rcount[a.roff[img] + (int64_t)by * nbx + bx], 1);
        atomicAdd(&a.ccount[a.coff[img] + (int64_t)bx * nby + by], 1);
    }
}

__global__ void grid_scatter_kernel(GridBuildArgs a) {
    // GRID_SPLIT CTAs per image (a range of 8 images would otherwise run on 8 SMs)
    const int img = a.img0 + blockIdx.x / GRID_SPLIT;
    const int part = blockIdx.x % GRID_SPLIT;
    const int64_t off = a.img_off[img];
    const int n = a.img_n[img];
    const int nbx = a.dims[2 * img], nby = a.dims[2 * img + 1];
    for (int f = part * blockDim.x + threadIdx.x; f < n; f += GRID_SPLIT * blockDim.x) {
        float2 p = a.xy[off + f];
        int bx = bucket_of(p.x, a.D, nbx), by = bucket_of(p.y, a.D, nby);
        int r = atomicAdd(&a.rcur[a.roff[img] + (int64_t)by * nbx + bx], 1);
        int c = atomicAdd(&a.ccur[a.coff[img] + (int64_t)bx * nby + by], 1);
        a.rmem[r] = f;
        a.cmem[c] = f;
        const int4 rec = make_int4(__float_as_int(p.x), __float_as_int(p.y), a.norm2[off + f], f);
        a.rrec[r] = rec;
        a.crec[c] = rec;
    }
}


// ------------------------------------------------------------------ matching
// Per-group context, computed once by prep_kernel (one thread per group) so the
// warp-per-group match kernel starts from fp32 values and never divides in fp64.
// The first 32 bytes are what the setup kernel re-reads after writing the record;
// the rest is only read by the match kernel (stored evict-first).
struct alignas(16) GroupRec {
    int rep, cnt, moff, K;                 // rep slot, members, member offset; K<0: the rep
                                           // line misses the padded image (C' empty)
    float maxdev, ar, br, cr;              // max member-band deviation; rep line (fp32)
    int p, pad1;                           // chunk-local pair
    float hsure, len;                      // sure-in-C' radius
    float pbx, pby, dirx, diry;            // padded segment origin (pb) and direction
    float spacing, invK, invD, dxf;
    float dyf, slack;
    int pad2, pad3;
    double pax, pay, pbx64, pby64;         // exact sample interpolation (guided.py:187)
    double sl0, sl1, sl2, spare;           // singleton member's own (dgemv) line
};
static_assert(sizeof(GroupRec) == 160, "GroupRec: 32 hot bytes + 128 match-only bytes");

// Per-member epilogue constants (prep_kernel), indexed like members[].
struct MemberRec {
    float a, b, c, lo;    // member line (fp32) and sure-in-band threshold d - eps
    float hi;             // d + eps: above it the fp32 value is surely out of band
    unsigned qn9;         // |q|^2 << 9
    int fid;              // query feature id
    int slotgi;           // chunk-local slot | (group index within its super-group << SLOT_BITS)
};

// A super-group: up to SG_MEMBERS consecutive members (groups ordered by line
// angle) that share one strip gather and full n8 tiles (sg_prep_kernel).
struct alignas(16) SGRec {
    int p, m0, mcnt, g0;                   // pair, member range, first group (dense gid)
    int gcnt, horiz, rlo, rhi;             // groups, strip orientation, bucket-row range
    float ar, br, cr, R;                   // base line (fp32) and strip half-width
    float delta, hsure, border, invD;      // max rep-vs-base deviation, sure radius, border
    float alpha, beta, inv_alpha, Pmax;    // strip row math in the chosen orientation
    float W, H;
    int nalong, pad0;                      // buckets along a strip row
    long long toff, qoff;                  // first bank feature of the target / query image
    long long toffb, dbase;                // first bucket of the strip table, dedupe base
};

// Per group, the view the match kernel bulk-copies: rep line (fp32), member-band
// reach, first member position (sg_prep_kernel).
struct alignas(16) GView {
    float a, b, c, reach;
    int moff, pad0, pad1, pad2;
};

#ifndef MSFM_SG_NT
#define MSFM_SG_NT 2
#endif
constexpr int SG_NT = MSFM_SG_NT;          // n8 member tiles per super-group
constexpr int SG_MEMBERS = 8 * SG_NT;
// member records pack the chunk-local query slot with the group index within its
// super-group (< SG_MEMBERS <= 16: 4 bits) into one word
constexpr int SLOT_BITS = 28;
constexpr unsigned SLOT_MASK = (1u << SLOT_BITS) - 1u;
constexpr int64_t AUTO_CHUNK_SLOTS = 48ll << 20;    // query slots per automatic chunk
// per-candidate C' bits are one 16-bit mask over the super-group's groups (<= members)
static_assert(SG_MEMBERS <= 16, "MSFM_SG_NT > 2 needs wider per-candidate group masks");
#ifndef MSFM_MATCH_MINB
#define MSFM_MATCH_MINB (SG_NT == 1 ? 6 : 4)
#endif
constexpr int MATCH_MINB = MSFM_MATCH_MINB;   // resident CTAs (4 warps) per SM
constexpr float SG_TAU = 24.0f;
constexpr int SG_MAX_GROUPS = SG_MEMBERS;

struct ChunkArgs {
    // bank
    const float2* xy; const uint8_t* desc; const int32_t* norm2;
    const int64_t* img_off; const int32_t* img_n; const int32_t* img_wh;
    // index
    const int32_t* sub; const int32_t* dims; const int64_t* roff; const int64_t* coff;
    const int32_t* rstart; const int32_t* cstart; const int32_t* rmem; const int32_t* cmem;
    const int4* rrec; const int4* crec;   // bucket-ordered (x, y, |desc|^2, id)
    double D, d;
    float ratio, single_cap;
    int tie_fid;                 // ratio > 1: ties at the minimum resolve to the lowest target id
    int stats_mode;              // 1: one super-group per group (exact SearchStats)
    int strategy;                // 0 grid, 1 linear, 2 radial (msfm_match_params)
    double r2;                   // radial: (d * sqrt(2))^2 as the reference rounds it
    float sg_tau;                // super-group line tolerance (px)
    // pairs
    const int32_t* pair_q; const int32_t* pair_t; const double* pair_F;
    const int64_t* qlist_off; const int32_t* qlist;
    const int64_t* qlist_src;    // optional: per-pair start of its list inside qlist
    int32_t* q_fid;              // chunk-local query feature ids (filled by setup_kernel)
    int32_t p0, npairs; int64_t qbase;
    // chunk workspace
    int64_t* tab_off; int64_t* tbase;
    int32_t* sg_total;           // super-groups queued by the chunk's setup (atomic)
    int32_t* sg_next;            // match kernel's queue head
    unsigned long long* tab_key; unsigned* tab_rep; unsigned* tab_cnt;
    int32_t* q_tab; double* q_line;
    float4* q_lf;                // per clipped query: its line in f32 + |q|^2 bits (setup re-reads)
    int2* gtmp; float* gkey; int32_t* gpos; float4* gline; float4* gend; int2* sglist;
    int4* grec; int32_t* gfill; int32_t* members; GroupRec* grp; MemberRec* mrec; SGRec* sg;
    int32_t* mgid;               // per member position: the pair's (sorted) group index
    int32_t* msg;                // per member position: the pair's super-group index
    unsigned* gfit;              // per group: first member position past its tau-fit run
    unsigned long long* sgdev;   // per super-group: max member-band deviation (f64 bits)
    GView* gview;                // per group: rep line (fp32), member-band reach, first member
    int32_t* jmp_a; int32_t* jmp_b; int32_t* jmark;   // super-group walk (large pairs)
    unsigned long long* mstate;  // per member slot: best (d2<<32 | tid)
    unsigned* mstate2;           // per member slot: second d2
    int32_t* res_tid; float* res_dist; float* res_ratio;
    unsigned long long* dedupe;
    unsigned long long* stats;   // [2*n_pairs] (global pair index) or null
    unsigned long long* dbg;     // optional workload counters (msfm_debug_counters)
    // outputs
    int32_t* out_q; int32_t* out_t; float* out_dist; float* out_ratio; int32_t* out_count;
};

__device__ __forceinline__ int nextpow2(int v) {
    int p = 2;
    while (p < v) p <<= 1;
    return p;
}

constexpr int GB = 8192;   // angle buckets of the per-pair group order

// Upper bound of |dist_m(f) - dist_r(f)| over the image rectangle restricted to
// the member's band (|dist_m| <= d + 0.5): the difference is affine, so its
// maximum over that convex polygon sits at one of its vertices.
// band_deviation of one member line against two lines at once: the points where
// the member band is extremal (corners, band-edge / border crossings, with their
// divisions) depend only on m and are evaluated once for both.
__device__ void band_deviation2(const double m[3], const double r[3], const double b[3],
                                double W, double H, double d, double& dev_r, double& dev_b) {
    const double ra = m[0] - r[0], rb = m[1] - r[1], rc = m[2] - r[2];
    const double ba = m[0] - b[0], bb = m[1] - b[1], bc = m[2] - b[2];
    const double B = d + 0.5;
    dev_r = 0.0;
    dev_b = 0.0;
    const double cx[4] = {0.0, W, 0.0, W}, cy[4] = {0.0, 0.0, H, H};
    for (int k = 0; k < 4; k++) {
        double dm = m[0] * cx[k] + m[1] * cy[k] + m[2];
        if (fabs(dm) <= B) {
            dev_r = fmax(dev_r, fabs(ra * cx[k] + rb * cy[k] + rc));
            dev_b = fmax(dev_b, fabs(ba * cx[k] + bb * cy[k] + bc));
        }
    }
    const double i1 = fabs(m[1]) > 1e-12 ? 1.0 / m[1] : 0.0;
    const double i0 = fabs(m[0]) > 1e-12 ? 1.0 / m[0] : 0.0;
    for (int s = -1; s <= 1; s += 2) {
        if (i1 != 0.0) {
            for (int e = 0; e < 2; e++) {
                double x = e ? W : 0.0;
                double y = (s * B - m[2] - m[0] * x) * i1;
                if (y >= -1e-6 && y <= H + 1e-6) {
                    dev_r = fmax(dev_r, fabs(ra * x + rb * y + rc));
                    dev_b = fmax(dev_b, fabs(ba * x + bb * y + bc));
                }
            }
        }
        if (i0 != 0.0) {
            for (int e = 0; e < 2; e++) {
                double y = e ? H : 0.0;
                double x = (s * B - m[2] - m[1] * y) * i0;
                if (x >= -1e-6 && x <= W + 1e-6) {
                    dev_r = fmax(dev_r, fabs(ra * x + rb * y + rc));
                    dev_b = fmax(dev_b, fabs(ba * x + bb * y + bc));
                }
            }
        }
    }
}

__device__ double band_deviation(const double m[3], const double r[3], double W, double H,
                                 double d) {
    const double da = m[0] - r[0], db = m[1] - r[1], dc = m[2] - r[2];
    const double B = d + 0.5;
    double dev = 0.0;
    const double cx[4] = {0.0, W, 0.0, W}, cy[4] = {0.0, 0.0, H, H};
    for (int k = 0; k < 4; k++) {
        double dm = m[0] * cx[k] + m[1] * cy[k] + m[2];
        if (fabs(dm) <= B) dev = fmax(dev, fabs(da * cx[k] + db * cy[k] + dc));
    }
    const double i1 = fabs(m[1]) > 1e-12 ? 1.0 / m[1] : 0.0;
    const double i0 = fabs(m[0]) > 1e-12 ? 1.0 / m[0] : 0.0;
    for (int s = -1; s <= 1; s += 2) {
        if (i1 != 0.0) {
            for (int e = 0; e < 2; e++) {
                double x = e ? W : 0.0;
                double y = (s * B - m[2] - m[0] * x) * i1;
                if (y >= -1e-6 && y <= H + 1e-6) dev = fmax(dev, fabs(da * x + db * y + dc));
            }
        }
        if (i0 != 0.0) {
            for (int e = 0; e < 2; e++) {
                double y = e ? H : 0.0;
                double x = (s * B - m[2] - m[1] * y) * i0;
                if (x >= -1e-6 && x <= W + 1e-6) dev = fmax(dev, fabs(da * x + db * y + dc));
            }
        }
    }
    return dev;
}

#include "guided_setup.cuh"

// mma.sync m16n8k32 u8 x u8 -> s32 (rows = candidates, cols = members)
__device__ __forceinline__ void mma_u8(int (&c)[4], unsigned a0, unsigned a1, unsigned a2,
                                       unsigned a3, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void top2_push(unsigned key, unsigned& b1, unsigned& b2) {
    unsigned lo = min(key, b1), hi = max(key, b1);
    b1 = lo;
    b2 = min(b2, hi);
}

__device__ __forceinline__ void top2_merge(unsigned& b1, unsigned& b2, unsigned o1, unsigned o2) {
    unsigned lo = min(b1, o1), hi = max(b1, o1);
    b1 = lo;
    b2 = min(hi, min(b2, o2));
}

// Exact subcell of sample k of a rep line (guided.py:173-187 + cell_indices):
// fp32 interpolation, exact fp64 evaluation only near a subcell boundary.
__device__ __forceinline__ void sample_subcell(const GroupRec& G, double D, int k, int& u, int& v) {
    const float t = (float)k * G.invK;
    const float sx = fmaf(t, G.dxf, G.pbx), sy = fmaf(t, G.dyf, G.pby);
    const float qx = sx * G.invD, qy = sy * G.invD;
    const float fx = floorf(qx), fy = floorf(qy);
    const float rx = qx - fx, ry = qy - fy;
    if (rx > G.slack && rx < 1.0f - G.slack && ry > G.slack && ry < 1.0f - G.slack) {
        u = (int)fx; v = (int)fy;
        return;
    }
    const double kd = (double)k, rk = (double)(G.K - k), Kd = (double)G.K;
    const double ex = (kd * G.pax + rk * G.pbx64) / Kd;
    const double ey = (kd * G.pay + rk * G.pby64) / Kd;
    u = exact_subcell(ex, D);
    v = exact_subcell(ey, D);
}

// f in C'(rep): some sample subcell is within Chebyshev distance 1 of f's.
__device__ bool in_cprime_exact(const GroupRec& G, double D, float fx, float fy, int fu, int fv) {
    if (G.K < 0) return false;
    const float tau = (fx - G.pbx) * G.dirx + (fy - G.pby) * G.diry;
    const float reach = 2.0f * 1.41421356f * (float)D + 1.0f;
    const float inv_sp = 1.0f / G.spacing;
    int klo = (int)floorf((tau - reach) * inv_sp) - 1;
    int khi = (int)ceilf((tau + reach) * inv_sp) + 1;
    if (klo < 0) klo = 0;
    if (khi > G.K) khi = G.K;
    for (int k = klo; k <= khi; k++) {
        int u, v;
        sample_subcell(G, D, k, u, v);
        if (abs(u - fu) <= 1 && abs(v - fv) <= 1) return true;
    }
    return false;
}

// C' membership of f for group G, using the sure zone first
// the reference's float64 band value for one (member, target) element, guided.py:447
__device__ __forceinline__ bool band_exact(double A, double B, double C, bool gemv, double x,
                                           double y, double d) {
    double v = gemv ? fma(A, x, B * y) : fma(B, y, A * x);
    v = v + C;
    return fabs(v) <= d;
}

// radial (guided.py:273-285): some sample within r of f, squared distance in f64
// exactly as scipy's cKDTree.query_ball_point compares it (dx*dx + dy*dy <= r*r)
__device__ bool in_radial_exact(const GroupRec& G, double r2, float fx, float fy) {
    if (G.K < 0) return false;
    const float tau = (fx - G.pbx) * G.dirx + (fy - G.pby) * G.diry;
    const float reach = (float)sqrt(r2) + 1.0f;
    const float inv_sp = 1.0f / G.spacing;
    int klo = (int)floorf((tau - reach) * inv_sp) - 1;
    int khi = (int)ceilf((tau + reach) * inv_sp) + 1;
    if (klo < 0) klo = 0;
    if (khi > G.K) khi = G.K;
    const double x = (double)fx, y = (double)fy, Kd = (double)G.K;
    for (int k = klo; k <= khi; k++) {
        const double kd = (double)k, rk = (double)(G.K - k);
        const double sx = (kd * G.pax + rk * G.pbx64) / Kd;
        const double sy = (kd * G.pay + rk * G.pby64) / Kd;
        const double dx = x - sx, dy = y - sy;
        if (dx * dx + dy * dy <= r2) return true;
    }
    return false;
}

__device__ __forceinline__ bool in_cprime(const ChunkArgs& a, const GroupRec& G, const SGRec& S,
                                          float fx, float fy, int64_t toff, int f) {
    if (a.strategy == 1) {
        // linear (guided.py:190-194): |xy @ [a, b] + c| <= d, a dgemv (fma(a, x, b*y))
        const float dg = fabsf(fmaf(G.ar, fx, fmaf(G.br, fy, G.cr)));
        if (dg <= S.hsure) return true;
        const double* L = a.q_line + 3 * (int64_t)G.rep;
        return band_exact(L[0], L[1], L[2], true, (double)fx, (double)fy, a.d);
    }
    if (G.K < 0) return false;
    const float dg = fabsf(fmaf(G.ar, fx, fmaf(G.br, fy, G.cr)));
    if (dg <= S.hsure && fx >= S.border && fx <= S.W - S.border && fy >= S.border &&
        fy <= S.H - S.border)
        return true;
    if (a.strategy == 2) return in_radial_exact(G, a.r2, fx, fy);
    const int su = a.sub[toff + f];
    return in_cprime_exact(G, a.D, fx, fy, (short)(su & 0xffff), su >> 16);
}

#include "guided_match.cuh"

constexpr int CT = 1024;   // compact_kernel threads (one pair per CTA)
__global__ void __launch_bounds__(CT) compact_kernel(ChunkArgs a) {
    __shared__ int sm[CT / 32 + 1];
    const int p = blockIdx.x, pg = a.p0 + p;
    const int64_t q0 = a.qlist_off[pg];
    const int nq = (int)(a.qlist_off[pg + 1] - q0);
    const int64_t s0 = q0 - a.qbase;
    const int64_t db = a.tbase[p];
    int carry = 0;
    for (int i0 = 0; i0 < nq; i0 += CT) {
        const int i = i0 + threadIdx.x;
        bool keep = false;
        int tid = -1, qid = 0;
        float dist = 0.f, ratio = 0.f;
        if (i < nq) {
            // the slot's four fields load together (no dependence on tid)
            tid = a.res_tid[s0 + i];
            qid = a.q_fid[s0 + i];
            dist = a.res_dist[s0 + i];
            ratio = a.res_ratio[s0 + i];
            if (tid >= 0) {
                const unsigned long long key =
                    ((unsigned long long)__float_as_uint(dist) << 32) | (unsigned)qid;
                keep = a.dedupe[db + tid] == key;
            }
        }
        int tot;
        const int ex = block_exclusive_scan<CT>(keep ? 1 : 0, &tot, sm);
        if (keep) {
            const int64_t o = q0 + carry + ex;
            a.out_q[o] = qid;
            a.out_t[o] = tid;
            a.out_dist[o] = dist;
            a.out_ratio[o] = ratio;
        }
        carry += tot;
    }
    if (threadIdx.x == 0) a.out_count[pg] = carry;
}

// pack the per-pair match segments into contiguous 16-B rows:
// (pair, q | t << 16, dist bits, ratio bits)
__global__ void pack_scan_kernel(const int32_t* __restrict__ count, int n_pairs,
                                 int64_t* __restrict__ out_off) {
    __shared__ int sm[SCAN_T / 32 + 1];
    long long carry = 0;
    for (int b0 = 0; b0 < n_pairs; b0 += SCAN_T) {
        const int p = b0 + threadIdx.x;
        const int v = p < n_pairs ? count[p] : 0;
        int tot;
        const int ex = block_exclusive_scan<SCAN_T>(v, &tot, sm);
        if (p < n_pairs) out_off[p] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) out_off[n_pairs] = carry;
}

// chunk c of a pipelined packing: pairs [p0, p0 + np); meta[2c] = first row of the
// chunk (after chunk c-1), meta[2c+1] = rows in the chunk
__global__ void pack_chunk_scan_kernel(const int32_t* __restrict__ count, int p0, int np, int c,
                                       int64_t* __restrict__ out_off, int64_t* __restrict__ meta) {
    __shared__ int sm[SCAN_T / 32 + 1];
    const long long base = c > 0 ? meta[2 * (c - 1)] + meta[2 * (c - 1) + 1] : 0;
    long long carry = 0;
    for (int b0 = 0; b0 < np; b0 += SCAN_T) {
        const int k = b0 + threadIdx.x;
        const int v = k < np ? count[p0 + k] : 0;
        int tot;
        const int ex = block_exclusive_scan<SCAN_T>(v, &tot, sm);
        if (k < np) out_off[p0 + k] = base + carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) { meta[2 * c] = base; meta[2 * c + 1] = carry; }
}

__global__ void pack_kernel(const int64_t* __restrict__ qlist_off, const int32_t* __restrict__ count,
                            const int64_t* __restrict__ out_off, const int32_t* __restrict__ q,
                            const int32_t* __restrict__ t, const float* __restrict__ dist,
                            const float* __restrict__ ratio, int4* __restrict__ rows, int p0 = 0) {
    const int p = p0 + blockIdx.x;
    const int64_t src = qlist_off[p], dst = out_off[p];
    const int c = count[p];
    for (int i = threadIdx.x; i < c; i += blockDim.x)
        rows[dst + i] = make_int4(p, (q[src + i] & 0xffff) | (t[src + i] << 16),
                                  __float_as_int(dist[src + i]), __float_as_int(ratio[src + i]));
}

// workspace plan for one chunk
struct ChunkSizes {
    int64_t P, Q, T, NT;
};

size_t chunk_bytes(const ChunkSizes& c) {
    size_t b = 0;
    b += aligned_bytes<int64_t>(c.P + 1) * 2;          // tab_off, tbase
    b += 256 * 2;                                      // sg_total, sg_next
    b += aligned_bytes<float4>(c.Q) * 2 + aligned_bytes<int2>(c.Q);   // gline, gend, sglist
    b += aligned_bytes<unsigned long long>(c.T);       // tab_key
    b += aligned_bytes<unsigned>(c.T) * 2;             // tab_rep, tab_cnt
    b += aligned_bytes<int32_t>(c.Q) * 2;              // q_tab, q_fid
    b += aligned_bytes<int32_t>(c.Q) * 2;              // mgid, msg
    b += aligned_bytes<unsigned>(c.Q);                 // gfit
    b += aligned_bytes<unsigned long long>(c.Q);       // sgdev
    b += aligned_bytes<int32_t>(c.Q + c.P + 1) * 3;    // jmp_a, jmp_b, jmark (pairs past TS_SMEM)
    b += aligned_bytes<GView>(c.Q);                    // gview
    b += aligned_bytes<double>(3 * c.Q);               // q_line
    b += aligned_bytes<float4>(c.Q);                   // q_lf
    b += aligned_bytes<int4>(c.Q);                     // grec
    b += aligned_bytes<int32_t>(c.Q) * 2;              // gfill, members
    b += aligned_bytes<GroupRec>(c.Q);                 // grp
    b += aligned_bytes<MemberRec>(c.Q);                // mrec
    b += aligned_bytes<SGRec>(c.Q);                    // sg
    b += aligned_bytes<int2>(c.Q) + aligned_bytes<float>(c.Q) + aligned_bytes<int32_t>(c.Q);  // gtmp, gkey, gpos
    b += aligned_bytes<unsigned long long>(c.Q);       // mstate
    b += aligned_bytes<unsigned>(c.Q);                 // mstate2
    b += aligned_bytes<int32_t>(c.Q) * 3;              // res_tid/dist/ratio
    b += aligned_bytes<unsigned long long>(c.NT);      // dedupe
    return b + 4096;
}

}  // namespace
}  // namespace msfm

using namespace msfm;

static unsigned long long* g_dbg = nullptr;

extern "C" int msfm_debug_counters(int enable, int64_t* out16) {
    if (enable && !g_dbg) {
        MSFM_CUDA_TRY(cudaMalloc(&g_dbg, 16 * sizeof(unsigned long long)));
        MSFM_CUDA_TRY(cudaMemset(g_dbg, 0, 16 * sizeof(unsigned long long)));
    }
    if (out16 && g_dbg) {
        MSFM_CUDA_TRY(cudaMemcpy(out16, g_dbg, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        MSFM_CUDA_TRY(cudaMemset(g_dbg, 0, 16 * sizeof(unsigned long long)));
    }
    if (!enable && g_dbg) {
        cudaFree(g_dbg);
        g_dbg = nullptr;
    }
    return MSFM_OK;
}

extern "C" int msfm_feature_norms(const uint8_t* d_desc, int64_t n, int32_t* d_norm2, void* stream) {
    if (n < 0 || (n > 0 && (!d_desc || !d_norm2))) {
        set_error("msfm_feature_norms: bad arguments");
        return MSFM_EINVAL;
    }
    if (n == 0) return MSFM_OK;
    norms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_desc, n, d_norm2);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

extern "C" int msfm_pack_matches(int32_t n_pairs, const int64_t* d_qlist_off,
                                 const int32_t* d_count, const int32_t* d_q, const int32_t* d_t,
                                 const float* d_dist, const float* d_ratio, int64_t* d_out_off,
                                 int32_t* d_rows, void* stream) {
    if (n_pairs < 0) {
        set_error("msfm_pack_matches: bad arguments");
        return MSFM_EINVAL;
    }
    if (n_pairs == 0) return MSFM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    pack_scan_kernel<<<1, SCAN_T, 0, st>>>(d_count, n_pairs, d_out_off);
    pack_kernel<<<n_pairs, 128, 0, st>>>(d_qlist_off, d_count, d_out_off, d_q, d_t, d_dist, d_ratio,
                                         reinterpret_cast<int4*>(d_rows));
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    return MSFM_OK;
}

extern "C" int msfm_grid_dims(int32_t width, int32_t height, double D, int32_t dims_out[2]) {
    if (!(D > 0) || width < 0 || height < 0 || !dims_out) {
        set_error("msfm_grid_dims: cell half-size D must be positive, got %g", D);
        return MSFM_EINVAL;
    }
    dims_out[0] = (int32_t)floor((double)width / D) + 1;
    dims_out[1] = (int32_t)floor((double)height / D) + 1;
    return MSFM_OK;
}

extern "C" size_t msfm_grid_workspace_bytes(int64_t n_buckets_total) {
    int64_t nb = (n_buckets_total + 1 + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER) + 1;
    return aligned_bytes<int32_t>(n_buckets_total + 1) * 2 + aligned_bytes<int32_t>(nb) * 2 +
           1024;
}

// the range build; with norms, the count pass also writes the range's |desc|^2 (the
// staged matcher's per-range indexing: one pass over the rows instead of two)
static int grid_build_range_impl(const msfm_bank* bank, const int32_t* d_dims,
                                 const int64_t* d_roff, const int64_t* d_coff,
                                 int64_t n_buckets_total, int32_t img0, int32_t img1,
                                 int64_t bucket0, int64_t bucket1, int64_t feat0, double D,
                                 int32_t* d_sub, int32_t* d_rstart, int32_t* d_cstart,
                                 int32_t* d_rmem, int32_t* d_cmem, int32_t* d_rrec,
                                 int32_t* d_crec, void* d_workspace, size_t workspace_bytes,
                                 void* stream, int32_t* norm_out) {
    if (!bank || !(D > 0) || n_buckets_total < 0 || img0 < 0 || img1 < img0 ||
        img1 > bank->n_images || bucket0 < 0 || bucket1 < bucket0 || bucket1 > n_buckets_total ||
        feat0 < 0 || feat0 > INT32_MAX) {
        set_error("msfm_grid_build_range: bad arguments (D=%g, images [%d, %d))", D, img0, img1);
        return MSFM_EINVAL;
    }
    if (workspace_bytes < msfm_grid_workspace_bytes(n_buckets_total)) {
        set_error("msfm_grid_build: workspace too small");
        return MSFM_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar(d_workspace, workspace_bytes);
    int32_t* rcur = ar.take<int32_t>(n_buckets_total + 1);
    int32_t* ccur = ar.take<int32_t>(n_buckets_total + 1);
    int64_t nb = (n_buckets_total + 1 + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER) + 1;
    int32_t* bsum0 = ar.take<int32_t>(nb);
    int32_t* bsum1 = ar.take<int32_t>(nb);
    // counts go to the cursor arrays; the scan writes the CSR starts [bucket0, bucket1]
    // (the closing start included, = the next range's first start) without ever
    // touching a start another range already published
    const int64_t n = bucket1 - bucket0 + 1;
    MSFM_CUDA_TRY(cudaMemsetAsync(rcur + bucket0, 0, sizeof(int32_t) * n, st));
    MSFM_CUDA_TRY(cudaMemsetAsync(ccur + bucket0, 0, sizeof(int32_t) * n, st));
    GridBuildArgs a{reinterpret_cast<const float2*>(bank->d_xy), bank->d_img_off, bank->d_img_n,
                    bank->d_img_wh, d_dims, d_roff, d_coff, d_sub, rcur, ccur, rcur, ccur,
                    d_rmem, d_cmem, reinterpret_cast<int4*>(d_rrec),
                    reinterpret_cast<int4*>(d_crec), bank->d_norm2, D, img0, bank->d_desc, norm_out};
    if (img1 > img0) {
        grid_count_kernel<<<(img1 - img0) * GRID_SPLIT, 256, 0, st>>>(a);
        MSFM_LAUNCH_CHECK();
        count_launches(1);
    }
    // row and column tables in one scan launch set
    Scan2 sc;
    sc.data[0] = rcur + bucket0; sc.data[1] = ccur + bucket0;
    sc.copy[0] = d_rstart + bucket0; sc.copy[1] = d_cstart + bucket0;
    sc.bsum[0] = bsum0; sc.bsum[1] = bsum1;
    sc.n = n; sc.base0 = (int32_t)feat0;
    int rc = exclusive_scan2(sc, st);
    if (rc) return rc;
    if (img1 > img0) {
        grid_scatter_kernel<<<(img1 - img0) * GRID_SPLIT, 256, 0, st>>>(a);
        MSFM_LAUNCH_CHECK();
        count_launches(1);
    }
    return MSFM_OK;
}

extern "C" int msfm_grid_build_range(const msfm_bank* bank, const int32_t* d_dims,
                                     const int64_t* d_roff, const int64_t* d_coff,
                                     int64_t n_buckets_total, int32_t img0, int32_t img1,
                                     int64_t bucket0, int64_t bucket1, int64_t feat0, double D,
                                     int32_t* d_sub, int32_t* d_rstart, int32_t* d_cstart,
                                     int32_t* d_rmem, int32_t* d_cmem, int32_t* d_rrec,
                                     int32_t* d_crec, void* d_workspace, size_t workspace_bytes,
                                     void* stream) {
    return grid_build_range_impl(bank, d_dims, d_roff, d_coff, n_buckets_total, img0, img1,
                                 bucket0, bucket1, feat0, D, d_sub, d_rstart, d_cstart, d_rmem,
                                 d_cmem, d_rrec, d_crec, d_workspace, workspace_bytes, stream,
                                 nullptr);
}

extern "C" int msfm_grid_build(const msfm_bank* bank, const int32_t* d_dims, const int64_t* d_roff,
                               const int64_t* d_coff, int64_t n_buckets_total, int64_t n_total,
                               double D, int32_t* d_sub, int32_t* d_rstart, int32_t* d_cstart,
                               int32_t* d_rmem, int32_t* d_cmem, int32_t* d_rrec, int32_t* d_crec,
                               void* d_workspace,
                               size_t workspace_bytes, void* stream) {
    if (!bank || !(D > 0) || n_buckets_total < 0 || n_total < 0) {
        set_error("msfm_grid_build: bad arguments (D=%g)", D);
        return MSFM_EINVAL;
    }
    return msfm_grid_build_range(bank, d_dims, d_roff, d_coff, n_buckets_total, 0, bank->n_images,
                                 0, n_buckets_total, 0, D, d_sub, d_rstart, d_cstart, d_rmem,
                                 d_cmem, d_rrec, d_crec, d_workspace, workspace_bytes, stream);
}

static void plan_chunks(int32_t n_pairs, const int64_t* h_qlist_off, const msfm_match_params* prm,
                        std::vector<int>& bounds, ChunkSizes& worst) {
    // A chunk holds at most cp pairs, 2^SLOT_BITS query slots (member records pack
    // the chunk-local slot into SLOT_BITS bits), AUTO_CHUNK_SLOTS slots, and as many
    // slots as keep its workspace within the byte budget — explicit chunk_pairs
    // included.  Auto mode: large chunks (fewer kernel tails per stage: a C3 step in
    // one chunk is 3.7% faster than in six).
    const int cp = prm->chunk_pairs > 0 ? prm->chunk_pairs : 8192;
    int64_t budget = prm->max_workspace_bytes;
    if (budget <= 0) {
        // a quarter of the device memory free at the first planning on this device:
        // cudaMemGetInfo itself can stall a step for tens of ms (measured 2-74 ms in
        // the staged e2e loop), so it is asked once per device and process
        static int64_t cached[64];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || cached[dev] <= 0) {
            size_t fr = 0, tot = 0;
            const int64_t b = (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0) ? (int64_t)(fr / 4)
                                                                                 : (int64_t)16 << 30;
            if (dev >= 0 && dev < 64) cached[dev] = b;
            budget = b;
        } else {
            budget = cached[dev];
        }
    }
    const int64_t qmax = std::min<int64_t>((int64_t)1 << SLOT_BITS, AUTO_CHUNK_SLOTS);
    auto bytes_of = [&](int64_t P, int64_t Q) {
        ChunkSizes c{P, Q, 2 * (Q + P) + 2 * P, P * (int64_t)prm->max_nt};
        return (int64_t)chunk_bytes(c);
    };
    bounds.clear();
    worst = {0, 0, 0, 0};
    int p = 0;
    bounds.push_back(0);
    // pipelined (first_chunk_pairs > 0): chunk sizes ramp first, 4 first, 16 first, ...
    // up to chunk_pairs, so each chunk's compute covers the upload of the next one's
    // images and the matcher starts after a few images instead of a chunk's worth
    int ramp = prm->first_chunk_pairs > 0 ? prm->first_chunk_pairs : cp;
    while (p < n_pairs) {
        int e = p + 1;
        const int cap = std::min(cp, ramp);
        if (ramp < cp) ramp = ramp > cp / 4 ? cp : ramp * 4;
        while (e < n_pairs && e - p < cap && h_qlist_off[e + 1] - h_qlist_off[p] <= qmax &&
               bytes_of(e + 1 - p, h_qlist_off[e + 1] - h_qlist_off[p]) <= budget)
            e++;
        ChunkSizes c;
        c.P = e - p;
        c.Q = h_qlist_off[e] - h_qlist_off[p];
        c.T = 2 * (c.Q + c.P) + 2 * c.P;
        c.NT = c.P * (int64_t)prm->max_nt;
        if (c.P > worst.P) worst.P = c.P;
        if (c.Q > worst.Q) worst.Q = c.Q;
        if (c.T > worst.T) worst.T = c.T;
        if (c.NT > worst.NT) worst.NT = c.NT;
        bounds.push_back(e);
        p = e;
    }
    // pipelined (first_chunk_pairs > 0): the last chunk ramps down too (pieces of 16,
    // 4 and 1 first_chunk_pairs cut from its end), so each chunk's readback hides
    // behind the next chunk's compute and the one no chunk hides is small (a split
    // chunk only shrinks: the worst sizes hold)
    const int first = prm->first_chunk_pairs;
    if (first > 0 && bounds.size() >= 2) {
        const int b0 = bounds[bounds.size() - 2];
        int end = bounds.back();
        std::vector<int> cuts;
        for (int64_t sz = first; sz <= 16 * (int64_t)first; sz *= 4)   // last piece first
            if (end - b0 > 2 * sz) {
                end -= (int)sz;
                cuts.push_back(end);
            }
        std::reverse(cuts.begin(), cuts.end());
        bounds.insert(bounds.end() - 1, cuts.begin(), cuts.end());
    }
}

extern "C" int32_t msfm_guided_chunk_bounds(int32_t n_pairs, const int64_t* h_qlist_off,
                                            const msfm_match_params* prm, int32_t* out_bounds,
                                            int32_t capacity) {
    if (!prm || !h_qlist_off || n_pairs < 0) return -1;
    std::vector<int> bounds;
    ChunkSizes w;
    plan_chunks(n_pairs, h_qlist_off, prm, bounds, w);
    const int32_t nc = (int32_t)bounds.size() - 1;
    if (out_bounds)
        for (int32_t k = 0; k <= nc && k < capacity; k++) out_bounds[k] = bounds[k];
    return nc < 0 ? 0 : nc;
}

extern "C" size_t msfm_guided_workspace_bytes(int32_t n_pairs, const int64_t* h_qlist_off,
                                              const msfm_match_params* prm) {
    if (!prm || !h_qlist_off || n_pairs < 0) return 0;
    std::vector<int> bounds;
    ChunkSizes w;
    plan_chunks(n_pairs, h_qlist_off, prm, bounds, w);
    return chunk_bytes(w);
}

// after each chunk: hook(chunk index, first pair, end pair) -> status
typedef int (*ChunkHookFn)(void* ctx, int c, int p0, int p1);

static int guided_match_impl(const msfm_bank* bank, const msfm_grids* grids, int32_t n_pairs,
                             const int32_t* d_pair_q, const int32_t* d_pair_t,
                             const double* d_pair_F, const int64_t* d_qlist_off,
                             const int32_t* d_qlist, const int64_t* d_qlist_src,
                             const int64_t* h_qlist_off,
                             const msfm_match_params* prm, int32_t* d_out_q, int32_t* d_out_t,
                             float* d_out_dist, float* d_out_ratio, int32_t* d_out_count,
                             int64_t* d_stats, void* d_workspace, size_t workspace_bytes,
                             void* stream, ChunkHookFn hook, void* hook_ctx,
                             const msfm_stage_plan* plan = nullptr) {
    if (!bank || !grids || !prm || n_pairs < 0 || !h_qlist_off) {
        set_error("msfm_guided_match: null argument");
        return MSFM_EINVAL;
    }
    if (!(prm->d > 0)) {
        set_error("msfm_guided_match: band d must be positive, got %g", prm->d);
        return MSFM_EINVAL;
    }
    if (!(grids->D > 0)) {
        set_error("msfm_guided_match: grid cell half-size must be positive, got %g", grids->D);
        return MSFM_EINVAL;
    }
    if (prm->max_nt > 65536) {
        set_error("msfm_guided_match: images with more than 65536 features are not supported");
        return MSFM_EINVAL;
    }
    if (prm->ratio != prm->ratio) {
        set_error("msfm_guided_match: ratio is NaN");
        return MSFM_EINVAL;
    }
    if (n_pairs == 0) return MSFM_OK;
    std::vector<int> bounds;
    ChunkSizes w;
    plan_chunks(n_pairs, h_qlist_off, prm, bounds, w);
    if (workspace_bytes < chunk_bytes(w)) {
        set_error("msfm_guided_match: workspace too small (%zu < %zu)", workspace_bytes, chunk_bytes(w));
        return MSFM_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (d_stats) MSFM_CUDA_TRY(cudaMemsetAsync(d_stats, 0, sizeof(int64_t) * 2 * n_pairs, st));
    Arena ar(d_workspace, workspace_bytes);
    ChunkArgs a;
    a.xy = reinterpret_cast<const float2*>(bank->d_xy);
    a.desc = bank->d_desc; a.norm2 = bank->d_norm2;
    a.img_off = bank->d_img_off; a.img_n = bank->d_img_n; a.img_wh = bank->d_img_wh;
    a.sub = grids->d_sub; a.dims = grids->d_dims; a.roff = grids->d_roff; a.coff = grids->d_coff;
    a.rstart = grids->d_rstart; a.cstart = grids->d_cstart; a.rmem = grids->d_rmem; a.cmem = grids->d_cmem;
    a.rrec = reinterpret_cast<const int4*>(grids->d_rrec);
    a.crec = reinterpret_cast<const int4*>(grids->d_crec);
    a.D = grids->D; a.d = prm->d; a.ratio = prm->ratio; a.single_cap = prm->single_cap;
    a.tie_fid = prm->ratio > 1.0f ? 1 : 0;
    if (prm->strategy < 0 || prm->strategy > 2) {
        set_error("msfm_guided_match: unknown strategy %d", prm->strategy);
        return MSFM_EINVAL;
    }
    a.strategy = prm->strategy;
    {
        const double r = prm->d * sqrt(2.0);      // guided.py:275 radius_factor=np.sqrt(2.0)
        a.r2 = r * r;
    }
    a.stats_mode = d_stats ? 1 : 0;
    {
        const char* e = getenv("MSFM_SG_TAU");
        a.sg_tau = e ? (float)atof(e) : SG_TAU;
    }
    a.pair_q = d_pair_q; a.pair_t = d_pair_t; a.pair_F = d_pair_F;
    a.qlist_off = d_qlist_off; a.qlist = d_qlist; a.qlist_src = d_qlist_src;
    a.q_fid = ar.take<int32_t>(w.Q);
    a.mgid = ar.take<int32_t>(w.Q); a.msg = ar.take<int32_t>(w.Q);
    a.gfit = ar.take<unsigned>(w.Q); a.sgdev = ar.take<unsigned long long>(w.Q);
    a.jmp_a = ar.take<int32_t>(w.Q + w.P + 1); a.jmp_b = ar.take<int32_t>(w.Q + w.P + 1);
    a.jmark = ar.take<int32_t>(w.Q + w.P + 1);
    a.gview = ar.take<GView>(w.Q);
    a.tab_off = ar.take<int64_t>(w.P + 1); a.tbase = ar.take<int64_t>(w.P + 1);
    a.sg_total = ar.take<int32_t>(1);
    a.sg_next = ar.take<int32_t>(1);
    a.gline = ar.take<float4>(w.Q); a.gend = ar.take<float4>(w.Q); a.sglist = ar.take<int2>(w.Q);
    a.tab_key = ar.take<unsigned long long>(w.T);
    a.tab_rep = ar.take<unsigned>(w.T); a.tab_cnt = ar.take<unsigned>(w.T);
    a.q_tab = ar.take<int32_t>(w.Q); a.q_line = ar.take<double>(3 * w.Q);
    a.q_lf = ar.take<float4>(w.Q);
    a.grec = ar.take<int4>(w.Q);
    a.gfill = ar.take<int32_t>(w.Q); a.members = ar.take<int32_t>(w.Q);
    a.grp = ar.take<GroupRec>(w.Q);
    a.mrec = ar.take<MemberRec>(w.Q);
    a.sg = ar.take<SGRec>(w.Q);
    a.gtmp = ar.take<int2>(w.Q); a.gkey = ar.take<float>(w.Q); a.gpos = ar.take<int32_t>(w.Q);
    a.mstate = ar.take<unsigned long long>(w.Q); a.mstate2 = ar.take<unsigned>(w.Q);
    a.res_tid = ar.take<int32_t>(w.Q); a.res_dist = ar.take<float>(w.Q); a.res_ratio = ar.take<float>(w.Q);
    a.dedupe = ar.take<unsigned long long>(w.NT);
    a.stats = reinterpret_cast<unsigned long long*>(d_stats);
    a.dbg = g_dbg;
    a.out_q = d_out_q; a.out_t = d_out_t; a.out_dist = d_out_dist; a.out_ratio = d_out_ratio;
    a.out_count = d_out_count;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    MSFM_CUDA_TRY(cudaFuncSetAttribute(setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SETUP_SMEM));
    if (getenv("MSFM_OCC")) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, setup_kernel, ST, SETUP_SMEM);
        fprintf(stderr, "setup_kernel: %d CTAs/SM (%zu B smem)\n", nb, (size_t)SETUP_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, match_ms_kernel<false, false>, MS_WARPS * 32, sizeof(MSmem) * MS_WARPS);
        fprintf(stderr, "match_ms_kernel: %d CTAs/SM\n", nb);
    }
    const size_t ms_smem = sizeof(MSmem) * MS_WARPS;
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<true, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<false, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<true, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<false, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    const bool sync_dbg = getenv("MSFM_SYNC_CHECK") && atoi(getenv("MSFM_SYNC_CHECK")) != 0;
    // Staged plans: every range is indexed on a high-priority side stream as soon as
    // its rows land, so range r + 1's grid build runs beside chunk c's kernels (in the
    // tail of its persistent match kernel) instead of between chunks on `st`; chunk c
    // waits only for the builds of the ranges it reads.  Ranges write disjoint bucket
    // and |desc|^2 rows, and the builds share the plan's workspace in stream order.
    std::vector<cudaEvent_t> built;
    struct EvGuard {
        std::vector<cudaEvent_t>& v;
        ~EvGuard() { for (cudaEvent_t e : v) cudaEventDestroy(e); }
    } ev_guard{built};
    if (plan && plan->n_ranges > 0) {
        static cudaStream_t side[64];
        if (dev < 0 || dev >= 64) {
            set_error("msfm_guided_match_rows: device index %d out of range", dev);
            return MSFM_EINVAL;
        }
        if (!side[dev]) {
            int lo = 0, hi = 0;
            MSFM_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            MSFM_CUDA_TRY(cudaStreamCreateWithPriority(&side[dev], cudaStreamNonBlocking, hi));
        }
        cudaStream_t ix = side[dev];
        cudaEvent_t e0;
        MSFM_CUDA_TRY(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
        built.push_back(e0);
        MSFM_CUDA_TRY(cudaEventRecord(e0, st));        // everything `st` did before
        MSFM_CUDA_TRY(cudaStreamWaitEvent(ix, e0, 0));
        for (int r = 0; r < plan->n_ranges; r++) {
            if (plan->landed && plan->landed[r])
                MSFM_CUDA_TRY(cudaStreamWaitEvent(ix, (cudaEvent_t)plan->landed[r], 0));
            const int64_t f0 = plan->feat0[r], f1 = plan->feat1[r];
            if (f1 < f0 || f1 > bank->n_total) {
                set_error("msfm_guided_match_rows: stage range %d rows [%lld, %lld)", r,
                          (long long)f0, (long long)f1);
                return MSFM_EINVAL;
            }
            // a plan hands the matcher the (otherwise read-only) |desc|^2 and index
            // arrays of its ranges to fill
            auto w32 = [](const int32_t* p) { return const_cast<int32_t*>(p); };
            // |desc|^2 of the range computed by the build's count pass
            int rc = grid_build_range_impl(bank, grids->d_dims, grids->d_roff, grids->d_coff,
                                           plan->n_buckets_total, plan->img0[r], plan->img1[r],
                                           plan->bucket0[r], plan->bucket1[r], f0, grids->D,
                                           w32(grids->d_sub), w32(grids->d_rstart),
                                           w32(grids->d_cstart), w32(grids->d_rmem),
                                           w32(grids->d_cmem), w32(grids->d_rrec),
                                           w32(grids->d_crec), plan->grid_workspace,
                                           plan->grid_workspace_bytes, ix, w32(bank->d_norm2));
            if (rc) return rc;
            cudaEvent_t e;
            MSFM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            built.push_back(e);
            MSFM_CUDA_TRY(cudaEventRecord(e, ix));
        }
    }
    int next_range = 0;
    for (size_t c = 0; c + 1 < bounds.size(); c++) {
        const int p0 = bounds[c], p1 = bounds[c + 1];
        a.p0 = p0;
        a.npairs = p1 - p0;
        a.qbase = h_qlist_off[p0];
        // bank ranges first read by this chunk: wait for their grid builds
        for (; plan && next_range < plan->n_ranges && plan->chunk[next_range] <= (int32_t)c;
             next_range++)
            MSFM_CUDA_TRY(cudaStreamWaitEvent(st, built[next_range + 1], 0));
        // MSFM_SYNC_CHECK=1: synchronize after every kernel and name the one that failed
        auto sync_check = [&](const char* what) -> int {
            if (!sync_dbg) return MSFM_OK;
            const cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) {
                set_error("msfm_guided_match: %s (chunk %d): %s", what, (int)c, cudaGetErrorString(e));
                return MSFM_ECUDA;
            }
            return MSFM_OK;
        };
        plan_kernel<<<1, SCAN_T, 0, st>>>(a);
        if (int rc = sync_check("plan_kernel")) return rc;
        { ProfScope ps("setup_kernel", st); setup_kernel<<<a.npairs, ST, SETUP_SMEM, st>>>(a); }
        if (int rc = sync_check("setup_kernel")) return rc;
        {
            ProfScope ps("match_kernel", st);
            const dim3 grid(nsm * MS_MINB), block(MS_WARPS * 32);
            if (a.tie_fid) {
                if (d_stats) match_ms_kernel<true, true><<<grid, block, ms_smem, st>>>(a);
                else         match_ms_kernel<false, true><<<grid, block, ms_smem, st>>>(a);
            } else {
                if (d_stats) match_ms_kernel<true, false><<<grid, block, ms_smem, st>>>(a);
                else         match_ms_kernel<false, false><<<grid, block, ms_smem, st>>>(a);
            }
        }
        if (int rc = sync_check("match_kernel")) return rc;
        { ProfScope ps("compact_kernel", st); compact_kernel<<<a.npairs, CT, 0, st>>>(a); }
        if (int rc = sync_check("compact_kernel")) return rc;
        MSFM_LAUNCH_CHECK();
        count_launches(4);
        if (hook) {
            const int rc = hook(hook_ctx, (int)c, p0, p1);
            if (rc) return rc;
        }
    }
    // later work on `st` (the next step's uploads into the bank) follows every build
    if (!built.empty()) MSFM_CUDA_TRY(cudaStreamWaitEvent(st, built.back(), 0));
    return MSFM_OK;
}

extern "C" int msfm_guided_match(const msfm_bank* bank, const msfm_grids* grids, int32_t n_pairs,
                                 const int32_t* d_pair_q, const int32_t* d_pair_t,
                                 const double* d_pair_F, const int64_t* d_qlist_off,
                                 const int32_t* d_qlist, const int64_t* d_qlist_src,
                                 const int64_t* h_qlist_off,
                                 const msfm_match_params* prm, int32_t* d_out_q, int32_t* d_out_t,
                                 float* d_out_dist, float* d_out_ratio, int32_t* d_out_count,
                                 int64_t* d_stats, void* d_workspace, size_t workspace_bytes,
                                 void* stream) {
    return guided_match_impl(bank, grids, n_pairs, d_pair_q, d_pair_t, d_pair_F, d_qlist_off,
                             d_qlist, d_qlist_src, h_qlist_off, prm, d_out_q, d_out_t, d_out_dist,
                             d_out_ratio, d_out_count, d_stats, d_workspace, workspace_bytes,
                             stream, nullptr, nullptr);
}

namespace {
// pipelined packing + device-to-host copy of every finished chunk
struct RowsCtx {
    cudaStream_t st, copy;
    const int64_t* qlist_off; const int32_t* count;
    const int32_t* q; const int32_t* t; const float* dist; const float* ratio;
    int64_t* out_off; int32_t* d_rows; int32_t* h_rows;
    int64_t* d_meta; int64_t* h_meta;
    std::vector<cudaEvent_t> ev;
    int flushed;
};

int rows_flush(RowsCtx& x, int c) {
    MSFM_CUDA_TRY(cudaEventSynchronize(x.ev[c]));
    const int64_t base = x.h_meta[2 * c], tot = x.h_meta[2 * c + 1];
    if (tot > 0) {
        MSFM_CUDA_TRY(cudaStreamWaitEvent(x.copy, x.ev[c], 0));
        MSFM_CUDA_TRY(cudaMemcpyAsync(x.h_rows + 4 * base, x.d_rows + 4 * base,
                                      (size_t)tot * 16, cudaMemcpyDeviceToHost, x.copy));
    }
    x.flushed = c + 1;
    return MSFM_OK;
}

int rows_hook(void* ctx, int c, int p0, int p1) {
    RowsCtx& x = *static_cast<RowsCtx*>(ctx);
    const int np = p1 - p0;
    pack_chunk_scan_kernel<<<1, SCAN_T, 0, x.st>>>(x.count, p0, np, c, x.out_off, x.d_meta);
    pack_kernel<<<np, 128, 0, x.st>>>(x.qlist_off, x.count, x.out_off, x.q, x.t, x.dist, x.ratio,
                                      reinterpret_cast<int4*>(x.d_rows), p0);
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    MSFM_CUDA_TRY(cudaMemcpyAsync(x.h_meta + 2 * c, x.d_meta + 2 * c, 2 * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, x.st));
    cudaEvent_t e;
    MSFM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MSFM_CUDA_TRY(cudaEventRecord(e, x.st));
    x.ev.push_back(e);
    // the previous chunk's rows go out while this chunk computes
    if (c > 0) return rows_flush(x, c - 1);
    return MSFM_OK;
}
}  // namespace

extern "C" int msfm_guided_match_rows(const msfm_bank* bank, const msfm_grids* grids,
                                      int32_t n_pairs, const int32_t* d_pair_q,
                                      const int32_t* d_pair_t, const double* d_pair_F,
                                      const int64_t* d_qlist_off, const int32_t* d_qlist,
                                      const int64_t* d_qlist_src, const int64_t* h_qlist_off,
                                      const msfm_match_params* prm, int32_t* d_out_q,
                                      int32_t* d_out_t, float* d_out_dist, float* d_out_ratio,
                                      int32_t* d_out_count, int64_t* d_out_off, int32_t* d_rows,
                                      int64_t* d_meta, int64_t* h_meta, int32_t* h_rows,
                                      int64_t* h_total, void* d_workspace,
                                      size_t workspace_bytes, void* stream, void* copy_stream,
                                      const msfm_stage_plan* plan) {
    if (!d_out_off || !d_rows || !d_meta || !h_meta || !h_rows || !h_total || !copy_stream) {
        set_error("msfm_guided_match_rows: null argument");
        return MSFM_EINVAL;
    }
    *h_total = 0;
    RowsCtx x;
    x.st = (cudaStream_t)stream; x.copy = (cudaStream_t)copy_stream;
    x.qlist_off = d_qlist_off; x.count = d_out_count;
    x.q = d_out_q; x.t = d_out_t; x.dist = d_out_dist; x.ratio = d_out_ratio;
    x.out_off = d_out_off; x.d_rows = d_rows; x.h_rows = h_rows;
    x.d_meta = d_meta; x.h_meta = h_meta; x.flushed = 0;
    int rc = guided_match_impl(bank, grids, n_pairs, d_pair_q, d_pair_t, d_pair_F, d_qlist_off,
                               d_qlist, d_qlist_src, h_qlist_off, prm, d_out_q, d_out_t,
                               d_out_dist, d_out_ratio, d_out_count, nullptr, d_workspace,
                               workspace_bytes, stream, rows_hook, &x, plan);
    if (rc == MSFM_OK && !x.ev.empty()) rc = rows_flush(x, (int)x.ev.size() - 1);
    if (rc == MSFM_OK) {
        cudaError_t e = cudaStreamSynchronize(x.copy);
        if (e != cudaSuccess) {
            set_error("msfm_guided_match_rows: %s", cudaGetErrorString(e));
            rc = MSFM_ECUDA;
        }
    }
    if (rc == MSFM_OK && !x.ev.empty()) {
        const int last = (int)x.ev.size() - 1;
        *h_total = h_meta[2 * last] + h_meta[2 * last + 1];
    }
    for (cudaEvent_t e : x.ev) cudaEventDestroy(e);
    return rc;
}
