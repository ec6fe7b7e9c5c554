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
    return np_hypot(pb[0] - pa[0], pb[1] - pa[1]) > 1e-12;
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
    return !(np_hypot(pb[0] - pa[0], pb[1] - pa[1]) < 1e-12);
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
    const int img = a.img0 + blockIdx.x;
    const int64_t off = a.img_off[img];
    const int n = a.img_n[img];
    const int nbx = a.dims[2 * img], nby = a.dims[2 * img + 1];
    for (int f = threadIdx.x; f < n; f += blockDim.x) {
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
    const int img = a.img0 + blockIdx.x;
    const int64_t off = a.img_off[img];
    const int n = a.img_n[img];
    const int nbx = a.dims[2 * img], nby = a.dims[2 * img + 1];
    for (int f = threadIdx.x; f < n; f += blockDim.x) {
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
struct GroupRec {
    int p, rep, cnt, moff;                 // chunk-local pair, rep slot, members, member offset
    float ar, br, cr, hsure;               // rep line (fp32), sure-in-C' radius
    float pbx, pby, dirx, diry;            // padded segment origin (pb) and direction
    float len, spacing, invK, invD;
    float dxf, dyf, slack, maxdev;         // maxdev: max member-band deviation from the rep line
    int K, pad1, pad2, pad3;               // K<0: the rep line misses the padded image (C' empty)
    double pax, pay, pbx64, pby64;         // exact sample interpolation (guided.py:187)
    double sl0, sl1, sl2, spare;           // singleton member's own (dgemv) line
};

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
constexpr float SG_TAU = 16.0f;
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
    int stats_mode;              // 1: one super-group per group (exact SearchStats)
    int strategy;                // 0 grid, 1 linear, 2 radial (msfm_match_params)
    double r2;                   // radial: (d * sqrt(2))^2 as the reference rounds it
    float sg_tau;                // super-group line tolerance (px)
    // pairs
    const int32_t* pair_q; const int32_t* pair_t; const double* pair_F;
    const int64_t* qlist_off; const int32_t* qlist;
    const int64_t* qlist_src;    // optional: per-pair start of its list inside qlist
    int32_t* q_fid;              // chunk-local query feature ids (filled by lines_kernel)
    int32_t p0, npairs; int64_t qbase;
    // chunk workspace
    int64_t* tab_off; int64_t* tbase; int32_t* ngroups; int32_t* gstart; int32_t* nmem;
    int32_t* sgstart; int32_t* sg_next; int32_t* nsg;
    unsigned long long* tab_key; unsigned* tab_rep; unsigned* tab_cnt;
    int32_t* q_tab; double* q_line;
    int2* gtmp; float* gkey; int32_t* gpos; float4* gline; float4* gend; int2* sglist;
    int4* grec; int32_t* gfill; int32_t* members; GroupRec* grp; MemberRec* mrec; SGRec* sg;
    int32_t* mgid;               // per member position: dense group id (-1: unused position)
    int32_t* msg;                // per member position: super-group id
    unsigned* gfit;              // per sorted group: bit i = group g+1+i fits g's line (tau)
    unsigned long long* sgdev;   // per super-group: max member-band deviation (f64 bits)
    float4* gl4;                 // per dense group: rep line (fp32) + member-band reach
    int32_t* gmoff;              // per dense group: first member position
    GView* gview;                // per dense group: the two above as one 32-B record
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

__global__ void plan_kernel(ChunkArgs a) {
    __shared__ int sm[SCAN_T / 32 + 1];
    long long carry_t = 0, carry_d = 0;
    for (int b0 = 0; b0 < a.npairs; b0 += SCAN_T) {
        int p = b0 + threadIdx.x;
        int ts = 0, nt = 0;
        if (p < a.npairs) {
            int pg = a.p0 + p;
            int nq = (int)(a.qlist_off[pg + 1] - a.qlist_off[pg]);
            ts = nextpow2(nq + 1);
            nt = a.img_n[a.pair_t[pg]];
        }
        int tot_t, tot_d;
        int ex_t = block_exclusive_scan<SCAN_T>(ts, &tot_t, sm);
        int ex_d = block_exclusive_scan<SCAN_T>(nt, &tot_d, sm);
        if (p < a.npairs) {
            a.tab_off[p] = carry_t + ex_t;
            a.tbase[p] = carry_d + ex_d;
        }
        carry_t += tot_t;
        carry_d += tot_d;
    }
    if (threadIdx.x == 0) {
        a.tab_off[a.npairs] = carry_t;
        a.tbase[a.npairs] = carry_d;
    }
}

#ifndef MSFM_LINES_T
#define MSFM_LINES_T 1024
#endif
__global__ void __launch_bounds__(MSFM_LINES_T) lines_kernel(ChunkArgs a) {
    const int p = blockIdx.x, pg = a.p0 + p;
    const int64_t q0 = a.qlist_off[pg];
    const int nq = (int)(a.qlist_off[pg + 1] - q0);
    const int64_t s0 = q0 - a.qbase;
    const int64_t t0 = a.tab_off[p];
    const int tsize = (int)(a.tab_off[p + 1] - t0);
    const int ti = a.pair_t[pg], qi = a.pair_q[pg];
    const int nt = a.img_n[ti];
    const int64_t db = a.tbase[p];
    for (int e = threadIdx.x; e < tsize; e += blockDim.x) {
        a.tab_key[t0 + e] = EMPTY;
        a.tab_rep[t0 + e] = NONE;
        a.tab_cnt[t0 + e] = 0;
    }
    for (int e = threadIdx.x; e < nt; e += blockDim.x) a.dedupe[db + e] = EMPTY;
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
        a.res_tid[s0 + i] = -1;
        a.gfill[s0 + i] = 0;
        a.mgid[s0 + i] = -1;
    }
    if (threadIdx.x == 0) { a.ngroups[p] = 0; a.nmem[p] = 0; }
    __syncthreads();
    double F[9];
#pragma unroll
    for (int j = 0; j < 9; j++) F[j] = a.pair_F[9 * (int64_t)pg + j];
    if (isnan(F[0])) {
        for (int i = threadIdx.x; i < nq; i += blockDim.x) a.q_tab[s0 + i] = -1;
        return;
    }
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1];
    const int64_t qoff = a.img_off[qi];
    const unsigned mask = (unsigned)tsize - 1;
    const int64_t qs = a.qlist_src ? a.qlist_src[pg] : q0;
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
        const int fid = a.qlist[qs + i];
        a.q_fid[s0 + i] = fid;
        const float2 p2 = a.xy[qoff + fid];
        double l[3];
        epiline(F, (double)p2.x, (double)p2.y, nq == 1, l);
        const double nrm = np_hypot(l[0], l[1]);
        int slot = -1;
        if (nrm > 1e-12) {
            l[0] /= nrm; l[1] /= nrm; l[2] /= nrm;
            double pa[2], pb[2];
            if (clip_batch(l, W, H, pa, pb)) {
                const unsigned long long key = composite_key(pa, pb);
                unsigned h = (unsigned)mix64(key) & mask;
                while (true) {
                    unsigned long long prev = atomicCAS(&a.tab_key[t0 + h], EMPTY, key);
                    if (prev == EMPTY || prev == key) break;
                    h = (h + 1) & mask;
                }
                atomicMin(&a.tab_rep[t0 + h], (unsigned)i);
                atomicAdd(&a.tab_cnt[t0 + h], 1u);
                slot = (int)h;
                double* L = a.q_line + 3 * (s0 + i);
                L[0] = l[0]; L[1] = l[1]; L[2] = l[2];
            }
        }
        a.q_tab[s0 + i] = slot;
    }
}

// Groups of a pair: compact the occupied hash slots, then order the groups by
// the angle of their representative line (adaptive 4096-bucket counting sort)
// so consecutive groups have nearly identical lines, and lay out their member
// ranges in that order.  The order only affects how members are packed into
// super-groups, never any result.
constexpr int GB = 4096;
constexpr int GT = 1024;   // groups_kernel threads per pair
__global__ void __launch_bounds__(GT, 2) groups_kernel(ChunkArgs a) {
    __shared__ int sm[GT / 32 + 1];
    __shared__ int hist[GB];
    __shared__ float fmin_s[GT / 32], fmax_s[GT / 32];
    const int p = blockIdx.x, pg = a.p0 + p;
    const int64_t s0 = a.qlist_off[pg] - a.qbase;
    const int64_t t0 = a.tab_off[p];
    const int tsize = (int)(a.tab_off[p + 1] - t0);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int gcarry = 0;
    float lo = 1e30f, hi = -1e30f;
    for (int e0 = 0; e0 < tsize; e0 += GT) {
        const int e = e0 + threadIdx.x;
        bool occ = false;
        unsigned cnt = 0, rep = 0;
        if (e < tsize) {
            occ = a.tab_key[t0 + e] != EMPTY;
            if (occ) { cnt = a.tab_cnt[t0 + e]; rep = a.tab_rep[t0 + e]; }
        }
        int gtot;
        const int lg = block_exclusive_scan<GT>(occ ? 1 : 0, &gtot, sm);
        if (occ) {
            const int g = gcarry + lg;
            a.gtmp[s0 + g] = make_int2((int)rep, (int)cnt);
            const double* L = a.q_line + 3 * (s0 + rep);
            float la = (float)L[0], lb = (float)L[1];
            if (la < 0.f || (la == 0.f && lb < 0.f)) { la = -la; lb = -lb; }
            const float ang = atan2f(lb, la);
            a.gkey[s0 + g] = ang;
            lo = fminf(lo, ang);
            hi = fmaxf(hi, ang);
            a.tab_rep[t0 + e] = (unsigned)g;
        }
        gcarry += gtot;
    }
    const int ng = gcarry;
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
    }
    if (lane == 0) { fmin_s[wid] = lo; fmax_s[wid] = hi; }
    for (int b = threadIdx.x; b < GB; b += GT) hist[b] = 0;
    __syncthreads();
    lo = fmin_s[0]; hi = fmax_s[0];
    for (int w = 1; w < GT / 32; w++) { lo = fminf(lo, fmin_s[w]); hi = fmaxf(hi, fmax_s[w]); }
    const float scale = (float)GB / fmaxf(hi - lo, 1e-20f);
    for (int g = threadIdx.x; g < ng; g += GT) {
        const int b = min(GB - 1, max(0, (int)((a.gkey[s0 + g] - lo) * scale)));
        atomicAdd(&hist[b], 1);
    }
    __syncthreads();
    // exclusive scan of the histogram (16 buckets per thread)
    {
        int v[GB / GT];
        int s = 0;
        for (int k = 0; k < GB / GT; k++) { v[k] = hist[threadIdx.x * (GB / GT) + k]; s += v[k]; }
        int tot;
        int ex = block_exclusive_scan<GT>(s, &tot, sm);
        for (int k = 0; k < GB / GT; k++) { hist[threadIdx.x * (GB / GT) + k] = ex; ex += v[k]; }
    }
    __syncthreads();
    for (int g = threadIdx.x; g < ng; g += GT) {
        const int b = min(GB - 1, max(0, (int)((a.gkey[s0 + g] - lo) * scale)));
        a.gpos[s0 + g] = atomicAdd(&hist[b], 1);
    }
    __syncthreads();
    int mcarry = 0;
    // write grec in sorted order (scatter by gpos), then scan counts in that order
    for (int g = threadIdx.x; g < ng; g += GT) {
        const int2 r = a.gtmp[s0 + g];
        a.grec[s0 + a.gpos[s0 + g]] = make_int4(r.x, r.y, 0, 0);
    }
    __syncthreads();
    for (int i0 = 0; i0 < ng; i0 += GT) {
        const int i = i0 + threadIdx.x;
        const int cnt = i < ng ? a.grec[s0 + i].y : 0;
        int tot;
        const int ex = block_exclusive_scan<GT>(cnt, &tot, sm);
        if (i < ng) a.grec[s0 + i].z = (int)(s0 + mcarry + ex);
        mcarry += tot;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < tsize; e += GT) {
        if (a.tab_key[t0 + e] != EMPTY) a.tab_rep[t0 + e] = (unsigned)a.gpos[s0 + a.tab_rep[t0 + e]];
    }
    // boundary endpoints of every representative line (in sorted order)
    const int ti = a.pair_t[pg];
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1];
    for (int g = threadIdx.x; g < ng; g += GT) {
        const int4 gr = a.grec[s0 + g];
        const double* L = a.q_line + 3 * (s0 + gr.x);
        const double l[3] = {L[0], L[1], L[2]};
        double pa[2] = {0, 0}, pb[2] = {0, 0};
        clip_batch(l, W, H, pa, pb);
        a.gline[s0 + g] = make_float4((float)l[0], (float)l[1], (float)l[2], 0.f);
        a.gend[s0 + g] = make_float4((float)pa[0], (float)pa[1], (float)pb[0], (float)pb[1]);
    }
    __syncthreads();
    // super-groups: greedy walk over the angle-ordered groups; a super-group holds
    // at most SG_MEMBERS members and closes when the next group's line leaves the
    // base line by more than SG_TAU px inside the image (stats mode: one per group).
    // The tau tests run in parallel (gfit bit i: group g+1+i fits group g's line);
    // one thread then walks the groups with integer work only.
    if (a.stats_mode) {
        for (int g = threadIdx.x; g < ng; g += GT) {
            const int4 gr = a.grec[s0 + g];
            a.sglist[s0 + g] = make_int2(gr.z, gr.y);
        }
        if (threadIdx.x == 0) a.nsg[p] = ng;
    } else {
        for (int g = threadIdx.x; g < ng; g += GT) {
            const float4 ln = a.gline[s0 + g];
            unsigned bits = 0;
            const int lim = min(SG_MEMBERS, ng - 1 - g);
            for (int i = 0; i < lim; i++) {
                const float4 en = a.gend[s0 + g + 1 + i];
                const float d1 = fabsf(fmaf(ln.x, en.x, fmaf(ln.y, en.y, ln.z)));
                const float d2 = fabsf(fmaf(ln.x, en.z, fmaf(ln.y, en.w, ln.z)));
                if (fmaxf(d1, d2) <= a.sg_tau) bits |= 1u << i;
            }
            a.gfit[s0 + g] = bits;
        }
        __syncthreads();
        // The super-groups partition the member sequence into contiguous ranges, so the
        // greedy walk is a chain over member positions: end[q] = where the super-group
        // opened at position q closes (all q in parallel), then one thread follows the
        // chain from 0 through shared memory.
        extern __shared__ unsigned short send[];
        const int nm = mcarry;
        for (int g = threadIdx.x; g < ng; g += GT) {
            const int4 gr = a.grec[s0 + g];
            const int cnt = gr.y, rel0 = (int)(gr.z - s0);
            const unsigned fit = a.gfit[s0 + g];
            for (int k = 0; k < cnt; k++) {
                const int q = rel0 + k, r = cnt - k;
                int e;
                if (r > SG_MEMBERS) {
                    e = q + SG_MEMBERS;
                } else {
                    int cur = r, j = g + 1;
                    e = -1;
                    while (j < ng && cur < SG_MEMBERS && ((fit >> (j - g - 1)) & 1u)) {
                        const int4 gj = a.grec[s0 + j];
                        const int take = min(SG_MEMBERS - cur, gj.y);
                        cur += take;
                        if (take < gj.y) { e = (int)(gj.z - s0) + take; break; }
                        j++;
                    }
                    if (e < 0) e = j < ng ? (int)(a.grec[s0 + j].z - s0) : nm;
                }
                send[q] = (unsigned short)e;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int nsg = 0;
            for (int q = 0; q < nm;) {
                const int e = send[q];
                a.sglist[s0 + nsg++] = make_int2((int)s0 + q, e - q);
                q = e;
            }
            a.nsg[p] = nsg;
        }
    }
    if (threadIdx.x == 0) { a.ngroups[p] = ng; a.nmem[p] = mcarry; }
}

__global__ void gscan_kernel(ChunkArgs a) {
    __shared__ int sm[SCAN_T / 32 + 1];
    int carry = 0, carry_sg = 0;
    for (int b0 = 0; b0 < a.npairs; b0 += SCAN_T) {
        int p = b0 + threadIdx.x;
        int v = p < a.npairs ? a.ngroups[p] : 0;
        int vs = 0;
        if (p < a.npairs) vs = a.nsg[p];
        int total, total_sg;
        int ex = block_exclusive_scan<SCAN_T>(v, &total, sm);
        int exs = block_exclusive_scan<SCAN_T>(vs, &total_sg, sm);
        if (p < a.npairs) { a.gstart[p] = carry + ex; a.sgstart[p] = carry_sg + exs; }
        carry += total;
        carry_sg += total_sg;
    }
    if (threadIdx.x == 0) {
        a.gstart[a.npairs] = carry;
        a.sgstart[a.npairs] = carry_sg;
        *a.sg_next = 0;
    }
}

__global__ void __launch_bounds__(MSFM_LINES_T) scatter_kernel(ChunkArgs a) {
    const int p = blockIdx.x, pg = a.p0 + p;
    const int64_t q0 = a.qlist_off[pg];
    const int nq = (int)(a.qlist_off[pg + 1] - q0);
    const int64_t s0 = q0 - a.qbase;
    const int64_t t0 = a.tab_off[p];
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
        const int h = a.q_tab[s0 + i];
        if (h < 0) continue;
        const int lg = (int)a.tab_rep[t0 + h];
        const int4 g = a.grec[s0 + lg];
        const int pos = g.z + atomicAdd(&a.gfill[s0 + lg], 1);
        a.members[pos] = (int)(s0 + i);
        a.mgid[pos] = a.gstart[p] + lg;
    }
}

__device__ __forceinline__ int find_pair(const int32_t* gstart, int npairs, int gid) {
    int lo = 0, hi = npairs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (gstart[mid] <= gid) lo = mid; else hi = mid - 1;
    }
    return lo;
}

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

// |dist_g - dist_base| over the whole image rectangle (affine -> max at a corner)

// Per group: the C' geometry of its representative line + member constants.
__global__ void __launch_bounds__(128) prep_kernel(ChunkArgs a, int max_groups) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = a.gstart[a.npairs];
    if (gid >= total || gid >= max_groups) return;
    const int p = find_pair(a.gstart, a.npairs, gid);
    const int pg = a.p0 + p;
    const int64_t q0 = a.qlist_off[pg];
    const int64_t s0 = q0 - a.qbase;
    const int4 g = a.grec[s0 + (gid - a.gstart[p])];
    const int ti = a.pair_t[pg];
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1], D = a.D, d = a.d;
    const double* rl = a.q_line + 3 * (s0 + g.x);
    const double r[3] = {rl[0], rl[1], rl[2]};
    GroupRec o;
    o.p = p; o.rep = (int)(s0 + g.x); o.cnt = g.y; o.moff = g.z;
    o.sl0 = r[0]; o.sl1 = r[1]; o.sl2 = r[2]; o.spare = 0.0;
    o.pad1 = o.pad2 = o.pad3 = 0;
    double maxdev = 0.0;
    double pa[2] = {0, 0}, pb[2] = {0, 0}, len = 0.0;
    o.K = -1;
    if (clip_scalar(r[0], r[1], r[2], W, H, d, pa, pb)) {
        len = np_hypot(pb[0] - pa[0], pb[1] - pa[1]);
        long long K = (long long)ceil(len / d);
        o.K = (int)(K < 1 ? 1 : K);
    }
    o.pax = pa[0]; o.pay = pa[1]; o.pbx64 = pb[0]; o.pby64 = pb[1];
    o.ar = (float)r[0]; o.br = (float)r[1]; o.cr = (float)r[2];
    o.maxdev = (float)(maxdev + 0.05);   // raised by member_kernel (atomic max of f32 bits)
    const double hs2 = D * D - 0.25 * d * d;
    o.hsure = hs2 > 0 ? (float)(sqrt(hs2) - 0.075) : -1.0f;
    o.pbx = (float)pb[0]; o.pby = (float)pb[1];
    o.dirx = len > 0 ? (float)((pa[0] - pb[0]) / len) : 0.f;
    o.diry = len > 0 ? (float)((pa[1] - pb[1]) / len) : 0.f;
    o.len = (float)len;
    o.spacing = o.K > 0 ? fmaxf((float)(len / o.K), 1e-6f) : 1.0f;
    o.invK = o.K > 0 ? (float)(1.0 / o.K) : 0.f;
    o.dxf = (float)(pa[0] - pb[0]); o.dyf = (float)(pa[1] - pb[1]);
    o.slack = (float)(4e-6 * (W + H + 4.0 * d) / D) + 1e-4f;
    o.invD = (float)(1.0 / D);
    a.grp[gid] = o;
}

// Per super-group: member window, its groups, the base line and strip.
// Super-group shape (thread per super-group): group range and base line.
__global__ void __launch_bounds__(128) sg_shape_kernel(ChunkArgs a, int max_sg) {
    const int sid = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = a.sgstart[a.npairs];
    if (sid >= total || sid >= max_sg) return;
    const int p = find_pair(a.sgstart, a.npairs, sid);
    const int ls = sid - a.sgstart[p];
    const int pg = a.p0 + p;
    const int64_t s0 = a.qlist_off[pg] - a.qbase;
    const int ng = a.ngroups[p];
    SGRec o = {};
    o.p = p;
    int lg0, lg1;                       // group range [lg0, lg1] (sorted order)
    const int2 sgm = a.sglist[s0 + ls];
    o.m0 = sgm.x; o.mcnt = sgm.y;
    if (a.stats_mode) {
        lg0 = lg1 = ls;
    } else {
        // groups containing the first and last member (member offsets ascend with lg)
        auto group_of = [&](int m) {
            int lo = 0, hi = ng - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (a.grec[s0 + mid].z <= m) lo = mid; else hi = mid - 1;
            }
            return lo;
        };
        lg0 = group_of(o.m0);
        lg1 = group_of(o.m0 + o.mcnt - 1);
    }
    o.g0 = a.gstart[p] + lg0;
    o.gcnt = lg1 - lg0 + 1;
    // base line: the middle group's representative (its chunk-local slot in rlo)
    o.rlo = a.grp[a.gstart[p] + (lg0 + lg1) / 2].rep;
    for (int j = 0; j < o.mcnt; j++) a.msg[o.m0 + j] = sid;
    a.sgdev[sid] = 0ull;
    a.sg[sid] = o;
}

// Per member (thread per member position): epilogue constants, the member band's
// deviation from its group's representative line (-> GroupRec.maxdev) and from its
// super-group's base line (-> sgdev), both as atomic maxima.
__global__ void __launch_bounds__(128, 12) member_kernel(ChunkArgs a, int max_pos) {
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= max_pos) return;
    const int gid = a.mgid[pos];
    if (gid < 0) return;
    GroupRec& G = a.grp[gid];
    const int p = G.p, pg = a.p0 + p;
    const int ti = a.pair_t[pg], qi = a.pair_q[pg];
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1], d = a.d;
    const int64_t qoff = a.img_off[qi];
    const int slot = a.members[pos];
    const int fid = a.q_fid[slot];
    double m[3];
    if (G.cnt == 1) {
        // a singleton's own band uses the dgemv-rounded line (guided.py:443-446, m == 1)
        double F[9];
        for (int j = 0; j < 9; j++) F[j] = a.pair_F[9 * (int64_t)pg + j];
        const float2 p2 = a.xy[qoff + fid];
        epiline(F, (double)p2.x, (double)p2.y, true, m);
        double nrm = fmax(np_hypot(m[0], m[1]), 1e-15);
        m[0] /= nrm; m[1] /= nrm; m[2] /= nrm;
        G.sl0 = m[0]; G.sl1 = m[1]; G.sl2 = m[2];
    } else {
        const double* ml = a.q_line + 3 * (int64_t)slot;
        m[0] = ml[0]; m[1] = ml[1]; m[2] = ml[2];
    }
    const double* rl = a.q_line + 3 * (int64_t)G.rep;
    const double r[3] = {rl[0], rl[1], rl[2]};
    const int sid = a.msg[pos];
    const SGRec& SG = a.sg[sid];
    const double* bl = a.q_line + 3 * (int64_t)SG.rlo;
    const double b[3] = {bl[0], bl[1], bl[2]};
    double rdev, sdev;
    band_deviation2(m, r, b, W, H, d, rdev, sdev);
    const float gdev = (float)(rdev + 0.05);
    atomicMax(reinterpret_cast<unsigned*>(&G.maxdev), __float_as_uint(gdev));
    atomicMax(&a.sgdev[sid], (unsigned long long)__double_as_longlong(sdev));
    MemberRec mr;
    mr.a = (float)m[0]; mr.b = (float)m[1]; mr.c = (float)m[2];
    const float eps = (float)((fabs(m[0]) * W + fabs(m[1]) * H + fabs(m[2])) * 0x1p-20) + 1e-6f;
    mr.lo = (float)d - eps;
    mr.hi = (float)d + eps;
    mr.qn9 = (unsigned)a.norm2[qoff + fid] << 9;
    mr.fid = fid;
    mr.slotgi = (int)((unsigned)slot | ((unsigned)(gid - SG.g0) << SLOT_BITS));
    a.mrec[pos] = mr;
}

// Super-group strip geometry (thread per super-group), after member_kernel.
__global__ void __launch_bounds__(128) sg_prep_kernel(ChunkArgs a, int max_sg) {
    const int sid = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = a.sgstart[a.npairs];
    if (sid >= total || sid >= max_sg) return;
    SGRec o = a.sg[sid];
    const int pg = a.p0 + o.p;
    const int ti = a.pair_t[pg];
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1], D = a.D, d = a.d;
    const double* bl = a.q_line + 3 * (int64_t)o.rlo;
    const double r[3] = {bl[0], bl[1], bl[2]};
    const double dev = __longlong_as_double((long long)a.sgdev[sid]);
    bool all_k = true;
    const double R = d + dev + 0.05;
    double delta = 0.0;
    for (int g = o.g0; g < o.g0 + o.gcnt; g++) {
        const GroupRec& G = a.grp[g];
        const double* gl = a.q_line + 3 * (int64_t)G.rep;
        const double gr[3] = {gl[0], gl[1], gl[2]};
        // |dist_g - dist_base| over the strip |dist_base| <= R inside the image
        delta = fmax(delta, band_deviation(r, gr, W, H, R));
        all_k = all_k && G.K >= 0;
        // compact per-group view for the match kernel (groups shared by two
        // super-groups get the same values twice)
        a.gl4[g] = (G.K < 0 && a.strategy != 1) ? make_float4(0.f, 0.f, 1e30f, -1.f)
                           : make_float4(G.ar, G.br, G.cr, (float)a.d + G.maxdev + 0.05f);
        a.gmoff[g] = G.moff;
        const float4 v = a.gl4[g];
        GView gv;
        gv.a = v.x; gv.b = v.y; gv.c = v.z; gv.reach = v.w;
        gv.moff = G.moff; gv.pad0 = gv.pad1 = gv.pad2 = 0;
        a.gview[g] = gv;
    }
    o.ar = (float)r[0]; o.br = (float)r[1]; o.cr = (float)r[2]; o.R = (float)R;
    // sure-in-C' radius around the base line: grid, the 3x3 subcell block of the
    // nearest sample (half-size D); radial, the disk of radius r around it; both with the
    // sample spacing <= d.  Linear: the rep-line band itself (fp32 error << 0.05 px).
    const double DC = a.strategy == 2 ? sqrt(a.r2) : D;
    const double hs2 = DC * DC - 0.25 * d * d;
    const double hs = a.strategy == 1 ? d - 0.05 : (hs2 > 0 ? sqrt(hs2) - 0.075 : -1.0);
    o.hsure = (float)hs;
    o.delta = (all_k || a.strategy == 1) ? (float)(delta + 0.01) : 1e30f;
    o.border = a.strategy == 1 ? -1e30f : (float)(fmax(0.0, hs - d) + 0.05);
    o.invD = (float)(1.0 / D);
    o.W = (float)W; o.H = (float)H; o.pad0 = 0;
    const bool horiz = fabs(r[1]) >= fabs(r[0]);
    const int qi = a.pair_q[pg];
    o.toff = a.img_off[ti]; o.qoff = a.img_off[qi];
    o.nalong = horiz ? a.dims[2 * ti] : a.dims[2 * ti + 1];
    o.toffb = horiz ? a.roff[ti] : a.coff[ti];
    o.dbase = a.tbase[o.p];
    const double al = horiz ? r[0] : r[1], be = horiz ? r[1] : r[0];
    const double Pm = horiz ? W : H, Qm = horiz ? H : W;
    const int nrows = horiz ? a.dims[2 * ti + 1] : a.dims[2 * ti];
    double qv[4] = {(-R - r[2]) / be, (R - r[2]) / be, (-R - r[2] - al * Pm) / be, (R - r[2] - al * Pm) / be};
    double qlo = fmin(fmin(qv[0], qv[1]), fmin(qv[2], qv[3]));
    double qhi = fmax(fmax(qv[0], qv[1]), fmax(qv[2], qv[3]));
    int rlo = (int)floor((fmax(qlo, 0.0) - 0.01) / D), rhi = (int)floor((fmin(qhi, Qm) + 0.01) / D);
    o.horiz = horiz;
    o.rlo = rlo < 0 ? 0 : rlo;
    o.rhi = rhi > nrows - 1 ? nrows - 1 : rhi;
    o.alpha = (float)al; o.beta = (float)be;
    o.inv_alpha = fabs(al) > 1e-6 ? (float)(1.0 / al) : 0.f;
    o.Pmax = (float)Pm;
    a.sg[sid] = o;
}

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

struct alignas(16) WarpSmem {
    float2 xy[CAP];              // candidate positions (from the bucket-ordered records)
    unsigned nrm[CAP];           // candidate |desc|^2
    unsigned short list[CAP];    // candidate feature ids (target-local)
    unsigned short cmask[CAP];   // per candidate: groups (bit gi) whose C' contains it
    unsigned short ulist[CAP];   // positions still to decide
    unsigned sure[CAP / 32];     // candidate in C' of every group of the super-group
    unsigned anyb[CAP / 8];      // stats: candidate inside some member band
    SGRec sg;                    // this warp's super-group (broadcast reads)
    float4 gl[SG_MAX_GROUPS];    // per group: rep line (fp32), member-band reach
    MemberRec mr[SG_MEMBERS];    // the super-group's members (when mcnt <= SG_MEMBERS)
    int gbeg[SG_MAX_GROUPS + 1]; // member range of each group within the super-group
};
static_assert(offsetof(WarpSmem, mr) % 16 == 0, "member records must be 16-B aligned");
static_assert(sizeof(MemberRec) == 32, "MemberRec is read as two 16-B shared loads");


__device__ __forceinline__ bool member_band(const ChunkArgs& a, int gid, const MemberRec& M,
                                            float x, float y) {
    const float v = fabsf(fmaf(M.a, x, fmaf(M.b, y, M.c)));
    if (v <= M.lo) return true;
    if (v > M.hi) return false;
    const GroupRec& G = a.grp[gid];
    if (G.cnt == 1) return band_exact(G.sl0, G.sl1, G.sl2, true, x, y, a.d);
    const double* L = a.q_line + 3 * (int64_t)(M.slotgi & SLOT_MASK);
    return band_exact(L[0], L[1], L[2], false, x, y, a.d);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// volatile shared loads: re-read per tile instead of pinning registers across the loop
__device__ __forceinline__ float4 lds_f4(const void* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_addr(p)));
    return v;
}
__device__ __forceinline__ uint4 lds_u4(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_addr(p)));
    return v;
}

// member block [mt0, mt0 + SG_MEMBERS) of the super-group into S.mr; columns past the
// last member get a line that never passes the band test
__device__ __forceinline__ void stage_members(const ChunkArgs& a, WarpSmem& S, int m0, int m, int mt0) {
    const int lane = threadIdx.x & 31;
    if (lane < SG_MEMBERS) {
        MemberRec M;
        if (mt0 + lane < m) {
            M = a.mrec[m0 + mt0 + lane];
        } else {
            M.a = 0.f; M.b = 0.f; M.c = 1e30f; M.lo = -1.f; M.hi = -1.f;
            M.qn9 = 0; M.fid = 0; M.slotgi = 0;
        }
        S.mr[lane] = M;
    }
}

template <bool STATS>
__device__ void process_round(const ChunkArgs& a, WarpSmem& S, int n, int64_t toff, int64_t qoff,
                              bool first_round, int& cols_total) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const SGRec& SG = S.sg;
    const int m = SG.mcnt;
    const MemberRec* MR = m <= SG_MEMBERS ? S.mr : a.mrec + SG.m0;
    const unsigned all_groups = (1u << SG.gcnt) - 1u;
    // ---- per-group C' bits of the candidates not surely inside every group's C'
    int nu = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        const bool sure = j < n && ((S.sure[j >> 5] >> (j & 31)) & 1u);
        if (j < n) S.cmask[j] = sure ? (unsigned short)all_groups : 0;
        const bool need = j < n && !sure;
        const unsigned bal = __ballot_sync(FULL, need);
        if (need) S.ulist[nu + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)j;
        nu += __popc(bal);
    }
    __syncwarp();
    if (a.dbg && lane == 0) {
        atomicAdd(&a.dbg[5], (unsigned long long)nu);
        atomicAdd(&a.dbg[7], (unsigned long long)((n + 15) >> 4) * ((m + 15) >> 4));
        atomicAdd(&a.dbg[9], 1ull);
    }
    for (int u0 = 0; u0 < nu; u0 += 32) {
        const int uj = u0 + lane;
        if (uj < nu) {
            const int j = S.ulist[uj];
            const int f = S.list[j];
            const float2 p2 = S.xy[j];
            const bool inner = p2.x >= SG.border && p2.x <= SG.W - SG.border &&
                               p2.y >= SG.border && p2.y <= SG.H - SG.border;
            unsigned bits = 0;
            for (int gi = 0; gi < SG.gcnt; gi++) {
                // gl: rep line and member reach; a group whose line misses the image
                // (K < 0) has gl = (0, 0, 1e30) and is never taken
                const float4 gl = S.gl[gi];
                const float dg = fabsf(fmaf(gl.x, p2.x, fmaf(gl.y, p2.y, gl.z)));
                if (dg <= SG.hsure && inner) { bits |= 1u << gi; continue; }
                // outside every member band of this group: the bit is never consulted
                if (dg > gl.w) continue;
                bool any = false;
                for (int k = S.gbeg[gi]; k < S.gbeg[gi + 1] && !any; k++)
                    any = member_band(a, SG.g0 + gi, MR[k], p2.x, p2.y);
                if (any && a.dbg) atomicAdd(&a.dbg[6], 1ull);
                if (any && in_cprime(a, a.grp[SG.g0 + gi], SG, p2.x, p2.y, toff, f))
                    bits |= 1u << gi;
            }
            S.cmask[j] = (unsigned short)bits;
        }
    }
    if (STATS) {
        for (int w = lane; w < CAP / 8; w += 32) S.anyb[w] = 0;
    }
    __syncwarp();
    const int ntiles = (n + 15) >> 4;
    for (int mt0 = 0; mt0 < m; mt0 += SG_MEMBERS) {
        if (m > SG_MEMBERS) {
            __syncwarp();
            stage_members(a, S, SG.m0, m, mt0);
            __syncwarp();
        }
        // B fragments: member mt0 + 8 nt + g of n-tile nt, bytes [32t, 32t+32)
        unsigned bw[SG_NT][8];
#pragma unroll
        for (int nt = 0; nt < SG_NT; nt++) {
            const int j = mt0 + nt * 8 + g;
            if (j < m) {
                const int fid = S.mr[nt * 8 + g].fid;
                const uint4* row = reinterpret_cast<const uint4*>(a.desc + (qoff + fid) * 128) + 2 * t;
                const uint4 v0 = __ldg(row), v1 = __ldg(row + 1);
                bw[nt][0] = v0.x; bw[nt][1] = v0.y; bw[nt][2] = v0.z; bw[nt][3] = v0.w;
                bw[nt][4] = v1.x; bw[nt][5] = v1.y; bw[nt][6] = v1.z; bw[nt][7] = v1.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; k++) bw[nt][k] = 0;
            }
        }
        // epilogue columns: (nt, 2t + c) -> member mt0 + 8 nt + 2t + c; their constants
        // are re-read from S.mr every tile (two 16-B shared loads per column)
        constexpr int NC = 2 * SG_NT;    // epilogue columns per lane
        unsigned b1[NC], b2[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) { b1[c] = NONE; b2[c] = NONE; }
        // candidate tile loads, double-buffered in registers so the next tile's
        // L2 traffic overlaps this tile's mma + epilogue
        struct Tile {
            uint4 x00, x01, x10, x11;
            unsigned tb0, tb1;
        };
        const uint4* tdesc = reinterpret_cast<const uint4*>(a.desc + toff * 128) + 2 * t;
        auto load_tile = [&](int mt, Tile& T) {
            const int r0 = mt * 16 + g, r1 = r0 + 8;
            const bool v0 = r0 < n, v1 = r1 < n;
            const int f0 = v0 ? S.list[r0] : 0, f1 = v1 ? S.list[r1] : 0;
            const uint4* row0 = tdesc + 8 * f0;
            const uint4* row1 = tdesc + 8 * f1;
            T.x00 = __ldg(row0); T.x01 = __ldg(row0 + 1);
            T.x10 = __ldg(row1); T.x11 = __ldg(row1 + 1);
            T.tb0 = (S.nrm[v0 ? r0 : 0] << 9) | (unsigned)r0;
            T.tb1 = (S.nrm[v1 ? r1 : 0] << 9) | (unsigned)r1;
        };
        auto do_tile = [&](int mt, const Tile& cur) {
            const uint4 x00 = cur.x00, x01 = cur.x01, x10 = cur.x10, x11 = cur.x11;
            const unsigned tb0 = cur.tb0, tb1 = cur.tb1;
            const int r0 = mt * 16 + g, r1 = r0 + 8;
            const unsigned cm0 = r0 < n ? S.cmask[r0] : 0u, cm1 = r1 < n ? S.cmask[r1] : 0u;
            const float2 p0 = S.xy[r0 < n ? r0 : 0], p1 = S.xy[r1 < n ? r1 : 0];
            int acc[SG_NT][4];
#pragma unroll
            for (int nt = 0; nt < SG_NT; nt++) {
                acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
                mma_u8(acc[nt], x00.x, x10.x, x00.y, x10.y, bw[nt][0], bw[nt][1]);
                mma_u8(acc[nt], x00.z, x10.z, x00.w, x10.w, bw[nt][2], bw[nt][3]);
                mma_u8(acc[nt], x01.x, x11.x, x01.y, x11.y, bw[nt][4], bw[nt][5]);
                mma_u8(acc[nt], x01.z, x11.z, x01.w, x11.w, bw[nt][6], bw[nt][7]);
            }
            // Fast path: elements surely inside the member band (fp32 value <= d - eps) and
            // inside the group's C' go straight into the top-2; elements within eps of the
            // band edge are collected in ucm and decided with the reference's fp64 value
            // afterwards (rare; top-2 is insensitive to the push order).
            constexpr int NE = 4 * SG_NT;
            unsigned ucm = 0;
#ifdef MSFM_MATCH_TILE_STATS
            unsigned inb = 0;
#endif
            bool any0 = false, any1 = false;
            // column by column: one member's constants (two 16-B shared loads) live at a
            // time, used by its two elements of this lane
#pragma unroll
            for (int c = 0; c < NC; c++) {
              const MemberRec* Mc = &S.mr[(c >> 1) * 8 + 2 * t + (c & 1)];
              const float4 MLc = lds_f4(&Mc->a);      // a, b, c, lo
              const uint4 MHc = lds_u4(&Mc->hi);      // hi, qn9, fid, slotgi
#pragma unroll
              for (int rh = 0; rh < 2; rh++) {
                const int nt = c >> 1, q = (c & 1) + 2 * rh, e = nt * 4 + q;
                const bool rowhi = rh != 0;
                const float2 P = rowhi ? p1 : p0;
                const float av = fabsf(fmaf(MLc.x, P.x, fmaf(MLc.y, P.y, MLc.z)));
#ifdef MSFM_MATCH_TILE_STATS
                if (a.dbg && av <= __uint_as_float(MHc.x) && (rowhi ? r1 : r0) < n) inb |= 1u << e;
#endif
                const bool cbit = ((rowhi ? cm1 : cm0) >> (MHc.w >> SLOT_BITS)) & 1u;
                const bool sure_in = av <= MLc.w && cbit;
                if (!(av <= MLc.w) && av <= __uint_as_float(MHc.x) && cbit) ucm |= 1u << e;
                if (STATS) { if (rowhi) any1 |= sure_in; else any0 |= sure_in; }
                const unsigned key = (rowhi ? tb1 : tb0) + MHc.y - ((unsigned)acc[nt][q] << 10);
                top2_push(sure_in ? key : NONE, b1[c], b2[c]);
              }
            }
#ifdef MSFM_MATCH_TILE_STATS
            if (a.dbg) {
                // band-reach occupancy of the tile: elements near some member band, and
                // (tile, 8-member block)s with none (MMA + epilogue work a skip could save)
                int blk_empty = 0, blk = 0;
#pragma unroll
                for (int nt = 0; nt < SG_NT; nt++) {
                    if (mt0 + nt * 8 >= m) continue;
                    blk++;
                    if (!__any_sync(FULL, ((inb >> (4 * nt)) & 0xFu) != 0)) blk_empty++;
                }
                unsigned ne = __popc(inb);
#pragma unroll
                for (int o = 16; o; o >>= 1) ne += __shfl_xor_sync(FULL, ne, o);
                if (lane == 0) {
                    const int rv = min(16, n - mt * 16), cv = min(16, m - mt0);
                    atomicAdd(&a.dbg[10], (unsigned long long)(rv * cv));
                    atomicAdd(&a.dbg[11], (unsigned long long)ne);
                    atomicAdd(&a.dbg[12], (unsigned long long)blk_empty);
                    atomicAdd(&a.dbg[13], (unsigned long long)blk);
                }
            }
#endif
            if (__any_sync(FULL, ucm != 0)) {
#pragma unroll
                for (int e = 0; e < NE; e++) {
                    if (!((ucm >> e) & 1u)) continue;
                    const int nt = e >> 2, q = e & 3, c = nt * 2 + (q & 1);
                    const bool rowhi = q >= 2;
                    const float2 P = rowhi ? p1 : p0;
                    const uint4 MHc = lds_u4(&S.mr[(c >> 1) * 8 + 2 * t + (c & 1)].hi);
                    const GroupRec& Gc = a.grp[SG.g0 + (int)(MHc.w >> SLOT_BITS)];
                    const bool gemv = Gc.cnt == 1;
                    const double* L = gemv ? &Gc.sl0 : a.q_line + 3 * (int64_t)(MHc.w & SLOT_MASK);
                    if (band_exact(L[0], L[1], L[2], gemv, (double)P.x, (double)P.y, a.d)) {
                        if (STATS) { if (rowhi) any1 = true; else any0 = true; }
                        const unsigned key = (rowhi ? tb1 : tb0) + MHc.y - ((unsigned)acc[nt][q] << 10);
                        top2_push(key, b1[c], b2[c]);
                    }
                }
            }
            if (STATS) {
                unsigned m0 = __ballot_sync(FULL, any0);
                unsigned m1 = __ballot_sync(FULL, any1);
                if (lane == 0) {
                    m0 |= m0 >> 1; m0 |= m0 >> 2;
                    m1 |= m1 >> 1; m1 |= m1 >> 2;
                    S.anyb[2 * mt] |= m0 & 0x11111111u;
                    S.anyb[2 * mt + 1] |= m1 & 0x11111111u;
                }
            }
        };
        // two register tiles in flight: tile mt+1's loads overlap tile mt's mma + epilogue
        Tile nxt;
        if (ntiles > 0) load_tile(0, nxt);
        for (int mt = 0; mt < ntiles; mt++) {
            const Tile cur = nxt;
            if (mt + 1 < ntiles) load_tile(mt + 1, nxt);
            do_tile(mt, cur);
        }
        // reduce across the 8 lanes sharing t
#pragma unroll
        for (int c = 0; c < NC; c++) {
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                unsigned o1 = __shfl_xor_sync(FULL, b1[c], o);
                unsigned o2 = __shfl_xor_sync(FULL, b2[c], o);
                top2_merge(b1[c], b2[c], o1, o2);
            }
        }
        if (g == 0) {
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const int jj = (c >> 1) * 8 + 2 * t + (c & 1);
                if (mt0 + jj >= m) continue;
                const int mslot = S.mr[jj].slotgi & SLOT_MASK;
                unsigned long long best = ~0ull;
                unsigned sec = NONE;
                if (b1[c] != NONE) {
                    const unsigned d2 = b1[c] >> 9;
                    const int tid = S.list[b1[c] & 511u];
                    best = ((unsigned long long)d2 << 32) | (unsigned)tid;
                }
                if (b2[c] != NONE) sec = b2[c] >> 9;
                if (!first_round) {
                    const unsigned long long ob = a.mstate[mslot];
                    const unsigned os = a.mstate2[mslot];
                    const unsigned bd = (unsigned)(best >> 32), od = (unsigned)(ob >> 32);
                    const unsigned nh = max(bd, od);
                    const unsigned long long nbest = (bd < od) ? best : ob;
                    sec = min(nh, min(sec, os));
                    best = nbest;
                }
                a.mstate[mslot] = best;
                a.mstate2[mslot] = sec;
            }
        }
    }
    if (STATS) {
        __syncwarp();
        int cnt = 0;
        for (int w = lane; w < ntiles * 2; w += 32) cnt += __popc(S.anyb[w]);
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        cols_total += cnt;
    }
    __syncwarp();
}

template <bool STATS>
__global__ void __launch_bounds__(WARPS * 32, MATCH_MINB) match_kernel(ChunkArgs a) {
    __shared__ WarpSmem smem[WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& S = smem[warp];
    const int total = a.sgstart[a.npairs];
    const float Df = (float)a.D;
    static_assert(sizeof(SGRec) % 16 == 0, "SGRec must be 16-byte granular");
    constexpr int SG_CHUNKS = (int)(sizeof(SGRec) / 16);
    // the next super-group's id and record are fetched while the current one runs
    int nsid = 0;
    if (lane == 0) nsid = atomicAdd(a.sg_next, 1);
    nsid = __shfl_sync(FULL, nsid, 0);
    uint4 nrec = make_uint4(0, 0, 0, 0);
    if (nsid < total && lane < SG_CHUNKS) nrec = __ldg(reinterpret_cast<const uint4*>(a.sg + nsid) + lane);
    for (;;) {
        const int sid = nsid;
        if (sid >= total) break;
        if (lane < SG_CHUNKS) reinterpret_cast<uint4*>(&S.sg)[lane] = nrec;
        __syncwarp();
        if (lane == 0) nsid = atomicAdd(a.sg_next, 1);
        nsid = __shfl_sync(FULL, nsid, 0);
        if (nsid < total && lane < SG_CHUNKS)
            nrec = __ldg(reinterpret_cast<const uint4*>(a.sg + nsid) + lane);
        const SGRec& SG = S.sg;
        if (a.dbg && lane == 0) {
            atomicAdd(&a.dbg[0], 1ull);
            atomicAdd(&a.dbg[1], (unsigned long long)SG.mcnt);
            atomicAdd(&a.dbg[8], (unsigned long long)SG.gcnt);
        }
        if (lane <= SG.gcnt) {
            S.gbeg[lane] = lane < SG.gcnt ? max(a.gmoff[SG.g0 + lane] - SG.m0, 0) : SG.mcnt;
            if (lane < SG.gcnt) S.gl[lane] = a.gl4[SG.g0 + lane];
        }
        stage_members(a, S, SG.m0, SG.mcnt, 0);
        __syncwarp();
        const int pg = a.p0 + SG.p;
        const int64_t toff = SG.toff, qoff = SG.qoff;
        const int nalong = SG.nalong;
        const int64_t toffb = SG.toffb;
        const int32_t* start = SG.horiz ? a.rstart : a.cstart;
        const int4* mrec4 = SG.horiz ? a.rrec : a.crec;
        int n = 0;
        bool first_round = true;
        int cols_total = 0;
        if (lane < CAP / 32) S.sure[lane] = 0;
        __syncwarp();
        // ---- strip gather: bucket rows of the strip |dist_base| <= R.  The CSR starts of
        // the next 32 rows are loaded while the current rows' entries are processed.
        auto row_span = [&](int r, int& bs, int& e1) {
            bs = 0; e1 = 0;
            if (r <= SG.rhi) {
                int blo = 0, bhi = nalong - 1;
                if (SG.inv_alpha != 0.f) {
                    const float y0 = r * Df - 0.01f, y1 = (r + 1) * Df + 0.01f;
                    const float e00 = (-SG.R - SG.beta * y0 - SG.cr) * SG.inv_alpha;
                    const float e01 = (SG.R - SG.beta * y0 - SG.cr) * SG.inv_alpha;
                    const float e10 = (-SG.R - SG.beta * y1 - SG.cr) * SG.inv_alpha;
                    const float e11 = (SG.R - SG.beta * y1 - SG.cr) * SG.inv_alpha;
                    const float plo = fminf(fminf(e00, e01), fminf(e10, e11));
                    const float phi = fmaxf(fmaxf(e00, e01), fmaxf(e10, e11));
                    blo = max(blo, (int)floorf(fmaxf(plo - 0.02f, -1.f) * SG.invD));
                    bhi = min(bhi, (int)floorf(fminf(phi + 0.02f, SG.Pmax + 1.f) * SG.invD));
                }
                if (blo <= bhi) {
                    const int64_t cb = toffb + (int64_t)r * nalong;
                    bs = __ldg(start + cb + blo);
                    e1 = __ldg(start + cb + bhi + 1);
                }
            }
        };
        int nbs, ne1;
        row_span(SG.rlo + lane, nbs, ne1);
        for (int r0 = SG.rlo; r0 <= SG.rhi; r0 += 32) {
            const int bs = nbs, len = ne1 - nbs;
            row_span(r0 + 32 + lane, nbs, ne1);
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const int tot = __shfl_sync(FULL, incl, 31);
            if (a.dbg && lane == 0) atomicAdd(&a.dbg[2], (unsigned long long)tot);
            for (int j0 = 0; j0 < tot; j0 += 32) {
                const int j = j0 + lane;
                int o = 0;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) {
                    int v = __shfl_sync(FULL, incl, o + s - 1);
                    if (v <= j) o += s;
                }
                const int ob = __shfl_sync(FULL, bs, o & 31);
                const int oex = __shfl_sync(FULL, incl - len, o & 31);
                bool pass = false, sure = false;
                int f = 0;
                unsigned nrm = 0;
                float2 p2 = make_float2(0.f, 0.f);
                if (j < tot) {
                    const int4 rec = __ldg(mrec4 + ob + (j - oex));
                    f = rec.w;
                    p2 = make_float2(__int_as_float(rec.x), __int_as_float(rec.y));
                    nrm = (unsigned)rec.z;
                    const float adr = fabsf(fmaf(SG.ar, p2.x, fmaf(SG.br, p2.y, SG.cr)));
                    pass = adr <= SG.R;
                    sure = adr + SG.delta <= SG.hsure && p2.x >= SG.border &&
                           p2.x <= SG.W - SG.border && p2.y >= SG.border && p2.y <= SG.H - SG.border;
                }
                const unsigned bal = __ballot_sync(FULL, pass);
                const int cnt = __popc(bal);
                if (a.dbg && lane == 0) {
                    atomicAdd(&a.dbg[3], (unsigned long long)cnt);
                    atomicAdd(&a.dbg[4], (unsigned long long)__popc(__ballot_sync(FULL, pass && sure)));
                } else if (a.dbg) {
                    __ballot_sync(FULL, pass && sure);
                }
                if (n + cnt > CAP) {
                    __syncwarp();
                    process_round<STATS>(a, S, n, toff, qoff, first_round, cols_total);
                    first_round = false;
                    n = 0;
                    if (lane < CAP / 32) S.sure[lane] = 0;
                    __syncwarp();
                }
                const int k = __popc(bal & ((1u << lane) - 1u));
                if (pass) {
                    S.list[n + k] = (unsigned short)f;
                    S.xy[n + k] = p2;
                    S.nrm[n + k] = nrm;
                }
                const unsigned bits = __reduce_or_sync(FULL, (pass && sure) ? (1u << k) : 0u);
                if (lane == 0 && cnt) {
                    const int w = n >> 5, sh = n & 31;
                    S.sure[w] |= bits << sh;
                    if (sh && sh + cnt > 32) S.sure[w + 1] |= bits >> (32 - sh);
                }
                n += cnt;
                __syncwarp();
            }
        }
        if (n > 0) {
            __syncwarp();
            process_round<STATS>(a, S, n, toff, qoff, first_round, cols_total);
            first_round = false;
        }
        __syncwarp();
        // ---- ratio test + dedupe per member (ratio_filter / _dedupe_targets)
        if (!first_round) {
            for (int j = lane; j < SG.mcnt; j += 32) {
                const MemberRec& M = a.mrec[SG.m0 + j];
                const int slot = M.slotgi & SLOT_MASK;
                const unsigned long long best = a.mstate[slot];
                const unsigned sec = a.mstate2[slot];
                if (best == ~0ull) continue;
                const unsigned bd2 = (unsigned)(best >> 32);
                const int tid = (int)(best & 0xffffffffu);
                const float db = sqrtf((float)bd2);
                float rr;
                bool acc;
                if (sec == NONE) {
                    acc = db < a.single_cap;
                    rr = 0.0f;
                } else {
                    const float ds = sqrtf((float)sec);
                    rr = ds > 0.0f ? db / ds : 1.0f;
                    acc = rr < a.ratio;
                }
                if (!acc) continue;
                a.res_tid[slot] = tid;
                a.res_dist[slot] = db;
                a.res_ratio[slot] = rr;
                const unsigned long long key =
                    ((unsigned long long)__float_as_uint(db) << 32) | (unsigned)M.fid;
                atomicMin(&a.dedupe[SG.dbase + tid], key);
            }
        }
        if (STATS && lane == 0 && cols_total > 0) {
            atomicAdd(&a.stats[2 * pg], (unsigned long long)SG.mcnt);
            atomicAdd(&a.stats[2 * pg + 1], (unsigned long long)SG.mcnt * (unsigned long long)cols_total);
        }
        __syncwarp();
    }
}

#include "guided_match.cuh"

__global__ void __launch_bounds__(256) compact_kernel(ChunkArgs a) {
    __shared__ int sm[256 / 32 + 1];
    const int p = blockIdx.x, pg = a.p0 + p;
    const int64_t q0 = a.qlist_off[pg];
    const int nq = (int)(a.qlist_off[pg + 1] - q0);
    const int64_t s0 = q0 - a.qbase;
    const int64_t db = a.tbase[p];
    int carry = 0;
    for (int i0 = 0; i0 < nq; i0 += 256) {
        const int i = i0 + threadIdx.x;
        bool keep = false;
        int tid = -1, qid = 0;
        float dist = 0.f;
        if (i < nq) {
            tid = a.res_tid[s0 + i];
            if (tid >= 0) {
                qid = a.q_fid[s0 + i];
                dist = a.res_dist[s0 + i];
                const unsigned long long key =
                    ((unsigned long long)__float_as_uint(dist) << 32) | (unsigned)qid;
                keep = a.dedupe[db + tid] == key;
            }
        }
        int tot;
        const int ex = block_exclusive_scan<256>(keep ? 1 : 0, &tot, sm);
        if (keep) {
            const int64_t o = q0 + carry + ex;
            a.out_q[o] = qid;
            a.out_t[o] = tid;
            a.out_dist[o] = dist;
            a.out_ratio[o] = a.res_ratio[s0 + i];
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
    b += aligned_bytes<int32_t>(c.P + 1) * 5 + 256;    // ngroups, gstart, nmem, sgstart, nsg, sg_next
    b += aligned_bytes<float4>(c.Q) * 2 + aligned_bytes<int2>(c.Q);   // gline, gend, sglist
    b += aligned_bytes<unsigned long long>(c.T);       // tab_key
    b += aligned_bytes<unsigned>(c.T) * 2;             // tab_rep, tab_cnt
    b += aligned_bytes<int32_t>(c.Q) * 2;              // q_tab, q_fid
    b += aligned_bytes<int32_t>(c.Q) * 2;              // mgid, msg
    b += aligned_bytes<unsigned>(c.Q);                 // gfit
    b += aligned_bytes<unsigned long long>(c.Q);       // sgdev
    b += aligned_bytes<float4>(c.Q) + aligned_bytes<int32_t>(c.Q);   // gl4, gmoff
    b += aligned_bytes<GView>(c.Q);                    // gview
    b += aligned_bytes<double>(3 * c.Q);               // q_line
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
        grid_count_kernel<<<img1 - img0, 256, 0, st>>>(a);
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
        grid_scatter_kernel<<<img1 - img0, 256, 0, st>>>(a);
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
        size_t fr = 0, tot = 0;
        budget = (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0) ? (int64_t)(fr / 4)
                                                                       : (int64_t)16 << 30;
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
    while (p < n_pairs) {
        int e = p + 1;
        const int cap = (p == 0 && prm->first_chunk_pairs > 0) ? std::min(cp, prm->first_chunk_pairs) : cp;
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
    if (!(prm->ratio <= 1.0f)) {
        set_error("msfm_guided_match: ratio > 1 is not supported (got %g)", (double)prm->ratio);
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
    a.gl4 = ar.take<float4>(w.Q); a.gmoff = ar.take<int32_t>(w.Q);
    a.gview = ar.take<GView>(w.Q);
    a.tab_off = ar.take<int64_t>(w.P + 1); a.tbase = ar.take<int64_t>(w.P + 1);
    a.ngroups = ar.take<int32_t>(w.P + 1); a.gstart = ar.take<int32_t>(w.P + 1);
    a.nmem = ar.take<int32_t>(w.P + 1); a.sgstart = ar.take<int32_t>(w.P + 1);
    a.sg_next = ar.take<int32_t>(1);
    a.nsg = ar.take<int32_t>(w.P + 1);
    a.gline = ar.take<float4>(w.Q); a.gend = ar.take<float4>(w.Q); a.sglist = ar.take<int2>(w.Q);
    a.tab_key = ar.take<unsigned long long>(w.T);
    a.tab_rep = ar.take<unsigned>(w.T); a.tab_cnt = ar.take<unsigned>(w.T);
    a.q_tab = ar.take<int32_t>(w.Q); a.q_line = ar.take<double>(3 * w.Q);
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
    MSFM_CUDA_TRY(cudaFuncSetAttribute(groups_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       2 * 65536 + 16));
    // MSFM_MATCH_V1=1 selects the round-1 kernel (A/B comparisons)
    const bool use_v1 = getenv("MSFM_MATCH_V1") && atoi(getenv("MSFM_MATCH_V1")) != 0;
    const size_t ms_smem = sizeof(MSmem) * MS_WARPS;
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    MSFM_CUDA_TRY(cudaFuncSetAttribute(match_ms_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
    int next_range = 0;
    for (size_t c = 0; c + 1 < bounds.size(); c++) {
        const int p0 = bounds[c], p1 = bounds[c + 1];
        a.p0 = p0;
        a.npairs = p1 - p0;
        a.qbase = h_qlist_off[p0];
        const int64_t Q = h_qlist_off[p1] - h_qlist_off[p0];
        // bank ranges first read by this chunk: wait for their rows, then index them
        for (; plan && next_range < plan->n_ranges && plan->chunk[next_range] <= (int32_t)c;
             next_range++) {
            const int r = next_range;
            if (plan->landed && plan->landed[r])
                MSFM_CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)plan->landed[r], 0));
            const int64_t f0 = plan->feat0[r], f1 = plan->feat1[r];
            const int i1 = plan->img1[r];
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
                                           plan->n_buckets_total, plan->img0[r], i1,
                                           plan->bucket0[r], plan->bucket1[r], f0, grids->D,
                                           w32(grids->d_sub), w32(grids->d_rstart),
                                           w32(grids->d_cstart), w32(grids->d_rmem),
                                           w32(grids->d_cmem), w32(grids->d_rrec),
                                           w32(grids->d_crec), plan->grid_workspace,
                                           plan->grid_workspace_bytes, st, w32(bank->d_norm2));
            if (rc) return rc;
        }
        plan_kernel<<<1, SCAN_T, 0, st>>>(a);
        { ProfScope ps("lines_kernel", st); lines_kernel<<<a.npairs, MSFM_LINES_T, 0, st>>>(a); }
        {
            int64_t max_nq = 1;
            for (int k = p0; k < p1; k++) max_nq = std::max(max_nq, h_qlist_off[k + 1] - h_qlist_off[k]);
            ProfScope ps("groups_kernel", st);
            groups_kernel<<<a.npairs, GT, (size_t)(2 * max_nq + 16), st>>>(a);
        }
        gscan_kernel<<<1, SCAN_T, 0, st>>>(a);
        { ProfScope ps("scatter_kernel", st); scatter_kernel<<<a.npairs, MSFM_LINES_T, 0, st>>>(a); }
        if (Q > 0) {
            const unsigned nb = (unsigned)((Q + 127) / 128);
            { ProfScope ps("prep_kernel", st); prep_kernel<<<nb, 128, 0, st>>>(a, (int)Q); }
            { ProfScope ps("sg_shape_kernel", st); sg_shape_kernel<<<nb, 128, 0, st>>>(a, (int)Q); }
            { ProfScope ps("member_kernel", st); member_kernel<<<nb, 128, 0, st>>>(a, (int)Q); }
            { ProfScope ps("sg_prep_kernel", st); sg_prep_kernel<<<nb, 128, 0, st>>>(a, (int)Q); }
        }
        if (use_v1) {
            ProfScope ps("match_kernel", st);
            if (d_stats) match_kernel<true><<<nsm * MATCH_MINB, WARPS * 32, 0, st>>>(a);
            else         match_kernel<false><<<nsm * MATCH_MINB, WARPS * 32, 0, st>>>(a);
        } else {
            ProfScope ps("match_kernel", st);
            if (d_stats) match_ms_kernel<true><<<nsm * MS_MINB, MS_WARPS * 32, ms_smem, st>>>(a);
            else         match_ms_kernel<false><<<nsm * MS_MINB, MS_WARPS * 32, ms_smem, st>>>(a);
        }
        { ProfScope ps("compact_kernel", st); compact_kernel<<<a.npairs, 256, 0, st>>>(a); }
        MSFM_LAUNCH_CHECK();
        count_launches(7 + (Q > 0 ? 4 : 0));
        if (hook) {
            const int rc = hook(hook_ctx, (int)c, p0, p1);
            if (rc) return rc;
        }
    }
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
