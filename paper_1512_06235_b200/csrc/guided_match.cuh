// Member-stationary match kernel (included by guided.cu inside msfm::<anon>).
//
// The K4/K5 core of guided_match_pair (guided.py:393-480 + ratio_filter /
// _dedupe_targets, matching.py:82-113), one warp per super-group (SG: <= 16
// members of angle-adjacent groups sharing one candidate strip, guided.cu §SGRec):
//
//   * the SG's inputs — its record, member records, group views and the 16
//     members' descriptor rows — arrive in a per-warp shared-memory slot through
//     the async (TMA) proxy: cp.async.bulk copies completing on mbarriers, issued
//     two SGs ahead of the one being matched (slot ring of 2 + the SG record of
//     the one after), so the gathers' L2/HBM latency overlaps the current SG's
//     tiles;
//   * members are the M = 16 rows of mma.sync.m16n8k32 u8 tiles and stay in
//     registers (descriptor fragments + band constants), candidates stream as
//     the n8 columns: each lane owns 2 members x 2 candidates per tile, so the
//     per-element epilogue (fp32 band value, C' bit, key, branch-free top-2) is
//     ~12 instructions with no shared-memory reload of member constants;
//   * keys are signed 32-bit (s << 8 | local), s = |t|^2 - 2 q.t = d2 - |q|^2:
//     one IMAD per element, exact integer ranking per member (CAP = 256 per round).
//
// Bit-exactness rules are those of the v1 kernel: fp32 band value
// with a proven error bound and the reference's fp64 value inside [d-eps, d+eps];
// exact C' membership; f32 sqrt / ratio; (f32 dist, qid) dedupe.

constexpr int MS_WARPS = 4;            // warps per CTA
#ifndef MSFM_MS_MINB
#define MSFM_MS_MINB 5
#endif
constexpr int MS_MINB = MSFM_MS_MINB;  // resident CTAs per SM
constexpr int MS_CAP = 192;            // candidates per round (local index < 256)
constexpr int KEY_NONE = 0x7fffffff;

struct alignas(16) MSlot {
    SGRec sg;                  // 128 B
    MemberRec mr[16];          // first 16 members
    GView gv[SG_MAX_GROUPS];   // per group: rep line + member reach, member offset
    uint8_t desc[16][128];     // the first 16 members' descriptor rows
};
static_assert(sizeof(SGRec) == 128, "SGRec is bulk-copied as 128 B");
static_assert(sizeof(GView) == 32, "GView is bulk-copied as 32-B records");
static_assert(offsetof(MSlot, mr) % 16 == 0 && offsetof(MSlot, gv) % 16 == 0 &&
              offsetof(MSlot, desc) % 16 == 0, "bulk-copy destinations must be 16-B aligned");

struct alignas(16) MSmem {
    MSlot slot[2];
    SGRec sgq;                 // record of the SG after next
    int4 cand[MS_CAP];         // per candidate: x, y (f32 bits), tb = |t|^2 << 8 | local, C' bits
    unsigned short cid[MS_CAP];    // target-local feature id
    unsigned short ulist[MS_CAP];  // candidates whose C' bits are still to be decided
    unsigned anyb[MS_CAP / 32];    // stats: candidate inside some member band
    uint64_t bar_q, bar_rec[2], bar_desc[2];
};

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ms_bar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
}
__device__ __forceinline__ void ms_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ms_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}
// bounded parity wait: a protocol bug traps instead of hanging the GPU
__device__ __forceinline__ void ms_wait(uint64_t* b, uint32_t parity) {
    const uint32_t addr = su32(b);
    for (long long it = 0; it < (1LL << 30); it++) {
        uint32_t done;
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
__device__ __forceinline__ void ms_fence_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// member records + group views of the SG in slot L (lane 0 issues; bar gets one phase)
__device__ __forceinline__ void ms_issue_rec(const ChunkArgs& a, MSlot& L, uint64_t* bar) {
    const SGRec& SG = L.sg;
    const int nm = min(SG.mcnt, 16), ng = SG.gcnt;
    ms_expect(bar, (uint32_t)(nm * sizeof(MemberRec) + ng * sizeof(GView)));
    if (nm) ms_bulk(L.mr, a.mrec + SG.m0, nm * sizeof(MemberRec), bar);
    if (ng) ms_bulk(L.gv, a.gview + SG.g0, ng * sizeof(GView), bar);
}

// descriptor rows of the slot's first 16 members (lanes < 16 issue one 128-B copy each)
__device__ __forceinline__ void ms_issue_desc(const ChunkArgs& a, MSlot& L, uint64_t* bar) {
    const int lane = threadIdx.x & 31;
    const int nm = min(L.sg.mcnt, 16);
    if (lane == 0) ms_expect(bar, (uint32_t)(nm * 128));
    __syncwarp();
    if (lane < nm) ms_bulk(L.desc[lane], a.desc + (L.sg.qoff + L.mr[lane].fid) * 128, 128, bar);
}

__device__ __forceinline__ void ms_top2(int key, int& b1, int& b2) {
    const int lo = min(key, b1), hi = max(key, b1);
    b1 = lo;
    b2 = min(b2, hi);
}

// the reference's float64 band decision for one (member, candidate) element
__device__ __forceinline__ bool ms_band_exact(const ChunkArgs& a, const SGRec& SG, const MemberRec& M,
                                              float x, float y) {
    const GroupRec& G = a.grp[SG.g0 + (int)((unsigned)M.slotgi >> SLOT_BITS)];
    if (G.cnt == 1) return band_exact(G.sl0, G.sl1, G.sl2, true, x, y, a.d);
    const double* L = a.q_line + 3 * (int64_t)(M.slotgi & SLOT_MASK);
    return band_exact(L[0], L[1], L[2], false, x, y, a.d);
}

// fp32 prefilter, then the exact value near the edge (member_band of the v1 kernel)
__device__ __forceinline__ bool ms_member_band(const ChunkArgs& a, const SGRec& SG, const MemberRec& M,
                                               float x, float y) {
    const float v = fabsf(fmaf(M.a, x, fmaf(M.b, y, M.c)));
    if (v <= M.lo) return true;
    if (v > M.hi) return false;
    return ms_band_exact(a, SG, M, x, y);
}

// C' membership of candidate (x, y, f) for group G (in_cprime of the v1 kernel)
__device__ __forceinline__ bool ms_in_cprime(const ChunkArgs& a, const GroupRec& G, const SGRec& S,
                                             float fx, float fy, int f) {
    return in_cprime(a, G, S, fx, fy, S.toff, f);
}

// One round: C' bits of the unsure candidates, then the distance tiles of every
// member block against the round's n candidates; per-member top-2 merged into
// mstate / mstate2 (first_round: written).
template <bool STATS>
__device__ void ms_round(const ChunkArgs& a, MSmem& S, const MSlot& L, int n, int nu,
                         bool first_round, int& cols_total) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const SGRec& SG = L.sg;
    const int m = SG.mcnt;
    // ---- C' bits of the candidates not surely inside every group's C'
    for (int u0 = 0; u0 < nu; u0 += 32) {
        const int uj = u0 + lane;
        if (uj < nu) {
            const int j = S.ulist[uj];
            const int f = S.cid[j];
            const int4 c = S.cand[j];
            const float px = __int_as_float(c.x), py = __int_as_float(c.y);
            const bool inner = px >= SG.border && px <= SG.W - SG.border && py >= SG.border &&
                               py <= SG.H - SG.border;
            unsigned bits = 0;
            for (int gi = 0; gi < SG.gcnt; gi++) {
                const GView gv = L.gv[gi];
                const float dg = fabsf(fmaf(gv.a, px, fmaf(gv.b, py, gv.c)));
                if (dg <= SG.hsure && inner) { bits |= 1u << gi; continue; }
                if (dg > gv.reach) continue;   // outside every member band of the group
                const int k0 = max(gv.moff - SG.m0, 0);
                const int k1 = gi + 1 < SG.gcnt ? max(L.gv[gi + 1].moff - SG.m0, 0) : m;
                bool any = false;
                for (int k = k0; k < k1 && !any; k++) {
                    const MemberRec M = k < 16 ? L.mr[k] : a.mrec[SG.m0 + k];
                    any = ms_member_band(a, SG, M, px, py);
                }
                if (any && ms_in_cprime(a, a.grp[SG.g0 + gi], SG, px, py, f)) bits |= 1u << gi;
            }
            S.cand[j].w = (int)bits;
        }
    }
    // ---- pad the last n8 tile with candidates no member accepts
    const int ntile = (n + 7) >> 3;
    if (lane < ntile * 8 - n) {
        S.cand[n + lane] = make_int4(0, 0, 0, 0);
        S.cid[n + lane] = 0;
    }
    if (STATS)
        for (int w = lane; w < MS_CAP / 32; w += 32) S.anyb[w] = 0;
    __syncwarp();
    const uint4* tdesc = reinterpret_cast<const uint4*>(a.desc + SG.toff * 128) + 2 * t;
    for (int mb0 = 0; mb0 < m; mb0 += 16) {
        // ---- member rows g, g+8 of this block: band constants + descriptor fragments
        float ma[2], mbv[2], mc[2], mlo[2], mhi[2];
        unsigned gb[2];
        unsigned aw[2][8];
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int j = mb0 + g + 8 * r;
            if (j < m) {
                const MemberRec M = (j < 16) ? L.mr[j] : a.mrec[SG.m0 + j];
                ma[r] = M.a; mbv[r] = M.b; mc[r] = M.c; mlo[r] = M.lo; mhi[r] = M.hi;
                gb[r] = 1u << ((unsigned)M.slotgi >> SLOT_BITS);
                uint4 w0, w1;
                if (j < 16) {
                    const uint4* row = reinterpret_cast<const uint4*>(L.desc[j]) + 2 * t;
                    w0 = row[0]; w1 = row[1];
                } else {
                    const uint4* row = reinterpret_cast<const uint4*>(a.desc + (SG.qoff + M.fid) * 128) + 2 * t;
                    w0 = __ldg(row); w1 = __ldg(row + 1);
                }
                aw[r][0] = w0.x; aw[r][1] = w0.y; aw[r][2] = w0.z; aw[r][3] = w0.w;
                aw[r][4] = w1.x; aw[r][5] = w1.y; aw[r][6] = w1.z; aw[r][7] = w1.w;
            } else {
                ma[r] = 0.f; mbv[r] = 0.f; mc[r] = 1e30f; mlo[r] = -1.f; mhi[r] = -1.f; gb[r] = 0;
#pragma unroll
                for (int k = 0; k < 8; k++) aw[r][k] = 0;
            }
        }
        int k1[2] = {KEY_NONE, KEY_NONE}, k2[2] = {KEY_NONE, KEY_NONE};
        // candidate descriptor fragments, one n8 tile ahead
        uint4 nx0, nx1;
        {
            const int f = S.cid[g];
            nx0 = __ldg(tdesc + 8 * f);
            nx1 = __ldg(tdesc + 8 * f + 1);
        }
        for (int nt = 0; nt < ntile; nt++) {
            const uint4 x0 = nx0, x1 = nx1;
            if (nt + 1 < ntile) {
                const int f = S.cid[8 * (nt + 1) + g];
                nx0 = __ldg(tdesc + 8 * f);
                nx1 = __ldg(tdesc + 8 * f + 1);
            }
            int acc[4] = {0, 0, 0, 0};
            mma_u8(acc, aw[0][0], aw[1][0], aw[0][1], aw[1][1], x0.x, x0.y);
            mma_u8(acc, aw[0][2], aw[1][2], aw[0][3], aw[1][3], x0.z, x0.w);
            mma_u8(acc, aw[0][4], aw[1][4], aw[0][5], aw[1][5], x1.x, x1.y);
            mma_u8(acc, aw[0][6], aw[1][6], aw[0][7], aw[1][7], x1.z, x1.w);
            const int4 c0 = S.cand[8 * nt + 2 * t], c1 = S.cand[8 * nt + 2 * t + 1];
            unsigned ucm = 0;
            bool any0 = false, any1 = false;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int r = e >> 1;               // member row (g, g+8)
                const int4 c = (e & 1) ? c1 : c0;   // candidate column (2t, 2t+1)
                const float px = __int_as_float(c.x), py = __int_as_float(c.y);
                const float av = fabsf(fmaf(ma[r], px, fmaf(mbv[r], py, mc[r])));
                const bool cb = ((unsigned)c.w & gb[r]) != 0u;
                const bool in = av <= mlo[r] && cb;
                if (!(av <= mlo[r]) && av <= mhi[r] && cb) ucm |= 1u << e;
                if (STATS) { if (e & 1) any1 |= in; else any0 |= in; }
                const int key = c.z - acc[e] * 512;
                ms_top2(in ? key : KEY_NONE, k1[r], k2[r]);
            }
            if (__any_sync(FULL, ucm != 0)) {
                // within eps of the band edge: the reference's fp64 band value decides
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if (!((ucm >> e) & 1u)) continue;
                    const int r = e >> 1;
                    const int4 c = (e & 1) ? c1 : c0;
                    const int j = mb0 + g + 8 * r;
                    const MemberRec M = (j < 16) ? L.mr[j] : a.mrec[SG.m0 + j];
                    if (ms_band_exact(a, SG, M, __int_as_float(c.x), __int_as_float(c.y))) {
                        if (STATS) { if (e & 1) any1 = true; else any0 = true; }
                        ms_top2(c.z - acc[e] * 512, k1[r], k2[r]);
                    }
                }
            }
            if (STATS) {
                const unsigned b0 = __ballot_sync(FULL, any0), b1 = __ballot_sync(FULL, any1);
                if (lane == 0) {
                    unsigned bits = 0;
#pragma unroll
                    for (int tt = 0; tt < 4; tt++) {
                        if (b0 & (0x11111111u << tt)) bits |= 1u << (2 * tt);
                        if (b1 & (0x11111111u << tt)) bits |= 1u << (2 * tt + 1);
                    }
                    const int c8 = 8 * nt;
                    S.anyb[c8 >> 5] |= bits << (c8 & 31);
                }
            }
        }
        // ---- reduce the per-lane top-2 over the 4 lanes (t) sharing a member row
#pragma unroll
        for (int r = 0; r < 2; r++) {
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                const int o1 = __shfl_xor_sync(FULL, k1[r], o), o2 = __shfl_xor_sync(FULL, k2[r], o);
                const int lo = min(k1[r], o1), hi = max(k1[r], o1);
                k1[r] = lo;
                k2[r] = min(hi, min(k2[r], o2));
            }
        }
        if (t == 0) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const int j = mb0 + g + 8 * r;
                if (j >= m) continue;
                const MemberRec M = (j < 16) ? L.mr[j] : a.mrec[SG.m0 + j];
                const int mslot = M.slotgi & SLOT_MASK;
                const unsigned q2 = (unsigned)M.qn9 >> 9;
                unsigned long long best = ~0ull;
                unsigned sec = NONE;
                if (k1[r] != KEY_NONE) {
                    const unsigned d2 = q2 + (unsigned)(k1[r] >> 8);
                    best = ((unsigned long long)d2 << 32) | (unsigned)S.cid[k1[r] & 255];
                }
                if (k2[r] != KEY_NONE) sec = q2 + (unsigned)(k2[r] >> 8);
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
        int cnt = lane < MS_CAP / 32 ? __popc(S.anyb[lane]) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        cols_total += cnt;
    }
    __syncwarp();
}

template <bool STATS>
__global__ void __launch_bounds__(MS_WARPS * 32, MS_MINB) match_ms_kernel(ChunkArgs a) {
    extern __shared__ __align__(128) unsigned char ms_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    MSmem& S = reinterpret_cast<MSmem*>(ms_raw)[warp];
    const int total = a.sgstart[a.npairs];
    const float Df = (float)a.D;
    if (lane == 0) {
        ms_bar_init(&S.bar_q);
        ms_bar_init(&S.bar_rec[0]); ms_bar_init(&S.bar_rec[1]);
        ms_bar_init(&S.bar_desc[0]); ms_bar_init(&S.bar_desc[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t ph_q = 0, ph_rec = 0, ph_desc = 0;   // phase bits (per slot: bit s)
    auto claim = [&]() {
        int s = 0;
        if (lane == 0) s = atomicAdd(a.sg_next, 1);
        return __shfl_sync(FULL, s, 0);
    };
    auto load_sg = [&](MSlot& L, int sid) {
        if (lane < 8)
            reinterpret_cast<uint4*>(&L.sg)[lane] = __ldg(reinterpret_cast<const uint4*>(a.sg + sid) + lane);
        __syncwarp();
    };
    // prologue: slots 0 and 1 get the first two SGs (records + member data in flight)
    int sid_s[2];
    sid_s[0] = claim();
    sid_s[1] = claim();
#pragma unroll
    for (int s = 0; s < 2; s++) {
        if (sid_s[s] < total) {
            load_sg(S.slot[s], sid_s[s]);
            if (lane == 0) ms_issue_rec(a, S.slot[s], &S.bar_rec[s]);
        }
    }
    if (sid_s[0] < total) {
        ms_wait(&S.bar_rec[0], 0);
        ph_rec ^= 1u;
        ms_issue_desc(a, S.slot[0], &S.bar_desc[0]);
    }
    int cur = 0;
    for (;;) {
        const int sid = sid_s[cur];
        if (sid >= total) break;
        const int nxt = cur ^ 1;
        MSlot& L = S.slot[cur];
        // the SG after next: its record goes to sgq
        const int sid2 = claim();
        if (sid2 < total && lane == 0) {
            ms_expect(&S.bar_q, (uint32_t)sizeof(SGRec));
            ms_bulk(&S.sgq, a.sg + sid2, sizeof(SGRec), &S.bar_q);
        }
        // this SG's member records / group views / member descriptors have landed
        ms_wait(&S.bar_desc[cur], (ph_desc >> cur) & 1u);
        ph_desc ^= 1u << cur;
        const SGRec& SG = L.sg;
        if (a.dbg && lane == 0) {
            atomicAdd(&a.dbg[0], 1ull);
            atomicAdd(&a.dbg[1], (unsigned long long)SG.mcnt);
            atomicAdd(&a.dbg[8], (unsigned long long)SG.gcnt);
        }
        const unsigned all_groups = (1u << SG.gcnt) - 1u;
        const int nalong = SG.nalong;
        const int64_t toffb = SG.toffb;
        const int32_t* start = SG.horiz ? a.rstart : a.cstart;
        const int4* mrec4 = SG.horiz ? a.rrec : a.crec;
        int n = 0, nu = 0;
        bool first_round = true;
        int cols_total = 0;
        bool nxt_desc_issued = false;
        auto issue_next_desc = [&]() {
            if (!nxt_desc_issued && sid_s[nxt] < total) {
                ms_wait(&S.bar_rec[nxt], (ph_rec >> nxt) & 1u);
                ph_rec ^= 1u << nxt;
                ms_fence_async();
                ms_issue_desc(a, S.slot[nxt], &S.bar_desc[nxt]);
            }
            nxt_desc_issued = true;
        };
        // ---- strip gather: bucket rows of |dist_base| <= R (CSR starts of the next 32
        // rows and the next batch of records are loaded ahead of their use)
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
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const int tot = __shfl_sync(FULL, incl, 31);
            if (a.dbg && lane == 0) atomicAdd(&a.dbg[2], (unsigned long long)tot);
            auto rec_at = [&](int j) {
                int o = 0;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) {
                    const int v = __shfl_sync(FULL, incl, o + s - 1);
                    if (v <= j) o += s;
                }
                const int ob = __shfl_sync(FULL, bs, o & 31);
                const int oex = __shfl_sync(FULL, incl - len, o & 31);
                return ob + (j - oex);
            };
            int4 nrec = make_int4(0, 0, 0, 0);
            {
                const int ri = rec_at(lane);
                if (lane < tot) nrec = __ldg(mrec4 + ri);
            }
            for (int j0 = 0; j0 < tot; j0 += 32) {
                const int j = j0 + lane;
                const int4 rec = nrec;
                {
                    const int ri = rec_at(j + 32);
                    if (j + 32 < tot) nrec = __ldg(mrec4 + ri);
                }
                bool pass = false, sure = false;
                const float px = __int_as_float(rec.x), py = __int_as_float(rec.y);
                if (j < tot) {
                    const float adr = fabsf(fmaf(SG.ar, px, fmaf(SG.br, py, SG.cr)));
                    pass = adr <= SG.R;
                    sure = adr + SG.delta <= SG.hsure && px >= SG.border &&
                           px <= SG.W - SG.border && py >= SG.border && py <= SG.H - SG.border;
                }
                const unsigned bal = __ballot_sync(FULL, pass);
                const int cnt = __popc(bal);
                if (a.dbg && lane == 0) {
                    atomicAdd(&a.dbg[3], (unsigned long long)cnt);
                    atomicAdd(&a.dbg[4], (unsigned long long)__popc(__ballot_sync(FULL, pass && sure)));
                } else if (a.dbg) {
                    __ballot_sync(FULL, pass && sure);
                }
                if (n + cnt > MS_CAP) {
                    issue_next_desc();
                    ms_round<STATS>(a, S, L, n, nu, first_round, cols_total);
                    first_round = false;
                    n = 0;
                    nu = 0;
                }
                const int k = __popc(bal & ((1u << lane) - 1u));
                const unsigned ubal = __ballot_sync(FULL, pass && !sure);
                if (pass) {
                    const int pos = n + k;
                    S.cand[pos] = make_int4(rec.x, rec.y, (rec.z << 8) | pos, sure ? (int)all_groups : 0);
                    S.cid[pos] = (unsigned short)rec.w;
                    if (!sure) S.ulist[nu + __popc(ubal & ((1u << lane) - 1u))] = (unsigned short)pos;
                }
                n += cnt;
                nu += __popc(ubal);
                __syncwarp();
            }
        }
        issue_next_desc();
        if (n > 0) {
            ms_round<STATS>(a, S, L, n, nu, first_round, cols_total);
            first_round = false;
        }
        __syncwarp();
        // ---- ratio test + dedupe per member (ratio_filter / _dedupe_targets)
        if (!first_round) {
            for (int j = lane; j < SG.mcnt; j += 32) {
                const MemberRec M = j < 16 ? L.mr[j] : a.mrec[SG.m0 + j];
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
            const int pg = a.p0 + SG.p;
            atomicAdd(&a.stats[2 * pg], (unsigned long long)SG.mcnt);
            atomicAdd(&a.stats[2 * pg + 1], (unsigned long long)SG.mcnt * (unsigned long long)cols_total);
        }
        __syncwarp();
        // ---- slot `cur` is free: it takes the SG after next
        sid_s[cur] = sid2;
        if (sid2 < total) {
            ms_wait(&S.bar_q, ph_q);
            ph_q ^= 1u;
            if (lane < 8) reinterpret_cast<uint4*>(&L.sg)[lane] = reinterpret_cast<const uint4*>(&S.sgq)[lane];
            __syncwarp();
            ms_fence_async();
            if (lane == 0) ms_issue_rec(a, L, &S.bar_rec[cur]);
        }
        __syncwarp();
        cur = nxt;
    }
}
