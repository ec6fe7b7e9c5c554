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
#define MSFM_MS_MINB 4
#endif
constexpr int MS_MINB = MSFM_MS_MINB;  // resident CTAs per SM
constexpr int MS_CAP = 192;            // candidates per round (local index < 256)
constexpr int MS_RING = 3;             // n8 tiles of candidate rows in flight (cp.async ring)
constexpr int KEY_NONE = 0x7fffffff;
#ifndef MSFM_PF3
#define MSFM_PF3 0
#endif

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
    uint4 bring[MS_RING][64];      // candidate descriptor rows of the next tiles (swizzled 16-B chunks)
    int rbs[32], rex[32];          // gather batch: CSR start / batch start of the k-th non-empty row
    unsigned long long mbest[16];  // running best (d2 << 32 | target) of the slot's first 16 members
    unsigned msec[16];             // and second d2 (members past 16: a.mstate / a.mstate2)
    uint64_t bar_q, bar_rec[2];
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
// the same with an L2 evict-first policy: per-super-group records are read once
__device__ __forceinline__ void ms_bulk_ef(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
        " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], pol;\n}\n" ::"r"(su32(dst)),
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
    if (nm) ms_bulk_ef(L.mr, a.mrec + SG.m0, nm * sizeof(MemberRec), bar);
    if (ng) {
        ms_bulk_ef(L.gv, a.gview + SG.g0, ng * sizeof(GView), bar);
        // the groups' full records (exact C' samples, singleton lines) into L2: the rare
        // exact paths then wait on an L2 hit instead of DRAM
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.grp + SG.g0),
                     "r"((uint32_t)(ng * sizeof(GroupRec)))
                     : "memory");
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_u32(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ uint4 lds128_u32(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// descriptor rows of the slot's first 16 members: 128 16-B cp.async, 4 per lane
// (completion: cp.async.wait_all before the SG starts)
__device__ __forceinline__ void ms_issue_desc(const ChunkArgs& a, MSlot& L) {
    const int lane = threadIdx.x & 31;
    const int nm = min(L.sg.mcnt, 16);
    const int part = lane & 7, j0 = lane >> 3;      // lane copies chunk `part` of rows j0 + 4q
    uint64_t src;                                   // opaque: one IMAD.WIDE per copy
    asm("mov.b64 %0, %1;" : "=l"(src) : "l"(reinterpret_cast<uint64_t>(a.desc + L.sg.qoff * 128 + part * 16)));
    const uint32_t dst = su32(L.desc[j0] + 16 * part);
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int j = j0 + 4 * q;
        if (j < nm)
            cp_async16_u32(dst + q * 4 * 128, reinterpret_cast<const void*>(src + (unsigned)L.mr[j].fid * 128ull));
    }
    // the members' f64 lines into L2 (the exact band fallback near a band edge reads
    // them; written by the setup kernel long before, they are back in DRAM by now)
    if (lane < nm)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q_line + 3 * (int64_t)(L.mr[lane].slotgi & SLOT_MASK)));
}

__device__ __forceinline__ void ms_top2(int key, int& b1, int& b2) {
    const int lo = min(key, b1), hi = max(key, b1);
    b1 = lo;
    b2 = min(b2, hi);
}

// the reference's float64 band decision for one (member, candidate) element
__device__ __noinline__ bool ms_band_exact(const GroupRec* grp, const double* q_line, double d,
                                           int g0, int slotgi, float x, float y) {
    // the group record's singleton line and the slot's own line are loaded together
    // (one round trip; q_line holds every slot's line, singletons included)
    const GroupRec& G = grp[g0 + (int)((unsigned)slotgi >> SLOT_BITS)];
    const double* L = q_line + 3 * (int64_t)(slotgi & SLOT_MASK);
    const int cnt = G.cnt;
    const double s0 = G.sl0, s1 = G.sl1, s2 = G.sl2;
    const double l0 = L[0], l1 = L[1], l2 = L[2];
    return cnt == 1 ? band_exact(s0, s1, s2, true, x, y, d) : band_exact(l0, l1, l2, false, x, y, d);
}

// fp32 prefilter, then the exact value near the edge
__device__ __forceinline__ bool ms_member_band(const ChunkArgs& a, const SGRec& SG, const MemberRec& M,
                                               float x, float y) {
    const float v = fabsf(fmaf(M.a, x, fmaf(M.b, y, M.c)));
    if (v <= M.lo) return true;
    if (v > M.hi) return false;
    return ms_band_exact(a.grp, a.q_line, a.d, SG.g0, M.slotgi, x, y);
}

// C' membership of candidate (x, y, f) for group G (in_cprime of the v1 kernel)
__device__ __forceinline__ bool ms_in_cprime(const ChunkArgs& a, const GroupRec& G, const SGRec& S,
                                             float fx, float fy, int f) {
    return in_cprime(a, G, S, fx, fy, S.toff, f);
}

__device__ __forceinline__ MemberRec ms_member(const ChunkArgs& a, const MSlot& L, int j) {
    return j < 16 ? L.mr[j] : a.mrec[L.sg.m0 + j];
}

// per-lane state of one member block: rows g, g+8 (band constants, descriptor
// fragments in mma order, running top-2 keys)
struct MsRows {
    float ma0, mb0, mc0, lo0, hi0, ma1, mb1, mc1, lo1, hi1;
    unsigned gb0, gb1;
    unsigned af[4][4];
    int k1a, k2a, k1b, k2b;
};

__device__ __forceinline__ void ms_ldB(const MSmem& S, const uint4* tdesc, int nt, int g, uint4& u0,
                                       uint4& u1) {
    const int f = S.cid[8 * nt + g];
    u0 = __ldg(tdesc + 8 * f);
    u1 = __ldg(tdesc + 8 * f + 1);
}

// one n8 tile: 4 mma k-steps, then the 4 elements of this lane
__device__ __forceinline__ uint4 lds128v(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(su32(p)));
    return v;
}

template <bool CB, bool STATS, bool SLOTA>
__device__ __forceinline__ void ms_tile(const ChunkArgs& a, MSmem& S, const MSlot& L, MsRows& R,
                                        int mb0, int nt, const uint4& u0, const uint4& u1) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    int acc[4] = {0, 0, 0, 0};
    if (SLOTA) {
        const uint4* qd = reinterpret_cast<const uint4*>(&L.desc[0][0]) + lane;
        uint4 q = lds128v(qd);
        mma_u8(acc, q.x, q.y, q.z, q.w, u0.x, u0.y);
        q = lds128v(qd + 32);
        mma_u8(acc, q.x, q.y, q.z, q.w, u0.z, u0.w);
        q = lds128v(qd + 64);
        mma_u8(acc, q.x, q.y, q.z, q.w, u1.x, u1.y);
        q = lds128v(qd + 96);
        mma_u8(acc, q.x, q.y, q.z, q.w, u1.z, u1.w);
    } else {
        mma_u8(acc, R.af[0][0], R.af[0][1], R.af[0][2], R.af[0][3], u0.x, u0.y);
        mma_u8(acc, R.af[1][0], R.af[1][1], R.af[1][2], R.af[1][3], u0.z, u0.w);
        mma_u8(acc, R.af[2][0], R.af[2][1], R.af[2][2], R.af[2][3], u1.x, u1.y);
        mma_u8(acc, R.af[3][0], R.af[3][1], R.af[3][2], R.af[3][3], u1.z, u1.w);
    }
    const int4 c0 = S.cand[8 * nt + 2 * t], c1 = S.cand[8 * nt + 2 * t + 1];
    const float x0 = __int_as_float(c0.x), y0 = __int_as_float(c0.y);
    const float x1 = __int_as_float(c1.x), y1 = __int_as_float(c1.y);
    // elements: e0 (g, 2t), e1 (g, 2t+1), e2 (g+8, 2t), e3 (g+8, 2t+1)
    const float v0 = fabsf(fmaf(R.ma0, x0, fmaf(R.mb0, y0, R.mc0)));
    const float v1 = fabsf(fmaf(R.ma0, x1, fmaf(R.mb0, y1, R.mc0)));
    const float v2 = fabsf(fmaf(R.ma1, x0, fmaf(R.mb1, y0, R.mc1)));
    const float v3 = fabsf(fmaf(R.ma1, x1, fmaf(R.mb1, y1, R.mc1)));
    bool i0 = v0 <= R.lo0, i1 = v1 <= R.lo0, i2 = v2 <= R.lo1, i3 = v3 <= R.lo1;
    // branch-free: some element in (lo, hi]
    const bool edge = ((v0 <= R.hi0) & !i0) | ((v1 <= R.hi0) & !i1) | ((v2 <= R.hi1) & !i2) |
                      ((v3 <= R.hi1) & !i3);
    if (CB) {
        i0 = i0 && ((unsigned)c0.w & R.gb0); i1 = i1 && ((unsigned)c1.w & R.gb0);
        i2 = i2 && ((unsigned)c0.w & R.gb1); i3 = i3 && ((unsigned)c1.w & R.gb1);
    }
    ms_top2(i0 ? c0.z - acc[0] * 512 : KEY_NONE, R.k1a, R.k2a);
    ms_top2(i1 ? c1.z - acc[1] * 512 : KEY_NONE, R.k1a, R.k2a);
    ms_top2(i2 ? c0.z - acc[2] * 512 : KEY_NONE, R.k1b, R.k2b);
    ms_top2(i3 ? c1.z - acc[3] * 512 : KEY_NONE, R.k1b, R.k2b);
    bool any0 = false, any1 = false;
    if (STATS) { any0 = i0 || i2; any1 = i1 || i3; }
    if (__any_sync(FULL, edge)) {
        // within eps of the band edge: the reference's fp64 band value decides
#pragma unroll 1
        for (int e = 0; e < 4; e++) {
            const float v = e == 0 ? v0 : e == 1 ? v1 : e == 2 ? v2 : v3;
            const float lo = e < 2 ? R.lo0 : R.lo1, hi = e < 2 ? R.hi0 : R.hi1;
            if (!(v > lo && v <= hi)) continue;
            const int4 c = (e & 1) ? c1 : c0;
            if (CB && !((unsigned)c.w & (e < 2 ? R.gb0 : R.gb1))) continue;
            const MemberRec M = ms_member(a, L, mb0 + g + 8 * (e >> 1));
            if (!ms_band_exact(a.grp, a.q_line, a.d, L.sg.g0, M.slotgi, __int_as_float(c.x),
                               __int_as_float(c.y)))
                continue;
            const int av = e == 0 ? acc[0] : e == 1 ? acc[1] : e == 2 ? acc[2] : acc[3];
            if (e < 2) ms_top2(c.z - av * 512, R.k1a, R.k2a);
            else       ms_top2(c.z - av * 512, R.k1b, R.k2b);
            if (STATS) { if (e & 1) any1 = true; else any0 = true; }
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
            S.anyb[(8 * nt) >> 5] |= bits << ((8 * nt) & 31);
        }
    }
}

// One member block's tiles: lane (g, t) owns member rows g, g+8 (registers) and
// candidate columns 2t, 2t+1 of every n8 tile.  CB: consult the candidates' C' bits.
template <bool CB, bool STATS, bool SLOTA>
__device__ __forceinline__ void ms_block(const ChunkArgs& a, MSmem& S, const MSlot& L, int mb0, int m,
                                         int ntile, bool first_round) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const SGRec& SG = L.sg;
    MsRows R;
    R.ma0 = 0.f; R.mb0 = 0.f; R.mc0 = 1e30f; R.lo0 = -1.f; R.hi0 = -1.f;
    R.ma1 = 0.f; R.mb1 = 0.f; R.mc1 = 1e30f; R.lo1 = -1.f; R.hi1 = -1.f;
    R.gb0 = 0; R.gb1 = 0;
    {
        const int j0 = mb0 + g, j1 = mb0 + g + 8;
        if (j0 < m) {
            const MemberRec M = ms_member(a, L, j0);
            R.ma0 = M.a; R.mb0 = M.b; R.mc0 = M.c; R.lo0 = M.lo; R.hi0 = M.hi;
            R.gb0 = 1u << ((unsigned)M.slotgi >> SLOT_BITS);
        }
        if (j1 < m) {
            const MemberRec M = ms_member(a, L, j1);
            R.ma1 = M.a; R.mb1 = M.b; R.mc1 = M.c; R.lo1 = M.lo; R.hi1 = M.hi;
            R.gb1 = 1u << ((unsigned)M.slotgi >> SLOT_BITS);
        }
        if (!SLOTA) {
            // member blocks past the slot (one group of > 16 members, stats mode)
            uint4 w00 = make_uint4(0, 0, 0, 0), w01 = w00, w10 = w00, w11 = w00;
            if (j0 < m) {
                const uint4* row = reinterpret_cast<const uint4*>(
                    a.desc + (SG.qoff + ms_member(a, L, j0).fid) * 128) + 2 * t;
                w00 = __ldg(row); w01 = __ldg(row + 1);
            }
            if (j1 < m) {
                const uint4* row = reinterpret_cast<const uint4*>(
                    a.desc + (SG.qoff + ms_member(a, L, j1).fid) * 128) + 2 * t;
                w10 = __ldg(row); w11 = __ldg(row + 1);
            }
            R.af[0][0] = w00.x; R.af[0][1] = w10.x; R.af[0][2] = w00.y; R.af[0][3] = w10.y;
            R.af[1][0] = w00.z; R.af[1][1] = w10.z; R.af[1][2] = w00.w; R.af[1][3] = w10.w;
            R.af[2][0] = w01.x; R.af[2][1] = w11.x; R.af[2][2] = w01.y; R.af[2][3] = w11.y;
            R.af[3][0] = w01.z; R.af[3][1] = w11.z; R.af[3][2] = w01.w; R.af[3][3] = w11.w;
        }
    }
    R.k1a = KEY_NONE; R.k2a = KEY_NONE; R.k1b = KEY_NONE; R.k2b = KEY_NONE;
    // Candidate descriptor rows go through a ring of MS_RING tiles in shared memory:
    // tile nt + 2's rows are copied (cp.async, 16-B chunks, chunk p of row r at slot
    // p ^ r so a lane quad's reads spread over the banks) while tile nt is matched,
    // so the tile loop never waits on an L2 round trip.
    // Per-lane constants of the ring addressing: lane copies chunk `part` of rows prow
    // and prow + 4 of every tile; ring slots are 1 KB apart (offsets rotate, no modulo).
    const int prow = lane >> 3, part = lane & 7;
    // opaque copy: keeps the per-lane row base in one register pair, so each copy's
    // address is a single 64-bit multiply-add (f * 128 + base) instead of being
    // re-derived from SG.toff
    uint64_t src;
    asm("mov.b64 %0, %1;" : "=l"(src) : "l"(reinterpret_cast<uint64_t>(a.desc + SG.toff * 128 + part * 16)));
    const uint32_t ring0 = su32(&S.bring[0][0]);
    const uint32_t dst0 = ring0 + (uint32_t)(prow * 8 + (part ^ prow)) * 16u;
    const uint32_t dst1 = ring0 + (uint32_t)((prow + 4) * 8 + (part ^ (prow + 4))) * 16u;
    const uint32_t rd0 = ring0 + (uint32_t)(g * 8 + ((2 * t) ^ g)) * 16u;
    const uint32_t rd1 = ring0 + (uint32_t)(g * 8 + ((2 * t + 1) ^ g)) * 16u;
    constexpr uint32_t SLOT = 64 * 16, RING_END = MS_RING * SLOT;
    auto issue = [&](int nt, uint32_t k) {
        const unsigned f0 = S.cid[8 * nt + prow], f1 = S.cid[8 * nt + prow + 4];
        cp_async16_u32(dst0 + k, reinterpret_cast<const void*>(src + f0 * 128ull));
        cp_async16_u32(dst1 + k, reinterpret_cast<const void*>(src + f1 * 128ull));
    };
    issue(0, 0);
    cp_async_commit();
    if (1 < ntile) issue(1, SLOT);
    cp_async_commit();
    uint32_t kin = 2 * SLOT, kout = 0;
    for (int nt = 0; nt < ntile; nt++) {
        if (nt + 2 < ntile) issue(nt + 2, kin);
        kin = kin + SLOT == RING_END ? 0 : kin + SLOT;
        cp_async_commit();
        cp_async_wait_group<2>();
        __syncwarp();
        const uint4 u0 = lds128_u32(rd0 + kout), u1 = lds128_u32(rd1 + kout);
        kout = kout + SLOT == RING_END ? 0 : kout + SLOT;
        ms_tile<CB, STATS, SLOTA>(a, S, L, R, mb0, nt, u0, u1);
        __syncwarp();
    }
    // ---- reduce the per-lane top-2 over the 4 lanes (t) sharing a member row
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        int o1 = __shfl_xor_sync(FULL, R.k1a, o), o2 = __shfl_xor_sync(FULL, R.k2a, o);
        int lo = min(R.k1a, o1), hi = max(R.k1a, o1);
        R.k1a = lo; R.k2a = min(hi, min(R.k2a, o2));
        o1 = __shfl_xor_sync(FULL, R.k1b, o); o2 = __shfl_xor_sync(FULL, R.k2b, o);
        lo = min(R.k1b, o1); hi = max(R.k1b, o1);
        R.k1b = lo; R.k2b = min(hi, min(R.k2b, o2));
    }
    if (t == 0) {
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const int j = mb0 + g + 8 * r;
            if (j >= m) continue;
            const int k1 = r ? R.k1b : R.k1a, k2 = r ? R.k2b : R.k2a;
            const MemberRec M = ms_member(a, L, j);
            const int mslot = M.slotgi & SLOT_MASK;
            const unsigned q2 = (unsigned)M.qn9 >> 9;
            unsigned long long best = ~0ull;
            unsigned sec = NONE;
            if (k1 != KEY_NONE)
                best = ((unsigned long long)(q2 + (unsigned)(k1 >> 8)) << 32) | (unsigned)S.cid[k1 & 255];
            if (k2 != KEY_NONE) sec = q2 + (unsigned)(k2 >> 8);
            unsigned long long* pb = j < 16 ? &S.mbest[j] : &a.mstate[mslot];
            unsigned* ps = j < 16 ? &S.msec[j] : &a.mstate2[mslot];
            if (!first_round) {
                const unsigned long long ob = *pb;
                const unsigned os = *ps;
                const unsigned bd = (unsigned)(best >> 32), od = (unsigned)(ob >> 32);
                const unsigned nh = max(bd, od);
                // (d2, target) order: a tie across rounds keeps the lower target id
                const unsigned long long nbest = best < ob ? best : ob;
                sec = min(nh, min(sec, os));
                best = nbest;
            }
            *pb = best;
            *ps = sec;
        }
    }
}

// Rearrange the slot's 16 member rows in place into per-lane mma A quads: lane
// (g, t), k-step s gets {row g word 2s, row g+8 word 2s, row g word 2s+1, row g+8
// word 2s+1} of its 32-byte column block [32t, 32t+32) — one LDS.128 per k-step.
__device__ __forceinline__ void ms_quads(MSlot& L) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const uint4* r0 = reinterpret_cast<const uint4*>(L.desc[g]) + 2 * t;
    const uint4* r1 = reinterpret_cast<const uint4*>(L.desc[g + 8]) + 2 * t;
    const uint4 a0 = r0[0], a1 = r0[1], b0 = r1[0], b1 = r1[1];
    __syncwarp();
    uint4* q = reinterpret_cast<uint4*>(&L.desc[0][0]) + lane;     // [k-step][lane]
    q[0] = make_uint4(a0.x, b0.x, a0.y, b0.y);
    q[32] = make_uint4(a0.z, b0.z, a0.w, b0.w);
    q[64] = make_uint4(a1.x, b1.x, a1.y, b1.y);
    q[96] = make_uint4(a1.z, b1.z, a1.w, b1.w);
    __syncwarp();
}

// ratio > 1 only: the round's candidates reordered by target id (their rank among the
// round's unique ids), the key's local index rewritten to the new position
__device__ __forceinline__ void ms_order_by_target(MSmem& S, int n) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    int4 rc[MS_CAP / 32];
    unsigned short rid[MS_CAP / 32];
    int rank[MS_CAP / 32];
#pragma unroll
    for (int q = 0; q < MS_CAP / 32; q++) {
        const int j = lane + 32 * q;
        rank[q] = -1;
        if (j < n) {
            rc[q] = S.cand[j];
            rid[q] = S.cid[j];
            int r = 0;
            for (int i = 0; i < n; i++) r += S.cid[i] < rid[q];
            rank[q] = r;
        }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < MS_CAP / 32; q++) {
        if (rank[q] >= 0) {
            int4 c = rc[q];
            c.z = (c.z & ~0xff) | rank[q];
            S.cand[rank[q]] = c;
            S.cid[rank[q]] = rid[q];
        }
    }
    __syncwarp();
}

// One round: C' bits of the unsure candidates, then the distance tiles of every
// member block against the round's n candidates; per-member top-2 merged into
// mstate / mstate2 (first_round: written).
template <bool STATS, bool TIE>
__device__ __forceinline__ int ms_round(const ChunkArgs& a, MSmem& S, const MSlot& L, int n, int nu,
                                     bool first_round) {
    int cols_total = 0;
    const int lane = threadIdx.x & 31;
    const SGRec& SG = L.sg;
    const int m = SG.mcnt;
    const unsigned all_groups = (1u << SG.gcnt) - 1u;
    // ---- C' bits: "0" only where some member band of the group holds the candidate
    // and C'(group) does not; everywhere else the bit is never consulted (don't care)
    bool partial = false;
#ifdef MSFM_MATCH_CLOCKS
    const long long c_cb0 = clock64();
#endif
    const float c_x0 = SG.border, c_x1 = SG.W - SG.border, c_y1 = SG.H - SG.border;
    const float c_hs = SG.hsure;
    const int c_gcnt = SG.gcnt, c_m0 = SG.m0, c_g0 = SG.g0;
    int nany = 0;                      // (candidate, group) pairs decided exactly (counter)
    for (int u0 = 0; u0 < nu; u0 += 32) {
        const int uj = u0 + lane;
        if (uj < nu) {
            const int j = S.ulist[uj];
            const int f = S.cid[j];
            const int4 c = S.cand[j];
            const float px = __int_as_float(c.x), py = __int_as_float(c.y);
            const bool inner = (px >= c_x0) & (px <= c_x1) & (py >= c_x0) & (py <= c_y1);
            unsigned bits = all_groups;
            for (int gi = 0; gi < c_gcnt; gi++) {
                const GView gv = L.gv[gi];
                const float dg = fabsf(fmaf(gv.a, px, fmaf(gv.b, py, gv.c)));
                if ((dg <= c_hs && inner) || dg > gv.reach) continue;
                const int k0 = max(gv.moff - c_m0, 0);
                const int k1 = gi + 1 < c_gcnt ? max(L.gv[gi + 1].moff - c_m0, 0) : m;
                bool any = false;
                for (int k = k0; k < k1 && !any; k++) any = ms_member_band(a, SG, ms_member(a, L, k), px, py);
                nany += any;
                if (any && !in_cprime(a, a.grp[c_g0 + gi], SG, px, py, SG.toff, f)) bits &= ~(1u << gi);
            }
            S.cand[j].w = (int)bits;
            partial |= bits != all_groups;
        }
    }
#ifdef MSFM_MATCH_CLOCKS
    if (a.dbg && lane == 0) atomicAdd(&a.dbg[9], (unsigned long long)(clock64() - c_cb0));
    const long long c_t0 = clock64();
#else
    if (a.dbg && nany) atomicAdd(&a.dbg[6], (unsigned long long)nany);
#endif
    // ---- ratio > 1 accepts a tie at the minimum (ratio 1), and the reference's argmin
    // then names the lowest target id among the tied candidates: order the round's
    // candidates by target id so the key's local index (the tie-break) follows it
    // (target ids are unique within a super-group's strip)
    if (TIE) ms_order_by_target(S, n);
    // ---- pad the last n8 tile with candidates no member accepts (NaN position: never
    // inside a band, never near its edge)
    const int ntile = (n + 7) >> 3;
    if (lane < ntile * 8 - n) {
        S.cand[n + lane] = make_int4(0x7fc00000, 0x7fc00000, 0, 0);
        S.cid[n + lane] = 0;
    }
    if (STATS)
        for (int w = lane; w < MS_CAP / 32; w += 32) S.anyb[w] = 0;
    partial = __any_sync(FULL, partial);
    __syncwarp();
    if (partial) ms_block<true, STATS, true>(a, S, L, 0, m, ntile, first_round);
    else         ms_block<false, STATS, true>(a, S, L, 0, m, ntile, first_round);
    // member blocks past the slot (one group of > 16 members, stats mode only)
    for (int mb0 = 16; mb0 < m; mb0 += 16) ms_block<true, STATS, false>(a, S, L, mb0, m, ntile, first_round);
#ifdef MSFM_MATCH_CLOCKS
    if (a.dbg && lane == 0) atomicAdd(&a.dbg[6], (unsigned long long)(clock64() - c_t0));
#endif
    if (STATS) {
        __syncwarp();
        int cnt = lane < MS_CAP / 32 ? __popc(S.anyb[lane]) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        cols_total += cnt;
    }
    __syncwarp();
    return cols_total;
}

// TIE (ratio > 1): candidates of a round ordered by target id before the tiles
template <bool STATS, bool TIE>
__global__ void __launch_bounds__(MS_WARPS * 32, MS_MINB) match_ms_kernel(const __grid_constant__ ChunkArgs a) {
    extern __shared__ __align__(128) unsigned char ms_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    MSmem& S = reinterpret_cast<MSmem*>(ms_raw)[warp];
    const int total = *a.sg_total;
    const float Df = (float)a.D;
    if (lane == 0) {
        ms_bar_init(&S.bar_q);
        ms_bar_init(&S.bar_rec[0]); ms_bar_init(&S.bar_rec[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t ph_q = 0, ph_rec = 0;     // phase bits (per slot: bit s)
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
    int sid_cur = claim(), sid_nxt = claim();
    if (sid_cur < total) {
        load_sg(S.slot[0], sid_cur);
        if (lane == 0) ms_issue_rec(a, S.slot[0], &S.bar_rec[0]);
    }
    if (sid_nxt < total) {
        load_sg(S.slot[1], sid_nxt);
        if (lane == 0) ms_issue_rec(a, S.slot[1], &S.bar_rec[1]);
    }
    if (sid_cur < total) {
        ms_wait(&S.bar_rec[0], 0);
        ph_rec ^= 1u;
        ms_issue_desc(a, S.slot[0]);
    }
    int cur = 0;
    for (;;) {
        const int sid = sid_cur;
        if (sid >= total) break;
#ifdef MSFM_MATCH_CLOCKS
        const long long c0 = clock64();
        long long c_round = 0;
#endif
        const int nxt = cur ^ 1;
        MSlot& L = S.slot[cur];
        // the SG after next: its record goes to sgq
        const int sid2 = claim();
        if (sid2 < total && lane == 0) {
            ms_expect(&S.bar_q, (uint32_t)sizeof(SGRec));
            ms_bulk_ef(&S.sgq, a.sg + sid2, sizeof(SGRec), &S.bar_q);
        }
        // this SG's member descriptor rows (cp.async issued during the last SG)
        cp_async_wait_all();
        __syncwarp();
        ms_quads(L);
#ifdef MSFM_MATCH_CLOCKS
        const long long c1 = clock64();
#endif
        const SGRec& SG = L.sg;
        if (a.dbg && lane == 0) {
            atomicAdd(&a.dbg[0], 1ull);
            atomicAdd(&a.dbg[1], (unsigned long long)SG.mcnt);
            atomicAdd(&a.dbg[8], (unsigned long long)SG.gcnt);
#ifndef MSFM_MATCH_CLOCKS
            atomicAdd(&a.dbg[5], (unsigned long long)(SG.rhi - SG.rlo + 1));   // strip rows
#endif
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
            if (!nxt_desc_issued && sid_nxt < total) {
                ms_wait(&S.bar_rec[nxt], (ph_rec >> nxt) & 1u);
                ph_rec ^= 1u << nxt;
                ms_issue_desc(a, S.slot[nxt]);
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
        // Resumable gather state: the current 32-row batch (per-lane CSR span bs, len
        // and its inclusive prefix), the next record index j0 in it, the prefetched
        // record of j0 + lane, and the next batch's spans (prefetched).  A full
        // candidate list suspends the gather for a round; the round runs outside the
        // gather loop, so the two never compete for registers.
        int r0 = SG.rlo, bs = 0, len = 0, incl = 0, tot = 0, j0 = 0;
        int nbs, ne1;
        int4 nrec = make_int4(0, 0, 0, 0);
        // record index of batch position j = w0 + lane: the row holding j is the last
        // non-empty row starting at or before j.  Non-empty rows' starts are distinct, so
        // the window's starts form one bit mask (OR-reduction); rows are ranked among the
        // non-empty ones, whose (CSR start, batch start) open_batch keeps in shared memory.
        auto rec_at = [&](int w0) {
            const int excl = incl - len;
            const bool ne = len > 0;
            const unsigned bit = (ne && excl >= w0 && excl < w0 + 32) ? 1u << (excl - w0) : 0u;
            const unsigned mask = __reduce_or_sync(FULL, bit);
            const int before = __popc(__ballot_sync(FULL, ne && excl < w0));
            const int k = max(before + __popc(mask & (0xffffffffu >> (31 - lane))) - 1, 0);
            return S.rbs[k] + (w0 + lane - S.rex[k]);
        };
        auto open_batch = [&]() {
            bs = nbs;
            len = ne1 - nbs;
            row_span(r0 + 32 + lane, nbs, ne1);
            incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            tot = __shfl_sync(FULL, incl, 31);
            {
                const unsigned nem = __ballot_sync(FULL, len > 0);
                if (len > 0) {
                    const int rk = __popc(nem & ((1u << lane) - 1u));
                    S.rbs[rk] = bs;
                    S.rex[rk] = incl - len;
                }
                __syncwarp();
            }
#ifndef MSFM_MATCH_CLOCKS
            if (a.dbg && lane == 0) atomicAdd(&a.dbg[2], (unsigned long long)tot);
#endif
            j0 = 0;
            const int ri = rec_at(0);
            nrec = lane < tot ? __ldg(mrec4 + ri) : make_int4(0, 0, 0, 0);
        };
        row_span(SG.rlo + lane, nbs, ne1);
        if (r0 <= SG.rhi) open_batch();
        for (;;) {
            // the strip and "sure" constants in registers for this gather pass (SG lives
            // in shared memory, which the candidate stores below could alias: the
            // compiler would reload it per batch); not live across the round
            const float g_ar = SG.ar, g_br = SG.br, g_cr = SG.cr, g_R = SG.R;
            const float g_delta = SG.delta, g_hs = SG.hsure;
            const float g_x0 = SG.border, g_x1 = SG.W - SG.border, g_y1 = SG.H - SG.border;
            const int g_rhi = SG.rhi;
            // ---- gather until the strip ends or the next record batch would overflow
            bool full = false;
            while (r0 <= g_rhi) {
                if (j0 >= tot) {
                    r0 += 32;
                    if (r0 > g_rhi) break;
                    open_batch();
                    continue;
                }
                const int j = j0 + lane;
                const int4 rec = nrec;
                bool pass = false, sure = false;
                const float px = __int_as_float(rec.x), py = __int_as_float(rec.y);
                if (j < tot) {
                    const float adr = fabsf(fmaf(g_ar, px, fmaf(g_br, py, g_cr)));
                    pass = adr <= g_R;
                    sure = (adr + g_delta <= g_hs) & (px >= g_x0) & (px <= g_x1) & (py >= g_x0) & (py <= g_y1);
                }
                const unsigned bal = __ballot_sync(FULL, pass);
                const int cnt = __popc(bal);
                if (n + cnt > MS_CAP) { full = true; break; }
                {
                    const int ri = rec_at(j0 + 32);
                    if (j + 32 < tot) nrec = __ldg(mrec4 + ri);
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
                j0 += 32;
                __syncwarp();
            }
            __syncwarp();
            issue_next_desc();
#ifndef MSFM_MATCH_CLOCKS
            // counters once per round: passing = n, surely in every C' = n - nu
            if (a.dbg && lane == 0) {
                atomicAdd(&a.dbg[3], (unsigned long long)n);
                atomicAdd(&a.dbg[4], (unsigned long long)(n - nu));
            }
#endif
            if (n > 0) {
#ifdef MSFM_MATCH_CLOCKS
                const long long cr = clock64();
#endif
                cols_total += ms_round<STATS, TIE>(a, S, L, n, nu, first_round);
#ifdef MSFM_MATCH_CLOCKS
                c_round += clock64() - cr;
#endif
                first_round = false;
                n = 0;
                nu = 0;
            }
            if (!full) break;
        }
        __syncwarp();
#ifdef MSFM_MATCH_CLOCKS
        const long long c2 = clock64();
#endif
        // ---- ratio test + dedupe per member (ratio_filter / _dedupe_targets)
        if (!first_round) {
            for (int j = lane; j < SG.mcnt; j += 32) {
                const MemberRec M = j < 16 ? L.mr[j] : a.mrec[SG.m0 + j];
                const int slot = M.slotgi & SLOT_MASK;
                const unsigned long long best = j < 16 ? S.mbest[j] : a.mstate[slot];
                const unsigned sec = j < 16 ? S.msec[j] : a.mstate2[slot];
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
        sid_cur = sid_nxt;
        sid_nxt = sid2;
        if (sid2 < total) {
            ms_wait(&S.bar_q, ph_q);
            ph_q ^= 1u;
            if (lane < 8) reinterpret_cast<uint4*>(&L.sg)[lane] = reinterpret_cast<const uint4*>(&S.sgq)[lane];
            __syncwarp();
            ms_fence_async();
            if (lane == 0) ms_issue_rec(a, L, &S.bar_rec[cur]);
        }
        __syncwarp();
#ifdef MSFM_MATCH_CLOCKS
        if (a.dbg && lane == 0) {
            const long long c3 = clock64();
            atomicAdd(&a.dbg[5], (unsigned long long)(c1 - c0));                // SG setup
            atomicAdd(&a.dbg[7], (unsigned long long)(c2 - c1 - c_round));      // gather
            atomicAdd(&a.dbg[10], (unsigned long long)(c3 - c2));               // ratio + rotation
        }
#endif
        cur = nxt;
    }
}
