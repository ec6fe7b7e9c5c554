// Per-pair matcher setup (included by guided.cu inside msfm::<anon>).
//
// One CTA per pair runs the whole front half of guided_match_pair
// (guided.py:393-446) for that pair and leaves the super-group records the
// match kernel consumes:
//
//   lines     epipolar line of every query (dgemm rounding), normalise, clip,
//             composite bucket key (group_queries guided.py:340-390), insert into
//             the pair's hash table (shared memory up to TS_SMEM slots)
//   groups    compact the occupied slots, order the groups by representative-line
//             angle (pseudo-angle key, GB-bucket counting sort, each bucket sorted
//             by (key, group)), member ranges, boundary endpoints
//   scatter   member lists; per group the padded clip / sample geometry (GroupRec,
//             equidistant_line_points guided.py:173-187)
//   chain     super-groups: e(q) = min(q + 16, B(g(q))) per member position (B: the
//             first group that stops fitting g's line, or the end), the greedy walk
//             from position 0 found in three segmented passes, compacted in order
//   shape     per super-group: group range, base line (middle group's rep)
//   members   per member: epilogue constants, band deviation from its group's rep
//             and its super-group's base (shared-memory / L2 atomic maxima)
//   strips    per (super-group, group): rep deviation from the base, group views;
//             per super-group: strip half-width, sure radius, bucket-row range
//
// Everything a pair needs stays in one CTA: the intermediates are written and
// re-read while L2-hot, the hash table lives in shared memory, and the only
// cross-pair step is one atomicAdd that places the pair's super-groups in the
// chunk-wide queue (their order only schedules work; results never depend on it).
// All arrays are indexed in chunk slot space (s0 + local index), which bounds
// groups / super-groups / members of a pair by its query count.

constexpr int ST = 1024;          // setup threads per pair
constexpr int TS_SMEM = 8192;     // hash tables up to this many slots live in shared memory
// table: key u64, rep u32, count u32 per slot; histogram; scan scratch
constexpr size_t SETUP_SMEM = (size_t)TS_SMEM * 16 + (size_t)GB * 4 + 512;

// Upper bounds of |dist_m - dist_r| (and - dist_b) over the member band (|dist_m| <=
// B = d + 0.5) inside the image, in fp32 (lines rounded to f32: < 1e-3 px on 3k-px
// images): the polygon's vertices (image corners inside
// the band, band-edge crossings of the borders) with every inclusion test widened by
// half a pixel and the result raised by 0.01 px.  Extra evaluation points only raise
// the maximum, and the fp32 errors (~1e-3 px on 3k-px images) are far below the
// margins, so these stay upper bounds; the deviations only size strips and C'-test
// reaches, never decide a match.
__device__ void band_deviation2_f(const float m[3], const float r[3], const float b[3], float W,
                                  float H, float d, float& dev_r, float& dev_b) {
    const float m0 = m[0], m1 = m[1], m2 = m[2];
    const float ra = m0 - r[0], rb = m1 - r[1], rc = m2 - r[2];
    const float ba = m0 - b[0], bb = m1 - b[1], bc = m2 - b[2];
    const float B = d + 0.5f, Bc = B + 0.01f, tol = 0.5f;
    float vr = 0.f, vb = 0.f;
    const float cx[4] = {0.f, W, 0.f, W}, cy[4] = {0.f, 0.f, H, H};
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (fabsf(fmaf(m0, cx[k], fmaf(m1, cy[k], m2))) <= Bc) {
            vr = fmaxf(vr, fabsf(fmaf(ra, cx[k], fmaf(rb, cy[k], rc))));
            vb = fmaxf(vb, fabsf(fmaf(ba, cx[k], fmaf(bb, cy[k], bc))));
        }
    }
    const float i1 = fabsf(m1) > 1e-12f ? 1.0f / m1 : 0.f;
    const float i0 = fabsf(m0) > 1e-12f ? 1.0f / m0 : 0.f;
#pragma unroll
    for (int s = -1; s <= 1; s += 2) {
        if (i1 != 0.f) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float x = e ? W : 0.f;
                const float y = (s * B - m2 - m0 * x) * i1;
                if (y >= -tol && y <= H + tol) {
                    vr = fmaxf(vr, fabsf(fmaf(ra, x, fmaf(rb, y, rc))));
                    vb = fmaxf(vb, fabsf(fmaf(ba, x, fmaf(bb, y, bc))));
                }
            }
        }
        if (i0 != 0.f) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float y = e ? H : 0.f;
                const float x = (s * B - m2 - m1 * y) * i0;
                if (x >= -tol && x <= W + tol) {
                    vr = fmaxf(vr, fabsf(fmaf(ra, x, fmaf(rb, y, rc))));
                    vb = fmaxf(vb, fabsf(fmaf(ba, x, fmaf(bb, y, bc))));
                }
            }
        }
    }
    dev_r = vr + 0.01f;
    dev_b = vb + 0.01f;
}

// max |dist_g - dist_base| over the strip |dist_base| <= R inside the image (fp32
// upper bound, as above)
__device__ float band_deviation_f(const float b[3], const float g[3], float W, float H, float R) {
    const float m0 = b[0], m1 = b[1], m2 = b[2];
    const float da = m0 - g[0], db = m1 - g[1], dc = m2 - g[2];
    const float Rc = R + 0.01f, tol = 0.5f;
    float v = 0.f;
    const float cx[4] = {0.f, W, 0.f, W}, cy[4] = {0.f, 0.f, H, H};
#pragma unroll
    for (int k = 0; k < 4; k++)
        if (fabsf(fmaf(m0, cx[k], fmaf(m1, cy[k], m2))) <= Rc)
            v = fmaxf(v, fabsf(fmaf(da, cx[k], fmaf(db, cy[k], dc))));
    const float i1 = fabsf(m1) > 1e-12f ? 1.0f / m1 : 0.f;
    const float i0 = fabsf(m0) > 1e-12f ? 1.0f / m0 : 0.f;
#pragma unroll
    for (int s = -1; s <= 1; s += 2) {
        if (i1 != 0.f) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float x = e ? W : 0.f;
                const float y = (s * R - m2 - m0 * x) * i1;
                if (y >= -tol && y <= H + tol) v = fmaxf(v, fabsf(fmaf(da, x, fmaf(db, y, dc))));
            }
        }
        if (i0 != 0.f) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float y = e ? H : 0.f;
                const float x = (s * R - m2 - m1 * y) * i0;
                if (x >= -tol && x <= W + tol) v = fmaxf(v, fabsf(fmaf(da, x, fmaf(db, y, dc))));
            }
        }
    }
    return v + 0.01f;
}

__global__ void __launch_bounds__(ST, 1) setup_kernel(const __grid_constant__ ChunkArgs a) {
    extern __shared__ __align__(16) unsigned char su_raw[];
    const int p = blockIdx.x, pg = a.p0 + p;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t q0 = a.qlist_off[pg];
    const int nq = (int)(a.qlist_off[pg + 1] - q0);
    const int64_t s0 = q0 - a.qbase;
    const int64_t t0 = a.tab_off[p];
    const int tsize = (int)(a.tab_off[p + 1] - t0);
    const int ti = a.pair_t[pg], qi = a.pair_q[pg];
    const int nt = a.img_n[ti];
    const int64_t db = a.tbase[p];
    int* hist = reinterpret_cast<int*>(su_raw + (size_t)TS_SMEM * 16);
    int* ssm = hist + GB;                                   // block-scan scratch (33)
    float* fmn = reinterpret_cast<float*>(ssm + 40);
    float* fmx = fmn + 32;
    int* sv = reinterpret_cast<int*>(fmx + 32);             // [0] ng [1] nm [2] nsg [3] base [4] done
    const bool small = tsize <= TS_SMEM;
    long long tmark[5] = {0, 0, 0, 0, 0};    // phase clocks (msfm_debug_counters)
    // after the compaction trep holds the group id
    unsigned long long* tkey = small ? reinterpret_cast<unsigned long long*>(su_raw) : a.tab_key + t0;
    unsigned* trep = small ? reinterpret_cast<unsigned*>(su_raw + (size_t)TS_SMEM * 8) : a.tab_rep + t0;
    unsigned* tcnt = small ? reinterpret_cast<unsigned*>(su_raw + (size_t)TS_SMEM * 12) : a.tab_cnt + t0;
    // small pairs keep the per-position / per-group indices the later phases re-read
    // as u16 in shared memory the table and histogram free up: the member's group
    // (from the scatter on, over the count array), its query (over the histogram),
    // each group's fit boundary (chain phase) and then each member's super-group
    // (both over the count array's second half)
    unsigned short* mg16 = reinterpret_cast<unsigned short*>(su_raw + (size_t)TS_SMEM * 12);
    unsigned short* fit16 = mg16 + TS_SMEM;
    unsigned short* sg16 = mg16 + TS_SMEM;
    unsigned short* mq16 = reinterpret_cast<unsigned short*>(su_raw + (size_t)TS_SMEM * 16);
    auto MGID = [&](int k) { return small ? (int)mg16[k] : a.mgid[s0 + k]; };
    auto MSG = [&](int k) { return small ? (int)sg16[k] : a.msg[s0 + k]; };
    auto MSLOT = [&](int k) { return small ? (int)(s0 + mq16[k]) : a.members[s0 + k]; };
    auto GFIT = [&](int g) { return small ? (int)fit16[g] : (int)a.gfit[s0 + g]; };

    // ---------------- init
    for (int e = tid; e < tsize; e += ST) {
        tkey[e] = EMPTY;
        trep[e] = NONE;
        tcnt[e] = 0;
    }
    // outputs the setup never re-reads are stored evict-first (st.global.cs) so they
    // do not push the phases' re-read data (lines, group records) out of L2
    for (int e = tid; e < nt; e += ST) __stcs(reinterpret_cast<unsigned long long*>(a.dedupe + db + e), EMPTY);
    for (int i = tid; i < nq; i += ST) {
        __stcs(a.res_tid + s0 + i, -1);
        if (!small) a.gfill[s0 + i] = 0;
    }
    if (isnan(a.pair_F[9 * (int64_t)pg]) || nq == 0) return;   // no groups: nothing queued
    __syncthreads();
    if (a.dbg && tid == 0) tmark[0] = clock64();

    // ---------------- lines (lines_kernel of round 1; guided.py:353-373)
    const double W = a.img_wh[2 * ti], H = a.img_wh[2 * ti + 1];
    const int64_t qoff = a.img_off[qi];
    const unsigned mask = (unsigned)tsize - 1;
    const int64_t qs = a.qlist_src ? a.qlist_src[pg] : q0;
    double F[9];
#pragma unroll
    for (int j = 0; j < 9; j++) F[j] = a.pair_F[9 * (int64_t)pg + j];
    // the next query's id, position and |q|^2 are loaded while this one's fp64
    // geometry runs (the loads are a two-deep dependent chain through qlist)
    int fid_n = 0, n2_n = 0;
    float2 p2_n = make_float2(0.f, 0.f);
    if (tid < nq) {
        fid_n = __ldg(a.qlist + qs + tid);
        p2_n = __ldg(a.xy + qoff + fid_n);
        n2_n = __ldg(a.norm2 + qoff + fid_n);
    }
    for (int i = tid; i < nq; i += ST) {
        const int fid = fid_n;
        const float2 p2 = p2_n;
        const int qn2 = n2_n;
        if (i + ST < nq) {
            fid_n = __ldg(a.qlist + qs + i + ST);
            p2_n = __ldg(a.xy + qoff + fid_n);
            n2_n = __ldg(a.norm2 + qoff + fid_n);
        }
        a.q_fid[s0 + i] = fid;
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
                    const unsigned long long prev = atomicCAS(&tkey[h], EMPTY, key);
                    if (prev == EMPTY || prev == key) break;
                    h = (h + 1) & mask;
                }
                atomicMin(&trep[h], (unsigned)i);
                atomicAdd(&tcnt[h], 1u);
                slot = (int)h;
                double* L = a.q_line + 3 * (s0 + i);
                L[0] = l[0]; L[1] = l[1]; L[2] = l[2];
                a.q_lf[s0 + i] = make_float4((float)l[0], (float)l[1], (float)l[2], __int_as_float(qn2));
            }
        }
        a.q_tab[s0 + i] = slot;
    }
    __syncthreads();
    if (a.dbg && tid == 0) tmark[1] = clock64();

    // ---------------- groups: compaction, angle order, member ranges, endpoints
    // one block scan: thread tid owns slots tid, tid + ST, ...; group ids are handed
    // out thread-major (any order: groups are re-ordered by angle below)
    float lo = 1e30f, hi = -1e30f;
    int gcarry;
    {
        int mine = 0;
        for (int e = tid; e < tsize; e += ST) mine += tkey[e] != EMPTY;
        const int gbase = block_exclusive_scan<ST>(mine, &gcarry, ssm);
        int g = gbase;
        for (int e = tid; e < tsize; e += ST) {
            if (tkey[e] == EMPTY) continue;
            const unsigned cnt = tcnt[e], rep = trep[e];
            a.gtmp[s0 + g] = make_int2((int)rep, (int)cnt);
            const double* L = a.q_line + 3 * (s0 + rep);
            float la = (float)L[0], lb = (float)L[1];
            if (la < 0.f || (la == 0.f && lb < 0.f)) { la = -la; lb = -lb; }
            // a monotone pseudo-angle of the direction (la >= 0 half-plane): the key
            // only buckets groups for the angle order, any monotone map of atan2 will do
            const float ang = lb / fmaxf(fabsf(la) + fabsf(lb), 1e-30f);
            a.gkey[s0 + g] = ang;
            lo = fminf(lo, ang);
            hi = fmaxf(hi, ang);
            trep[e] = (unsigned)g;
            g++;
        }
    }
    const int ng = gcarry;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
    }
    if (lane == 0) { fmn[wid] = lo; fmx[wid] = hi; }
    for (int b = tid; b < GB; b += ST) hist[b] = 0;
    __syncthreads();
    lo = fmn[0]; hi = fmx[0];
    for (int w = 1; w < ST / 32; w++) { lo = fminf(lo, fmn[w]); hi = fmaxf(hi, fmx[w]); }
    const float scale = (float)GB / fmaxf(hi - lo, 1e-20f);
    for (int g = tid; g < ng; g += ST) {
        const int b = min(GB - 1, max(0, (int)((a.gkey[s0 + g] - lo) * scale)));
        atomicAdd(&hist[b], 1);
    }
    __syncthreads();
    {
        int v[GB / ST];
        int s = 0;
#pragma unroll
        for (int k = 0; k < GB / ST; k++) { v[k] = hist[tid * (GB / ST) + k]; s += v[k]; }
        int tot;
        int ex = block_exclusive_scan<ST>(s, &tot, ssm);
#pragma unroll
        for (int k = 0; k < GB / ST; k++) { hist[tid * (GB / ST) + k] = ex; ex += v[k]; }
    }
    __syncthreads();
    for (int g = tid; g < ng; g += ST) {
        const float key = a.gkey[s0 + g];
        const int b = min(GB - 1, max(0, (int)((key - lo) * scale)));
        const int pos = atomicAdd(&hist[b], 1);
        a.gpos[s0 + g] = pos;
        const int2 r = a.gtmp[s0 + g];
        // .z: the key, .w: the group (for the sort below; .z becomes the member offset)
        a.grec[s0 + pos] = make_int4(r.x, r.y, __float_as_int(key), g);
    }
    __syncthreads();
    // the atomics leave a bucket's few groups in arbitrary order: sort each bucket by
    // (key, group) so the super-group walk sees the exact angle order (fewer breaks)
    auto before = [](const int4& u, const int4& v) {   // (key, group) order
        const float ku = __int_as_float(u.z), kv = __int_as_float(v.z);
        return ku < kv || (ku == kv && u.w < v.w);
    };
    for (int b = tid; b < GB; b += ST) {
        const int e = hist[b], st = b == 0 ? 0 : hist[b - 1];
        if (e - st < 2) continue;
        if (e - st == 2) {                                  // the common case: one swap
            int4 u = a.grec[s0 + st], v = a.grec[s0 + st + 1];
            if (before(v, u)) {
                a.grec[s0 + st] = v; a.grec[s0 + st + 1] = u;
                a.gpos[s0 + v.w] = st; a.gpos[s0 + u.w] = st + 1;
            }
            continue;
        }
        for (int i = st + 1; i < e; i++) {
            const int4 v = a.grec[s0 + i];
            const float kv = __int_as_float(v.z);
            int j = i - 1;
            for (; j >= st; j--) {
                const int4 u = a.grec[s0 + j];
                const float ku = __int_as_float(u.z);
                if (ku < kv || (ku == kv && u.w < v.w)) break;
                a.grec[s0 + j + 1] = u;
            }
            a.grec[s0 + j + 1] = v;
        }
        for (int i = st; i < e; i++) a.gpos[s0 + a.grec[s0 + i].w] = i;
    }
    __syncthreads();
    int mcarry = 0;
    for (int i0 = 0; i0 < ng; i0 += ST) {
        const int i = i0 + tid;
        const int cnt = i < ng ? a.grec[s0 + i].y : 0;
        int tot;
        const int ex = block_exclusive_scan<ST>(cnt, &tot, ssm);
        if (i < ng) a.grec[s0 + i].z = (int)(s0 + mcarry + ex);
        mcarry += tot;
    }
    const int nm = mcarry;
    for (int e = tid; e < tsize; e += ST)
        if (tkey[e] != EMPTY) trep[e] = (unsigned)a.gpos[s0 + trep[e]];
    __syncthreads();
    if (a.dbg && tid == 0) tmark[2] = clock64();

    // ---------------- scatter + per-group geometry (GroupRec, endpoints)
    // member fill counters: shared memory over the dead key array (small pairs)
    unsigned* gfill = small ? reinterpret_cast<unsigned*>(su_raw) : reinterpret_cast<unsigned*>(a.gfill + s0);
    if (small) {
        for (int g = tid; g < ng; g += ST) gfill[g] = 0u;
        __syncthreads();
    }
    for (int i = tid; i < nq; i += ST) {
        const int h = a.q_tab[s0 + i];
        if (h < 0) continue;
        const int lg = (int)trep[h];
        const int4 g = a.grec[s0 + lg];
        const int pos = g.z + (int)atomicAdd(&gfill[lg], 1u);
        if (small) {
            mg16[pos - s0] = (unsigned short)lg;
            mq16[pos - s0] = (unsigned short)i;
        } else {
            a.members[pos] = (int)(s0 + i);
            a.mgid[pos] = lg;
        }
    }
    const double D = a.D, d = a.d;
    for (int lg = tid; lg < ng; lg += ST) {
        const int4 g = a.grec[s0 + lg];
        const double* rl = a.q_line + 3 * (s0 + g.x);
        const double r[3] = {rl[0], rl[1], rl[2]};
        // boundary endpoints of the representative (group_queries' pa, pb)
        {
            double pa[2] = {0, 0}, pb[2] = {0, 0};
            clip_batch(r, W, H, pa, pb);
            a.gline[s0 + lg] = make_float4((float)r[0], (float)r[1], (float)r[2], 0.f);
            a.gend[s0 + lg] = make_float4((float)pa[0], (float)pa[1], (float)pb[0], (float)pb[1]);
        }
        // C' geometry of the representative (prep_kernel of round 1)
        GroupRec o;
        o.p = p; o.rep = (int)(s0 + g.x); o.cnt = g.y; o.moff = g.z;
        o.sl0 = r[0]; o.sl1 = r[1]; o.sl2 = r[2]; o.spare = 0.0;
        if (g.y == 1) {
            // a singleton's own band uses the dgemv-rounded line (guided.py:443-446,
            // m == 1): computed here, once per group, for the exact fallbacks
            const int fid = a.q_fid[s0 + g.x];
            const float2 p2 = a.xy[qoff + fid];
            double Fm[9], m[3];
#pragma unroll
            for (int j = 0; j < 9; j++) Fm[j] = a.pair_F[9 * (int64_t)pg + j];
            epiline(Fm, (double)p2.x, (double)p2.y, true, m);
            const double nrm = fmax(np_hypot(m[0], m[1]), 1e-15);
            o.sl0 = m[0] / nrm; o.sl1 = m[1] / nrm; o.sl2 = m[2] / nrm;
        }
        o.pad1 = o.pad2 = o.pad3 = 0;
        double pa[2] = {0, 0}, pb[2] = {0, 0}, len = 0.0;
        o.K = -1;
        if (clip_scalar(r[0], r[1], r[2], W, H, d, pa, pb)) {
            len = np_hypot(pb[0] - pa[0], pb[1] - pa[1]);
            const long long K = (long long)ceil(len / d);
            o.K = (int)(K < 1 ? 1 : K);
        }
        o.pax = pa[0]; o.pay = pa[1]; o.pbx64 = pb[0]; o.pby64 = pb[1];
        o.ar = (float)r[0]; o.br = (float)r[1]; o.cr = (float)r[2];
        o.maxdev = 0.05f;                     // raised per member (atomic max of f32 bits)
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
        {
            // hot 32 B (re-read by the later phases): normal stores; the rest evict-first
            int4* dst = reinterpret_cast<int4*>(a.grp + s0 + lg);
            const int4* w = reinterpret_cast<const int4*>(&o);
            dst[0] = w[0];
            dst[1] = w[1];
#pragma unroll
            for (int k = 2; k < 10; k++) __stcs(dst + k, w[k]);
        }
    }
    __syncthreads();
    if (a.dbg && tid == 0) tmark[3] = clock64();

    // ---------------- super-groups
    // J / mark arrays: shared memory (reusing the table) for small pairs, else global
    // (global: nm + 1 entries per pair, so pair p's range starts at s0 + p)
    int* Ja = small ? reinterpret_cast<int*>(su_raw) : a.jmp_a + s0 + p;
    int* Jb = small ? reinterpret_cast<int*>(su_raw) + TS_SMEM : a.jmp_b + s0 + p;
    int* mk = small ? reinterpret_cast<int*>(su_raw) + 2 * TS_SMEM : a.jmark + s0 + p;
    int nsg;
    if (a.stats_mode) {
        // one super-group per group (exact SearchStats)
        for (int g = tid; g < ng; g += ST) {
            const int4 gr = a.grec[s0 + g];
            a.sglist[s0 + g] = make_int2(gr.z, gr.y);
        }
        nsg = ng;
    } else {
        // B(g): first member position of the first group after g that does not fit
        // g's line within tau (bit i of the fit mask: group g+1+i fits), or nm
        for (int g = tid; g < ng; g += ST) {
            const float4 ln = a.gline[s0 + g];
            unsigned bits = 0;
            const int lim = min(SG_MEMBERS, ng - 1 - g);
            // all the following groups' endpoints in flight at once (no early exit)
#pragma unroll
            for (int i = 0; i < SG_MEMBERS; i++) {
                if (i < lim) {
                    const float4 en = a.gend[s0 + g + 1 + i];
                    const float d1 = fabsf(fmaf(ln.x, en.x, fmaf(ln.y, en.y, ln.z)));
                    const float d2 = fabsf(fmaf(ln.x, en.z, fmaf(ln.y, en.w, ln.z)));
                    if (fmaxf(d1, d2) <= a.sg_tau) bits |= 1u << i;
                }
            }
            const int j = g + 1 + __ffs(~bits) - 1;
            const int bnd = j < ng ? (int)(a.grec[s0 + j].z - s0) : nm;
            if (small) fit16[g] = (unsigned short)bnd;
            else a.gfit[s0 + g] = bnd;
        }
        __syncthreads();
        // e(q) = min(q + 16, B(g(q))) is where the super-group opened at q closes
        // (members are contiguous in group order); J = e, J(nm) = nm
        for (int q = tid; q <= nm; q += ST) {
            int e = nm;
            if (q < nm) e = min(q + SG_MEMBERS, GFIT(MGID(q)));
            Ja[q] = e;
            mk[q] = q == 0 ? 1 : 0;
        }
        __syncthreads();
        // The walk 0 -> e(0) -> e(e(0)) ... in three passes.  Positions are cut into
        // segments of S >= 16; a step moves at most 16, so the walk enters segment w at
        // one of its first 16 positions.  (A) each warp walks its segment from all 16
        // possible entries (a lane each) and records where each leaves it; (B) one
        // thread chains the segments' entries; (C) each warp re-walks its segment from
        // the resolved entry and marks the super-group starts.
        {
            __shared__ int cx_exit[ST / 32][16];
            __shared__ int cx_entry[ST / 32];
            constexpr int NSEG = ST / 32;
            const int S = max(SG_MEMBERS, (nm + NSEG - 1) / NSEG);
            const int nseg = (nm + S - 1) / S;
            if (wid < nseg && lane < 16) {
                const int lo = wid * S, hi = min(lo + S, nm);
                int q = lo + lane;
                while (q < hi) q = Ja[q];
                cx_exit[wid][lane] = q;
            }
            __syncthreads();
            if (tid == 0) {
                int q = 0;
                for (int w = 0; w < nseg; w++) {
                    cx_entry[w] = q;
                    q = cx_exit[w][q - w * S];
                }
            }
            __syncthreads();
            if (wid < nseg && lane == 0) {
                const int hi = min((wid + 1) * S, nm);
                for (int q = cx_entry[wid]; q < hi; q = Ja[q]) mk[q] = 1;
            }
            __syncthreads();
        }
        // the marks are the walk's starts; compact them in order (e from the q + 16 /
        // B rule again, since the J arrays were overwritten)
        // (one block scan: thread tid owns positions tid, tid + ST, ...; super-group
        // ids thread-major — their order only schedules work)
        int carry;
        {
            int mine = 0;
            for (int q = tid; q < nm; q += ST) mine += mk[q] != 0;
            int k = block_exclusive_scan<ST>(mine, &carry, ssm);
            for (int q = tid; q < nm; q += ST) {
                if (!mk[q]) continue;
                const int e = min(q + SG_MEMBERS, GFIT(MGID(q)));
                a.sglist[s0 + k] = make_int2((int)s0 + q, e - q);
                k++;
            }
        }
        nsg = carry;
    }
    if (tid == 0) sv[3] = atomicAdd(a.sg_total, nsg);     // this pair's slice of the queue
    __syncthreads();
    const int sgbase = sv[3];

    // per super-group: max member-band deviation from the base line (f32 bits rounded
    // up: the strip only has to be a superset), in the J array once the walk is done
    unsigned* sgdevf = reinterpret_cast<unsigned*>(Ja);
    unsigned* sgbl = reinterpret_cast<unsigned*>(Jb);     // base group | first group << 16
    unsigned* sgdelf = reinterpret_cast<unsigned*>(mk);   // max rep deviation (f32 bits; inf: a rep misses)

    // ---------------- super-group shape (base line = middle group's representative)
    for (int ls = tid; ls < nsg; ls += ST) {
        SGRec o = {};
        o.p = p;
        const int2 sgm = a.sglist[s0 + ls];
        o.m0 = sgm.x; o.mcnt = sgm.y;
        const int lg0 = a.stats_mode ? ls : MGID(o.m0 - (int)s0);
        const int lg1 = a.stats_mode ? ls : MGID(o.m0 + o.mcnt - 1 - (int)s0);
        o.g0 = (int)s0 + lg0;
        o.gcnt = lg1 - lg0 + 1;
        o.rlo = a.grp[s0 + (lg0 + lg1) / 2].rep;         // base line's slot (until strips)
        for (int j = 0; j < o.mcnt; j++) {
            if (small) sg16[o.m0 - s0 + j] = (unsigned short)ls;
            else a.msg[o.m0 + j] = ls;
        }
        sgdevf[ls] = 0u;
        sgbl[ls] = (unsigned)((lg0 + lg1) / 2) | ((unsigned)lg0 << 16);
        sgdelf[ls] = 0u;
        a.sg[sgbase + ls] = o;
    }
    __syncthreads();
    if (a.dbg && tid == 0) tmark[4] = clock64();

    // ---------------- members: epilogue constants, band deviations
    for (int k = tid; k < nm; k += ST) {
        const int64_t pos = s0 + k;
        const int lg = MGID(k);
        GroupRec& G = a.grp[s0 + lg];
        const int slot = MSLOT(k);
        const int fid = a.q_fid[slot];
        const int ls = MSG(k);
        const unsigned bl2 = sgbl[ls];
        const GroupRec& GB = a.grp[s0 + (bl2 & 0xffffu)];     // the super-group's base group
        const int g0 = (int)s0 + (int)(bl2 >> 16);
        const float4 lf = a.q_lf[slot];       // the member's line (f32) and |q|^2
        // the member's line in f32 (a singleton's dgemv-rounded line differs from it by
        // an ulp of the f64 value, far inside the fp32 band's error bound eps; the
        // exact fallbacks read the dgemv line from the group record)
        const float mf[3] = {lf.x, lf.y, lf.z};
        // (the group's and the base's rep lines as the f32 copies of their records)
        const float r[3] = {G.ar, G.br, G.cr};
        const float b[3] = {GB.ar, GB.br, GB.cr};
        float rdev, sdev;
        band_deviation2_f(mf, r, b, (float)W, (float)H, (float)d, rdev, sdev);
        const float gdev = rdev + 0.05f;
        // members of a group / super-group sit in consecutive lanes: reduce each run in
        // the warp first, one atomic per run (the shared-memory maxima serialised up to
        // 16 ways per super-group otherwise)
        {
            const unsigned act = __activemask();
            const unsigned below = (1u << lane) - 1u;
            const unsigned mg = __match_any_sync(act, lg);
            const unsigned gmax = __reduce_max_sync(mg, __float_as_uint(gdev));
            if (!(mg & below)) atomicMax(reinterpret_cast<unsigned*>(&G.maxdev), gmax);
            const unsigned ms = __match_any_sync(act, ls);
            const unsigned smax = __reduce_max_sync(ms, __float_as_uint(sdev));
            if (!(ms & below)) atomicMax(&sgdevf[ls], smax);
        }
        MemberRec mr;
        mr.a = mf[0]; mr.b = mf[1]; mr.c = mf[2];
        // fp32 band-value error bound (from the f32 line: the bound's own
        // relative change is ~1e-7, far inside its slack)
        const float eps = (fabsf(mf[0]) * (float)W + fabsf(mf[1]) * (float)H + fabsf(mf[2])) * 0x1p-20f * 1.0001f + 1e-6f;
        mr.lo = (float)d - eps;
        mr.hi = (float)d + eps;
        mr.qn9 = (unsigned)__float_as_int(lf.w) << 9;
        mr.fid = fid;
        mr.slotgi = (int)((unsigned)slot | ((unsigned)(s0 + lg - g0) << SLOT_BITS));
        {
            const int4* w = reinterpret_cast<const int4*>(&mr);
            __stcs(reinterpret_cast<int4*>(a.mrec + pos), w[0]);
            __stcs(reinterpret_cast<int4*>(a.mrec + pos) + 1, w[1]);
        }
    }
    __syncthreads();

    // ---------------- strips.  (a) per (super-group, group) — the first member of each
    // group within its super-group: |dist_g - dist_base| over the strip (atomic max in
    // shared memory) and the group's view (groups shared by two super-groups get the
    // same view twice)
    // Per group: its member run [gm0, gm1) meets at most two super-groups when it has
    // <= 16 members (a super-group opened inside a group runs at least to the group's
    // end), the ones holding its first and last member; longer groups walk their run.
    auto strip_head = [&](int lg, int ls) {
        const GroupRec& G = a.grp[s0 + lg];
        const GroupRec& GB = a.grp[s0 + (sgbl[ls] & 0xffffu)];
        const float R = (float)d + __uint_as_float(sgdevf[ls]) + 0.05f;
        const float bf[3] = {GB.ar, GB.br, GB.cr};
        const float gr[3] = {G.ar, G.br, G.cr};
        const float dlt = (G.K < 0 && a.strategy != 1) ? __int_as_float(0x7f800000)
                                                        : band_deviation_f(bf, gr, (float)W, (float)H, R);
        atomicMax(&sgdelf[ls], __float_as_uint(dlt));
        GView gv;
        if (G.K < 0 && a.strategy != 1) {
            gv.a = 0.f; gv.b = 0.f; gv.c = 1e30f; gv.reach = -1.f;
        } else {
            gv.a = G.ar; gv.b = G.br; gv.c = G.cr; gv.reach = (float)a.d + G.maxdev + 0.05f;
        }
        gv.moff = G.moff; gv.pad0 = gv.pad1 = gv.pad2 = 0;
        const int4* w = reinterpret_cast<const int4*>(&gv);
        __stcs(reinterpret_cast<int4*>(a.gview + s0 + lg), w[0]);
        __stcs(reinterpret_cast<int4*>(a.gview + s0 + lg) + 1, w[1]);
    };
    for (int lg = tid; lg < ng; lg += ST) {
        const int gm0 = a.grec[s0 + lg].z - (int)s0;
        const int gm1 = lg + 1 < ng ? a.grec[s0 + lg + 1].z - (int)s0 : nm;
        if (gm1 <= gm0) continue;
        const int ls0 = MSG(gm0), ls1 = MSG(gm1 - 1);
        if (gm1 - gm0 <= SG_MEMBERS) {
            strip_head(lg, ls0);
            if (ls1 != ls0) strip_head(lg, ls1);
        } else {
            for (int k = gm0; k < gm1; k++)
                if (k == gm0 || MSG(k) != MSG(k - 1)) strip_head(lg, MSG(k));
        }
    }
    __syncthreads();
    // (b) per super-group: strip half-width, sure radius, bucket-row range (sg_prep_kernel
    // of round 1)
    for (int ls = tid; ls < nsg; ls += ST) {
        SGRec o = a.sg[sgbase + ls];
        const double* bl = a.q_line + 3 * (int64_t)o.rlo;
        const double r[3] = {bl[0], bl[1], bl[2]};
        const double R = d + (double)__uint_as_float(sgdevf[ls]) + 0.05;
        const float dlt = __uint_as_float(sgdelf[ls]);
        const bool all_k = !isinf(dlt);
        const double delta = all_k ? (double)dlt : 0.0;
        o.ar = (float)r[0]; o.br = (float)r[1]; o.cr = (float)r[2]; o.R = (float)R;
        // sure-in-C' radius around the base line: grid, the 3x3 subcell block of the
        // nearest sample (half-size D); radial, the disk of radius r around it; both with
        // the sample spacing <= d.  Linear: the rep-line band itself.
        const double DC = a.strategy == 2 ? sqrt(a.r2) : D;
        const double hs2 = DC * DC - 0.25 * d * d;
        const double hs = a.strategy == 1 ? d - 0.05 : (hs2 > 0 ? sqrt(hs2) - 0.075 : -1.0);
        o.hsure = (float)hs;
        o.delta = (all_k || a.strategy == 1) ? (float)(delta + 0.01) : 1e30f;
        o.border = a.strategy == 1 ? -1e30f : (float)(fmax(0.0, hs - d) + 0.05);
        o.invD = (float)(1.0 / D);
        o.W = (float)W; o.H = (float)H; o.pad0 = 0;
        const bool horiz = fabs(r[1]) >= fabs(r[0]);
        o.toff = a.img_off[ti]; o.qoff = qoff;
        o.nalong = horiz ? a.dims[2 * ti] : a.dims[2 * ti + 1];
        o.toffb = horiz ? a.roff[ti] : a.coff[ti];
        o.dbase = db;
        const double al = horiz ? r[0] : r[1], be = horiz ? r[1] : r[0];
        const double Pm = horiz ? W : H, Qm = horiz ? H : W;
        const int nrows = horiz ? a.dims[2 * ti + 1] : a.dims[2 * ti];
        const double qv[4] = {(-R - r[2]) / be, (R - r[2]) / be, (-R - r[2] - al * Pm) / be,
                              (R - r[2] - al * Pm) / be};
        const double qlo = fmin(fmin(qv[0], qv[1]), fmin(qv[2], qv[3]));
        const double qhi = fmax(fmax(qv[0], qv[1]), fmax(qv[2], qv[3]));
        const int rlo = (int)floor((fmax(qlo, 0.0) - 0.01) / D);
        const int rhi = (int)floor((fmin(qhi, Qm) + 0.01) / D);
        o.horiz = horiz;
        o.rlo = rlo < 0 ? 0 : rlo;
        o.rhi = rhi > nrows - 1 ? nrows - 1 : rhi;
        o.alpha = (float)al; o.beta = (float)be;
        o.inv_alpha = fabs(al) > 1e-6 ? (float)(1.0 / al) : 0.f;
        o.Pmax = (float)Pm;
        {
            int4* dst = reinterpret_cast<int4*>(a.sg + sgbase + ls);
            const int4* w = reinterpret_cast<const int4*>(&o);
#pragma unroll
            for (int k = 0; k < 8; k++) __stcs(dst + k, w[k]);
        }
    }
    if (a.dbg) {
        __syncthreads();
        if (tid == 0) {
            const long long t5 = clock64();
            atomicAdd(&a.dbg[11], (unsigned long long)(tmark[1] - tmark[0]));   // lines
            atomicAdd(&a.dbg[12], (unsigned long long)(tmark[2] - tmark[1]));   // groups
            atomicAdd(&a.dbg[13], (unsigned long long)(tmark[3] - tmark[2]));   // scatter + geometry
            atomicAdd(&a.dbg[14], (unsigned long long)(tmark[4] - tmark[3]));   // chain + shape
            atomicAdd(&a.dbg[15], (unsigned long long)(t5 - tmark[4]));         // members + strips
        }
    }
}

// chunk setup: table / dedupe offsets (scan over pairs) and the queue counters
__global__ void plan_kernel(ChunkArgs a) {
    __shared__ int sm[SCAN_T / 32 + 1];
    long long carry_t = 0, carry_d = 0;
    for (int b0 = 0; b0 < a.npairs; b0 += SCAN_T) {
        const int p = b0 + threadIdx.x;
        int ts = 0, nt = 0;
        if (p < a.npairs) {
            const int pg = a.p0 + p;
            const int nq = (int)(a.qlist_off[pg + 1] - a.qlist_off[pg]);
            ts = nextpow2(nq + 1);
            nt = a.img_n[a.pair_t[pg]];
        }
        int tot_t, tot_d;
        const int ex_t = block_exclusive_scan<SCAN_T>(ts, &tot_t, sm);
        const int ex_d = block_exclusive_scan<SCAN_T>(nt, &tot_d, sm);
        if (p < a.npairs) {
            // tables that fit the setup kernel's shared memory take no global slots
            a.tab_off[p] = carry_t + ex_t;
            a.tbase[p] = carry_d + ex_d;
        }
        carry_t += tot_t;
        carry_d += tot_d;
    }
    if (threadIdx.x == 0) {
        a.tab_off[a.npairs] = carry_t;
        a.tbase[a.npairs] = carry_d;
        *a.sg_total = 0;
        *a.sg_next = 0;
    }
}
