// Host-side RANSAC hypothesis generator: the exact draw sequence of
//   rng = np.random.default_rng(seed); rng.choice(n, size=6, replace=False)
// repeated, as msfm.reconstruct.pnp_ransac does (reconstruct.py:185-194).
// numpy 2.x internals restated: PCG64 (XSL-RR 128/64, step-then-output),
// buffered next_uint32, Lemire bounded ints (random_bounded_uint64 with
// use_masked=0), Generator.choice's Floyd branch with a linear-probing hash
// set of size nextpow2(1.2*size), then the in-place Fisher-Yates _shuffle_int.
// The initial state is either numpy's own (rng.bit_generator.state) or, for the
// batched entry, numpy's SeedSequence(seed) -> PCG64 seeding restated below
// (bit_generator.pyx hashmix/mix/generate_state, pcg64_set_seed).  Validated
// draw-for-draw and state-for-state in tests/test_sampler.py.
#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>
#include <stdint.h>
#include <string.h>

#include "msfm_b200.h"

namespace {
typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
    int has32;
    uint32_t u32;
    uint64_t next64() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
        state = state * mult + inc;
        uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        unsigned rot = (unsigned)(hi >> 58);
        uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    uint32_t next32() {
        if (has32) {
            has32 = 0;
            return u32;
        }
        uint64_t n = next64();
        has32 = 1;
        u32 = (uint32_t)(n >> 32);
        return (uint32_t)(n & 0xffffffffu);
    }
    // random_bounded_uint64(off=0, rng, mask=0, use_masked=0)
    uint64_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng <= 0xFFFFFFFFULL) {
            if (rng == 0xFFFFFFFFULL) return next32();
            const uint32_t r = (uint32_t)rng, rexcl = r + 1;
            uint64_t m = (uint64_t)next32() * rexcl;
            uint32_t left = (uint32_t)m;
            if (left < rexcl) {
                const uint32_t thr = (UINT32_MAX - r) % rexcl;
                while (left < thr) {
                    m = (uint64_t)next32() * rexcl;
                    left = (uint32_t)m;
                }
            }
            return m >> 32;
        }
        // 64-bit Lemire (ranges beyond 2^32 never occur for pnp sample sizes)
        const uint64_t rexcl = rng + 1;
        u128 m = (u128)next64() * rexcl;
        uint64_t left = (uint64_t)m;
        if (left < rexcl) {
            const uint64_t thr = (UINT64_MAX - rng) % rexcl;
            while (left < thr) {
                m = (u128)next64() * rexcl;
                left = (uint64_t)m;
            }
        }
        return (uint64_t)(m >> 64);
    }
};

uint64_t gen_mask(uint64_t v) {
    v |= v >> 1; v |= v >> 2; v |= v >> 4; v |= v >> 8; v |= v >> 16; v |= v >> 32;
    return v;
}

// Generator.choice(pop, size, replace=False, shuffle=True), Floyd branch
bool choice_floyd(Pcg64& g, int64_t pop, int size, int64_t* out) {
    if (pop > 10000 && size > pop / 50) return false;  // tail-shuffle branch: not restated
    uint64_t set_size = (uint64_t)(1.2 * size);
    const uint64_t mask = gen_mask(set_size);
    set_size = mask + 1;
    uint64_t hs[64];
    if (set_size > 64) return false;
    for (uint64_t i = 0; i < set_size; i++) hs[i] = ~0ULL;
    for (int64_t j = pop - size; j < pop; j++) {
        uint64_t val = g.bounded((uint64_t)j);
        uint64_t loc = val & mask;
        while (hs[loc] != ~0ULL && hs[loc] != val) loc = (loc + 1) & mask;
        if (hs[loc] == ~0ULL) {
            hs[loc] = val;
            out[j - pop + size] = (int64_t)val;
        } else {
            loc = (uint64_t)j & mask;
            while (hs[loc] != ~0ULL) loc = (loc + 1) & mask;
            hs[loc] = (uint64_t)j;
            out[j - pop + size] = j;
        }
    }
    // _shuffle_int(size, first=1): for i in reversed(range(1, size))
    for (int64_t i = size - 1; i >= 1; i--) {
        int64_t k = (int64_t)g.bounded((uint64_t)i);
        int64_t tmp = out[k];
        out[k] = out[i];
        out[i] = tmp;
    }
    return true;
}
}  // namespace

namespace {
// numpy SeedSequence (bit_generator.pyx), pool size 4, 32-bit words
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;

inline uint32_t hashmix(uint32_t value, uint32_t& hash_const) {
    value ^= hash_const;
    hash_const *= MULT_A;
    value *= hash_const;
    value ^= value >> 16;
    return value;
}

inline uint32_t mixw(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> 16;
    return r;
}

// PCG64 state of np.random.default_rng(seed) for 0 <= seed < 2^64
void seed_pcg64(uint64_t seed, Pcg64& g) {
    uint32_t ent[2];
    int ne = 0;
    if (seed == 0) ent[ne++] = 0;
    while (seed > 0) { ent[ne++] = (uint32_t)(seed & 0xffffffffu); seed >>= 32; }
    uint32_t pool[4];
    uint32_t hc = INIT_A;
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < ne ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
    // generate_state(4, uint64): 8 words, cycling the pool
    uint32_t w[8];
    uint32_t hb = INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    uint64_t v64[4];
    for (int i = 0; i < 4; i++) v64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const u128 initstate = ((u128)v64[0] << 64) | v64[1];
    const u128 initseq = ((u128)v64[2] << 64) | v64[3];
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    g.state = 0;
    g.inc = (initseq << 1) | 1u;
    g.state = g.state * mult + g.inc;
    g.state += initstate;
    g.state = g.state * mult + g.inc;
    g.has32 = 0;
    g.u32 = 0;
}
}  // namespace

namespace msfm { void set_error(const char* fmt, ...); }

extern "C" int msfm_rng_seed_state(uint64_t seed, uint64_t state_out[6]) {
    if (!state_out) return MSFM_EINVAL;
    Pcg64 g;
    seed_pcg64(seed, g);
    state_out[0] = (uint64_t)(g.state >> 64);
    state_out[1] = (uint64_t)g.state;
    state_out[2] = (uint64_t)(g.inc >> 64);
    state_out[3] = (uint64_t)g.inc;
    state_out[4] = 0;
    state_out[5] = 0;
    return MSFM_OK;
}

extern "C" int msfm_ransac_samples_seeded(int32_t n_items, const uint64_t* seeds, const int64_t* n,
                                          int32_t sample_size, int32_t count, int32_t* out,
                                          uint64_t* state_out) {
    if (n_items < 0 || !seeds || !n || !out || sample_size < 1 || sample_size > 48 || count < 0) {
        msfm::set_error("msfm_ransac_samples_seeded: bad arguments");
        return MSFM_EINVAL;
    }
    for (int32_t it = 0; it < n_items; it++) {
        if (n[it] < sample_size) {
            msfm::set_error("msfm_ransac_samples_seeded: item %d has %lld < %d rows", it,
                            (long long)n[it], sample_size);
            return MSFM_EINVAL;
        }
    }
    // items are independent streams: host threads over items (output order fixed)
    std::atomic<int32_t> next{0};
    std::atomic<int64_t> bad_n{-1};
    auto work = [&]() {
        int64_t tmp[48];
        for (;;) {
            const int32_t it = next.fetch_add(1);
            if (it >= n_items) return;
            Pcg64 g;
            seed_pcg64(seeds[it], g);
            int32_t* o = out + (int64_t)it * count * sample_size;
            for (int32_t h = 0; h < count; h++) {
                if (!choice_floyd(g, n[it], sample_size, tmp)) {
                    bad_n.store(n[it]);
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
    };
    const int64_t draws = (int64_t)n_items * count;
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 16);
    nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, draws / 2048));
    nt = std::min(nt, std::max(n_items, 1));
    std::vector<std::thread> pool;
    for (int k = 1; k < nt; k++) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (bad_n.load() >= 0) {
        msfm::set_error("msfm_ransac_samples_seeded: population %lld outside the Floyd branch",
                        (long long)bad_n.load());
        return MSFM_EINVAL;
    }
    return MSFM_OK;
}

extern "C" int msfm_ransac_samples(const uint64_t state_inc[4], int32_t has_uint32,
                                   uint32_t uinteger, int64_t n, int32_t sample_size,
                                   int32_t count, int32_t* out, uint64_t state_out[6]) {
    if (!state_inc || !out || n < sample_size || sample_size < 1 || sample_size > 48 || count < 0) {
        msfm::set_error("msfm_ransac_samples: bad arguments (n=%lld, size=%d)", (long long)n,
                        sample_size);
        return MSFM_EINVAL;
    }
    Pcg64 g;
    g.state = ((u128)state_inc[0] << 64) | state_inc[1];
    g.inc = ((u128)state_inc[2] << 64) | state_inc[3];
    g.has32 = has_uint32 ? 1 : 0;
    g.u32 = uinteger;
    int64_t tmp[48];
    for (int32_t h = 0; h < count; h++) {
        if (!choice_floyd(g, n, sample_size, tmp)) {
            msfm::set_error("msfm_ransac_samples: population %lld outside the Floyd branch",
                            (long long)n);
            return MSFM_EINVAL;
        }
        for (int k = 0; k < sample_size; k++) out[(int64_t)h * sample_size + k] = (int32_t)tmp[k];
    }
    if (state_out) {
        state_out[0] = (uint64_t)(g.state >> 64);
        state_out[1] = (uint64_t)g.state;
        state_out[2] = (uint64_t)(g.inc >> 64);
        state_out[3] = (uint64_t)g.inc;
        state_out[4] = (uint64_t)g.has32;
        state_out[5] = (uint64_t)g.u32;
    }
    return MSFM_OK;
}
