// numpy 2.x Generator internals used by the RANSAC samplers, restated once for the
// host (sampler.cpp) and the device (pnp.cu): PCG64 (XSL-RR 128/64, step then
// output), buffered next_uint32, Lemire bounded ints (random_bounded_uint64,
// use_masked=0), Generator.choice's Floyd branch + _shuffle_int, and the
// SeedSequence(seed) -> PCG64 seeding of np.random.default_rng (bit_generator.pyx).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define MSFM_HD __host__ __device__ __forceinline__
#else
#define MSFM_HD inline
#endif

namespace msfm_rng {
typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
    int has32;
    uint32_t u32;
    MSFM_HD uint64_t next64() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
        state = state * mult + inc;
        uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        unsigned rot = (unsigned)(hi >> 58);
        uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    MSFM_HD uint32_t next32() {
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
    MSFM_HD uint64_t bounded(uint64_t rng) {
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

MSFM_HD uint64_t gen_mask(uint64_t v) {
    v |= v >> 1; v |= v >> 2; v |= v >> 4; v |= v >> 8; v |= v >> 16; v |= v >> 32;
    return v;
}

// Generator.choice(pop, size, replace=False, shuffle=True), Floyd branch
MSFM_HD bool choice_floyd(Pcg64& g, int64_t pop, int size, int64_t* out) {
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
// numpy SeedSequence (bit_generator.pyx), pool size 4, 32-bit words
static constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
static constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
static constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;

MSFM_HD uint32_t hashmix(uint32_t value, uint32_t& hash_const) {
    value ^= hash_const;
    hash_const *= MULT_A;
    value *= hash_const;
    value ^= value >> 16;
    return value;
}

MSFM_HD uint32_t mixw(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> 16;
    return r;
}

// PCG64 state of np.random.default_rng(seed) for 0 <= seed < 2^64
MSFM_HD void seed_pcg64(uint64_t seed, Pcg64& g) {
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
// numpy's pcg64_advance (pcg_advance_lcg_128): the LCG state `delta` steps later
MSFM_HD u128 pcg_advance(u128 state, u128 delta, u128 inc) {
    u128 cur_mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    u128 cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

// A generator positioned at 32-bit draw `i` of the stream that starts at (state0,
// inc) with no buffered half: draw i is the low half of 64-bit output i/2 when i
// is even, the high half of output (i-1)/2 when odd; output m comes from the state
// advanced m+1 steps (step, then output).
MSFM_HD void pcg_at_draw(u128 state0, u128 inc, uint64_t i, Pcg64& g) {
    g.inc = inc;
    if ((i & 1) == 0) {
        g.state = pcg_advance(state0, (u128)(i / 2), inc);
        g.has32 = 0;
        g.u32 = 0;
    } else {
        g.state = pcg_advance(state0, (u128)((i - 1) / 2 + 1), inc);
        const uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
        const unsigned rot = (unsigned)(hi >> 58);
        const uint64_t x = hi ^ lo;
        const uint64_t o = (x >> rot) | (x << ((64 - rot) & 63));
        g.has32 = 1;
        g.u32 = (uint32_t)(o >> 32);
    }
}

// Pcg64::bounded for ranges below 2^32 - 1 drawing exactly one 32-bit value; sets
// `rej` where Lemire's method would reject and draw again (probability ~ rng/2^32)
MSFM_HD uint64_t bounded_once(Pcg64& g, uint64_t rng, bool& rej) {
    if (rng == 0) return 0;
    const uint32_t r = (uint32_t)rng, rexcl = r + 1;
    const uint64_t m = (uint64_t)g.next32() * rexcl;
    const uint32_t left = (uint32_t)m;
    if (left < rexcl && left < (UINT32_MAX - r) % rexcl) rej = true;
    return m >> 32;
}

// choice_floyd drawing one value per bounded call with a non-zero range;
// `rej` flags a draw the sequential stream would have repeated
MSFM_HD void choice_floyd_once(Pcg64& g, int64_t pop, int size, int64_t* out, bool& rej) {
    uint64_t set_size = (uint64_t)(1.2 * size);
    const uint64_t mask = gen_mask(set_size);
    uint64_t hs[64];
    for (uint64_t i = 0; i <= mask; i++) hs[i] = ~0ULL;
    for (int64_t j = pop - size; j < pop; j++) {
        uint64_t val = bounded_once(g, (uint64_t)j, rej);
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
    for (int64_t i = size - 1; i >= 1; i--) {
        int64_t k = (int64_t)bounded_once(g, (uint64_t)i, rej);
        int64_t tmp = out[k];
        out[k] = out[i];
        out[i] = tmp;
    }
}
}  // namespace msfm_rng
