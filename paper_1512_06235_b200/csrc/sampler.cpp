// Host-side RANSAC hypothesis generator: the exact draw sequence of
//   rng = np.random.default_rng(seed); rng.choice(n, size=6, replace=False)
// repeated, as msfm.reconstruct.pnp_ransac does (reconstruct.py:185-194).
// numpy 2.x internals restated: PCG64 (XSL-RR 128/64, step-then-output),
// buffered next_uint32, Lemire bounded ints (random_bounded_uint64 with
// use_masked=0), Generator.choice's Floyd branch with a linear-probing hash
// set of size nextpow2(1.2*size), then the in-place Fisher-Yates _shuffle_int.
// The initial state comes from numpy itself (rng.bit_generator.state), so
// SeedSequence is not restated.  Validated draw-for-draw in tests/test_sampler.py.
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

namespace msfm { void set_error(const char* fmt, ...); }

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
