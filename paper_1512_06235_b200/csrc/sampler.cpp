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

#include "rng.cuh"
using namespace msfm_rng;

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
