// Native staging of .msft feature files (features.py:98-130): header and size
// validation, bounds check, stable descending-scale order, written straight into
// caller buffers (typically the pinned host bank), many files on host threads.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "msfm_b200.h"

namespace {

constexpr int HEADER_BYTES = 24;          // "<4sIIIII"
constexpr int RECORD_BYTES = 16 + 128;

bool read_file(const char* path, std::vector<uint8_t>& buf) {
    FILE* f = fopen(path, "rb");
    if (!f) return false;
    if (fseek(f, 0, SEEK_END) != 0) { fclose(f); return false; }
    const long n = ftell(f);
    if (n < 0) { fclose(f); return false; }
    rewind(f);
    buf.resize((size_t)n);
    const size_t got = n ? fread(buf.data(), 1, (size_t)n, f) : 0;
    fclose(f);
    return got == (size_t)n;
}

uint32_t le32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

float lef(const uint8_t* p) {
    const uint32_t u = le32(p);
    float f;
    memcpy(&f, &u, 4);
    return f;
}

// header + size checks; info->count etc. filled as far as they are known
int parse_header(const std::vector<uint8_t>& d, msfm_msft_info* info) {
    info->file_bytes = (int64_t)d.size();
    if (d.size() < (size_t)HEADER_BYTES) return info->status = MSFM_MSFT_TRUNCATED;
    memcpy(info->magic, d.data(), 4);
    info->version = le32(d.data() + 4);
    info->image_id = (int32_t)le32(d.data() + 8);
    info->width = (int32_t)le32(d.data() + 12);
    info->height = (int32_t)le32(d.data() + 16);
    info->count = (int64_t)le32(d.data() + 20);
    if (memcmp(info->magic, "MSFT", 4) != 0) return info->status = MSFM_MSFT_BAD_MAGIC;
    if (info->version != 1) return info->status = MSFM_MSFT_BAD_VERSION;
    if ((int64_t)d.size() != HEADER_BYTES + info->count * RECORD_BYTES)
        return info->status = MSFM_MSFT_BAD_SIZE;
    return info->status = MSFM_MSFT_OK;
}

// capacity: records the caller's buffers hold (sized from an earlier header read);
// a file whose count no longer matches is rejected before anything is written
int load_one(const char* path, msfm_msft_info* info, float* xy, float* scale, float* orient,
             uint8_t* desc, int64_t capacity) {
    memset(info, 0, sizeof(*info));
    info->bad_record = -1;
    std::vector<uint8_t> d;
    if (!read_file(path, d)) return info->status = MSFM_MSFT_IO;
    if (parse_header(d, info) != MSFM_MSFT_OK) return info->status;
    if (!xy) return info->status;          // header probe only
    const int64_t n = info->count;
    if (n != capacity) return info->status = MSFM_MSFT_CHANGED;
    const uint8_t* rec = d.data() + HEADER_BYTES;
    // the reference's bounds test (x < 0 | x >= w | y < 0 | y >= h | scale <= 0), first hit
    const float W = (float)info->width, H = (float)info->height;
    for (int64_t i = 0; i < n; i++) {
        const uint8_t* r = rec + i * RECORD_BYTES;
        const float x = lef(r), y = lef(r + 4), s = lef(r + 8);
        if (x < 0.f || x >= W || y < 0.f || y >= H || s <= 0.f) {
            info->bad_record = i;
            info->bad_x = x; info->bad_y = y; info->bad_scale = s;
            return info->status = MSFM_MSFT_BOUNDS;
        }
    }
    // np.argsort(-scale, kind="stable"): descending scale, ties in file order, NaN last
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; i++) order[(size_t)i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        const float sa = lef(rec + a * RECORD_BYTES + 8), sb = lef(rec + b * RECORD_BYTES + 8);
        if (isnan(sa)) return false;
        if (isnan(sb)) return true;
        return sa > sb;
    });
    for (int64_t k = 0; k < n; k++) {
        const uint8_t* r = rec + order[(size_t)k] * RECORD_BYTES;
        xy[2 * k] = lef(r);
        xy[2 * k + 1] = lef(r + 4);
        if (scale) scale[k] = lef(r + 8);
        if (orient) orient[k] = lef(r + 12);
        memcpy(desc + k * 128, r + 16, 128);
    }
    return info->status;
}

}  // namespace

extern "C" int msfm_msft_load(const char* path, msfm_msft_info* info, float* xy, float* scale,
                              float* orientation, uint8_t* desc, int64_t capacity) {
    if (!path || !info) return MSFM_EINVAL;
    load_one(path, info, xy, scale, orientation, desc, capacity);
    return MSFM_OK;
}

extern "C" int msfm_msft_load_many(int32_t n_files, const char* const* paths, const int64_t* row_off,
                                   msfm_msft_info* infos, float* xy, float* scale,
                                   float* orientation, uint8_t* desc, int32_t n_threads) {
    if (n_files < 0 || (n_files > 0 && (!paths || !row_off || !infos || !xy || !desc)))
        return MSFM_EINVAL;
    const int T = std::max(1, std::min<int>(n_threads > 0 ? n_threads : 1, n_files > 0 ? n_files : 1));
    std::atomic<int> next(0);
    auto work = [&]() {
        for (int i = next++; i < n_files; i = next++) {
            const int64_t o = row_off[i];
            load_one(paths[i], infos + i, xy + 2 * o, scale ? scale + o : nullptr,
                     orientation ? orientation + o : nullptr, desc + 128 * o, row_off[i + 1] - o);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; t++) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    return MSFM_OK;
}
