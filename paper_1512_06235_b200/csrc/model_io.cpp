// Host-only native reader of the reference's model snapshot (.msfm text,
// msfm.io.read_model io.py:51-84) straight into the CSR arrays the device stages
// consume (cameras + point positions + track CSR), with the reference's record
// validation and Model rules (model.py:114-156: duplicate registration, tracks of
// >= 2 distinct registered images, one owner per feature) reported as a status,
// the offending line and the reference's message text.
//
// Two calls: a probe (buffers NULL) returns the counts; the fill call checks them
// against the caller's capacities before writing (MSFM_MODEL_CHANGED otherwise).
#include <ctype.h>
#include <errno.h>
#include <stdarg.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "msfm_b200.h"

namespace {

bool read_file(const char* path, std::string& out) {
    FILE* f = fopen(path, "rb");
    if (!f) return false;
    char buf[1 << 16];
    size_t k;
    while ((k = fread(buf, 1, sizeof(buf), f)) > 0) out.append(buf, k);
    const bool ok = !ferror(f);
    fclose(f);
    return ok;
}

// Python str.split(): runs of whitespace separate, no empty tokens
void split_ws(const char* a, const char* b, std::vector<std::string>& out) {
    out.clear();
    while (a < b) {
        while (a < b && isspace((unsigned char)*a)) a++;
        const char* s = a;
        while (a < b && !isspace((unsigned char)*a)) a++;
        if (a > s) out.emplace_back(s, a - s);
    }
}

// Python's int() / float() accept '_' between digits
bool strip_underscores(const std::string& t, std::string& o) {
    o.clear();
    for (size_t i = 0; i < t.size(); i++) {
        if (t[i] == '_') {
            if (i == 0 || i + 1 == t.size() || !isdigit((unsigned char)t[i - 1]) ||
                !isdigit((unsigned char)t[i + 1]))
                return false;
            continue;
        }
        o.push_back(t[i]);
    }
    return true;
}

bool py_int(const std::string& t, long long& v) {
    std::string s;
    if (!strip_underscores(t, s) || s.empty()) return false;
    size_t i = 0;
    if (s[0] == '+' || s[0] == '-') i = 1;
    if (i == s.size()) return false;
    for (size_t k = i; k < s.size(); k++)
        if (!isdigit((unsigned char)s[k])) return false;
    errno = 0;
    v = strtoll(s.c_str(), nullptr, 10);
    return errno == 0;
}

bool py_float(const std::string& t, double& v) {
    std::string s;
    if (!strip_underscores(t, s) || s.empty()) return false;
    // reject hex floats and other strtod extensions Python's float() refuses
    for (char c : s)
        if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
    char* end = nullptr;
    v = strtod(s.c_str(), &end);
    return end == s.c_str() + s.size();
}

struct Reader {
    msfm_model_info* info;
    void fail(int status, int line, const char* fmt, ...) __attribute__((format(printf, 4, 5))) {
        info->status = status;
        info->line = line;
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(info->message, sizeof(info->message), fmt, ap);
        va_end(ap);
    }
};

}  // namespace

extern "C" int msfm_model_read(const char* path, msfm_model_info* info, int32_t* cam_id,
                               double* cam_fcc, double* cam_R, double* cam_t, int32_t* cam_line,
                               double* pt_xyz, int64_t* track_ptr, int32_t* track_img,
                               int32_t* track_fid, int32_t* pt_line, int64_t cap_cams,
                               int64_t cap_points, int64_t cap_obs) {
    if (!path || !info) return MSFM_EINVAL;
    memset(info, 0, sizeof(*info));
    Reader rd{info};
    std::string text;
    if (!read_file(path, text)) {
        info->status = MSFM_MODEL_IO;
        return MSFM_OK;
    }
    const bool fill = cam_id != nullptr;
    std::vector<std::string> tok;
    // splitlines(): \n, \r\n, \r (and a few rarer separators, not written by write_model)
    std::vector<std::pair<const char*, const char*>> lines;
    {
        const char* p = text.data();
        const char* e = p + text.size();
        while (p < e) {
            const char* s = p;
            while (p < e && *p != '\n' && *p != '\r') p++;
            lines.emplace_back(s, p);
            if (p < e && *p == '\r' && p + 1 < e && p[1] == '\n') p += 2;
            else if (p < e) p++;
        }
    }
    // header: text[0].strip() == "MSFM-MODEL 1"
    bool head_ok = false;
    if (!lines.empty()) {
        const char* a = lines[0].first;
        const char* b = lines[0].second;
        while (a < b && isspace((unsigned char)*a)) a++;
        while (b > a && isspace((unsigned char)b[-1])) b--;
        head_ok = std::string(a, b) == "MSFM-MODEL 1";
    }
    if (!head_ok) {
        rd.fail(MSFM_MODEL_HEADER, 1, "missing 'MSFM-MODEL 1' header");
        return MSFM_OK;
    }
    std::unordered_set<long long> registered;
    std::unordered_map<unsigned long long, long long>* owner_map = nullptr;
    long long n_cams = 0, n_pts = 0, n_obs = 0;
    std::string stage;
    // owner point id per feature for the reference's "already belongs to point p"
    std::unordered_map<unsigned long long, long long> owners;
    owner_map = &owners;
    std::vector<long long> imgs;
    std::vector<long long> fids;
    for (size_t li = 1; li < lines.size(); li++) {
        const int lineno = (int)li + 1;
        split_ws(lines[li].first, lines[li].second, tok);
        if (tok.empty()) continue;
        const std::string& kind = tok[0];
        if (kind == "STAGE") {
            stage = tok.size() > 1 ? tok[1] : "";
        } else if (kind == "CAM") {
            long long id;
            if (tok.size() < 2) { rd.fail(MSFM_MODEL_RECORD, lineno, "list index out of range"); return MSFM_OK; }
            if (!py_int(tok[1], id)) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "invalid literal for int() with base 10: '%s'", tok[1].c_str());
                return MSFM_OK;
            }
            double v[15];
            int nv = 0;
            for (size_t k = 2; k < tok.size() && k < 17; k++) {
                if (!py_float(tok[k], v[nv])) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "could not convert string to float: '%s'",
                            tok[k].c_str());
                    return MSFM_OK;
                }
                nv++;
            }
            if (nv < 3) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "not enough values to unpack (expected 3, got %d)", nv);
                return MSFM_OK;
            }
            if (nv < 12) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "cannot reshape array of size %d into shape (3,3)", nv - 3);
                return MSFM_OK;
            }
            if (nv < 15) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "cannot reshape array of size %d into shape (3,)", nv - 12);
                return MSFM_OK;
            }
            const double* R = v + 3;
            const double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                               R[2] * (R[3] * R[7] - R[4] * R[6]);
            if (fabs(det - 1.0) > 1e-9) {
                // Camera.__post_init__ (model.py:38-39); numpy's det (LU) rounds differently
                // from this cofactor sum only ~1e-16 away from the 1e-9 gate
                rd.fail(MSFM_MODEL_DET, lineno, "camera %lld: det(R)", id);
                info->value = det;
                info->value_id = id;
                return MSFM_OK;
            }
            if (registered.count(id)) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "image %lld already registered", id);
                return MSFM_OK;
            }
            registered.insert(id);
            if (fill) {
                if (n_cams >= cap_cams) { info->status = MSFM_MODEL_CHANGED; return MSFM_OK; }
                cam_id[n_cams] = (int32_t)id;
                for (int k = 0; k < 3; k++) cam_fcc[3 * n_cams + k] = v[k];
                for (int k = 0; k < 9; k++) cam_R[9 * n_cams + k] = v[3 + k];
                for (int k = 0; k < 3; k++) cam_t[3 * n_cams + k] = v[12 + k];
                cam_line[n_cams] = lineno;
            }
            n_cams++;
        } else if (kind == "PT") {
            double pos[3];
            int np = 0;
            for (size_t k = 1; k < tok.size() && k < 4; k++) {
                if (!py_float(tok[k], pos[np])) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "could not convert string to float: '%s'",
                            tok[k].c_str());
                    return MSFM_OK;
                }
                np++;
            }
            if (tok.size() < 5) { rd.fail(MSFM_MODEL_RECORD, lineno, "list index out of range"); return MSFM_OK; }
            long long n;
            if (!py_int(tok[4], n)) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "invalid literal for int() with base 10: '%s'", tok[4].c_str());
                return MSFM_OK;
            }
            imgs.clear();
            fids.clear();
            for (long long k = 0; k < n; k++) {
                if ((size_t)(6 + 2 * k) >= tok.size()) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "list index out of range");
                    return MSFM_OK;
                }
                long long im, fi;
                if (!py_int(tok[5 + 2 * k], im)) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "invalid literal for int() with base 10: '%s'",
                            tok[5 + 2 * k].c_str());
                    return MSFM_OK;
                }
                if (!py_int(tok[6 + 2 * k], fi)) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "invalid literal for int() with base 10: '%s'",
                            tok[6 + 2 * k].c_str());
                    return MSFM_OK;
                }
                imgs.push_back(im);
                fids.push_back(fi);
            }
            // Model.add_point (model.py:140-156)
            std::unordered_set<long long> distinct(imgs.begin(), imgs.end());
            if (imgs.size() < 2 || distinct.size() < imgs.size()) {
                rd.fail(MSFM_MODEL_RECORD, lineno, "a track needs >= 2 features from distinct images");
                return MSFM_OK;
            }
            for (size_t k = 0; k < imgs.size(); k++) {
                if (!registered.count(imgs[k])) {
                    rd.fail(MSFM_MODEL_RECORD, lineno, "image %lld is not registered", imgs[k]);
                    return MSFM_OK;
                }
                const unsigned long long key = ((unsigned long long)(uint32_t)imgs[k] << 32) | (unsigned long long)(uint32_t)fids[k];
                auto it = owner_map->find(key);
                if (it != owner_map->end()) {
                    rd.fail(MSFM_MODEL_RECORD, lineno,
                            "FeatureRef(image_id=%lld, feature_id=%lld) already belongs to point %lld",
                            imgs[k], fids[k], it->second);
                    return MSFM_OK;
                }
            }
            if (np < 3) {
                // np.asarray(position) of < 3 values is accepted by add_point itself; the
                // reference stores it as is, which no stage can use: reject it here
                rd.fail(MSFM_MODEL_POSITION, lineno, "point position has %d coordinates", np);
                return MSFM_OK;
            }
            for (size_t k = 0; k < imgs.size(); k++) {
                const unsigned long long key = ((unsigned long long)(uint32_t)imgs[k] << 32) | (unsigned long long)(uint32_t)fids[k];
                (*owner_map)[key] = n_pts;
            }
            if (fill) {
                if (n_pts >= cap_points || n_obs + (long long)imgs.size() > cap_obs) {
                    info->status = MSFM_MODEL_CHANGED;
                    return MSFM_OK;
                }
                for (int k = 0; k < 3; k++) pt_xyz[3 * n_pts + k] = pos[k];
                track_ptr[n_pts] = n_obs;
                for (size_t k = 0; k < imgs.size(); k++) {
                    track_img[n_obs + k] = (int32_t)imgs[k];
                    track_fid[n_obs + k] = (int32_t)fids[k];
                }
                pt_line[n_pts] = lineno;
            }
            n_pts++;
            n_obs += (long long)imgs.size();
        } else {
            rd.fail(MSFM_MODEL_RECORD, lineno, "unknown record '%s'", kind.c_str());
            // the reference re-raises this FormatError without the wrapping below
            info->status = MSFM_MODEL_UNKNOWN;
            return MSFM_OK;
        }
    }
    if (fill) {
        if (n_cams != cap_cams || n_pts != cap_points || n_obs != cap_obs) {
            info->status = MSFM_MODEL_CHANGED;
            return MSFM_OK;
        }
        track_ptr[n_pts] = n_obs;
    }
    info->n_cams = n_cams;
    info->n_points = n_pts;
    info->n_obs = n_obs;
    snprintf(info->stage, sizeof(info->stage), "%s", stage.c_str());
    info->stage_truncated = stage.size() >= sizeof(info->stage);
    return MSFM_OK;
}
