// Track merge of the densification stage (densify.py:68-158) on the device.
//
// Nodes are bank feature rows; the bank holds its images in ascending image id,
// so node order equals the reference's (image << 32 | feature) key order.  One
// stage's matches are the edges; the model tracks that touch them are unioned in
// as well (every point's refs are unioned: untouched points end up alone in
// their own component and produce nothing).  Per component (root = smallest
// node, i.e. the reference's `min` key):
//   - two or more owning points: ambiguous bridge, dropped;
//   - per image: the owner's own refs are kept (not fresh) and other nodes of
//     that image dropped; otherwise the node with the smallest (support, key)
//     is kept, support = its smallest incident match distance;
//   - owner present: the kept fresh nodes extend it; no owner: a new track when
//     at least two images remain.
// Output: fresh nodes grouped by component in ascending root order, ascending
// within a component, plus one segment (owner or -1, offset) per component.
#include <stdint.h>

#include "common.cuh"
#include "scan.cuh"

namespace msfm {
namespace {

constexpr uint32_t NO_SUPPORT = 0xffffffffu;
constexpr unsigned long long EMPTY_KEY = ~0ull;

struct MergeArgs {
    int64_t n_nodes, n_edges;
    const int32_t* u; const int32_t* v; const float* dist;
    int32_t n_points; const int64_t* tptr; const int32_t* tnode;
    const int64_t* img_off; int32_t n_images;
    int32_t* parent; int32_t* root; uint32_t* support; int32_t* owner; int32_t* conflict;
    int32_t* fresh_cnt; int32_t* fresh; int32_t* seg_idx; int32_t* seg_off; int32_t* fill;
    unsigned long long* hkey; unsigned long long* hval; int64_t hmask;
    int32_t* out_node; int32_t* seg_owner; int64_t* seg_off_out; int64_t* counts;
    int32_t* tmp_node;           // scratch for the segment sort (touched_bound)
};

__device__ __forceinline__ int find_root(int32_t* parent, int x) {
    int p = __ldcg(parent + x);
    while (p != x) {
        const int gp = __ldcg(parent + p);
        if (gp != p) parent[x] = gp;     // path halving (benign race: gp is an ancestor)
        x = p;
        p = __ldcg(parent + x);
    }
    return x;
}

// link the larger root under the smaller one, so every root is its component's
// smallest node
__device__ void unite(int32_t* parent, int a, int b) {
    while (true) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicCAS(parent + b, b, a);
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ int image_of(const MergeArgs& a, int node) {
    int lo = 0, hi = a.n_images - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.img_off[mid] <= node) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void merge_init_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        a.parent[i] = (int32_t)i;
        a.support[i] = NO_SUPPORT;
        a.owner[i] = -1;
        a.conflict[i] = 0;
        a.fresh_cnt[i] = 0;
        a.fresh[i] = 0;
        a.fill[i] = 0;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= a.hmask;
         i += (int64_t)gridDim.x * blockDim.x) {
        a.hkey[i] = EMPTY_KEY;
        a.hval[i] = EMPTY_KEY;
    }
}

__global__ void merge_edges_kernel(MergeArgs a) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n_edges;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int u = a.u[e], v = a.v[e];
        const uint32_t d = __float_as_uint(a.dist[e]);   // >= 0: bit order = value order
        atomicMin(a.support + u, d);
        atomicMin(a.support + v, d);
        unite(a.parent, u, v);
    }
}

__global__ void merge_tracks_kernel(MergeArgs a) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.n_points) return;
    const int64_t b = a.tptr[p], e = a.tptr[p + 1];
    for (int64_t j = b + 1; j < e; j++) unite(a.parent, a.tnode[b], a.tnode[j]);
}

// roots into their own array: path-halving stores of concurrent finds could
// overwrite an in-place compression with an intermediate ancestor
__global__ void merge_compress_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x)
        a.root[i] = find_root(a.parent, (int)i);
}

// owning point of every component; a second distinct owner marks a bridge
__global__ void merge_owner_kernel(MergeArgs a) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.n_points) return;
    const int64_t b = a.tptr[p], e = a.tptr[p + 1];
    if (b == e) return;
    const int c = a.root[a.tnode[b]];
    const int old = atomicCAS(a.owner + c, -1, p);
    if (old != -1 && old != p) a.conflict[c] = 1;
}

// true if node i competes for its (component, image) slot
__device__ __forceinline__ bool contender(const MergeArgs& a, int i, int& c, int& img) {
    if (a.support[i] == NO_SUPPORT) return false;       // not a matched node
    c = a.root[i];
    if (a.conflict[c]) return false;
    img = image_of(a, i);
    const int o = a.owner[c];
    if (o >= 0) {
        // an image holding one of the owner's refs keeps those refs only
        for (int64_t j = a.tptr[o]; j < a.tptr[o + 1]; j++)
            if (image_of(a, a.tnode[j]) == img) return false;
    }
    return true;
}

__device__ __forceinline__ int64_t slot_of(const MergeArgs& a, unsigned long long key, bool insert) {
    int64_t h = (int64_t)(mix64(key) & (unsigned long long)a.hmask);
    while (true) {
        const unsigned long long k = a.hkey[h];
        if (k == key) return h;
        if (k == EMPTY_KEY) {
            if (!insert) return -1;
            const unsigned long long old = atomicCAS(a.hkey + h, EMPTY_KEY, key);
            if (old == EMPTY_KEY || old == key) return h;
        }
        h = (h + 1) & a.hmask;
    }
}

__global__ void merge_select_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c, img;
        if (!contender(a, (int)i, c, img)) continue;
        const unsigned long long key = ((unsigned long long)(uint32_t)c << 16) | (uint32_t)img;
        const int64_t h = slot_of(a, key, true);
        atomicMin(a.hval + h, ((unsigned long long)a.support[i] << 32) | (uint32_t)i);
    }
}

__global__ void merge_winner_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c, img;
        if (!contender(a, (int)i, c, img)) continue;
        const unsigned long long key = ((unsigned long long)(uint32_t)c << 16) | (uint32_t)img;
        const int64_t h = slot_of(a, key, false);
        if (a.hval[h] == (((unsigned long long)a.support[i] << 32) | (uint32_t)i)) {
            a.fresh[i] = 1;
            atomicAdd(a.fresh_cnt + c, 1);
        }
    }
}

// per root: emits a segment?  seg_idx <- 0/1, seg_off <- fresh count (scanned next)
__global__ void merge_flag_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool root = a.root[i] == (int32_t)i;
        const int f = a.fresh_cnt[i];
        const bool seg = root && !a.conflict[i] && (a.owner[i] >= 0 ? f >= 1 : f >= 2);
        a.seg_idx[i] = seg ? 1 : 0;
        a.seg_off[i] = seg ? f : 0;
    }
}

__global__ void merge_emit_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n_nodes;
         i += (int64_t)gridDim.x * blockDim.x) {
        // segment table (roots that emit)
        const bool root = a.root[i] == (int32_t)i;
        const int f = a.fresh_cnt[i];
        const bool seg = root && !a.conflict[i] && (a.owner[i] >= 0 ? f >= 1 : f >= 2);
        if (seg) {
            const int s = a.seg_idx[i];
            a.seg_owner[s] = a.owner[i];
            a.seg_off_out[s] = a.seg_off[i];
        }
        // fresh nodes of emitting components
        if (a.fresh[i]) {
            const int c = a.root[i];
            const int fc = a.fresh_cnt[c];
            const bool cseg = !a.conflict[c] && (a.owner[c] >= 0 ? fc >= 1 : fc >= 2);
            if (cseg) a.out_node[a.seg_off[c] + atomicAdd(a.fill + c, 1)] = (int32_t)i;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // totals: the scans are exclusive, add the last element back
        const int64_t n = a.n_nodes;
        const int last = (int)(n - 1);
        const bool root = a.root[last] == last;
        const int f = a.fresh_cnt[last];
        const bool seg = root && !a.conflict[last] && (a.owner[last] >= 0 ? f >= 1 : f >= 2);
        const int64_t nseg = (int64_t)a.seg_idx[last] + (seg ? 1 : 0);
        const int64_t nout = (int64_t)a.seg_off[last] + (seg ? f : 0);
        a.counts[0] = nseg;
        a.counts[1] = nout;
        a.seg_off_out[nseg] = nout;
    }
}

// ascending node order inside every segment (one node per image: short segments):
// one warp per segment, every element placed at its rank (node ids are distinct)
__global__ void merge_sort_kernel(MergeArgs a) {
    const int64_t nseg = a.counts[0];
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = w0; s < nseg; s += nw) {
        const int64_t b = a.seg_off_out[s], e = a.seg_off_out[s + 1];
        const int L = (int)(e - b);
        for (int i = lane; i < L; i += 32) {
            const int x = a.out_node[b + i];
            int r = 0;
            for (int j = 0; j < L; j++) r += a.out_node[b + j] < x;
            a.tmp_node[b + r] = x;
        }
        __syncwarp();
        for (int i = lane; i < L; i += 32) a.out_node[b + i] = a.tmp_node[b + i];
        __syncwarp();
    }
}

// covisibility counts (model.py:105-110 for every image pair): one thread per
// point adds 1 to C[a][b] for every ordered pair of distinct images on its track
__global__ void covis_kernel(int32_t n_points, const int64_t* __restrict__ ptr,
                            const int32_t* __restrict__ img, int32_t n_images,
                            int32_t* __restrict__ C) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_points) return;
    const int64_t b = ptr[p], e = ptr[p + 1];
    for (int64_t i = b; i < e; i++)
        for (int64_t j = i + 1; j < e; j++) {
            const int x = img[i], y = img[j];
            if (x == y) continue;
            atomicAdd(C + (int64_t)x * n_images + y, 1);
            atomicAdd(C + (int64_t)y * n_images + x, 1);
        }
}

// nodes the merge can emit: every fresh node is a distinct bank row touched by an
// edge, so min(2 * edges, nodes) bounds the (component, image) keys, the output
// nodes and their segments alike
int64_t touched_bound(int64_t n_nodes, int64_t n_edges) {
    const int64_t b = 2 * n_edges < n_nodes ? 2 * n_edges : n_nodes;
    return b > 0 ? b : 1;
}

// open addressing at load <= 1/2 over at most `keys` keys
int64_t hash_size(int64_t keys) {
    int64_t h = 1024;
    while (h < 2 * keys) h <<= 1;
    return h;
}

}  // namespace
}  // namespace msfm

using namespace msfm;

extern "C" int msfm_covisibility(int32_t n_points, const int64_t* d_track_ptr,
                                 const int32_t* d_track_img, int32_t n_images, int32_t* d_counts,
                                 void* stream) {
    if (n_points < 0 || n_images < 0 || (n_points > 0 && (!d_track_ptr || !d_track_img)) ||
        (n_images > 0 && !d_counts)) {
        set_error("msfm_covisibility: bad arguments");
        return MSFM_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n_images == 0) return MSFM_OK;
    MSFM_CUDA_TRY(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * (size_t)n_images * n_images, st));
    if (n_points == 0) return MSFM_OK;
    covis_kernel<<<(n_points + 255) / 256, 256, 0, st>>>(n_points, d_track_ptr, d_track_img,
                                                         n_images, d_counts);
    MSFM_LAUNCH_CHECK();
    count_launches(1);
    return MSFM_OK;
}

extern "C" size_t msfm_merge_workspace_bytes(int64_t n_nodes, int64_t n_edges) {
    const int64_t n = n_nodes > 0 ? n_nodes : 1;
    const int64_t nb = (n + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER) + 1;
    return aligned_bytes<int32_t>(n) * 10 + aligned_bytes<int32_t>(nb) +
           aligned_bytes<unsigned long long>(hash_size(touched_bound(n, n_edges))) * 2 +
           aligned_bytes<int32_t>(touched_bound(n, n_edges)) + 4096;
}

extern "C" int msfm_merge_tracks(const msfm_bank* bank, int64_t n_edges, const int32_t* d_u,
                                 const int32_t* d_v, const float* d_dist, int32_t n_points,
                                 const int64_t* d_track_ptr, const int32_t* d_track_node,
                                 int32_t* d_out_node, int32_t* d_seg_owner, int64_t* d_seg_off,
                                 int64_t* d_counts, void* d_workspace, size_t workspace_bytes,
                                 void* stream) {
    if (!bank || n_edges < 0 || n_points < 0 || !d_counts || (n_points > 0 && !d_track_ptr)) {
        set_error("msfm_merge_tracks: bad arguments");
        return MSFM_EINVAL;
    }
    const int64_t n = bank->n_total;
    if (n >= (1LL << 31) || bank->n_images >= (1 << 16)) {
        set_error("msfm_merge_tracks: bank too large for 32-bit nodes / 16-bit images");
        return MSFM_EINVAL;
    }
    if (workspace_bytes < msfm_merge_workspace_bytes(n, n_edges)) {
        set_error("msfm_merge_tracks: workspace too small");
        return MSFM_EWORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        MSFM_CUDA_TRY(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int64_t), st));
        MSFM_CUDA_TRY(cudaMemsetAsync(d_seg_off, 0, sizeof(int64_t), st));
        return MSFM_OK;
    }
    Arena ar(d_workspace, workspace_bytes);
    MergeArgs a;
    a.n_nodes = n; a.n_edges = n_edges; a.u = d_u; a.v = d_v; a.dist = d_dist;
    a.n_points = n_points; a.tptr = d_track_ptr; a.tnode = d_track_node;
    a.img_off = bank->d_img_off; a.n_images = bank->n_images;
    a.parent = ar.take<int32_t>(n); a.root = ar.take<int32_t>(n); a.support = ar.take<uint32_t>(n); a.owner = ar.take<int32_t>(n);
    a.conflict = ar.take<int32_t>(n); a.fresh_cnt = ar.take<int32_t>(n); a.fresh = ar.take<int32_t>(n);
    a.seg_idx = ar.take<int32_t>(n); a.seg_off = ar.take<int32_t>(n); a.fill = ar.take<int32_t>(n);
    const int64_t nb = (n + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER) + 1;
    int32_t* bsum = ar.take<int32_t>(nb);
    const int64_t hs = hash_size(touched_bound(n, n_edges));
    a.hkey = ar.take<unsigned long long>(hs); a.hval = ar.take<unsigned long long>(hs);
    a.hmask = hs - 1;
    a.tmp_node = ar.take<int32_t>(touched_bound(n, n_edges));
    a.out_node = d_out_node; a.seg_owner = d_seg_owner; a.seg_off_out = d_seg_off; a.counts = d_counts;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = nsm * 8;
    ProfScope ps("merge_tracks", st);
    merge_init_kernel<<<grid, 256, 0, st>>>(a);
    if (n_edges > 0) merge_edges_kernel<<<grid, 256, 0, st>>>(a);
    if (n_points > 0) merge_tracks_kernel<<<(n_points + 255) / 256, 256, 0, st>>>(a);
    merge_compress_kernel<<<grid, 256, 0, st>>>(a);
    if (n_points > 0) merge_owner_kernel<<<(n_points + 255) / 256, 256, 0, st>>>(a);
    merge_select_kernel<<<grid, 256, 0, st>>>(a);
    merge_winner_kernel<<<grid, 256, 0, st>>>(a);
    merge_flag_kernel<<<grid, 256, 0, st>>>(a);
    MSFM_LAUNCH_CHECK();
    count_launches(6 + (n_edges > 0) + 2 * (n_points > 0));
    int rc = exclusive_scan(a.seg_idx, n, nullptr, bsum, st);
    if (rc) return rc;
    rc = exclusive_scan(a.seg_off, n, nullptr, bsum, st);
    if (rc) return rc;
    merge_emit_kernel<<<grid, 256, 0, st>>>(a);
    merge_sort_kernel<<<grid, 256, 0, st>>>(a);
    MSFM_LAUNCH_CHECK();
    count_launches(2);
    return MSFM_OK;
}
