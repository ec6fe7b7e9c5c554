/*
 * msfm_b200 — C-ABI of the B200-native fine-stage hot path of Multistage SfM.
 *
 * The reference (pkg/src/msfm) is pure Python and has no FFI; its "plugin
 * surface" is the Python function set the stages call.  Each
 * entry point below is the native body of one of those functions, batched over
 * pairs / images / tracks.  The Python drop-in (paper_1512_06235_b200/) binds
 * them with ctypes exactly as a maintainer would from msfm.
 *
 * Conventions
 *   - every function returns 0 on success, a negative MSFM_E* code on error;
 *     msfm_last_error() returns the thread's last message.  No exceptions and
 *     no hidden state cross the ABI.
 *   - pointers named d_* are device pointers (caller-owned, e.g. torch
 *     tensors); h_* are host pointers.  `stream` is a cudaStream_t (void*).
 *   - all work is enqueued on `stream`; nothing synchronises the host unless
 *     stated.
 */
#ifndef MSFM_B200_H
#define MSFM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSFM_OK 0
#define MSFM_EINVAL (-1)      /* bad argument (ValueError in the Python layer) */
#define MSFM_ECUDA (-2)       /* CUDA runtime / launch failure */
#define MSFM_EWORKSPACE (-3)  /* workspace too small */
#define MSFM_ECAPACITY (-4)   /* an output capacity would be exceeded */

const char* msfm_last_error(void);
int msfm_version(void);

/* Number of kernels this library has launched so far (process-wide). */
int64_t msfm_launch_count(void);
/* Optional CUDA-event timing of the library's hot kernels, recorded on the
 * stream each kernel is launched on.  enable(1) clears previous records;
 * read() synchronises on the recorded events and sums their durations. */
int msfm_profile_enable(int on);
int msfm_profile_read(const char* kernel_name, double* total_ms, int64_t* launches);
/* Diagnostics: enable(1) allocates 16 device counters the matcher increments
 * (super-groups, members, gathered, passing, sure, unsure, exact-C' tests,
 * m-tiles, groups, rounds); read copies them to out16 and resets; enable(0) frees. */
int msfm_debug_counters(int enable, int64_t* out16);

/* ------------------------------------------------------------------------
 * Feature bank: all images' features concatenated (SoA, HBM-resident).
 *   xy    f32 [n_total][2]          FeatureSet.xy            features.py:55
 *   desc  u8  [n_total][128]        FeatureSet.descriptors   features.py:58
 *   norm2 i32 [n_total]             |desc|^2 (msfm_feature_norms)
 *   img_off i64 [n_images]          first feature of image i
 *   img_n   i32 [n_images]          feature count of image i
 *   img_wh  i32 [n_images][2]       width, height
 * ---------------------------------------------------------------------- */
typedef struct {
    const float* d_xy;
    const uint8_t* d_desc;
    const int32_t* d_norm2;
    const int64_t* d_img_off;
    const int32_t* d_img_n;
    const int32_t* d_img_wh;
    int32_t n_images;
    int64_t n_total;          /* total features (rows of d_xy / d_desc) */
} msfm_bank;

/* |desc|^2 per feature (exact int32). */
int msfm_feature_norms(const uint8_t* d_desc, int64_t n, int32_t* d_norm2, void* stream);

/* ------------------------------------------------------------------------
 * Spatial index of every target image (replaces msfm.guided.build_grid /
 * OverlapGrid, guided.py:46-137).
 *
 * The reference's union of the 4 containing cells (offset grids of cell size
 * 2D) of a line sample equals the 3x3 block of D-sized "subcells" around the
 * sample's subcell: cell_g(f) == cell_g(s) for some g  <=>  |u_f-u_s| <= 1 and
 * |v_f-v_s| <= 1, with u = 2*floor(x/2D) + [floor((x-D)/2D) == floor(x/2D)]
 * evaluated in the reference's float64 rounding.  The index therefore stores,
 * per feature, its subcell (u, v) (int16 each), and two CSR bucket tables of
 * D x D buckets (bucket = floor(x/D), floor(y/D)): row-major (rows of y) and
 * column-major (rows of x), used to enumerate the features near a line.
 *   d_sub    [n_total]       short2 (u, v)
 *   d_dims   [n_images][2]   nbx, nby buckets
 *   d_roff/d_coff [n_images] first bucket of image i in the row/col tables
 *   d_rstart/d_cstart [n_buckets_total+1] CSR starts (global feature index)
 *   d_rmem/d_cmem [n_total]  image-local feature ids in bucket order
 *   d_rrec/d_crec [n_total][4] int32 records in bucket order: x, y (f32
 *                            bits), |desc|^2, feature id, so a strip gather
 *                            reads one 16-B record per entry instead of
 *                            chasing the id
 * ---------------------------------------------------------------------- */
typedef struct {
    const int32_t* d_sub;        /* short2 packed: (u & 0xffff) | (v << 16)      */
    const int32_t* d_dims;
    const int64_t* d_roff;
    const int64_t* d_coff;
    const int32_t* d_rstart;
    const int32_t* d_cstart;
    const int32_t* d_rmem;
    const int32_t* d_cmem;
    const int32_t* d_rrec;
    const int32_t* d_crec;
    double D;                    /* cell half-size = d * inflation (grid.d)      */
} msfm_grids;

/* Host-only: bucket dims (nbx, nby) of one image for cell half-size D. */
int msfm_grid_dims(int32_t width, int32_t height, double D, int32_t dims_out[2]);

/* Build the index of all images.  Bucket totals: sum over images of
 * nbx*nby (row table and col table each).  Outputs are caller-allocated:
 * d_sub[n_total], d_rstart/d_cstart[n_buckets_total+1], d_rmem/d_cmem[n_total]. */
size_t msfm_grid_workspace_bytes(int64_t n_buckets_total);
int msfm_grid_build(const msfm_bank* bank, const int32_t* d_dims, const int64_t* d_roff,
                    const int64_t* d_coff, int64_t n_buckets_total, int64_t n_total, double D,
                    int32_t* d_sub, int32_t* d_rstart, int32_t* d_cstart, int32_t* d_rmem,
                    int32_t* d_cmem, int32_t* d_rrec, int32_t* d_crec, void* d_workspace,
                    size_t workspace_bytes, void* stream);

/* The same for the contiguous image range [img0, img1) only (bucket range
 * [bucket0, bucket1) = [roff[img0], roff[img1]), first feature row feat0 =
 * img_off[img0]; d_coff must equal d_roff): lets a bank be indexed range by range
 * as its rows arrive (staged uploads).  Writes the CSR starts [bucket0, bucket1]
 * and never rewrites a start another range published.  Ranges built on one stream
 * share one workspace. */
int msfm_grid_build_range(const msfm_bank* bank, const int32_t* d_dims, const int64_t* d_roff,
                          const int64_t* d_coff, int64_t n_buckets_total, int32_t img0,
                          int32_t img1, int64_t bucket0, int64_t bucket1, int64_t feat0,
                          double D, int32_t* d_sub, int32_t* d_rstart, int32_t* d_cstart,
                          int32_t* d_rmem, int32_t* d_cmem, int32_t* d_rrec, int32_t* d_crec,
                          void* d_workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Geometry-aware (epipolar-guided) matching of a batch of image pairs.
 * Replaces msfm.guided.guided_match_pair(strategy="grid") (guided.py:393-480)
 * + ratio_filter/_dedupe_targets (matching.py:82-113), batched over the pair
 * loop of densify_stage (densify.py:220-240).
 *
 * Pair k: query image d_pair_q[k], target image d_pair_t[k], fundamental
 * matrix d_pair_F[9k..9k+8] (row-major, p_t^T F p_q = 0, from
 * fundamental_from_poses geometry.py:69-83), query feature ids
 * d_qlist[d_qlist_off[k] .. d_qlist_off[k+1]) in ascending order.  When
 * d_qlist_src (optional, [n_pairs] int64) is given, pair k's list is read from
 * d_qlist[d_qlist_src[k] ..] instead (pairs sharing a query image share one
 * list); d_qlist_off still sizes the lists and places the output segments.
 * A pair whose F row starts with NaN is skipped (degenerate geometry,
 * densify.py:161-165).
 *
 * Output (device): the matches of pair k are written to positions
 * [qlist_off[k], qlist_off[k] + d_out_count[k]) of the four SoA arrays, sorted
 * by query id (one match per query at most, so capacity = total queries):
 *   out_q (query fid), out_t (target fid), out_dist (f32 L2 distance),
 *   out_ratio (f32 best/second ratio, 0 for single-candidate accepts).
 * d_stats (optional, [2*n_pairs] int64): SearchStats (queries, comparisons)
 * exactly as guided.py:459-460 counts them.
 * ---------------------------------------------------------------------- */
typedef struct {
    double d;            /* band half-width (BAND_D_PX = 8)                      */
    float ratio;         /* Lowe ratio, compared in f32 (RATIO_GUIDED = 0.8)     */
    float single_cap;    /* single-candidate cap (SINGLE_CANDIDATE_CAP = 45)     */
    int32_t max_nt;      /* max target feature count over the batch (<= 65536)   */
    int32_t chunk_pairs; /* pairs per internal chunk (workspace bound); 0 = auto:
                          * up to 8192 pairs and 48M query slots per chunk       */
    int32_t strategy;    /* candidate strategy of guided_match_pair (guided.py:425-431):
                          * 0 grid (cells of the samples, default), 1 linear
                          * (|rep line| <= d, guided.py:190-194), 2 radial (disks of
                          * radius d*sqrt(2) around the samples, guided.py:273-285) */
    int32_t first_chunk_pairs; /* when > 0 (pipelined / staged use): chunk sizes ramp
                          * first, 4x, 16x ... up to chunk_pairs, so matching starts
                          * after few images have landed, and pieces of 16x, 4x, 1x
                          * first are cut from the end of the last chunk (its
                          * readback is the one no later chunk hides)            */
    int64_t max_workspace_bytes; /* chunks are cut so one chunk's workspace stays
                          * within this many bytes; 0 = a quarter of the device's
                          * free memory at planning time (at most 48M query slots,
                          * 2^26 per chunk hard limit, explicit chunk_pairs too) */
} msfm_match_params;

/* Pack the per-pair segments of msfm_guided_match's output into contiguous
 * 16-byte rows (pair index, q_fid | t_fid << 16, f32 dist bits, f32 ratio bits)
 * in pair order; d_out_off [n_pairs+1] receives the row offsets (total last).
 * d_rows capacity: 4 * total queries int32. */
int msfm_pack_matches(int32_t n_pairs, const int64_t* d_qlist_off, const int32_t* d_count,
                      const int32_t* d_q, const int32_t* d_t, const float* d_dist,
                      const float* d_ratio, int64_t* d_out_off, int32_t* d_rows, void* stream);

size_t msfm_guided_workspace_bytes(int32_t n_pairs, const int64_t* h_qlist_off,
                                   const msfm_match_params* prm);
int msfm_guided_match(const msfm_bank* bank, const msfm_grids* grids, int32_t n_pairs,
                      const int32_t* d_pair_q, const int32_t* d_pair_t, const double* d_pair_F,
                      const int64_t* d_qlist_off, const int32_t* d_qlist,
                      const int64_t* d_qlist_src, const int64_t* h_qlist_off, const msfm_match_params* prm,
                      int32_t* d_out_q, int32_t* d_out_t, float* d_out_dist, float* d_out_ratio,
                      int32_t* d_out_count, int64_t* d_stats,
                      void* d_workspace, size_t workspace_bytes, void* stream);

/* Staged bank for msfm_guided_match_rows: the bank rows of image range r arrive
 * (uploaded by the caller on its own stream, event landed[r]) while earlier
 * chunks match; just before chunk chunk[r] the matcher's stream waits on
 * landed[r] and computes the range's |desc|^2 and spatial index
 * (msfm_grid_build_range with img0/img1, bucket0/bucket1, feat0), so the index
 * build never queues behind a running chunk.  chunk[] is non-decreasing. */
typedef struct {
    int32_t n_ranges;
    const int32_t* chunk;
    const int32_t* img0;
    const int32_t* img1;
    const int64_t* bucket0;
    const int64_t* bucket1;
    const int64_t* feat0;         /* first bank row of the range */
    const int64_t* feat1;         /* end bank row of the range */
    void* const* landed;          /* cudaEvent_t per range, or NULL entries */
    int64_t n_buckets_total;
    void* grid_workspace;         /* msfm_grid_workspace_bytes(n_buckets_total) */
    size_t grid_workspace_bytes;
} msfm_stage_plan;

/* The matcher's internal chunking: writes the first pair of every chunk and the
 * end (n_chunks + 1 values, at most `capacity`) and returns n_chunks. */
int32_t msfm_guided_chunk_bounds(int32_t n_pairs, const int64_t* h_qlist_off,
                                 const msfm_match_params* prm, int32_t* out_bounds,
                                 int32_t capacity);

/* msfm_guided_match followed by the packing of msfm_pack_matches, pipelined with
 * the device-to-host copy: after every internal chunk its packed rows are copied
 * on `copy_stream` into the pinned host buffer h_rows (16-B rows, pair order)
 * while the next chunk computes.  Scratch: d_out_off [n_pairs+1], d_rows
 * (4 * total queries int32), d_meta / h_meta (pinned) [2 * (n_pairs + 1)] int64.
 * Returns after the last copy; *h_total = rows written.  No SearchStats.
 * plan (optional): the bank is still arriving; see msfm_stage_plan. */
int msfm_guided_match_rows(const msfm_bank* bank, const msfm_grids* grids, int32_t n_pairs,
                           const int32_t* d_pair_q, const int32_t* d_pair_t,
                           const double* d_pair_F, const int64_t* d_qlist_off,
                           const int32_t* d_qlist, const int64_t* d_qlist_src,
                           const int64_t* h_qlist_off, const msfm_match_params* prm,
                           int32_t* d_out_q, int32_t* d_out_t, float* d_out_dist,
                           float* d_out_ratio, int32_t* d_out_count, int64_t* d_out_off,
                           int32_t* d_rows, int64_t* d_meta, int64_t* h_meta, int32_t* h_rows,
                           int64_t* h_total, void* d_workspace, size_t workspace_bytes,
                           void* stream, void* copy_stream, const msfm_stage_plan* plan);

/* ------------------------------------------------------------------------
 * Host-only: RANSAC hypothesis sets.  Emits `count` consecutive draws of
 * numpy's `rng.choice(n, size=sample_size, replace=False)` starting from the
 * PCG64 state of a numpy Generator (state hi/lo, inc hi/lo, has_uint32,
 * uinteger = rng.bit_generator.state), exactly as pnp_ransac consumes them
 * (reconstruct.py:185-194).  out: [count][sample_size] int32.  state_out
 * (optional) receives the generator state after the draws: state hi/lo,
 * inc hi/lo, has_uint32, uinteger — to continue the stream in a later call.
 * ---------------------------------------------------------------------- */
int msfm_ransac_samples(const uint64_t state_inc[4], int32_t has_uint32, uint32_t uinteger,
                        int64_t n, int32_t sample_size, int32_t count, int32_t* out,
                        uint64_t state_out[6]);
/* PCG64 state (layout of state_out above) of np.random.default_rng(seed):
 * numpy's SeedSequence -> PCG64 seeding restated (0 <= seed < 2^64). */
int msfm_rng_seed_state(uint64_t seed, uint64_t state_out[6]);
/* msfm_ransac_samples for n_items independent streams default_rng(seeds[i])
 * over populations n[i]: out [n_items][count][sample_size], state_out
 * (optional) [n_items][6] after the draws. */
int msfm_ransac_samples_seeded(int32_t n_items, const uint64_t* seeds, const int64_t* n,
                               int32_t sample_size, int32_t count, int32_t* out,
                               uint64_t* state_out);

/* ------------------------------------------------------------------------
 * 3D-2D localization kNN (DescriptorIndex.knn2 exact path, descriptors.py:35-72,
 * for the mean-descriptor queries of direct_3d2d_search, localize.py:99-122).
 * Points are given exactly: S [n_points][128] int32 track-descriptor sums and
 * n [n_points] track lengths (mean = S/n, localize.py:51-59).  For every query
 * image d_images[s] (bank image index) and point p the result is the top-2 of
 *     key = n_p |f|^2 - 2 S_p.f     (N = |S - n f|^2 = n_p*key + |S_p|^2)
 * over the image's features, lowest feature index winning ties:
 *     k1[s][p], i1[s][p] (image-local feature id, -1 if none), k2[s][p]
 * (INT64_MAX when the image has < 2 features).  Row stride = n_points rounded
 * up to 128.  2 S.f runs on tcgen05 kind::i8 over u8 digit planes: points with
 * track length <= 100 use two (2S = lo + 256 hi, lo = 2 (S mod 128), hi = S >> 7,
 * int32 keys in the epilogue), longer tracks three base-256 digits of 2S and int64
 * keys (any track length up to 32767; max_track > 100 enables that launch);
 * max_image_features bounds the feature count of every query image.
 * ---------------------------------------------------------------------- */
size_t msfm_knn_workspace_bytes(int32_t n_points, int32_t n_images, int32_t max_image_features);
int msfm_knn2_tracks(const msfm_bank* bank, int32_t n_points, const int32_t* d_S,
                     const int32_t* d_n, int32_t n_images, const int32_t* d_images,
                     int32_t max_track, int32_t max_image_features, int64_t* d_k1, int32_t* d_i1,
                     int64_t* d_k2, void* d_workspace, size_t workspace_bytes, void* stream);

/* K7 track sums (mean_descriptor localize.py:51-59 in exact integer form, the
 * query points of msfm_knn2_tracks): point p's track is bank rows
 * d_track_row[d_track_ptr[p] .. d_track_ptr[p+1]); outputs S [n_points][128] int32
 * (sum of the u8 rows), n [n_points] track lengths, SS [n_points] = |S|^2 int64. */
int msfm_track_sums(const msfm_bank* bank, int64_t n_points, const int64_t* d_track_ptr,
                    const int64_t* d_track_row, int32_t* d_S, int32_t* d_n, int64_t* d_SS,
                    void* stream);

/* Index of the second neighbour of msfm_knn2_tracks' output (the lowest feature
 * index other than i1 whose key equals k2, descriptors.py:61-63), -1 when there
 * is none: d_i2 [n_images][n_points rounded up to 128]. */
int msfm_knn2_second_index(const msfm_bank* bank, int32_t n_points, const int32_t* d_S,
                           const int32_t* d_n, int32_t n_images, const int32_t* d_images,
                           const int64_t* d_k1, const int32_t* d_i1, const int64_t* d_k2,
                           int32_t* d_i2, void* stream);

/* Real-valued 2-NN for float descriptor rows that are not integer-valued
 * (two_nearest_bruteforce descriptors.py:35-72 / DescriptorIndex.knn2
 * descriptors.py:123-139 with arbitrary float32 input): squared L2 as
 * sum((q-t)^2) in f64 (differences and squares exact for f32 inputs), top-2 per
 * query with the lowest target index winning ties.  d_d2 [n_queries][2] f64,
 * d_idx [n_queries][2] int64; (inf, -1) where fewer than 2 targets exist. */
int msfm_knn2_float(const float* d_q, int64_t n_queries, const float* d_t, int64_t n_targets,
                    int32_t dim, double* d_d2, int64_t* d_idx, void* stream);

/* direct_3d2d_search post-processing (localize.py:108-122 + ratio_filter
 * matching.py:82-103) on the knn2 output: ratio test sqrt(N_b/N_s) < p/q
 * evaluated exactly (q^2 N_b < p^2 N_s), single-feature images: sqrt(N_b)/n <
 * single_cap; then one point per feature (smallest exact distance N/n^2, lower
 * point row wins ties).  Output per image slot s: rows d_corr_row[s*stride ..]
 * (ascending point row) and d_corr_fid, count d_corr_n[s].  d_win is scratch of
 * sum over query images of their feature counts (int32), offsets d_win_off[s]. */
int msfm_direct_3d2d(const msfm_bank* bank, int32_t n_points, const int32_t* d_n,
                     const int64_t* d_SS, int32_t n_images, const int32_t* d_images,
                     const int64_t* d_k1, const int32_t* d_i1, const int64_t* d_k2,
                     int64_t ratio_p, int64_t ratio_q, double single_cap,
                     int32_t* d_win, const int64_t* d_win_off, int32_t* d_corr_row,
                     int32_t* d_corr_fid, int32_t* d_corr_n, void* stream);

/* The PnP inputs of selected images straight from msfm_direct_3d2d's output
 * (localize.py:203-211: X = the points' positions, uv = the features' pixels as
 * f64).  Selected image k: correspondence table row d_sel[k] (stride m_pad),
 * bank row of its feature 0 d_row0[k], output rows [d_out_off[k], d_out_off[k+1]):
 * d_X [.][3] = d_xyz[point row], d_uv [.][2] = bank xy[d_row0[k] + fid]. */
int msfm_gather_3d2d(const int32_t* d_corr_row, const int32_t* d_corr_fid, int32_t m_pad,
                     int32_t n_sel, const int64_t* d_sel, const int64_t* d_row0,
                     const int64_t* d_out_off, const double* d_xyz, const float* d_bank_xy,
                     double* d_X, double* d_uv, void* stream);

/* msfm_ransac_samples_seeded on the device, the same draws bit for bit (the
 * PCG64 / SeedSequence / choice restatement is shared with the host sampler,
 * rng.cuh): one thread per (stream, choice) positioned with PCG64's jump-ahead,
 * streams where Lemire's bounded draw would have redrawn are redone sequentially.
 * d_bad: 1 + n_items int32 of scratch; d_bad[0] is set to 1 (never cleared) when
 * an item is outside choice's Floyd branch (n > 10000 and size > n/50). */
int msfm_ransac_samples_seeded_device(int32_t n_items, const uint64_t* d_seeds, const int64_t* d_n,
                                      int32_t sample_size, int32_t count, int32_t* d_out,
                                      uint64_t* d_state_out, int32_t* d_bad, void* stream);

/* ------------------------------------------------------------------------
 * PnP-RANSAC (reconstruct.py:168-226), batched over images.  Correspondences of
 * image s: X [off[s]..off[s+1])[3] f64 world points, uv [..][2] f64 pixels,
 * K [s][9].  msfm_pnp_hypotheses scores n_hyp host-supplied 6-point samples per
 * image (d_samples [s][h][6], image-local indices; see msfm_ransac_samples):
 * d_hyp [s][h][12] = R (row-major) | t of dlt_pose (reconstruct.py:53-103),
 * d_count [s][h] = inliers (err < threshold, z > 0), -1 when the DLT fails.
 * The caller replays the adaptive stop (reconstruct.py:192-211) on the counts
 * and passes the winning pose to msfm_pnp_refit, which recomputes the inlier
 * mask, refits dlt_pose on it, runs refine_pose_lm (<= lm_iters LM iterations)
 * and writes the final R, t, mask (d_mask[off[s]..]) and inlier count;
 * d_ok[s] = final inliers >= min_inliers and the refit succeeded.  Only images
 * with d_status[s] != 0 are processed.
 * ---------------------------------------------------------------------- */
int msfm_pnp_hypotheses(const double* d_X, const double* d_uv, const int64_t* d_off,
                        const double* d_K, int32_t n_images, const int32_t* d_samples,
                        int32_t n_hyp, double threshold, double* d_hyp, int32_t* d_count,
                        void* stream);
int msfm_pnp_refit(const double* d_X, const double* d_uv, const int64_t* d_off, const double* d_K,
                   int32_t n_images, const double* d_hyp_best, const int32_t* d_status,
                   double threshold, int32_t min_inliers, int32_t lm_iters, double* d_R,
                   double* d_t, uint8_t* d_mask, int32_t* d_n_inliers, int32_t* d_ok,
                   void* stream);

/* ------------------------------------------------------------------------
 * Multi-view DLT triangulation (geometry.py:276-357) of n_tracks tracks.
 * Cameras: K [c][9], R [c][9], t [c][3] (x ~ K (R X + t)).  Track k has the
 * observations [ptr[k], ptr[k+1]): camera index d_cam[i], pixel d_pix[i][2].
 * Output X [k][3], mean reprojection error err [k], status [k]:
 *   1 accepted, 0 rejected by a gate (the reference returns None),
 *  -1 DegenerateGeometryError (shared centre / parallel rays),
 *  -2 InsufficientDataError (< 2 observations).
 * ---------------------------------------------------------------------- */
int msfm_triangulate_batch(const double* d_K, const double* d_R, const double* d_t,
                           int32_t n_tracks, const int64_t* d_ptr, const int32_t* d_cam,
                           const double* d_pix, double max_error, double min_angle_deg,
                           double* d_X, double* d_err, int32_t* d_status, void* stream);

/* ------------------------------------------------------------------------
 * Two-view geometry of the coarse match graph: estimate_fundamental_ransac
 * (geometry.py:153-198) batched over image pairs.  Pair p's correspondences
 * are rows [off[p], off[p+1]) of d_q (query pixels) and d_c (target pixels),
 * f64 [..][2].  msfm_fundamental_hypotheses fits the normalized 8-point F of
 * n_hyp host-supplied samples per pair (d_samples [p][h][8], pair-local rows;
 * msfm_ransac_samples with sample_size 8) into d_F [p][h][9] and counts the
 * Sampson inliers (< threshold) into d_count [p][h] (-1: non-finite fit).
 * The caller replays the adaptive stop (geometry.py:176-191, w**8) and passes
 * the winner to msfm_fundamental_refit, which refits on its inliers (pairs
 * with d_status[p] != 0) and writes F, the final inlier mask (d_mask, per row),
 * the inlier count and the design-matrix gap s[-2]/s[0] (0 below 9 rows).
 * ---------------------------------------------------------------------- */
int msfm_fundamental_hypotheses(const double* d_q, const double* d_c, const int64_t* d_off,
                                int32_t n_pairs, const int32_t* d_samples, int32_t n_hyp,
                                double threshold, double* d_F, int32_t* d_count, void* stream);
int msfm_fundamental_refit(const double* d_q, const double* d_c, const int64_t* d_off,
                           int32_t n_pairs, const double* d_F_best, const int32_t* d_status,
                           double threshold, double* d_F, uint8_t* d_mask, int32_t* d_count,
                           double* d_gap, void* stream);

/* ------------------------------------------------------------------------
 * Track merge of densify_stage (densify.py:68-158): connected components over
 * one stage's matches plus the model tracks, with the reference's conflict
 * rules (two owning points: dropped; an image holding an owner ref keeps the
 * ref; otherwise one node per image, smallest (support distance, key)).
 * Nodes are bank feature rows (bank images in ascending id: node order is the
 * reference's (image, feature) key order).
 *   d_u, d_v, d_dist [n_edges]      matched nodes and f32 distances
 *   d_track_ptr [n_points+1], d_track_node  model tracks as bank nodes
 * Output: fresh nodes grouped per emitting component (ascending smallest node),
 * ascending inside: d_out_node [<= min(2 n_edges, bank rows)]; per segment d_seg_owner (track
 * row extended, -1 = new track) and d_seg_off [n_seg+1]; d_counts = {n_seg, n_out}.
 * ---------------------------------------------------------------------- */
size_t msfm_merge_workspace_bytes(int64_t n_nodes, int64_t n_edges);
/* Covisibility of all image pairs (len(model.covisible_points(a, b)),
 * model.py:105-110, used by candidate_images densify.py:37-56): d_counts
 * [n_images][n_images] int32 (zeroed here) counts the points whose track
 * (d_track_img [track_ptr[p] .. track_ptr[p+1]), image slots) holds both. */
int msfm_covisibility(int32_t n_points, const int64_t* d_track_ptr, const int32_t* d_track_img,
                      int32_t n_images, int32_t* d_counts, void* stream);
int msfm_merge_tracks(const msfm_bank* bank, int64_t n_edges, const int32_t* d_u,
                      const int32_t* d_v, const float* d_dist, int32_t n_points,
                      const int64_t* d_track_ptr, const int32_t* d_track_node,
                      int32_t* d_out_node, int32_t* d_seg_owner, int64_t* d_seg_off,
                      int64_t* d_counts, void* d_workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Host-only staging of .msft feature files (features.py:98-130): the
 * reference's header / size / bounds validation (status codes below, with the
 * first offending record), then the records in np.argsort(-scale, "stable")
 * order written to caller buffers (xy [n][2], scale, orientation [n] f32,
 * desc [n][128] u8; scale / orientation may be NULL; xy = NULL probes the
 * header only).  ``capacity`` is the record count the buffers were sized for (from
 * a probe): a file whose header now says otherwise gets MSFM_MSFT_CHANGED and
 * nothing is written.  msfm_msft_load_many loads n_files into one set of buffers
 * at rows [row_off[i], row_off[i+1]) (n_files + 1 offsets; e.g. the pinned host
 * bank) on n_threads host threads.
 * ---------------------------------------------------------------------- */
#define MSFM_MSFT_OK 0
#define MSFM_MSFT_TRUNCATED 1     /* shorter than the 24-byte header */
#define MSFM_MSFT_BAD_MAGIC 2
#define MSFM_MSFT_BAD_VERSION 3
#define MSFM_MSFT_BAD_SIZE 4      /* payload != count * 144 bytes */
#define MSFM_MSFT_BOUNDS 5        /* x, y outside the image or scale <= 0 */
#define MSFM_MSFT_IO 6
#define MSFM_MSFT_CHANGED 7       /* record count differs from the caller's capacity */
typedef struct {
    int32_t status;
    char magic[4];
    uint32_t version;
    int32_t image_id, width, height;
    int64_t count, file_bytes;
    int64_t bad_record;
    float bad_x, bad_y, bad_scale;
} msfm_msft_info;
int msfm_msft_load(const char* path, msfm_msft_info* info, float* xy, float* scale,
                   float* orientation, uint8_t* desc, int64_t capacity);
int msfm_msft_load_many(int32_t n_files, const char* const* paths, const int64_t* row_off,
                        msfm_msft_info* infos, float* xy, float* scale, float* orientation,
                        uint8_t* desc, int32_t n_threads);

/* ------------------------------------------------------------------------
 * Host-only reader of the model snapshot text (.msfm, msfm.io.read_model
 * io.py:51-84) into CSR arrays: cameras (id, f cx cy, R row-major, t, source
 * line) and points (xyz, track CSR of (image, feature) in file order, source
 * line; point ids = record order).  Validation in the reference's order —
 * header, record syntax, Camera det(R) (model.py:38), Model.attach_camera /
 * add_point rules (model.py:114-156) — stops at the first failure with
 * status, line and the reference's message (MSFM_MODEL_DET: value/value_id carry
 * det and the camera id; the caller formats numpy's repr).  Buffers NULL probes
 * the counts; the fill call takes the probe's counts as capacities.
 * ---------------------------------------------------------------------- */
#define MSFM_MODEL_OK 0
#define MSFM_MODEL_HEADER 1      /* "missing 'MSFM-MODEL 1' header" (no line prefix) */
#define MSFM_MODEL_RECORD 2      /* "<line>: <message>" */
#define MSFM_MODEL_UNKNOWN 3     /* "<line>: unknown record '<kind>'" */
#define MSFM_MODEL_DET 4         /* "<line>: camera <id>: det(R) = <value>" */
#define MSFM_MODEL_POSITION 5    /* PT with < 3 coordinates (accepted, unusable, by the reference) */
#define MSFM_MODEL_IO 6
#define MSFM_MODEL_CHANGED 7     /* counts differ from the fill call's capacities */
typedef struct {
    int32_t status, line;
    char message[192];
    double value;
    int64_t value_id;
    int64_t n_cams, n_points, n_obs;
    char stage[128];
    int32_t stage_truncated;
} msfm_model_info;
int msfm_model_read(const char* path, msfm_model_info* info, int32_t* cam_id, double* cam_fcc,
                    double* cam_R, double* cam_t, int32_t* cam_line, double* pt_xyz,
                    int64_t* track_ptr, int32_t* track_img, int32_t* track_fid, int32_t* pt_line,
                    int64_t cap_cams, int64_t cap_points, int64_t cap_obs);

#ifdef __cplusplus
}
#endif
#endif /* MSFM_B200_H */
