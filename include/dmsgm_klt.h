/*
 * dmsgm_klt.h -- C ABI of the B200 (sm_100a) motion estimation that produces the
 * per-frame homographies the DMSGM step consumes.
 *
 * The paper estimates camera motion with OpenCV (App. F; §2.4 P:116,
 * §3.1.3):
 *     goodFeaturesToTrack(prev, ...)                     -- Shi-Tomasi corners
 *     calcOpticalFlowPyrLK(prev, next, ..., Size(20,20), 5)   -- pyramidal Lucas-Kanade
 *     findHomography(prev_pts, cur_pts, CV_RANSAC)       -- RANSAC homography
 * This library does the same chain on the GPU for a batch of S independent streams, with
 * the readings DESIGN.md §2 R38-R42 states where the paper only names the OpenCV calls:
 *   R38 corners: exact integer 3x3 Sobel gradients and 3x3 structure tensor (replicated
 *       borders), score = float32(lambda_min) computed in fp64 from the exact tensor; local
 *       maxima (>= their 8 neighbours) of the interior with score > 0 and score >=
 *       quality x max score; greedy in descending (score, ascending raster index) order
 *       with distance >= min_distance to every kept corner; at most max_corners;
 *   R39 pyramid: 2x2 box average rounded half up, levels while both sizes >= win;
 *   R40 Lucas-Kanade: win x win bilinear samples centred on the point (continuous
 *       coordinates, pixel centres at +0.5), central-difference gradients, Newton steps
 *       until |d| < eps or max_iters; a level whose lambda_min(G)/win^2 < min_eig is
 *       skipped, at level 0 the point is lost (also when it leaves the frame);
 *   R41 homography: normalized DLT (Hartley) over the inliers of the best RANSAC model;
 *   R42 RANSAC: iteration i samples 4 distinct matches from a SplitMix64 counter stream
 *       (seed, i); minimal model by an 8x8 solve (degenerate: 3 collinear points);
 *       inliers have squared reprojection error < thresh^2; most inliers wins, ties to
 *       the earliest iteration.
 * The CPU oracle is oracle/klt_oracle.py (test infrastructure, no shared code).
 *
 * Conventions as in dmsgm.h: int status returns (DMSGM_OK / DMSGM_E*), dmsgm_klt_last_error
 * for the message, DEVICE pointers owned by the caller unless stated, calls enqueue on
 * `cuda_stream` and return (asynchronous) unless stated; frames are u8 [S][height][pitch],
 * stream s at byte offset s*height*pitch, pitch >= width.
 */
#ifndef DMSGM_KLT_H
#define DMSGM_KLT_H

#include <stddef.h>
#include <stdint.h>

#include "dmsgm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int    num_streams;    /* 1 <= S <= 32767                                                   */
    int    max_corners;    /* goodFeaturesToTrack maxCorners, 4..1024                           */
    double quality;        /* qualityLevel in (0, 1]                                            */
    double min_distance;   /* minDistance >= 1 (px)                                             */
    int    win;            /* LK window (samples per side), 3..32; the paper's Size(20,20) = 20 */
    int    max_level;      /* LK maxLevel 0..5; the paper's 5                                    */
    int    max_iters;      /* LK iterations per level, >= 1 (30)                                */
    float  eps;            /* LK step tolerance in px (0.01)                                    */
    float  min_eig;        /* LK minimum lambda_min(G)/win^2 (1e-3)                              */
    int    ransac_iters;   /* RANSAC iterations, 1..4096 (500)                                  */
    double ransac_thresh;  /* RANSAC reprojection threshold in px (3)                           */
    unsigned long long seed;   /* RANSAC sampler seed (42)                                      */
} dmsgm_klt_params;

typedef struct dmsgm_klt_ctx dmsgm_klt_ctx;

/* Create a context for S streams of width x height frames on `device`; allocates the
 * candidate, pyramid and match buffers.  DMSGM_EINVAL for bad sizes / params. */
int dmsgm_klt_create(int width, int height, const dmsgm_klt_params* p, int device, dmsgm_klt_ctx** out);

/* The whole chain for every stream: corners of `prev` (frame t-1), tracked into `next`
 * (frame t), RANSAC homography of the tracked pairs.  H_out: f64 [S][9] row-major, mapping
 * frame-t continuous coordinates to frame-(t-1) ones (R3) -- exactly the homographies
 * dmsgm_step takes with the frames `next`; a stream whose estimate fails (fewer than 4
 * tracked pairs or no model with 4 inliers) gets the identity and ok_out[s] = 0 (else the
 * inlier count).  ok_out may be NULL.  7 kernel launches, no host synchronisation. */
int dmsgm_klt_estimate(dmsgm_klt_ctx* ctx, const uint8_t* prev, size_t prev_pitch, const uint8_t* next,
                       size_t next_pitch, double* H_out, int* ok_out, void* cuda_stream);

/* The same estimate for consecutive frame pairs of a video (App. F runs the chain once per
 * frame): identical H_out / ok_out to dmsgm_klt_estimate(prev, next).  When
 * `prev` is the buffer (same pointer and pitch) passed as `next` to the previous
 * dmsgm_klt_estimate_seq call on this context, and no other dmsgm_klt_* call that computes
 * corners or pyramids (estimate, corners, track) or dmsgm_klt_seq_reset came in between,
 * the corners and pyramid levels computed from that frame are reused -- the CALLER
 * guarantees the buffer's content is unchanged since that call (else call
 * dmsgm_klt_seq_reset first).  Otherwise everything is computed from `prev` as in
 * dmsgm_klt_estimate.  The corners of `next` (for the following call) are computed on an
 * internal stream beside this pair's tracking and fit, and joined back into `cuda_stream`
 * before the call's work ends there.  7 kernel launches (9 when prev is not cached), no
 * host synchronisation; errors as dmsgm_klt_estimate (the cache is dropped on any error). */
int dmsgm_klt_estimate_seq(dmsgm_klt_ctx* ctx, const uint8_t* prev, size_t prev_pitch, const uint8_t* next,
                           size_t next_pitch, double* H_out, int* ok_out, void* cuda_stream);

/* Forget the frame dmsgm_klt_estimate_seq cached (the next call recomputes from `prev`). */
int dmsgm_klt_seq_reset(dmsgm_klt_ctx* ctx);

/* Stage 1 alone (R38): corners_out int32 [S][max_corners][2] (x, y pixel indices, in
 * selection order), counts_out int32 [S]. */
int dmsgm_klt_corners(dmsgm_klt_ctx* ctx, const uint8_t* frames, size_t pitch, int* corners_out,
                      int* counts_out, void* cuda_stream);

/* Stage 2 alone (R39, R40): track corners int32 [S][max_corners][2] (counts [S]) from
 * prev to next: tracked_out f32 [S][max_corners][2] in continuous coordinates (NaN when
 * lost), status_out u8 [S][max_corners] (1 tracked, 0 lost). */
int dmsgm_klt_track(dmsgm_klt_ctx* ctx, const uint8_t* prev, size_t prev_pitch, const uint8_t* next,
                    size_t next_pitch, const int* corners, const int* counts, float* tracked_out,
                    uint8_t* status_out, void* cuda_stream);

/* Stage 3 alone (R41, R42): matches src -> dst, f64 [S][max_corners][2] with counts [S];
 * H_out f64 [S][9] maps src to dst (identity + ok_out 0 on failure); inliers_out u8
 * [S][max_corners] (the best model's inliers; may be NULL); iter_counts_out int32
 * [S][ransac_iters] (inliers of every iteration's model, -1 for a degenerate sample; may
 * be NULL); ok_out int32 [S] (may be NULL). */
int dmsgm_klt_ransac(dmsgm_klt_ctx* ctx, const double* src, const double* dst, const int* counts,
                     double* H_out, uint8_t* inliers_out, int* iter_counts_out, int* ok_out,
                     void* cuda_stream);

/* Synchronises the device; *out bit 0 = some stream had more 3x3-maximum corner
 * candidates than the context's buffer (width*height/4 per stream) since the last call
 * -- its corners may then differ from the definition; the flag is cleared. */
int dmsgm_klt_get_status(dmsgm_klt_ctx* ctx, unsigned* out);

/* Pyramid levels in use (R39) and kernel launches per dmsgm_klt_estimate. */
int dmsgm_klt_levels(const dmsgm_klt_ctx* ctx);
int dmsgm_klt_kernels_per_estimate(const dmsgm_klt_ctx* ctx);

const char* dmsgm_klt_last_error(const dmsgm_klt_ctx* ctx);
void dmsgm_klt_destroy(dmsgm_klt_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
