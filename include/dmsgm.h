/*
 * dmsgm.h -- C ABI of the B200 (sm_100a) grid-block Dual-Mode SGM motion-masking step.
 *
 * Method: Henderson & Vertescher, "An Analysis of Parallelized Motion Masking Using
 * Dual-Mode Single Gaussian Models" (arXiv 1702.05156), implementing Yi et al.'s
 * DMSGM.  Per frame and per N x N grid block G_i (Eq. 4 kept general, |G_i| = N^2):
 *   (1) warp + mix the previous models through the frame's homography into the
 *       "previous values after motion compensation" mu~, sigma~, alpha~ (§2.2 P:89,
 *       §2.4; readings R2-R7), with age decay (R7);
 *   (2) block mean M_i (Eq. 4);
 *   (3) dual-mode update: match tests Eqs. 8-9, mean/variance/age updates
 *       Eqs. 3, 5, 6, 7, candidate reset, swap Eq. 10;
 *   (4) per-pixel mask (App. E, variance reading R14).
 * DESIGN.md §2 lists every reading; §3 the HBM layout.
 *
 * Conventions
 *  - All calls return an int status (DMSGM_OK or a negative DMSGM_E* code).  On error
 *    a message is available from dmsgm_last_error(ctx) (or dmsgm_last_error(NULL) for
 *    dmsgm_create failures).  Argument errors are detected synchronously and enqueue
 *    nothing.  Asynchronous device faults surface as DMSGM_ECUDA at a later call.
 *  - Unless stated otherwise every buffer pointer is a DEVICE pointer on the context's
 *    device, owned by the caller; the library never frees or retains them.  The
 *    context owns its model state (two ping-pong buffers of 6 fp32 planes per stream),
 *    per-stream "fresh" flags, any captured CUDA graph and the staging buffers of
 *    dmsgm_step_host.
 *  - A context is not thread-safe; use one context per device and host thread.
 *  - Images are 8-bit grayscale, row-major, `width` pixels per row with a row pitch
 *    in bytes.  Pitches must be multiples of 16 and >= width; frame/mask base pointers
 *    must be 16-byte aligned; homography pointers 8-byte aligned.
 *  - Streams: `num_streams` (S) independent video streams are processed per call;
 *    stream s of a batch lives at byte offset s*height*pitch.
 */
#ifndef DMSGM_H
#define DMSGM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMSGM_OK       0
#define DMSGM_EINVAL  -1 /* null pointer, width%block or height%block != 0, width%4 != 0,
                            block not in {1,2,4,8,16}, bad params, misaligned pointer/pitch,
                            invalid state values in dmsgm_set_state                      */
#define DMSGM_ENOMEM  -2 /* device or host allocation failed                             */
#define DMSGM_ECUDA   -3 /* CUDA runtime error (no device, launch failure, async fault)   */
#define DMSGM_ESTATE  -4 /* stream index out of range; row band: halo too small, band/peer
                            configuration invalid                                         */

/* Parameters of the method (all explicit; there are no hidden defaults in the kernel). */
typedef struct {
    float theta_s;            /* match gate of Eqs. 8-9; paper gives no value, 4 (R15) */
    float theta_d;            /* classification gate THETA_D of App. E P:657 (R14); 4 (R15)          */
    float var_init;           /* variance of a reset / new model, 255 (App. E)          */
    float age_cap;            /* age cap, 30 (App. E AGE_THRESH P:616); must be in [1, 2^24]    */
    float var_floor_match;    /* variance floor in the match test, 0.1 (App. E)         */
    float var_floor_classify; /* variance floor in classification, 0.25 (App. E)               */
    float decay_lambda;       /* age-decay rate lambda (R7); 0 disables the decay bitwise             */
    float decay_var_thresh;   /* age-decay variance threshold theta_v (R7)                           */
    int   num_streams;        /* S >= 1: independent streams batched per call                         */
    int   update_rule;        /* 0: Eqs. 3/5/7 (R10); 1: App. E code rule alpha = 1/age (R27)         */
    int   classify_rule;      /* 0: theta_d*max(var_A, f_c) (R14); 1: App. E theta_d*max(f_c, I) (R28) */
} dmsgm_params;

typedef struct dmsgm_ctx dmsgm_ctx;

/* Static facts about a context (for the harness: bytes, launch counts). */
typedef struct {
    int width, height, block;      /* W, H, N                                   */
    int blocks_x, blocks_y;        /* Wb = W/N, Hb = H/N                        */
    int num_streams;               /* S                                         */
    int kernels_per_step;          /* kernel launches per step: 1 (+1 band sync with neighbours) */
    int band_row0, band_rows, band_halo; /* row band (0, Hb, 0 for the whole frame)    */
    size_t state_bytes;            /* one state buffer (internal chunk-SoA layout, padded to Wb%4) */
    double algorithmic_bytes_per_frame; /* frame read + mask write + state read+write, one stream
                                           (band: its rows + the halo rows sent to neighbours;
                                           DMSGM_MASK_BITS: the mask write is ceil(W/8) B/row) */
    char kernel[64];               /* the kernel dmsgm_step launches, e.g. "dmsgm_step_staged<4,2>" */
} dmsgm_info;

/* Create a context on CUDA device `device` (W, H in pixels, N = block).  Allocates two
 * state buffers (S*6*Hb*Wb fp32 each) and the fresh flags; all streams start "fresh"
 * (their first step initialises A = C = (M, var_init, 1), R8).  No kernel is launched. */
int dmsgm_create(int width, int height, int block, const dmsgm_params* p, int device,
                 dmsgm_ctx** out);

/* One frame for all S streams.  frames: u8 [S][height][frame_pitch] (device);
 * homographies: f64 [S][9] (device), row-major, mapping frame-t continuous pixel
 * coordinates to frame-(t-1) coordinates (R3), ignored for streams on their first
 * frame but always read; masks: u8 [S][height][mask_pitch] (device), written with
 * {0,255}.  Enqueued on `cuda_stream` (a cudaStream_t, NULL = legacy default stream);
 * returns after the enqueue (asynchronous).  Exactly one kernel launch.
 * Stream ordering: the launch uses programmatic dependent launch (it may start while the
 * previous kernel on `cuda_stream` drains), but every global-memory read of the step --
 * frames, homographies, state -- follows griddepcontrol.wait, so inputs written by ANY
 * earlier work on `cuda_stream` (a copy, a producer kernel, the previous step) are seen
 * exactly as with plain stream order. */
int dmsgm_step(dmsgm_ctx* ctx, const uint8_t* frames, size_t frame_pitch,
               const double* homographies, uint8_t* masks, size_t mask_pitch, void* cuda_stream);

/* T consecutive frames per stream: frames u8 [T][S][height][frame_pitch], homographies
 * f64 [T][S][9], masks u8 [T][S][height][mask_pitch] (device).  The T launches are
 * captured once into a CUDA graph (re-captured when T or a pointer/pitch changes) and
 * replayed on `cuda_stream`.  Asynchronous.  The graph as a whole is ordered after earlier
 * work on `cuda_stream`; inside it, step t+1's producer loads its first frame tile before
 * waiting for step t (the frames of all T steps are inputs of the graph, so nothing inside
 * it writes them) -- unless preprocessing or frame warping is on, whose kernels write the
 * frames the step reads.  The frames, homographies and masks must not alias. */
int dmsgm_step_n(dmsgm_ctx* ctx, int T, const uint8_t* frames, size_t frame_pitch,
                 const double* homographies, uint8_t* masks, size_t mask_pitch, void* cuda_stream);

/* End-to-end step from HOST memory: frames u8 [S][height][frame_pitch] and homographies
 * f64 [S][9] in host memory (pinned for full speed), masks u8 [S][height][mask_pitch]
 * written to host memory.  Streams are split into chunks whose H2D copy, kernel and
 * D2H copy are pipelined over internal CUDA streams ordered after `cuda_stream`.
 * SYNCHRONOUS: returns when the masks are in host memory.  Device staging buffers are
 * allocated on the first call, grown when the images get taller (dmsgm_set_band), and
 * kept until dmsgm_destroy. */
int dmsgm_step_host(dmsgm_ctx* ctx, const uint8_t* host_frames, size_t frame_pitch,
                    const double* host_homographies, uint8_t* host_masks, size_t mask_pitch,
                    void* cuda_stream);

/* The same, ASYNCHRONOUS: returns after enqueueing.  Consecutive async calls pipeline
 * (step t+1's uploads overlap step t's kernels and downloads; each chunk of streams
 * follows its own previous chunk); work enqueued later on `cuda_stream`, and a sync of
 * it, sees the step complete.  It is ordered after this context's earlier dmsgm_step /
 * dmsgm_step_n calls (it reads the state they write) and, on the context's first host
 * step, after all earlier work on `cuda_stream`; it does NOT wait for other earlier work
 * on `cuda_stream` (its inputs are host memory).  host_frames / host_homographies must
 * stay unchanged and host_masks unread until then. */
int dmsgm_step_host_async(dmsgm_ctx* ctx, const uint8_t* host_frames, size_t frame_pitch,
                          const double* host_homographies, uint8_t* host_masks, size_t mask_pitch,
                          void* cuda_stream);

/* Mark stream `stream` (or all, -1) fresh: its next step re-initialises (R8).
 * Synchronises the device first. */
int dmsgm_reset(dmsgm_ctx* ctx, int stream);

/* Copy stream `stream`'s current models to HOST memory: f32 [6][Hb][Wb], planes
 * mu_A, var_A, age_A, mu_C, var_C, age_C.  Synchronises the device first. */
int dmsgm_get_state(dmsgm_ctx* ctx, int stream, float* host_out);

/* Load stream `stream`'s models from HOST memory (same layout) and mark it initialised.
 * Values must be finite with 0 <= mu <= 255, var >= 0, 0 <= age <= age_cap (else
 * DMSGM_EINVAL, nothing written).  Synchronises the device first. */
int dmsgm_set_state(dmsgm_ctx* ctx, int stream, const float* host_in);

/* 1 if stream `stream` has been initialised (stepped at least once or set), else 0;
 * negative on error.  Synchronises the device first. */
int dmsgm_is_initialised(dmsgm_ctx* ctx, int stream);

int dmsgm_get_info(const dmsgm_ctx* ctx, dmsgm_info* out);

/* Last error message of `ctx` ("" if none); with ctx == NULL, the last create error of
 * the calling thread.  The string lives until the next call on the same context. */
const char* dmsgm_last_error(const dmsgm_ctx* ctx);

/* Free all device/host resources of the context (synchronises the device). */
void dmsgm_destroy(dmsgm_ctx* ctx);

/* ------------------------------------------------------------------------------------
 * Frame preprocessing: PAPER.md §2.1 pre-processes
 * the incoming frame with "a Gaussian filter and a median filter"; §3.3.1
 * and App. C/D give the implementation.  DESIGN.md readings R30-R34: separable Gaussian
 * of odd size gauss_size (1 = off, 3, 5, 7) and std gauss_sigma > 0 in fp32 (row pass,
 * then column pass rounded once to u8), then the clamped 3x3 median (median_radius 1;
 * 0 = off); image borders clamp.
 * ------------------------------------------------------------------------------------ */

/* Filter every step's frames before the step (the filtered frame replaces the frame for
 * S4 and S8).  Allocates a filtered-frame buffer of S * height * round_up(width, 16)
 * bytes; one extra kernel per step.  (1, *, 0) switches it off.  Not available in
 * row-band mode (DMSGM_ESTATE).  Synchronises the device. */
int dmsgm_set_prefilter(dmsgm_ctx* ctx, int gauss_size, float gauss_sigma, int median_radius);

/* Stand-alone filter of `count` frames: in u8 [count][height][in_pitch], out u8
 * [count][height][out_pitch] (device; width % 4 == 0; in, out 4-byte aligned, in_pitch % 4
 * == 0, out_pitch % 4 == 0).  Enqueued on cuda_stream; DMSGM_EINVAL for bad arguments. */
int dmsgm_prefilter(int width, int height, int count, const uint8_t* in, size_t in_pitch, uint8_t* out,
                    size_t out_pitch, int gauss_size, float gauss_sigma, int median_radius, void* cuda_stream);

/* ------------------------------------------------------------------------------------
 * Motion-compensation mode.  DMSGM_MC_MODELS (default, the
 * north_star and §2.4): the previous models are warped and mixed through H (S1-S3).
 * DMSGM_MC_FRAME: the paper's own code path (App. F, warpPerspective with
 * INTER_LINEAR | WARP_INVERSE_MAP; §3.1.3): the current frame is resampled into the
 * previous frame's coordinates (bilinear, borders repeated; R35-R37) and the
 * models are updated in place (H = I); masks are then in the previous frame's coordinates.
 * ------------------------------------------------------------------------------------ */
#define DMSGM_MC_MODELS 0
#define DMSGM_MC_FRAME  1

/* Select the mode (one extra kernel per step and a warped-frame buffer of S * height *
 * round_up(width, 16) bytes in DMSGM_MC_FRAME).  Not in row-band mode (DMSGM_ESTATE).
 * Synchronises the device. */
int dmsgm_set_motion(dmsgm_ctx* ctx, int mode);

/* ------------------------------------------------------------------------------------
 * Mask format.  DMSGM_MASK_BYTES (default): one byte per pixel, 0 or 255 (App. E
 * writes 255 for foreground).  DMSGM_MASK_BITS: one bit per pixel, 1 = foreground, row y
 * of stream s at masks + s*height*mask_pitch + y*mask_pitch, pixel x in byte x/8, bit x%8
 * (least significant first: numpy.packbits(mask > 0, bitorder="little")); mask_pitch >=
 * ceil(width / 8), a multiple of 16.  The same decisions, an eighth of the bytes -- what
 * dmsgm_step_host(_async) then copies back over PCIe.  Requires the staged kernel (block 4
 * or 8, width / block a multiple of 32) in whole-frame mode; DMSGM_EINVAL otherwise.
 * ------------------------------------------------------------------------------------ */
#define DMSGM_MASK_BYTES 0
#define DMSGM_MASK_BITS  1

/* Select the mask format of every later step call.  Synchronises the device. */
int dmsgm_set_mask_format(dmsgm_ctx* ctx, int format);

/* Stand-alone frame warp of `count` frames: in / out u8 [count][height][pitch] (device,
 * width % 4 == 0, 4-byte aligned pitches and bases), homographies f64 [count][9]
 * (device, frame t -> frame t-1 as for the step).  Enqueued on cuda_stream. */
int dmsgm_warp_frames(int width, int height, int count, const uint8_t* in, size_t in_pitch,
                      const double* homographies, uint8_t* out, size_t out_pitch, void* cuda_stream);

/* ------------------------------------------------------------------------------------
 * Row-band split of one large frame over several GPUs (
 * north_star: "a single very large frame may optionally be split into row bands with
 * a one-block-row halo exchanged over NVLink").  Only S1-S2 read neighbouring blocks
 * (the warp/mix of the previous models, §2.4), so a band needs the previous
 * state of `halo` block rows above and below it; S4-S8 touch only its own pixels.
 *
 * Every band context keeps the full-grid state layout (rows outside band + halo are
 * never read).  Its step kernel writes its first / last `halo` rows of the new state
 * into the upper / lower neighbour's next-state buffer as well (direct stores, peer
 * memory over NVLink / NVSwitch when the neighbour is on another GPU), and
 * dmsgm_band_sync then publishes "step done" to the neighbours and waits for theirs.
 * Results are bitwise equal to the whole-frame step.
 * ------------------------------------------------------------------------------------ */

/* Make `ctx` process block rows [row0, row0 + rows) only (0 <= row0, rows >= 1,
 * row0 + rows <= Hb; 0 <= halo <= rows).  Afterwards frames and masks passed to the step
 * calls hold the band's pixel rows only: u8 [S][rows*N][pitch], pixel row 0 = global
 * pixel row row0*N; homographies stay in whole-frame coordinates.  Detaches any
 * neighbour, zeroes the sync counters and status, marks every stream fresh.  (0, Hb, 0)
 * restores whole-frame mode.  All bands of one frame must use the same halo.
 * Synchronises the device. */
int dmsgm_set_band(dmsgm_ctx* ctx, int row0, int rows, int halo);

/* Device buffers a neighbour needs (same process). */
typedef struct {
    void* state[2];      /* the two state ping-pong buffers (internal layout)            */
    void* flags;         /* 3 x u32 sync words                                            */
    int parity;          /* index of the buffer holding the current state                */
    unsigned steps;      /* steps completed by this context                               */
    size_t row_bytes;    /* bytes of one block row of one stream in a state buffer        */
    size_t stream_bytes; /* bytes of one stream in a state buffer                         */
} dmsgm_buffers;
int dmsgm_get_buffers(const dmsgm_ctx* ctx, dmsgm_buffers* out);

/* Attach the neighbour band on `side` (0: the band above, ending at row0; 1: the band
 * below, starting at row0 + rows) from its dmsgm_get_buffers (pointers valid on this
 * context's device: same device, or peer access enabled); NULL detaches.  Both bands
 * must have the same width, block, num_streams and halo, and must be stepped in
 * lockstep (same number of steps) from their set_band on. */
int dmsgm_attach_peer(dmsgm_ctx* ctx, int side, const dmsgm_buffers* peer);

/* Cross-process form: DMSGM_IPC_BYTES bytes of CUDA IPC handles for the two state
 * buffers and the sync words (written to `out`), and the attach that opens them. */
#define DMSGM_IPC_BYTES 192
int dmsgm_get_ipc_handles(const dmsgm_ctx* ctx, void* out, size_t out_bytes);
int dmsgm_attach_peer_ipc(dmsgm_ctx* ctx, int side, const void* handles, size_t bytes);

/* After a step: publish this context's step count to its neighbours (signal), wait
 * until every attached neighbour has completed the same step (wait), or both in one
 * launch (sync).  One single-thread kernel on `cuda_stream`; asynchronous.  A wait
 * longer than DMSGM_BAND_TIMEOUT_MS (env, default 10000) gives up and records a
 * timeout in the status word.  dmsgm_step_n issues the sync after every step itself
 * when neighbours are attached.  With several bands on ONE stream, enqueue all steps,
 * then all signals, then all waits (a wait blocks the stream behind it). */
int dmsgm_band_signal(dmsgm_ctx* ctx, void* cuda_stream);
int dmsgm_band_wait(dmsgm_ctx* ctx, void* cuda_stream);
int dmsgm_band_sync(dmsgm_ctx* ctx, void* cuda_stream);

/* Status word (synchronises the device), then clears it: bit 0 = a positive-weight
 * source lay outside the band + halo (the masks / state of that step are not valid),
 * bit 1 = a neighbour wait timed out.  Any set bit also makes the next step call fail
 * (DMSGM_ESTATE / DMSGM_ECUDA) until it is read here or the band is set again. */
int dmsgm_get_status(dmsgm_ctx* ctx, unsigned* out);

/* Host helper: the halo (block rows) that band [row0, row0 + rows) needs for the given
 * HOST homographies f64 [count][9]: max distance of a positive-weight source row from
 * the band, by the same fp32 projection as the kernel (S1, R17). */
int dmsgm_band_halo_needed(int width, int height, int block, const double* host_homographies, int count,
                           int row0, int rows, int* out);

/* Library version string, e.g. "dmsgm-b200 0.1 sm_100a". */
const char* dmsgm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DMSGM_H */
