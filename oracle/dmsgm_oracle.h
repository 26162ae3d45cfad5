/*
 * dmsgm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle of the grid-block Dual-Mode SGM step
 * (Henderson & Vertescher, arXiv 1702.05156, §2.2-2.4, Eqs. 3-10, App. E; with
 * Yi et al.'s grid-block form kept general, |G_i| = N*N).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code, header or constant with the CUDA product
 * path (paper_1702_05156_b200/).  DESIGN.md §2 lists every reading (R1-R28)
 * the oracle follows where the paper is silent.
 *
 * All pointers are HOST pointers.  Return codes: 0 ok, -1 invalid argument,
 * -2 out of memory.
 */
#ifndef DMSGM_ORACLE_H
#define DMSGM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    float theta_s;            /* match gate theta_s, Eqs. 8-9              */
    float theta_d;            /* classification gate THETA_D, App. E P:657 (R14)      */
    float var_init;           /* candidate reset variance, 255         */
    float age_cap;            /* age cap, 30 (App. E AGE_THRESH P:616)          */
    float var_floor_match;    /* 0.1, App. E                              */
    float var_floor_classify; /* 0.25, App. E                                    */
    float decay_lambda;       /* age decay rate (R7); 0 disables                       */
    float decay_var_thresh;   /* age decay variance threshold theta_v (R7)             */
    int   num_streams;        /* S                                                     */
    int   update_rule;        /* 0 = Eqs. 3/5/7 (R10); 1 = App. E code rule (R27)      */
    int   classify_rule;      /* 0 = theta_d*max(var_A,f_c) (R14); 1 = App. E theta_d*max(f_c,I) (R28) */
    int   form;               /* arithmetic form: DMSGM_ORACLE_FORM_KERNEL_ORDER (dmsgm_oracle.c, the
                                 canonical fp32 order the CUDA path reproduces bitwise) or
                                 DMSGM_ORACLE_FORM_PLAIN (dmsgm_plain.c, SURVEY §8(c) literally) */
} dmsgm_oracle_params;

#define DMSGM_ORACLE_FORM_KERNEL_ORDER 0
#define DMSGM_ORACLE_FORM_PLAIN 1

typedef struct dmsgm_oracle_ctx dmsgm_oracle_ctx;

int  dmsgm_oracle_create(int width, int height, int block, const dmsgm_oracle_params* p,
                         dmsgm_oracle_ctx** out);
void dmsgm_oracle_destroy(dmsgm_oracle_ctx* ctx);

/* One frame for every stream.  frames: u8 [S][height][frame_pitch];
 * homographies: f64 [S][9] (frame t -> frame t-1, R3); masks: u8 [S][height][mask_pitch]. */
int dmsgm_oracle_step(dmsgm_oracle_ctx* ctx, const uint8_t* frames, size_t frame_pitch,
                      const double* homographies, uint8_t* masks, size_t mask_pitch);

/* One frame for ONE stream s (frame/H/mask pointers address that stream only).
 * Streams are independent; distinct s may be stepped from different threads.
 * The caller must step every stream once before calling dmsgm_oracle_commit(). */
int dmsgm_oracle_step_stream(dmsgm_oracle_ctx* ctx, int s, const uint8_t* frame, size_t frame_pitch,
                             const double* homography, uint8_t* mask, size_t mask_pitch);
/* Finish a frame stepped stream-by-stream: marks all streams initialised, flips buffers. */
int dmsgm_oracle_commit(dmsgm_oracle_ctx* ctx);

int dmsgm_oracle_reset(dmsgm_oracle_ctx* ctx, int stream /* -1 = all */);
/* [6][Hb][Wb] fp32: mu_A var_A age_A mu_C var_C age_C */
int dmsgm_oracle_get_state(const dmsgm_oracle_ctx* ctx, int stream, float* out);
int dmsgm_oracle_set_state(dmsgm_oracle_ctx* ctx, int stream, const float* in);
int dmsgm_oracle_is_initialised(const dmsgm_oracle_ctx* ctx, int stream);

/* Step S1 alone for block (bi, bj) under homography h[9] (exposed for the
 * polygon-overlap pin P12).  Returns 1 if the block is exposed (R5), else 0
 * (footprint inside the grid) or 2 (footprint clipped by the border: the step
 * renormalises by *sum_w, R6), and fills src_x[4], src_y[4] (source block
 * indices, order self/H/V/HV), weight[4] (raw overlap areas, out-of-range
 * sources zeroed) and *sum_w. */
int dmsgm_oracle_mix_weights(int width, int height, int block, const double* h, int bi, int bj,
                             int* src_x, int* src_y, float* weight, float* sum_w);

/* Test probe: while buf is set, every step also writes, per stream and block, the tilde
 * models after S1-S3 (mu~_A var~_A age~_A mu~_C var~_C age~_C), the block mean M and
 * 1/0 for live/exposed into buf [S][8][Hb][Wb] (host memory owned by the caller). */
int dmsgm_oracle_set_tilde_probe(dmsgm_oracle_ctx* ctx, float* buf);

/* The decay factor exp(-lambda * d) of reading R18 (form 0; exposed for its pin). */
float dmsgm_oracle_decay_factor(float lambda, float d);

/* Frame preprocessing of §2.1 / §3.3.1 / App. C-D (prefilter_oracle.c, readings R30-R34):
 * the normalised Gaussian taps (size odd <= 15, sigma > 0), and the separable Gaussian
 * (gauss_size 1 = off) followed by the clamped median of radius median_radius
 * (0 = off, <= 4) of one u8 frame. */
int dmsgm_oracle_gauss_taps(int size, float sigma, float* taps);
int dmsgm_oracle_prefilter(int width, int height, const uint8_t* in, size_t in_pitch, uint8_t* out,
                           size_t out_pitch, int gauss_size, float gauss_sigma, int median_radius);

/* Frame-warp motion compensation of App. F (warp_oracle.c, readings R35-R37): out
 * samples `in` (frame t) at H^-1 of every pixel centre, H = h[9] the step's homography
 * (frame t -> frame t-1, R3); bilinear, border pixels repeated. */
int dmsgm_oracle_warp_frame(int width, int height, const uint8_t* in, size_t in_pitch, const double* h,
                            uint8_t* out, size_t out_pitch);

#ifdef __cplusplus
}
#endif
#endif
