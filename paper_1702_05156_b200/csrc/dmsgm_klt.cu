// dmsgm_klt.cu -- host side of the C ABI declared in include/dmsgm_klt.h (SURVEY §8(f)
// NEXT-4: GPU estimation of the homographies the DMSGM step consumes).
//
// Owns the candidate keys, pyramids, tracked points and RANSAC scratch of a batch of S
// streams; every entry point only enqueues kernels on the caller's CUDA stream.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <functional>
#include <stdio.h>
#include <string.h>

#include <new>

#include "dmsgm_klt.h"
#include "dmsgm_klt.cuh"

using namespace dmsgm_klt;

namespace {
thread_local char g_klt_err[512] = "";
}

struct dmsgm_klt_ctx {
    int W, H, S, device;
    dmsgm_klt_params p;
    int nlev;                        // pyramid levels in use (R39)
    int lw[kMaxLevels], lh[kMaxLevels];
    uint8_t* pyr[kMaxLevels];        // level L >= 1: [2][S][lh][lw] (set 0 prev, set 1 next)
    unsigned long long* cand;        // [S][cap]
    int cap;
    unsigned* cand_count;            // [S] } one allocation, cleared per call
    unsigned* maxbits;               // [S] }
    unsigned* overflow;              // [1]
    uint16_t* grid_global;           // [S][gh][gw] or null (grid in shared memory)
    int cell, gw, gh;
    size_t sel_smem;
    int* corners;                    // [2][S][max][2] (slot 1: dmsgm_klt_estimate_seq only)
    int* counts;                     // [2][S]
    float* tracked;                  // [S][max][2]
    uint8_t* status;                 // [S][max]
    double* src;                     // [S][max][2]
    double* dst;
    int* mcount;                     // [S]
    int* iter_counts;                // [S][iters]
    // dmsgm_klt_estimate forks the pyramid (which needs only the frames) onto `side`, beside
    // the corner score / select kernels, and joins before LK
    cudaStream_t side;
    cudaEvent_t ev_fork, ev_pyr;
    // dmsgm_klt_estimate_seq: the frame last passed as `next` (pointer, pitch), the pyramid set
    // and the corner slot that hold its levels and corners
    bool seq_valid;
    const uint8_t* seq_ptr;
    size_t seq_pitch;
    int seq_set, seq_slot;
    char err[512];
};

namespace {

int kfail(dmsgm_klt_ctx* c, int code, const char* fmt, ...) {
    char* buf = c ? c->err : g_klt_err;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, 512, fmt, ap);
    va_end(ap);
    return code;
}

int kcuda(dmsgm_klt_ctx* c, cudaError_t e, const char* what) {
    return kfail(c, DMSGM_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

struct Dev {
    int prev = -1;
    bool ok = true;
    explicit Dev(int d) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != d && cudaSetDevice(d) != cudaSuccess) ok = false;
    }
    ~Dev() {
        int now;
        if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
    }
};

bool params_ok(const dmsgm_klt_params* p, char* why, size_t n) {
    if (!p) { snprintf(why, n, "params is NULL"); return false; }
    // (the pyramid kernel covers two images of every stream in one grid dimension: 2 S <= 65535)
    if (p->num_streams < 1 || p->num_streams > 32767) { snprintf(why, n, "num_streams must be in [1, 32767]"); return false; }
    if (p->max_corners < 4 || p->max_corners > kMaxCorners) { snprintf(why, n, "max_corners must be in [4, %d]", kMaxCorners); return false; }
    if (!(p->quality > 0.0 && p->quality <= 1.0)) { snprintf(why, n, "quality must be in (0, 1]"); return false; }
    if (!(p->min_distance >= 1.0 && p->min_distance <= 4096.0)) { snprintf(why, n, "min_distance must be in [1, 4096]"); return false; }
    if (p->win < 3 || p->win > 32) { snprintf(why, n, "win must be in [3, 32]"); return false; }
    if (p->max_level < 0 || p->max_level > kMaxLevels - 1) { snprintf(why, n, "max_level must be in [0, %d]", kMaxLevels - 1); return false; }
    if (p->max_iters < 1 || p->max_iters > 1000) { snprintf(why, n, "max_iters must be in [1, 1000]"); return false; }
    if (!(p->eps > 0.0f) || !(p->min_eig >= 0.0f)) { snprintf(why, n, "eps must be > 0, min_eig >= 0"); return false; }
    if (p->ransac_iters < 1 || p->ransac_iters > 4096) { snprintf(why, n, "ransac_iters must be in [1, 4096]"); return false; }
    if (!(p->ransac_thresh > 0.0)) { snprintf(why, n, "ransac_thresh must be > 0"); return false; }
    return true;
}

bool img_ok(const dmsgm_klt_ctx* c, const void* p, size_t pitch) { return p && pitch >= (size_t)c->W; }

cudaError_t launch_corners(dmsgm_klt_ctx* c, const uint8_t* frames, size_t pitch, int* corners, int* counts,
                           cudaStream_t st, const std::function<cudaError_t()>& after_score = nullptr) {
    cudaError_t e = cudaMemsetAsync(c->cand_count, 0, 2 * c->S * sizeof(unsigned), st);   // counts + maxbits
    if (e != cudaSuccess) return e;
    ScoreArgs a;
    a.frames = frames; a.fstride = (long long)c->H * (long long)pitch; a.pitch = (int)pitch;
    a.W = c->W; a.H = c->H; a.cand = c->cand; a.cap = c->cap; a.count = c->cand_count; a.maxbits = c->maxbits;
    if ((c->W & 3) == 0 && (pitch & 3) == 0 && ((uintptr_t)frames & 3) == 0) {
        // 4-byte aligned rows: the streaming kernel (the same scores and candidates)
        const int strips = (c->W + 119) / 120;
        klt_score_stream_kernel<<<dim3((strips + kScoreWarps - 1) / kScoreWarps, (c->H + kScoreBand - 1) / kScoreBand,
                                       c->S), 32 * kScoreWarps, 0, st>>>(a);
    } else {
        klt_score_kernel<<<dim3((c->W + kTX - 1) / kTX, (c->H + kTY - 1) / kTY, c->S), 256, 0, st>>>(a);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (after_score && (e = after_score()) != cudaSuccess) return e;
    SelectArgs b;
    b.cand = c->cand; b.cap = c->cap; b.count = c->cand_count; b.maxbits = c->maxbits;
    b.quality = c->p.quality; b.min_dist2 = c->p.min_distance * c->p.min_distance;
    b.W = c->W; b.max_corners = c->p.max_corners;
    b.cell = c->cell; b.gw = c->gw; b.gh = c->gh; b.grid_global = c->grid_global;
    b.corners_out = corners; b.counts_out = counts; b.overflow = c->overflow;
    klt_select_kernel<<<c->S, kSelThreads, c->sel_smem, st>>>(b);
    return cudaGetLastError();
}

// Pyramid levels 1.. of n = 1 or 2 images (each S streams) into pyramid sets dset[i].
cudaError_t launch_pyramid(dmsgm_klt_ctx* c, int n, const uint8_t* const* img, const size_t* pitch, const int* dset,
                           cudaStream_t st) {
    if (c->nlev <= 1) return cudaSuccess;
    PyrArgs pa;
    for (int i = 0; i < 2; ++i) {
        const int j = i < n ? i : 0;
        pa.img0[i] = img[j];
        pa.stride0[i] = (long long)c->H * (long long)pitch[j];
        pa.pitch0[i] = (int)pitch[j];
        pa.dset[i] = dset[j];
        pa.vec[i] = ((uintptr_t)img[j] & 15) == 0 && (pitch[j] & 15) == 0;
    }
    for (int L = 0; L < kMaxLevels; ++L) { pa.lev[L] = c->pyr[L]; pa.w[L] = c->lw[L]; pa.h[L] = c->lh[L]; }
    pa.nlev = c->nlev; pa.S = c->S;
    klt_pyramid_kernel<<<dim3((c->lw[1] + kPyrTX - 1) / kPyrTX, (c->lh[1] + kPyrTY - 1) / kPyrTY, n * c->S), 256, 0,
                         st>>>(pa);
    return cudaGetLastError();
}

// LK of corners from prev (pyramid set pset) to next (set nset); skip_pyramid: the levels
// are already built, else both images' levels are built here into sets 0 / 1
cudaError_t launch_track(dmsgm_klt_ctx* c, const uint8_t* prev, size_t ppitch, const uint8_t* next, size_t npitch,
                         const int* corners, const int* counts, float* tracked, uint8_t* status, cudaStream_t st,
                         bool skip_pyramid = false, int pset = 0, int nset = 1) {
    cudaError_t e;
    if (!skip_pyramid) {
        const uint8_t* img[2] = {prev, next};
        const size_t pit[2] = {ppitch, npitch};
        const int ds[2] = {0, 1};
        if ((e = launch_pyramid(c, 2, img, pit, ds, st)) != cudaSuccess) return e;
        pset = 0; nset = 1;
    }
    LkArgs la;
    for (int L = 0; L < kMaxLevels; ++L) {
        if (L == 0) {
            la.prev[0] = Img{prev, (long long)c->H * (long long)ppitch, (int)ppitch, c->W, c->H};
            la.next[0] = Img{next, (long long)c->H * (long long)npitch, (int)npitch, c->W, c->H};
        } else {
            const long long img = (long long)c->lw[L] * c->lh[L];
            la.prev[L] = Img{c->pyr[L] ? c->pyr[L] + img * c->S * pset : nullptr, img, c->lw[L], c->lw[L], c->lh[L]};
            la.next[L] = Img{c->pyr[L] ? c->pyr[L] + img * c->S * nset : nullptr, img, c->lw[L], c->lw[L], c->lh[L]};
        }
    }
    la.nlev = c->nlev; la.win = c->p.win; la.max_iters = c->p.max_iters; la.max_corners = c->p.max_corners;
    la.eps2 = c->p.eps * c->p.eps; la.min_eig = c->p.min_eig;
    la.corners = corners; la.counts = counts; la.tracked = tracked; la.status = status;
    const dim3 grid((c->p.max_corners + kLkWarps - 1) / kLkWarps, c->S);
    const int ns = (c->p.win * c->p.win + 31) / 32;
    if (ns <= 8) klt_lk_kernel<8><<<grid, 32 * kLkWarps, 0, st>>>(la);
#ifndef DMSGM_LK_WIN20
#define DMSGM_LK_WIN20 1
#endif
    else if (DMSGM_LK_WIN20 && c->p.win == 20) klt_lk_kernel<13, 20><<<grid, 32 * kLkWarps, 0, st>>>(la);   // App. F's Size(20,20)
    else if (ns <= 13) klt_lk_kernel<13><<<grid, 32 * kLkWarps, 0, st>>>(la);
    else klt_lk_kernel<32><<<grid, 32 * kLkWarps, 0, st>>>(la);
    return cudaGetLastError();
}

cudaError_t launch_ransac(dmsgm_klt_ctx* c, const double* src, const double* dst, const int* mcount, double* H,
                          uint8_t* inliers, int* iter_counts, int* ok, cudaStream_t st) {
    RansacArgs r;
    r.src = src; r.dst = dst; r.mcount = mcount; r.max_corners = c->p.max_corners; r.iters = c->p.ransac_iters;
    r.seed = c->p.seed; r.thresh2 = c->p.ransac_thresh * c->p.ransac_thresh; r.iter_counts = iter_counts;
    klt_ransac_kernel<<<dim3((c->p.ransac_iters + kRansacWarps * kRansacPerWarp - 1) / (kRansacWarps * kRansacPerWarp), c->S),
                        32 * kRansacWarps, 0, st>>>(r);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RefitArgs f;
    f.src = src; f.dst = dst; f.mcount = mcount; f.iter_counts = iter_counts; f.max_corners = c->p.max_corners;
    f.iters = c->p.ransac_iters; f.S = c->S; f.seed = c->p.seed; f.thresh2 = r.thresh2;
    f.H_out = H; f.inliers = inliers; f.ok_out = ok;
    klt_refit_kernel<<<(c->S + 3) / 4, 128, 0, st>>>(f);
    return cudaGetLastError();
}

}  // namespace

extern "C" {

int dmsgm_klt_create(int width, int height, const dmsgm_klt_params* p, int device, dmsgm_klt_ctx** out) {
    g_klt_err[0] = 0;
    if (!out) return kfail(nullptr, DMSGM_EINVAL, "out is NULL");
    *out = nullptr;
    char why[256];
    if (!params_ok(p, why, sizeof why)) return kfail(nullptr, DMSGM_EINVAL, "%s", why);
    if (width < 8 || height < 8 || width > 65535 || height > 65535)
        return kfail(nullptr, DMSGM_EINVAL, "frames must be 8..65535 pixels per side");
    Dev g(device);
    if (!g.ok) return kfail(nullptr, DMSGM_ECUDA, "cudaSetDevice(%d) failed", device);
    dmsgm_klt_ctx* c = new (std::nothrow) dmsgm_klt_ctx();
    if (!c) return kfail(nullptr, DMSGM_ENOMEM, "host allocation failed");
    c->W = width; c->H = height; c->S = p->num_streams; c->device = device; c->p = *p;
    // R39: levels while both sizes stay >= win
    c->lw[0] = width; c->lh[0] = height; c->nlev = 1;
    for (int L = 1; L < kMaxLevels; ++L) {
        c->lw[L] = c->lw[L - 1] / 2;
        c->lh[L] = c->lh[L - 1] / 2;
    }
    while (c->nlev <= p->max_level && c->lw[c->nlev] >= p->win && c->lh[c->nlev] >= p->win) ++c->nlev;
    // candidates: at most one 3x3 local maximum per 2x2 pixels unless scores tie on plateaus
    c->cap = (int)(((long long)width * height + 3) / 4);
    if (c->cap < 4096) c->cap = 4096;
    c->cell = (int)ceil(p->min_distance / sqrt(2.0));
    if (c->cell < 1) c->cell = 1;
    c->gw = (width + c->cell - 1) / c->cell;
    c->gh = (height + c->cell - 1) / c->cell;
    const size_t base_smem = (size_t)kBatch * 8 + 256 * 4 + (size_t)kMaxCorners * 8 + (size_t)kBatch * 8;
    const size_t grid_bytes = (size_t)c->gw * c->gh * 2;
    const bool grid_in_smem = base_smem + grid_bytes <= 200 * 1024;
    c->sel_smem = base_smem + (grid_in_smem ? grid_bytes : 0);
    const int M = p->max_corners, S = c->S;
    cudaError_t e = cudaSuccess;
#define KALLOC(ptr, bytes) \
    if (e == cudaSuccess) e = cudaMalloc((void**)&(ptr), (bytes))
    KALLOC(c->cand, (size_t)S * c->cap * sizeof(unsigned long long));
    KALLOC(c->cand_count, 2 * (size_t)S * sizeof(unsigned));
    KALLOC(c->overflow, sizeof(unsigned));
    KALLOC(c->corners, 2 * (size_t)S * M * 2 * sizeof(int));
    KALLOC(c->counts, 2 * (size_t)S * sizeof(int));
    KALLOC(c->tracked, (size_t)S * M * 2 * sizeof(float));
    KALLOC(c->status, (size_t)S * M);
    KALLOC(c->src, (size_t)S * M * 2 * sizeof(double));
    KALLOC(c->dst, (size_t)S * M * 2 * sizeof(double));
    KALLOC(c->mcount, (size_t)S * sizeof(int));
    KALLOC(c->iter_counts, (size_t)S * p->ransac_iters * sizeof(int));
    if (!grid_in_smem) KALLOC(c->grid_global, (size_t)S * grid_bytes);
    for (int L = 1; L < c->nlev; ++L) KALLOC(c->pyr[L], 2 * (size_t)S * c->lw[L] * c->lh[L]);
#undef KALLOC
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_pyr, cudaEventDisableTiming);
    if (e == cudaSuccess) c->maxbits = c->cand_count + S;
    if (e == cudaSuccess) e = cudaMemset(c->overflow, 0, sizeof(unsigned));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(klt_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->sel_smem);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        dmsgm_klt_destroy(c);
        return kfail(nullptr, DMSGM_ENOMEM, "dmsgm_klt_create: %s", cudaGetErrorString(e));
    }
    *out = c;
    return DMSGM_OK;
}

int dmsgm_klt_corners(dmsgm_klt_ctx* c, const uint8_t* frames, size_t pitch, int* corners_out, int* counts_out,
                      void* stream) {
    if (!c) return DMSGM_EINVAL;
    if (!img_ok(c, frames, pitch) || !corners_out || !counts_out) return kfail(c, DMSGM_EINVAL, "bad frames / outputs");
    Dev g(c->device);
    c->seq_valid = false;                        // the candidate buffers are shared
    cudaError_t e = launch_corners(c, frames, pitch, corners_out, counts_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_corners");
    return DMSGM_OK;
}

int dmsgm_klt_track(dmsgm_klt_ctx* c, const uint8_t* prev, size_t ppitch, const uint8_t* next, size_t npitch,
                    const int* corners, const int* counts, float* tracked_out, uint8_t* status_out, void* stream) {
    if (!c) return DMSGM_EINVAL;
    if (!img_ok(c, prev, ppitch) || !img_ok(c, next, npitch) || !corners || !counts || !tracked_out || !status_out)
        return kfail(c, DMSGM_EINVAL, "bad frames / corners / outputs");
    Dev g(c->device);
    c->seq_valid = false;                        // both pyramid sets are overwritten
    cudaError_t e = launch_track(c, prev, ppitch, next, npitch, corners, counts, tracked_out, status_out,
                                 (cudaStream_t)stream);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_track");
    return DMSGM_OK;
}

int dmsgm_klt_ransac(dmsgm_klt_ctx* c, const double* src, const double* dst, const int* counts, double* H_out,
                     uint8_t* inliers_out, int* iter_counts_out, int* ok_out, void* stream) {
    if (!c) return DMSGM_EINVAL;
    if (!src || !dst || !counts || !H_out || ((uintptr_t)src & 7) || ((uintptr_t)dst & 7) || ((uintptr_t)H_out & 7))
        return kfail(c, DMSGM_EINVAL, "bad matches / outputs");
    Dev g(c->device);
    cudaError_t e = launch_ransac(c, src, dst, counts, H_out, inliers_out, iter_counts_out ? iter_counts_out : c->iter_counts,
                                  ok_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_ransac");
    return DMSGM_OK;
}

namespace {
// compact -> RANSAC -> refit of the tracked pairs (corners / counts of the tracked slot)
cudaError_t launch_fit(dmsgm_klt_ctx* c, const int* corners, const int* counts, double* H_out, int* ok_out,
                       cudaStream_t st) {
    CompactArgs ca;
    ca.corners = corners; ca.counts = counts; ca.tracked = c->tracked; ca.status = c->status;
    ca.max_corners = c->p.max_corners; ca.S = c->S; ca.src = c->src; ca.dst = c->dst; ca.mcount = c->mcount;
    klt_compact_kernel<<<(c->S + 3) / 4, 128, 0, st>>>(ca);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = launch_ransac(c, c->src, c->dst, c->mcount, H_out, nullptr, c->iter_counts, ok_out, st);
    return e;
}
int* slot_corners(dmsgm_klt_ctx* c, int slot) { return c->corners + (size_t)slot * c->S * c->p.max_corners * 2; }
int* slot_counts(dmsgm_klt_ctx* c, int slot) { return c->counts + (size_t)slot * c->S; }
}  // namespace

int dmsgm_klt_estimate(dmsgm_klt_ctx* c, const uint8_t* prev, size_t ppitch, const uint8_t* next, size_t npitch,
                       double* H_out, int* ok_out, void* stream) {
    if (!c) return DMSGM_EINVAL;
    if (!img_ok(c, prev, ppitch) || !img_ok(c, next, npitch) || !H_out || ((uintptr_t)H_out & 7))
        return kfail(c, DMSGM_EINVAL, "bad frames / outputs");
    Dev g(c->device);
    c->seq_valid = false;                        // slot 0 and both pyramid sets are overwritten
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    // the pyramid of prev and next on the side stream, forked after the score kernel so that it
    // runs beside the select kernel (32 CTAs: most SMs idle); joined before LK
    auto fork_pyramid = [&]() -> cudaError_t {
        if (c->nlev <= 1) return cudaSuccess;
        cudaError_t fe = cudaEventRecord(c->ev_fork, st);
        if (fe == cudaSuccess) fe = cudaStreamWaitEvent(c->side, c->ev_fork, 0);
        if (fe != cudaSuccess) return fe;
        const uint8_t* img[2] = {prev, next};
        const size_t pit[2] = {ppitch, npitch};
        const int ds[2] = {0, 1};
        if ((fe = launch_pyramid(c, 2, img, pit, ds, c->side)) != cudaSuccess) return fe;
        return cudaEventRecord(c->ev_pyr, c->side);
    };
    if (e == cudaSuccess) e = launch_corners(c, prev, ppitch, c->corners, c->counts, st, fork_pyramid);
    if (e == cudaSuccess && c->nlev > 1) e = cudaStreamWaitEvent(st, c->ev_pyr, 0);
    if (e == cudaSuccess)
        e = launch_track(c, prev, ppitch, next, npitch, c->corners, c->counts, c->tracked, c->status, st, true);
    if (e == cudaSuccess) e = launch_fit(c, c->corners, c->counts, H_out, ok_out, st);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_estimate");
    return DMSGM_OK;
}

int dmsgm_klt_estimate_seq(dmsgm_klt_ctx* c, const uint8_t* prev, size_t ppitch, const uint8_t* next, size_t npitch,
                           double* H_out, int* ok_out, void* stream) {
    if (!c) return DMSGM_EINVAL;
    if (!img_ok(c, prev, ppitch) || !img_ok(c, next, npitch) || !H_out || ((uintptr_t)H_out & 7))
        return kfail(c, DMSGM_EINVAL, "bad frames / outputs");
    Dev g(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    const bool cached = c->seq_valid && c->seq_ptr == prev && c->seq_pitch == ppitch;
    c->seq_valid = false;
    const int pset = cached ? c->seq_set : 0, pslot = cached ? c->seq_slot : 0;
    const int nset = 1 - pset, nslot = 1 - pslot;
    if (!cached) {
        // first frame of a sequence (or a jump): corners and levels of prev, then next's levels
        const uint8_t* img[2] = {prev, next};
        const size_t pit[2] = {ppitch, npitch};
        const int ds[2] = {pset, nset};
        e = launch_corners(c, prev, ppitch, slot_corners(c, pslot), slot_counts(c, pslot), st);
        if (e == cudaSuccess) e = launch_pyramid(c, 2, img, pit, ds, st);
    }
    // the corners of next (the next call's prev) on the side stream, beside the pyramid, LK
    // and the fit of this pair (it waits only for the work already on `cuda_stream`: the
    // previous call read corner slot nslot there); joined at the end, so the call's work is
    // complete when `cuda_stream` is
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    if (e == cudaSuccess) e = launch_corners(c, next, npitch, slot_corners(c, nslot), slot_counts(c, nslot), c->side);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_pyr, c->side);
    if (e == cudaSuccess && cached) {
        const uint8_t* img[1] = {next};
        const size_t pit[1] = {npitch};
        const int ds[1] = {nset};
        e = launch_pyramid(c, 1, img, pit, ds, st);
    }
    if (e == cudaSuccess)
        e = launch_track(c, prev, ppitch, next, npitch, slot_corners(c, pslot), slot_counts(c, pslot), c->tracked,
                         c->status, st, true, pset, nset);
    if (e == cudaSuccess) e = launch_fit(c, slot_corners(c, pslot), slot_counts(c, pslot), H_out, ok_out, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c->ev_pyr, 0);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_estimate_seq");
    c->seq_valid = true;
    c->seq_ptr = next;
    c->seq_pitch = npitch;
    c->seq_set = nset;
    c->seq_slot = nslot;
    return DMSGM_OK;
}

int dmsgm_klt_seq_reset(dmsgm_klt_ctx* c) {
    if (!c) return DMSGM_EINVAL;
    c->seq_valid = false;
    return DMSGM_OK;
}

int dmsgm_klt_get_status(dmsgm_klt_ctx* c, unsigned* out) {
    if (!c || !out) return DMSGM_EINVAL;
    Dev g(c->device);
    unsigned ov = 0;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&ov, c->overflow, sizeof ov, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemset(c->overflow, 0, sizeof ov);
    if (e != cudaSuccess) return kcuda(c, e, "dmsgm_klt_get_status");
    *out = ov ? 1u : 0u;
    return DMSGM_OK;
}

int dmsgm_klt_levels(const dmsgm_klt_ctx* c) { return c ? c->nlev : DMSGM_EINVAL; }

int dmsgm_klt_kernels_per_estimate(const dmsgm_klt_ctx* c) {
    if (!c) return DMSGM_EINVAL;
    return 2 + (c->nlev > 1 ? 1 : 0) + 1 + 1 + 2;   // score, select, pyramid, LK, compact, ransac, refit
}

const char* dmsgm_klt_last_error(const dmsgm_klt_ctx* c) { return c ? c->err : g_klt_err; }

void dmsgm_klt_destroy(dmsgm_klt_ctx* c) {
    if (!c) return;
    Dev g(c->device);
    cudaDeviceSynchronize();
    void* ptrs[] = {c->cand, c->cand_count, c->overflow, c->corners, c->counts, c->tracked, c->status, c->src,
                    c->dst, c->mcount, c->iter_counts, c->grid_global};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    for (int L = 0; L < kMaxLevels; ++L)
        if (c->pyr[L]) cudaFree(c->pyr[L]);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_pyr) cudaEventDestroy(c->ev_pyr);
    delete c;
}

}  // extern "C"
