// dmsgm.cu -- host side of the C ABI declared in include/dmsgm.h.
//
// Owns the device-resident model state (two ping-pong buffers, SoA, fp32,
// [S][6][Hb][Wb]) and per-stream fresh flags (two ping-pong arrays [S]); launches
// the fused step kernel (dmsgm_kernel.cuh) once per frame batch; captures T-step
// batches into CUDA graphs; pipelines host<->device copies for dmsgm_step_host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include "dmsgm.h"
#include "dmsgm_kernel.cuh"
#include "dmsgm_prefilter.cuh"
#include "dmsgm_warp.cuh"

using namespace dmsgm;

namespace {

constexpr int kPipeStreams = 3;
constexpr int kCounterSlots = 64;   // slot 0: dmsgm_step / dmsgm_step_n; 1..: concurrent step_host chunks
constexpr int kRowsPerCta = 4;

struct GraphSlot {
    bool valid = false;
    int T = 0, parity = 0;
    const void* frames = nullptr;
    const void* H = nullptr;
    const void* masks = nullptr;
    size_t fpitch = 0, mpitch = 0;
    cudaGraphExec_t exec = nullptr;
};

thread_local char g_create_err[512] = "";

}  // namespace

struct dmsgm_ctx {
    int W, H, N, Wb, Hb, S, device;
    dmsgm_params p;
    float* state[2];
    uint8_t* fresh[2];
    int cur;
    cudaStream_t capture_stream;
    GraphSlot graphs[2];
    int graph_next;
    // dmsgm_step_host staging
    uint8_t* st_frames;
    uint8_t* st_masks;
    double* st_H;
    size_t st_bytes;   // capacity of st_frames / st_masks (a later dmsgm_set_band may need more)
    cudaEvent_t ev_dev;   // recorded after device-side steps once step_host is in use
    bool dev_pending;     // a device-side step was enqueued since the last step_host call
    cudaStream_t pipe[kPipeStreams];
    cudaEvent_t ev_start;
    cudaEvent_t ev_done[kPipeStreams];   // dmsgm_step_host_async: end of each pipe stream's work
    bool pipe_ready;
    int staged;        // 1: persistent TMA-staged kernel (N = 4, N = 8)
    int staged_ctas;   // resident CTAs of the staged kernel on this device
    int staged_occ;    // register-capped occupancy variant (3 or 4 CTAs/SM)
    unsigned* item_ctr;   // [kCounterSlots] dynamic item counters of the staged kernel (0 between launches)
    int pdl;           // programmatic dependent launch of consecutive steps (DMSGM_PDL=0 disables)
    int gen_bpt;       // register-path kernel at N = 4: forced blocks per thread (0 = automatic)
    int mask_bits;     // DMSGM_MASK_BITS: 1 bit per pixel (staged kernel, whole frame)
    CUtensorMap state_map[2];   // TMA descriptors of the two state buffers (4-D: 96-B chunks of 4 records)
    // row band; whole frame: row0 = 0, rows = Hb, halo = 0, band = 0
    int band, row0, rows, halo;
    int Hp;                      // pixel rows of the frames / masks passed to a step (rows * N)
    unsigned steps;              // completed steps (host count; the device epoch is flags[2])
    unsigned* flags;             // device [3]: from upper, from lower, own epoch (band sync)
    unsigned* status_host;       // host-mapped status word: bit 0 halo overflow, bit 1 peer timeout
    unsigned* status_dev;
    float* peer_state[2][2];     // [side][buffer]: neighbours' state buffers (side 0 upper, 1 lower)
    unsigned* peer_slot[2];      // neighbour's flag word that we signal
    void* ipc_open[2][3];        // IPC mappings to close at destroy
    // preprocessing: Gaussian radius, median radius, taps,
    // and the filtered-frame buffer the step reads ([S][Hp][pf_pitch])
    int pf_g, pf_m;
    float pf_taps[2 * kPfMaxG + 1];
    uint8_t* pf_buf;
    size_t pf_pitch;
    // frame-warp motion compensation: warped-frame buffer
    // ([S][H][pf_pitch-like pitch]) and S identity homographies for the step that follows
    uint8_t* wf_buf;
    size_t wf_pitch;
    double* id_H;
    char err[512];
};

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 4-D view of a state buffer: {24 floats of a chunk, chunks per row, block rows, streams}.
// 3-D view of a frame batch: {width bytes, rows, streams}; box (32 x N x BPT) B x rows x 1.
bool encode_frame_map(const dmsgm_ctx* c, const uint8_t* base, size_t pitch, int count, int box_cols,
                      int box_rows, CUtensorMap* out) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)c->W, (cuuint64_t)c->Hp, (cuuint64_t)count};
    cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * c->Hp};
    cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_state_map(const dmsgm_ctx* c, float* base, int xc, int wrows, CUtensorMap* out) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const int tx = (c->Wb + kTile - 1) / kTile;
    cuuint64_t dims[4] = {(cuuint64_t)kTileFloats, (cuuint64_t)tx, (cuuint64_t)c->Hb, (cuuint64_t)c->S};
    cuuint64_t strides[3] = {(cuuint64_t)kTileFloats * 4, (cuuint64_t)tx * kTileFloats * 4,
                             (cuuint64_t)c->Hb * tx * kTileFloats * 4};
    cuuint32_t box[4] = {(cuuint32_t)kTileFloats, (cuuint32_t)xc, (cuuint32_t)wrows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Persistent TMA-staged kernel (N = 4 / 8): grid = resident CTAs (computed once per context).
template <int N, int BPT, int MINB, bool RULES, bool BAND = false, bool MBITS = false>
cudaError_t launch_staged(dmsgm_ctx* c, const StepArgs& a, const uint8_t* frames, size_t fpitch, int s0,
                          int count, int parity, int slot, cudaStream_t stream, bool early_frames) {
    StagedArgs sa;
    sa.early_frames = early_frames ? 1 : 0;
    sa.tiles_xc = (c->Wb + Staged<N, BPT>::TWB - 1) / Staged<N, BPT>::TWB;
    sa.tiles_y = (c->rows + kCtaY - 1) / kCtaY;
    sa.items = count * sa.tiles_xc * sa.tiles_y;
    sa.s0 = s0;
    sa.ctr = c->item_ctr + slot;
    CUtensorMap fmap;
    if (!encode_frame_map(c, frames, fpitch, count, Staged<N, BPT>::FROW_BYTES, N * kCtaY, &fmap))
        return cudaErrorInvalidValue;
    const int grid = sa.items < c->staged_ctas ? sa.items : c->staged_ctas;
    // programmatic dependent launch: may begin while the previous step drains; the kernel
    // itself waits (griddepcontrol.wait) before touching the state the previous step wrote
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kCtaX, kCtaY + 1, 1);
    cfg.dynamicSmemBytes = Staged<N, BPT>::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, dmsgm_step_staged<N, BPT, MINB, RULES, BAND, MBITS>, a, sa, fmap,
                              c->state_map[parity]);
}

template <int N, int BPT, int MINB>
cudaError_t setup_staged(dmsgm_ctx* c) {
    cudaError_t e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, true, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
    if constexpr (MINB == 3 && (N == 4 || N == 8)) {   // the bit-mask variants (DMSGM_MASK_BITS)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, false, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
    }
    if constexpr (MINB == 3) {   // the band-mode variants (default configuration only)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dmsgm_step_staged<N, BPT, MINB, true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, Staged<N, BPT>::SMEM_BYTES);
    }
    if (e != cudaSuccess) return e;
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dmsgm_step_staged<N, BPT, MINB, false, false>,
                                                      kStagedThreads, Staged<N, BPT>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (e != cudaSuccess) return e;
    // DMSGM_STAGED_CTAS_PER_SM caps the resident CTAs per SM the persistent grid uses (leaves
    // room for a concurrent kernel on another stream; scripts/pf_overlap.py)
    const char* cap = getenv("DMSGM_STAGED_CTAS_PER_SM");
    if (cap && atoi(cap) > 0 && atoi(cap) < per_sm) per_sm = atoi(cap);
    c->staged_ctas = (per_sm > 0 ? per_sm : 1) * sms;
    for (int i = 0; i < 2; ++i)
        if (!encode_state_map(c, c->state[i], Staged<N, BPT>::XC, Staged<N, BPT>::WROWS, &c->state_map[i]))
            return cudaErrorInvalidValue;
    return cudaSuccess;
}

namespace {

int fail(dmsgm_ctx* c, int code, const char* fmt, ...) {
    char* buf = c ? c->err : g_create_err;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, 512, fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(dmsgm_ctx* c, cudaError_t e, const char* what) {
    return fail(c, DMSGM_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

// Scoped device switch (restores the caller's current device).
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int now;
        if (prev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
    }
};

bool params_ok(const dmsgm_params* p, char* why, size_t n) {
    if (!p) { snprintf(why, n, "params is NULL"); return false; }
    if (!(p->theta_s > 0.f) || !(p->theta_d > 0.f)) { snprintf(why, n, "theta_s, theta_d must be > 0"); return false; }
    if (!(p->age_cap >= 1.f) || !(p->age_cap <= 16777216.f)) { snprintf(why, n, "age_cap must be in [1, 2^24]"); return false; }
    if (!(p->var_init >= 0.f) || !isfinite(p->var_init)) { snprintf(why, n, "var_init must be >= 0"); return false; }
    if (!(p->var_floor_match > 0.f) || !(p->var_floor_classify > 0.f)) { snprintf(why, n, "variance floors must be > 0"); return false; }
    if (!(p->decay_lambda >= 0.f) || !(p->decay_var_thresh >= 0.f)) { snprintf(why, n, "decay params must be >= 0"); return false; }
    if (p->num_streams < 1 || p->num_streams > 65535) { snprintf(why, n, "num_streams must be in [1, 65535]"); return false; }
    if (p->update_rule < 0 || p->update_rule > 1) { snprintf(why, n, "update_rule must be 0 or 1"); return false; }
    if (p->classify_rule < 0 || p->classify_rule > 1) { snprintf(why, n, "classify_rule must be 0 or 1"); return false; }
    return true;
}

KParams kparams(const dmsgm_params& p) {
    KParams k;
    k.theta_s = p.theta_s; k.theta_d = p.theta_d; k.var_init = p.var_init; k.age_cap = p.age_cap;
    k.f_m = p.var_floor_match; k.f_c = p.var_floor_classify;
    k.lambda = p.decay_lambda; k.theta_v = p.decay_var_thresh;
    k.update_rule = p.update_rule; k.classify_rule = p.classify_rule;
    const float tmin = p.theta_d * p.var_floor_classify;   // the kernel's fp32 product
    k.interval_may_be_empty = (tmin >= 0.25f) ? 0 : 1;
    return k;
}

size_t plane_elems(const dmsgm_ctx* c) { return (size_t)c->Wb * (size_t)c->Hb; }
int tiles_x_of(const dmsgm_ctx* c) { return (c->Wb + kTile - 1) / kTile; }
// floats of one stream's state in the internal layout [Hb][4*tiles_x][6] (24-byte block records,
// slots mu_A mu_C var_A var_C age_A age_C)
size_t stream_floats(const dmsgm_ctx* c) { return (size_t)c->Hb * tiles_x_of(c) * kTileFloats; }

// public [6][Hb][Wb] <-> internal [Hb][4*tiles_x][6] (host side, not on the hot path)
void to_public(const dmsgm_ctx* c, const float* in, float* out) {
    const size_t pe = plane_elems(c);
    const int tx = tiles_x_of(c);
    for (int p = 0; p < 6; ++p)
        for (int by = 0; by < c->Hb; ++by)
            for (int bx = 0; bx < c->Wb; ++bx)
                out[p * pe + (size_t)by * c->Wb + bx] =
                    in[(size_t)by * tx * kTileFloats + (size_t)bx * kPlanes + rec_slot(p)];
}
void to_internal(const dmsgm_ctx* c, const float* in, float* out) {
    const size_t pe = plane_elems(c);
    const int tx = tiles_x_of(c);
    memset(out, 0, stream_floats(c) * sizeof(float));
    for (int p = 0; p < 6; ++p)
        for (int by = 0; by < c->Hb; ++by)
            for (int bx = 0; bx < c->Wb; ++bx)
                out[(size_t)by * tx * kTileFloats + (size_t)bx * kPlanes + rec_slot(p)] =
                    in[p * pe + (size_t)by * c->Wb + bx];
}

// Blocks per thread strip: a strip row must be 4, 8 or 16 bytes (N*BPT), and Wb % BPT == 0.
int bpt_of(const dmsgm_ctx* c) {
    switch (c->N) {
        case 1: return 4;
        case 2: return 2;
        case 4:
            // DMSGM_GENERIC_BPT = 1 / 2 / 4 at dmsgm_create: blocks per thread of the register-path
            // kernel at N = 4 (32- / 64- / 128-bit pixel-row loads; the SURVEY §8(d) ablation)
            if (c->gen_bpt && c->Wb % c->gen_bpt == 0) return c->gen_bpt;
            return (c->Wb % 2 == 0) ? 2 : 1;
        default: return 1;
    }
}

// R30: normalised Gaussian taps (fp64 exp and normalisation, rounded to fp32)
bool gauss_taps(int size, float sigma, float* taps) {
    if (size < 1 || size % 2 == 0 || size > 2 * kPfMaxG + 1 || !(sigma > 0.0f)) return false;
    const int c = (size - 1) / 2;
    double t[2 * kPfMaxG + 1], sum = 0.0;
    for (int i = 0; i < size; ++i) {
        const double x = (double)(i - c);
        t[i] = exp(-(x * x) / (2.0 * (double)sigma * (double)sigma));
        sum += t[i];
    }
    for (int i = 0; i < size; ++i) taps[i] = (float)(t[i] / sum);
    return true;
}

cudaError_t launch_warp(int W, int H, int count, const uint8_t* in, long long in_stride, size_t in_pitch,
                        const double* Hs, uint8_t* out, long long out_stride, size_t out_pitch, cudaStream_t stream) {
    WarpArgs a;
    a.in = in; a.in_stride = in_stride; a.in_pitch = (int)in_pitch;
    a.out = out; a.out_stride = out_stride; a.out_pitch = (int)out_pitch;
    a.H = Hs; a.W = W; a.Hh = H; a.count = count;
    // persistent: kWarpCtasPerSm CTAs per SM
    // (per device: the dynamic shared-memory opt-in is a per-device function attribute)
    static int sms_of[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& sms = sms_of[dev & 63];
    if (sms == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cudaError_t e = cudaFuncSetAttribute(dmsgm_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarpDynSmem);
        if (e != cudaSuccess) return e;
        sms = n;
    }
    const long long tiles = (long long)((W / 4 + kWarpThreadsX - 1) / kWarpThreadsX) *
                            ((H + kWarpTileY - 1) / kWarpTileY) * count;
    const long long resident = (long long)kWarpCtasPerSm * sms;   // every CTA resident: contiguous tile ranges
    const int grid = (int)(tiles < resident ? tiles : resident);
    if (grid == 0) return cudaSuccess;
    // the frame batch as u16 {W/2, H, streams} for the TMA box copies (16-byte aligned rows
    // and streams required; otherwise the kernel copies every box row by row)
    CUtensorMap map = {};
    a.tma = 0;
    auto enc = tensor_map_encoder();
    if (enc && (in_pitch & 15) == 0 && ((uintptr_t)in & 15) == 0 && (in_stride & 15) == 0) {
        cuuint64_t dims[3] = {(cuuint64_t)W / 2, (cuuint64_t)H, (cuuint64_t)count};
        cuuint64_t strides[2] = {(cuuint64_t)in_pitch, (cuuint64_t)in_stride};
        cuuint32_t box[3] = {(cuuint32_t)kWarpBoxPitch / 2, (cuuint32_t)kWarpTmaRows, 1};
        cuuint32_t es[3] = {1, 1, 1};
        a.tma = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, (void*)in, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    dmsgm_warp_kernel<<<grid, kWarpThreads, kWarpDynSmem, stream>>>(a, map);
    return cudaGetLastError();
}

cudaError_t launch_prefilter(int W, int H, int count, const uint8_t* in, long long in_stride, size_t in_pitch,
                             uint8_t* out, long long out_stride, size_t out_pitch, int g, int m, const float* taps,
                             cudaStream_t stream) {
    PrefilterArgs a;
    a.in = in; a.in_stride = in_stride; a.in_pitch = (int)in_pitch;
    a.out = out; a.out_stride = out_stride; a.out_pitch = (int)out_pitch;
    a.W = W; a.H = H; a.g = g; a.m = m;
    a.one = 1;
    for (int i = 0; i < 2 * kPfMaxG + 1; ++i) a.taps[i] = i < 2 * g + 1 ? taps[i] : 0.0f;
    const int strips = (W + kPfOutW - 1) / kPfOutW;
    const dim3 grid((strips + kPfWarps - 1) / kPfWarps, (H + kPfBand - 1) / kPfBand, count);
#define DMSGM_PF(GG, MM) dmsgm_prefilter_kernel<GG, MM><<<grid, 32 * kPfWarps, 0, stream>>>(a)
    switch (g * 2 + m) {
        case 0: DMSGM_PF(0, 0); break;
        case 1: DMSGM_PF(0, 1); break;
        case 2: DMSGM_PF(1, 0); break;
        case 3: DMSGM_PF(1, 1); break;
        case 4: DMSGM_PF(2, 0); break;
        case 5: DMSGM_PF(2, 1); break;
        case 6: DMSGM_PF(3, 0); break;
        case 7: DMSGM_PF(3, 1); break;
        default: return cudaErrorInvalidValue;
    }
#undef DMSGM_PF
    return cudaGetLastError();
}

template <int N, int BPT>
void launch_kernel(const StepArgs& a, dim3 grid, dim3 block, cudaStream_t stream) {
    dmsgm_step_kernel<N, BPT><<<grid, block, 0, stream>>>(a);
}

// Enqueue one kernel for streams [s0, s0+count) of the batch.  early_frames: the kernel
// preceding this launch on `stream` cannot have written `frames` (StagedArgs::early_frames;
// ignored, i.e. off, when a filter / warp kernel of this context produces the frames).
cudaError_t launch_step(dmsgm_ctx* c, const uint8_t* frames, size_t fpitch, const double* H,
                        uint8_t* masks, size_t mpitch, int s0, int count, int parity,
                        cudaStream_t stream, int slot = 0, bool early_frames = false) {
    if (c->pf_buf || c->wf_buf) early_frames = false;
    if (c->pf_buf) {
        // preprocessing (R34): the filtered frames replace the frames for the whole step
        uint8_t* pf = c->pf_buf + (size_t)s0 * c->Hp * c->pf_pitch;
        cudaError_t e = launch_prefilter(c->W, c->Hp, count, frames, (long long)c->Hp * fpitch, fpitch, pf,
                                         (long long)c->Hp * c->pf_pitch, c->pf_pitch, c->pf_g, c->pf_m, c->pf_taps,
                                         stream);
        if (e != cudaSuccess) return e;
        frames = pf;
        fpitch = c->pf_pitch;
    }
    if (c->wf_buf) {
        // frame-warp motion compensation (R35): frame t resampled into frame t-1's
        // coordinates, then the step with H = I (the models are not warped)
        uint8_t* wf = c->wf_buf + (size_t)s0 * c->Hp * c->wf_pitch;
        cudaError_t e = launch_warp(c->W, c->Hp, count, frames, (long long)c->Hp * fpitch, fpitch, H, wf,
                                    (long long)c->Hp * c->wf_pitch, c->wf_pitch, stream);
        if (e != cudaSuccess) return e;
        frames = wf;
        fpitch = c->wf_pitch;
        H = c->id_H + (size_t)s0 * 9;
    }
    StepArgs a;
    a.frames = frames;
    a.fstride = (long long)c->Hp * (long long)fpitch;
    a.fpitch = (int)fpitch;
    a.mpitch = (int)mpitch;
    a.H = H;
    a.masks = masks;
    a.mstride = (long long)c->Hp * (long long)mpitch;
    const size_t sstride = stream_floats(c);
    a.prev = c->state[parity] + (size_t)s0 * sstride;
    a.next = c->state[parity ^ 1] + (size_t)s0 * sstride;
    a.fresh_in = c->fresh[parity] + s0;
    a.fresh_out = c->fresh[parity ^ 1] + s0;
    a.Wb = c->Wb;
    a.Hb = c->Hb;
    a.row0 = c->row0;
    a.rows = c->rows;
    a.lo = c->band ? (c->row0 - c->halo > 0 ? c->row0 - c->halo : 0) : 0;
    a.hi = c->band ? (c->row0 + c->rows + c->halo < c->Hb ? c->row0 + c->rows + c->halo : c->Hb) : c->Hb;
    a.halo = c->halo;
    a.peer_up = c->peer_state[0][parity ^ 1] ? c->peer_state[0][parity ^ 1] + (size_t)s0 * sstride : nullptr;
    a.peer_dn = c->peer_state[1][parity ^ 1] ? c->peer_state[1][parity ^ 1] + (size_t)s0 * sstride : nullptr;
    a.status = c->status_dev;
    const int bpt = bpt_of(c);
    a.Wstrips = c->Wb / bpt;
    a.tiles_x = tiles_x_of(c);
    a.sstride = (int)sstride;
    a.kp = kparams(c->p);
    dim3 block(kCtaX, kCtaY, 1);
    // each CTA walks kRowsPerCta tile rows of one stream (prefetching the next one)
    const int tiles_y = (c->rows + kCtaY - 1) / kCtaY;
    dim3 grid((a.Wstrips + kCtaX - 1) / kCtaX, (tiles_y + kRowsPerCta - 1) / kRowsPerCta, count);
    if (c->staged) {
        // RULES = the App. E compatibility switches (R27/R28) are on: runtime-switched code;
        // otherwise the default rules are compiled in without branches.
        const bool rules = c->p.update_rule != 0 || c->p.classify_rule != 0;
#define DMSGM_BAND(NN, BB)                                                                                    \
    return rules ? launch_staged<NN, BB, 3, true, true>(c, a, frames, fpitch, s0, count, parity, slot, stream,   \
                                                        early_frames)                                          \
                 : launch_staged<NN, BB, 3, false, true>(c, a, frames, fpitch, s0, count, parity, slot, stream,  \
                                                         early_frames)
        if (c->band) {   // band mode: halo check + neighbour stores compiled in
            if (c->N == 1) { DMSGM_BAND(1, DMSGM_N1_BPT); }
            if (c->N == 2) { DMSGM_BAND(2, 2); }
            if (c->N == 4) { DMSGM_BAND(4, 2); }
            DMSGM_BAND(8, 1);
        }
#undef DMSGM_BAND
#define DMSGM_STAGED(NN, BB, OO)                                                                            \
    return rules ? launch_staged<NN, BB, OO, true>(c, a, frames, fpitch, s0, count, parity, slot, stream,       \
                                                   early_frames)                                               \
                 : launch_staged<NN, BB, OO, false>(c, a, frames, fpitch, s0, count, parity, slot, stream,      \
                                                    early_frames)
#define DMSGM_STAGED_BITS(NN, BB)                                                                          \
    return rules ? launch_staged<NN, BB, 3, true, false, true>(c, a, frames, fpitch, s0, count, parity, slot,  \
                                                              stream, early_frames)                          \
                 : launch_staged<NN, BB, 3, false, false, true>(c, a, frames, fpitch, s0, count, parity, slot, \
                                                               stream, early_frames)
#define DMSGM_STAGED_OCC(NN, BB)                      \
    if (c->mask_bits) { DMSGM_STAGED_BITS(NN, BB); }  \
    if (c->staged_occ == 3) { DMSGM_STAGED(NN, BB, 3); } \
    DMSGM_STAGED(NN, BB, 4)
        if (c->N == 1) { DMSGM_STAGED(1, DMSGM_N1_BPT, 3); }
        if (c->N == 2) { DMSGM_STAGED(2, 2, 3); }
        if (c->N == 4) { DMSGM_STAGED_OCC(4, 2); }
        if (c->N == 8) { DMSGM_STAGED_OCC(8, 1); }
#undef DMSGM_STAGED_OCC
#undef DMSGM_STAGED_BITS
#undef DMSGM_STAGED
    }
    switch (c->N * 16 + bpt) {
        case 1 * 16 + 4: launch_kernel<1, 4>(a, grid, block, stream); break;
        case 2 * 16 + 2: launch_kernel<2, 2>(a, grid, block, stream); break;
        case 4 * 16 + 2: launch_kernel<4, 2>(a, grid, block, stream); break;
        case 4 * 16 + 1: launch_kernel<4, 1>(a, grid, block, stream); break;
        case 4 * 16 + 4: launch_kernel<4, 4>(a, grid, block, stream); break;
        case 8 * 16 + 1: launch_kernel<8, 1>(a, grid, block, stream); break;
        case 16 * 16 + 1: launch_kernel<16, 1>(a, grid, block, stream); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int check_images(dmsgm_ctx* c, const void* frames, size_t fpitch, const void* H, const void* masks,
                 size_t mpitch) {
    if (!frames || !H || !masks) return fail(c, DMSGM_EINVAL, "null frames/homographies/masks pointer");
    if (((uintptr_t)frames & 15) || ((uintptr_t)masks & 15))
        return fail(c, DMSGM_EINVAL, "frames and masks must be 16-byte aligned");
    if ((uintptr_t)H & 7) return fail(c, DMSGM_EINVAL, "homographies must be 8-byte aligned");
    if (fpitch < (size_t)c->W || (fpitch & 15)) return fail(c, DMSGM_EINVAL, "frame_pitch must be >= width and a multiple of 16");
    const size_t mrow = c->mask_bits ? ((size_t)c->W + 7) / 8 : (size_t)c->W;     // bytes of one mask row
    if (mpitch < mrow || (mpitch & 15))
        return fail(c, DMSGM_EINVAL, "mask_pitch must be >= %zu (the mask row) and a multiple of 16", mrow);
    if ((double)fpitch * c->Hp > 2147483647.0 || (double)mpitch * c->Hp > 2147483647.0)
        return fail(c, DMSGM_EINVAL, "one image (pitch x height) must be < 2 GiB");
    return DMSGM_OK;
}

bool has_peers(const dmsgm_ctx* c) { return c->peer_slot[0] || c->peer_slot[1]; }

// Once dmsgm_step_host(_async) is in use, a device-side step records ev_dev so that a
// following dmsgm_step_host_async orders its kernels after it (they read the state it wrote).
int note_device_step(dmsgm_ctx* c, void* stream) {
    if (!c->pipe_ready) return DMSGM_OK;     // the first step_host call waits on the whole stream
    cudaError_t e = cudaEventRecord(c->ev_dev, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaEventRecord");
    c->dev_pending = true;
    return DMSGM_OK;
}


// Enqueue the band signal / wait kernel (one thread).
cudaError_t launch_sync(dmsgm_ctx* c, int signal, int wait, cudaStream_t stream) {
    SyncArgs sa;
    sa.flags = c->flags;
    sa.peer_slot[0] = c->peer_slot[0];
    sa.peer_slot[1] = c->peer_slot[1];
    sa.signal = signal;
    sa.wait = wait;
    const char* tenv = getenv("DMSGM_BAND_TIMEOUT_MS");
    sa.timeout_ns = (unsigned long long)(tenv ? atof(tenv) : 10000.0) * 1000000ull;
    sa.status = c->status_dev;
    dmsgm_band_sync_kernel<<<1, 32, 0, stream>>>(sa);
    return cudaGetLastError();
}

// A halo overflow / peer timeout recorded by an earlier step (host-mapped word, no sync).
int check_status(dmsgm_ctx* c) {
    const unsigned st = c->status_host ? *(volatile unsigned*)c->status_host : 0u;
    if (st & 1u) return fail(c, DMSGM_ESTATE, "row band: a source block lay outside the band's halo (halo too small)");
    if (st & 2u) return fail(c, DMSGM_ECUDA, "row band: timed out waiting for a neighbour's step");
    return DMSGM_OK;
}

void destroy_graphs(dmsgm_ctx* c) {
    for (auto& g : c->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = GraphSlot();
    }
}

}  // namespace

extern "C" {

const char* dmsgm_version(void) { return "dmsgm-b200 0.1 sm_100a"; }

int dmsgm_create(int width, int height, int block, const dmsgm_params* p, int device, dmsgm_ctx** out) {
    g_create_err[0] = 0;
    if (!out) return fail(nullptr, DMSGM_EINVAL, "out is NULL");
    *out = nullptr;
    char why[256];
    if (!params_ok(p, why, sizeof why)) return fail(nullptr, DMSGM_EINVAL, "%s", why);
    if (block != 1 && block != 2 && block != 4 && block != 8 && block != 16)
        return fail(nullptr, DMSGM_EINVAL, "block must be 1, 2, 4, 8 or 16 (got %d)", block);
    if (width <= 0 || height <= 0 || width % block || height % block)
        return fail(nullptr, DMSGM_EINVAL, "width/height must be positive multiples of block (R1)");
    if (width % 4) return fail(nullptr, DMSGM_EINVAL, "width must be a multiple of 4");
    if ((double)(height / block) * ((width / block + 31) / 32) * 192.0 > 2147483647.0)
        return fail(nullptr, DMSGM_EINVAL, "block grid too large (6*Wb*Hb must be < 2^31)");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return fail(nullptr, DMSGM_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, DMSGM_EINVAL, "device %d out of range (%d devices)", device, ndev);
    DeviceGuard g(device);
    if (!g.ok) return fail(nullptr, DMSGM_ECUDA, "cudaSetDevice(%d) failed", device);

    dmsgm_ctx* c = new (std::nothrow) dmsgm_ctx();
    if (!c) return fail(nullptr, DMSGM_ENOMEM, "host allocation failed");
    c->W = width; c->H = height; c->N = block;
    c->Wb = width / block; c->Hb = height / block;
    c->S = p->num_streams; c->device = device; c->p = *p;
    c->band = 0; c->row0 = 0; c->rows = c->Hb; c->halo = 0; c->Hp = c->H;
    const size_t sbytes = (size_t)c->S * stream_floats(c) * sizeof(float);
    for (int i = 0; i < 2; ++i) {
        if ((e = cudaMalloc(&c->state[i], sbytes)) != cudaSuccess ||
            (e = cudaMalloc(&c->fresh[i], (size_t)c->S)) != cudaSuccess) {
            dmsgm_destroy(c);
            return fail(nullptr, DMSGM_ENOMEM, "cudaMalloc of %zu B failed: %s", sbytes, cudaGetErrorString(e));
        }
    }
    {
        const char* kenv = getenv("DMSGM_KERNEL");           // "generic" forces the register-path kernel
        const bool want = !(kenv && strcmp(kenv, "generic") == 0);
        const char* benv = getenv("DMSGM_GENERIC_BPT");
        c->gen_bpt = benv ? atoi(benv) : 0;
        if (c->gen_bpt != 1 && c->gen_bpt != 2 && c->gen_bpt != 4) c->gen_bpt = 0;
        c->staged = 0;
        if (want && block != 16) {   // N = 16: a 512-byte frame row exceeds the TMA box limit
            const char* oenv = getenv("DMSGM_STAGED_OCC");   // 3 or 4 resident CTAs per SM (register cap)
            c->staged_occ = (oenv && atoi(oenv) == 4) ? 4 : 3;
            const char* penv = getenv("DMSGM_PDL");
            c->pdl = !(penv && atoi(penv) == 0);
#define DMSGM_SETUP(NN, BB) (c->staged_occ == 3 ? setup_staged<NN, BB, 3>(c) : setup_staged<NN, BB, 4>(c))
            if (block < 4) c->staged_occ = 3;   // (the 4-CTA variants exist for N = 4 and 8 only)
            e = block == 1 ? setup_staged<1, DMSGM_N1_BPT, 3>(c)
              : block == 2 ? setup_staged<2, 2, 3>(c)
              : block == 4 ? DMSGM_SETUP(4, 2) : DMSGM_SETUP(8, 1);
#undef DMSGM_SETUP
            if (e != cudaSuccess) {
                dmsgm_destroy(c);
                return fail(nullptr, DMSGM_ECUDA, "staged kernel setup: %s", cudaGetErrorString(e));
            }
            c->staged = 1;
        }
    }
    if ((e = cudaMalloc(&c->item_ctr, kCounterSlots * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemset(c->item_ctr, 0, kCounterSlots * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMalloc(&c->flags, 3 * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaHostAlloc(&c->status_host, sizeof(unsigned), cudaHostAllocMapped)) != cudaSuccess ||
        (e = cudaHostGetDevicePointer(&c->status_dev, c->status_host, 0)) != cudaSuccess) {
        dmsgm_destroy(c);
        return fail(nullptr, DMSGM_ENOMEM, "flag allocation failed: %s", cudaGetErrorString(e));
    }
    *c->status_host = 0;
    if ((e = cudaMemset(c->flags, 0, 3 * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemset(c->state[0], 0, sbytes)) != cudaSuccess ||
        (e = cudaMemset(c->state[1], 0, sbytes)) != cudaSuccess ||
        (e = cudaMemset(c->fresh[0], 1, (size_t)c->S)) != cudaSuccess ||
        (e = cudaMemset(c->fresh[1], 1, (size_t)c->S)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess) {
        dmsgm_destroy(c);
        return fail(nullptr, DMSGM_ECUDA, "context init: %s", cudaGetErrorString(e));
    }
    *out = c;
    return DMSGM_OK;
}

int dmsgm_step(dmsgm_ctx* c, const uint8_t* frames, size_t fpitch, const double* H, uint8_t* masks,
               size_t mpitch, void* cuda_stream) {
    if (!c) return DMSGM_EINVAL;
    int rc = check_images(c, frames, fpitch, H, masks, mpitch);
    if (rc) return rc;
    if ((rc = check_status(c))) return rc;
    DeviceGuard g(c->device);
    if (!g.ok) return fail(c, DMSGM_ECUDA, "cudaSetDevice(%d) failed", c->device);
    cudaError_t e = launch_step(c, frames, fpitch, H, masks, mpitch, 0, c->S, c->cur,
                                (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_step launch");
    if ((rc = note_device_step(c, cuda_stream))) return rc;
    c->cur ^= 1;
    c->steps += 1;
    return DMSGM_OK;
}

int dmsgm_step_n(dmsgm_ctx* c, int T, const uint8_t* frames, size_t fpitch, const double* H,
                 uint8_t* masks, size_t mpitch, void* cuda_stream) {
    if (!c) return DMSGM_EINVAL;
    if (T < 1) return fail(c, DMSGM_EINVAL, "T must be >= 1");
    int rc = check_images(c, frames, fpitch, H, masks, mpitch);
    if (rc) return rc;
    if ((rc = check_status(c))) return rc;
    DeviceGuard g(c->device);
    if (!g.ok) return fail(c, DMSGM_ECUDA, "cudaSetDevice(%d) failed", c->device);
    const size_t fframe = (size_t)c->S * c->Hp * fpitch, mframe = (size_t)c->S * c->Hp * mpitch;
    GraphSlot* slot = nullptr;
    for (auto& gs : c->graphs)
        if (gs.valid && gs.T == T && gs.parity == c->cur && gs.frames == frames && gs.H == H &&
            gs.masks == masks && gs.fpitch == fpitch && gs.mpitch == mpitch)
            slot = &gs;
    cudaError_t e;
    if (!slot) {
        slot = &c->graphs[c->graph_next];
        c->graph_next ^= 1;
        if (slot->exec) cudaGraphExecDestroy(slot->exec);
        *slot = GraphSlot();
        cudaGraph_t graph;
        e = cudaStreamBeginCapture(c->capture_stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamBeginCapture");
        int parity = c->cur;
        cudaError_t le = cudaSuccess;
        for (int t = 0; t < T && le == cudaSuccess; ++t) {
            // the frames are graph inputs (written before the graph is launched) and the
            // node before each step is the previous step or band-sync kernel: the producer
            // may load its first frame box before griddepcontrol.wait
            le = launch_step(c, frames + t * fframe, fpitch, H + (size_t)t * c->S * 9, masks + t * mframe,
                             mpitch, 0, c->S, parity, c->capture_stream, 0, true);
            // band mode with neighbours: every step ends with the signal / wait exchange
            if (le == cudaSuccess && has_peers(c)) le = launch_sync(c, 1, 1, c->capture_stream);
            parity ^= 1;
        }
        e = cudaStreamEndCapture(c->capture_stream, &graph);
        if (le != cudaSuccess) return cuda_fail(c, le, "dmsgm_step_n capture launch");
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&slot->exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
        slot->valid = true; slot->T = T; slot->parity = c->cur;
        slot->frames = frames; slot->H = H; slot->masks = masks;
        slot->fpitch = fpitch; slot->mpitch = mpitch;
    }
    e = cudaGraphLaunch(slot->exec, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphLaunch");
    if ((rc = note_device_step(c, cuda_stream))) return rc;
    if (T & 1) c->cur ^= 1;
    c->steps += (unsigned)T;
    return DMSGM_OK;
}

namespace {
int step_host_impl(dmsgm_ctx* c, const uint8_t* hf, size_t fpitch, const double* hH, uint8_t* hm, size_t mpitch,
                   void* cuda_stream, bool async) {
    if (!c) return DMSGM_EINVAL;
    if (!hf || !hH || !hm) return fail(c, DMSGM_EINVAL, "null host pointer");
    if (fpitch < (size_t)c->W) return fail(c, DMSGM_EINVAL, "frame_pitch must be >= width");
    DeviceGuard g(c->device);
    if (!g.ok) return fail(c, DMSGM_ECUDA, "cudaSetDevice(%d) failed", c->device);
    cudaError_t e;
    const size_t dpitch = ((size_t)c->W + 15) & ~(size_t)15;
    const size_t fimg = (size_t)c->Hp * dpitch;
    const size_t mrow = c->mask_bits ? ((size_t)c->W + 7) / 8 : (size_t)c->W;   // bytes per mask row
    const size_t dmpitch = (mrow + 15) & ~(size_t)15, mimg = (size_t)c->Hp * dmpitch;
    if (mpitch < mrow) return fail(c, DMSGM_EINVAL, "mask_pitch must be >= %zu (the mask row)", mrow);
    int rc = check_status(c);
    if (rc) return rc;
    bool first = false;
    if (!c->pipe_ready) {
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaStreamCreateWithFlags(&c->pipe[i], cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_fail(c, e, "cudaStreamCreate");
        if ((e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&c->ev_dev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(c, e, "cudaEventCreate");
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(c, e, "cudaEventCreate");
        c->pipe_ready = true;
        first = true;
    }
    const size_t nb = (size_t)c->S * fimg;
    if (nb > c->st_bytes) {
        // (re)allocate: the first call, or a band / whole-frame switch that made images taller;
        // earlier async steps may still read / write the old buffers
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaStreamSynchronize(c->pipe[i])) != cudaSuccess) return cuda_fail(c, e, "staging sync");
        if (c->st_frames) cudaFree(c->st_frames);
        if (c->st_masks) cudaFree(c->st_masks);
        c->st_frames = nullptr;
        c->st_masks = nullptr;
        c->st_bytes = 0;
        if ((e = cudaMalloc(&c->st_frames, nb)) != cudaSuccess || (e = cudaMalloc(&c->st_masks, nb)) != cudaSuccess) {
            if (c->st_frames) cudaFree(c->st_frames);
            c->st_frames = nullptr;
            c->st_masks = nullptr;
            return fail(c, DMSGM_ENOMEM, "staging cudaMalloc failed: %s", cudaGetErrorString(e));
        }
        c->st_bytes = nb;
    }
    if (!c->st_H && (e = cudaMalloc(&c->st_H, (size_t)c->S * 9 * sizeof(double))) != cudaSuccess) {
        c->st_H = nullptr;
        return fail(c, DMSGM_ENOMEM, "staging cudaMalloc failed: %s", cudaGetErrorString(e));
    }
    if (!async || first) {
        // ordered after the caller's earlier work on cuda_stream
        if ((e = cudaEventRecord(c->ev_start, (cudaStream_t)cuda_stream)) != cudaSuccess)
            return cuda_fail(c, e, "cudaEventRecord");
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaStreamWaitEvent(c->pipe[i], c->ev_start, 0)) != cudaSuccess)
                return cuda_fail(c, e, "cudaStreamWaitEvent");
    } else if (c->dev_pending) {
        // an async step after device-side steps: its kernels read the state those wrote
        // (waiting on the last one, not on all of cuda_stream, keeps consecutive async
        // steps pipelined)
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaStreamWaitEvent(c->pipe[i], c->ev_dev, 0)) != cudaSuccess)
                return cuda_fail(c, e, "cudaStreamWaitEvent");
    }
    c->dev_pending = false;
    // chunks of streams: H2D(k) || kernel(k-1) || D2H(k-2) across the pipe streams
    const char* cenv = getenv("DMSGM_HOST_CHUNKS");
    int nchunks = cenv ? atoi(cenv) : 8;
    if (nchunks < 1) nchunks = 1;
    if (nchunks > c->S) nchunks = c->S;
    const int per = (c->S + nchunks - 1) / nchunks;
    const int parity = c->cur;
    for (int s0 = 0, k = 0; s0 < c->S; s0 += per, ++k) {
        const int cnt = (c->S - s0) < per ? (c->S - s0) : per;
        cudaStream_t st = c->pipe[k % kPipeStreams];
        uint8_t* df = c->st_frames + (size_t)s0 * fimg;
        uint8_t* dm = c->st_masks + (size_t)s0 * mimg;
        if ((e = cudaMemcpy2DAsync(df, dpitch, hf + (size_t)s0 * c->Hp * fpitch, fpitch, c->W, (size_t)cnt * c->Hp,
                                   cudaMemcpyHostToDevice, st)) != cudaSuccess)
            return cuda_fail(c, e, "H2D frames");
        if ((e = cudaMemcpyAsync(c->st_H + (size_t)s0 * 9, hH + (size_t)s0 * 9, (size_t)cnt * 9 * sizeof(double),
                                 cudaMemcpyHostToDevice, st)) != cudaSuccess)
            return cuda_fail(c, e, "H2D homographies");
        // chunks run concurrently on the pipe streams: each its own item-counter slot
        if ((e = launch_step(c, df, dpitch, c->st_H + (size_t)s0 * 9, dm, dmpitch, s0, cnt, parity, st,
                             1 + k % (kCounterSlots - 1))) != cudaSuccess)
            return cuda_fail(c, e, "dmsgm_step_host launch");
        if ((e = cudaMemcpy2DAsync(hm + (size_t)s0 * c->Hp * mpitch, mpitch, dm, dmpitch, mrow, (size_t)cnt * c->Hp,
                                   cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return cuda_fail(c, e, "D2H masks");
    }
    if (async) {
        // work enqueued later on cuda_stream (and a sync on it) sees this step complete;
        // the next async step's chunk k follows this one's chunk k on the same pipe stream
        for (int i = 0; i < kPipeStreams; ++i) {
            if ((e = cudaEventRecord(c->ev_done[i], c->pipe[i])) != cudaSuccess ||
                (e = cudaStreamWaitEvent((cudaStream_t)cuda_stream, c->ev_done[i], 0)) != cudaSuccess)
                return cuda_fail(c, e, "dmsgm_step_host_async events");
        }
    } else {
        for (int i = 0; i < kPipeStreams; ++i)
            if ((e = cudaStreamSynchronize(c->pipe[i])) != cudaSuccess) return cuda_fail(c, e, "dmsgm_step_host sync");
    }
    c->cur ^= 1;
    c->steps += 1;
    return DMSGM_OK;
}
}  // namespace

int dmsgm_step_host(dmsgm_ctx* c, const uint8_t* hf, size_t fpitch, const double* hH, uint8_t* hm,
                    size_t mpitch, void* cuda_stream) {
    return step_host_impl(c, hf, fpitch, hH, hm, mpitch, cuda_stream, false);
}

int dmsgm_step_host_async(dmsgm_ctx* c, const uint8_t* hf, size_t fpitch, const double* hH, uint8_t* hm,
                          size_t mpitch, void* cuda_stream) {
    return step_host_impl(c, hf, fpitch, hH, hm, mpitch, cuda_stream, true);
}

int dmsgm_reset(dmsgm_ctx* c, int stream) {
    if (!c) return DMSGM_EINVAL;
    if (stream < -1 || stream >= c->S) return fail(c, DMSGM_ESTATE, "stream %d out of range", stream);
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_reset sync");
    if (stream == -1) e = cudaMemset(c->fresh[c->cur], 1, (size_t)c->S);
    else e = cudaMemset(c->fresh[c->cur] + stream, 1, 1);
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_reset memset");
    return DMSGM_OK;
}

int dmsgm_get_state(dmsgm_ctx* c, int stream, float* out) {
    if (!c || !out) return c ? fail(c, DMSGM_EINVAL, "null output") : DMSGM_EINVAL;
    if (stream < 0 || stream >= c->S) return fail(c, DMSGM_ESTATE, "stream %d out of range", stream);
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_get_state sync");
    const size_t n = stream_floats(c);
    float* tmp = (float*)malloc(n * sizeof(float));
    if (!tmp) return fail(c, DMSGM_ENOMEM, "host allocation failed");
    e = cudaMemcpy(tmp, c->state[c->cur] + (size_t)stream * n, n * sizeof(float), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) to_public(c, tmp, out);
    free(tmp);
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_get_state copy");
    return DMSGM_OK;
}

int dmsgm_set_state(dmsgm_ctx* c, int stream, const float* in) {
    if (!c || !in) return c ? fail(c, DMSGM_EINVAL, "null input") : DMSGM_EINVAL;
    if (stream < 0 || stream >= c->S) return fail(c, DMSGM_ESTATE, "stream %d out of range", stream);
    const size_t pe = plane_elems(c);
    for (int m = 0; m < 2; ++m) {
        const float* mu = in + (size_t)(3 * m) * pe;
        const float* var = mu + pe;
        const float* age = var + pe;
        for (size_t i = 0; i < pe; ++i) {
            if (!(mu[i] >= 0.f && mu[i] <= 255.f) || !(var[i] >= 0.f && isfinite(var[i])) ||
                !(age[i] >= 0.f && age[i] <= c->p.age_cap))
                return fail(c, DMSGM_EINVAL, "invalid state value at model %d index %zu", m, i);
        }
    }
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_state sync");
    const size_t n = stream_floats(c);
    float* tmp = (float*)malloc(n * sizeof(float));
    if (!tmp) return fail(c, DMSGM_ENOMEM, "host allocation failed");
    to_internal(c, in, tmp);
    e = cudaMemcpy(c->state[c->cur] + (size_t)stream * n, tmp, n * sizeof(float), cudaMemcpyHostToDevice);
    free(tmp);
    if (e == cudaSuccess) e = cudaMemset(c->fresh[c->cur] + stream, 0, 1);
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_state copy");
    return DMSGM_OK;
}

int dmsgm_is_initialised(dmsgm_ctx* c, int stream) {
    if (!c) return DMSGM_EINVAL;
    if (stream < 0 || stream >= c->S) return fail(c, DMSGM_ESTATE, "stream %d out of range", stream);
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "sync");
    uint8_t f = 1;
    e = cudaMemcpy(&f, c->fresh[c->cur] + stream, 1, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "copy");
    return f ? 0 : 1;
}

int dmsgm_get_info(const dmsgm_ctx* c, dmsgm_info* out) {
    if (!c || !out) return DMSGM_EINVAL;
    out->width = c->W; out->height = c->H; out->block = c->N;
    out->blocks_x = c->Wb; out->blocks_y = c->Hb; out->num_streams = c->S;
    out->kernels_per_step = (has_peers(c) ? 2 : 1) + (c->pf_buf ? 1 : 0) + (c->wf_buf ? 1 : 0);
    out->band_row0 = c->row0; out->band_rows = c->rows; out->band_halo = c->halo;
    out->state_bytes = (size_t)c->S * stream_floats(c) * sizeof(float);
    // frame read (1 B/px) + mask write (1 B/px) + state read + write (2 x 24 B per block)
    // (band mode: the band's rows, plus the halo rows stored into each neighbour)
    const int nb = (c->peer_slot[0] ? 1 : 0) + (c->peer_slot[1] ? 1 : 0);
    // (DMSGM_MASK_BITS: the mask write is ceil(W/8) B per row)
    const double mask_row = c->mask_bits ? (double)((c->W + 7) / 8) : (double)c->W;
    out->algorithmic_bytes_per_frame = ((double)c->W + mask_row) * c->Hp + 2.0 * 24.0 * (double)c->Wb * c->rows +
                                       24.0 * (double)c->Wb * c->halo * nb;
    // preprocessing as its own kernel: + read the frame + write the filtered frame
    if (c->pf_buf) out->algorithmic_bytes_per_frame += 2.0 * c->W * c->Hp;
    if (c->wf_buf) out->algorithmic_bytes_per_frame += 2.0 * c->W * c->Hp;     // frame warp: read + write
    if (c->staged)
        snprintf(out->kernel, sizeof out->kernel, "dmsgm_step_staged<%d,%d,%d%s> (TMA, persistent)", c->N,
                 c->N == 8 ? 1 : (c->N == 1 ? DMSGM_N1_BPT : 2), c->staged_occ, c->mask_bits ? ",bits" : "");
    else
        snprintf(out->kernel, sizeof out->kernel, "dmsgm_step_kernel<%d,%d>", c->N, bpt_of(c));
    if (c->staged && c->band)
        snprintf(out->kernel, sizeof out->kernel, "dmsgm_step_staged<%d,%d,3,band> (TMA, persistent)",
                 c->N, c->N == 8 ? 1 : (c->N == 1 ? DMSGM_N1_BPT : 2));
    return DMSGM_OK;
}

// ---- preprocessing ----

int dmsgm_prefilter(int width, int height, int count, const uint8_t* in, size_t in_pitch, uint8_t* out,
                    size_t out_pitch, int gauss_size, float gauss_sigma, int median_radius, void* stream) {
    float taps[2 * kPfMaxG + 1];
    if (!in || !out || width < 4 || width % 4 || height < 1 || count < 1 || in_pitch < (size_t)width ||
        out_pitch < (size_t)width || (out_pitch & 3) || ((uintptr_t)out & 3) || (in_pitch & 3) || ((uintptr_t)in & 3))
        return DMSGM_EINVAL;
    if (median_radius < 0 || median_radius > 1 || !gauss_taps(gauss_size, gauss_sigma, taps)) return DMSGM_EINVAL;
    cudaError_t e = launch_prefilter(width, height, count, in, (long long)height * in_pitch, in_pitch, out,
                                     (long long)height * out_pitch, out_pitch, (gauss_size - 1) / 2, median_radius,
                                     taps, (cudaStream_t)stream);
    return e == cudaSuccess ? DMSGM_OK : DMSGM_ECUDA;
}

int dmsgm_set_prefilter(dmsgm_ctx* c, int gauss_size, float gauss_sigma, int median_radius) {
    if (!c) return DMSGM_EINVAL;
    float taps[2 * kPfMaxG + 1];
    if (median_radius < 0 || median_radius > 1 || !gauss_taps(gauss_size, gauss_sigma, taps))
        return fail(c, DMSGM_EINVAL, "gauss_size must be 1, 3, 5 or 7, sigma > 0, median_radius 0 or 1");
    if (c->band) return fail(c, DMSGM_ESTATE, "preprocessing is not supported in row-band mode");
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_prefilter sync");
    destroy_graphs(c);
    const bool on = gauss_size > 1 || median_radius > 0;
    if (c->pf_buf && !on) {
        cudaFree(c->pf_buf);
        c->pf_buf = nullptr;
    }
    if (on && !c->pf_buf) {
        c->pf_pitch = ((size_t)c->W + 15) & ~(size_t)15;
        if ((e = cudaMalloc(&c->pf_buf, (size_t)c->S * c->H * c->pf_pitch)) != cudaSuccess) {
            c->pf_buf = nullptr;
            return fail(c, DMSGM_ENOMEM, "filtered-frame buffer: %s", cudaGetErrorString(e));
        }
    }
    c->pf_g = (gauss_size - 1) / 2;
    c->pf_m = median_radius;
    for (int i = 0; i < 2 * kPfMaxG + 1; ++i) c->pf_taps[i] = i < gauss_size ? taps[i] : 0.0f;
    return DMSGM_OK;
}

// ---- frame-warp motion compensation ----

int dmsgm_warp_frames(int width, int height, int count, const uint8_t* in, size_t in_pitch,
                      const double* homographies, uint8_t* out, size_t out_pitch, void* stream) {
    if (!in || !out || !homographies || width < 4 || width % 4 || height < 1 || count < 1 ||
        in_pitch < (size_t)width || out_pitch < (size_t)width || (in_pitch & 3) || (out_pitch & 3) ||
        ((uintptr_t)in & 3) || ((uintptr_t)out & 3) || ((uintptr_t)homographies & 7))
        return DMSGM_EINVAL;
    cudaError_t e = launch_warp(width, height, count, in, (long long)height * in_pitch, in_pitch, homographies, out,
                                (long long)height * out_pitch, out_pitch, (cudaStream_t)stream);
    return e == cudaSuccess ? DMSGM_OK : DMSGM_ECUDA;
}

int dmsgm_set_mask_format(dmsgm_ctx* c, int format) {
    if (!c) return DMSGM_EINVAL;
    if (format != DMSGM_MASK_BYTES && format != DMSGM_MASK_BITS)
        return fail(c, DMSGM_EINVAL, "format must be DMSGM_MASK_BYTES or DMSGM_MASK_BITS");
    if (format == DMSGM_MASK_BITS &&
        (!c->staged || c->staged_occ != 3 || (c->N != 4 && c->N != 8) || c->Wb % kCtaX != 0 || c->band))
        return fail(c, DMSGM_EINVAL, "bit masks need the staged kernel (block 4 or 8, width / block a multiple of "
                                     "32) in whole-frame mode");
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_mask_format sync");
    destroy_graphs(c);
    c->mask_bits = format == DMSGM_MASK_BITS ? 1 : 0;
    return DMSGM_OK;
}

int dmsgm_set_motion(dmsgm_ctx* c, int mode) {
    if (!c) return DMSGM_EINVAL;
    if (mode != DMSGM_MC_MODELS && mode != DMSGM_MC_FRAME)
        return fail(c, DMSGM_EINVAL, "mode must be DMSGM_MC_MODELS (0) or DMSGM_MC_FRAME (1)");
    if (mode == DMSGM_MC_FRAME && c->band) return fail(c, DMSGM_ESTATE, "frame warping is not supported in row-band mode");
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_motion sync");
    destroy_graphs(c);
    if (mode == DMSGM_MC_MODELS) {
        if (c->wf_buf) cudaFree(c->wf_buf);
        if (c->id_H) cudaFree(c->id_H);
        c->wf_buf = nullptr;
        c->id_H = nullptr;
        return DMSGM_OK;
    }
    if (!c->wf_buf) {
        c->wf_pitch = ((size_t)c->W + 15) & ~(size_t)15;
        double* hid = (double*)malloc((size_t)c->S * 9 * sizeof(double));
        if (!hid) return fail(c, DMSGM_ENOMEM, "host allocation failed");
        for (int s = 0; s < c->S; ++s)
            for (int i = 0; i < 9; ++i) hid[9 * s + i] = (i % 4 == 0) ? 1.0 : 0.0;
        if ((e = cudaMalloc(&c->wf_buf, (size_t)c->S * c->H * c->wf_pitch)) != cudaSuccess ||
            (e = cudaMalloc(&c->id_H, (size_t)c->S * 9 * sizeof(double))) != cudaSuccess ||
            (e = cudaMemcpy(c->id_H, hid, (size_t)c->S * 9 * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess) {
            free(hid);
            if (c->wf_buf) cudaFree(c->wf_buf);
            if (c->id_H) cudaFree(c->id_H);
            c->wf_buf = nullptr;
            c->id_H = nullptr;
            return fail(c, DMSGM_ENOMEM, "warped-frame buffer: %s", cudaGetErrorString(e));
        }
        free(hid);
    }
    return DMSGM_OK;
}

// ---- row band ----

namespace {
void detach(dmsgm_ctx* c, int side) {
    for (int k = 0; k < 3; ++k)
        if (c->ipc_open[side][k]) {
            cudaIpcCloseMemHandle(c->ipc_open[side][k]);
            c->ipc_open[side][k] = nullptr;
        }
    c->peer_state[side][0] = c->peer_state[side][1] = nullptr;
    c->peer_slot[side] = nullptr;
}

int band_side_ok(dmsgm_ctx* c, int side) {
    if (side != 0 && side != 1) return fail(c, DMSGM_EINVAL, "side must be 0 (above) or 1 (below)");
    if (!c->band) return fail(c, DMSGM_ESTATE, "dmsgm_set_band first");
    if (side == 0 && c->row0 == 0) return fail(c, DMSGM_ESTATE, "the band starts at row 0: no band above");
    if (side == 1 && c->row0 + c->rows == c->Hb) return fail(c, DMSGM_ESTATE, "the band ends at the last row: no band below");
    if (c->halo < 1) return fail(c, DMSGM_ESTATE, "a band with neighbours needs halo >= 1");
    return DMSGM_OK;
}
}  // namespace

int dmsgm_set_band(dmsgm_ctx* c, int row0, int rows, int halo) {
    if (!c) return DMSGM_EINVAL;
    if (row0 < 0 || rows < 1 || row0 + rows > c->Hb)
        return fail(c, DMSGM_EINVAL, "band rows [%d, %d) outside [0, %d)", row0, row0 + rows, c->Hb);
    if (halo < 0 || halo > rows) return fail(c, DMSGM_EINVAL, "halo must be in [0, rows]");
    if ((c->pf_buf || c->wf_buf) && !(row0 == 0 && rows == c->Hb && halo == 0))
        return fail(c, DMSGM_ESTATE, "preprocessing / frame warping is not supported in row-band mode");
    if (c->mask_bits && !(row0 == 0 && rows == c->Hb && halo == 0))
        return fail(c, DMSGM_ESTATE, "bit masks are not supported in row-band mode");
    DeviceGuard g(c->device);
    if (!g.ok) return fail(c, DMSGM_ECUDA, "cudaSetDevice(%d) failed", c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_set_band sync");
    destroy_graphs(c);
    detach(c, 0);
    detach(c, 1);
    const bool whole = row0 == 0 && rows == c->Hb && halo == 0;
    if (!whole && c->staged && c->staged_occ != 3) {
        // the band kernels exist in the default configuration only
        e = c->N == 4 ? setup_staged<4, 2, 3>(c) : setup_staged<8, 1, 3>(c);   // (N < 4 is always 3)
        if (e != cudaSuccess) return cuda_fail(c, e, "band kernel setup");
        c->staged_occ = 3;
    }
    c->band = whole ? 0 : 1;
    c->row0 = row0;
    c->rows = rows;
    c->halo = halo;
    c->Hp = rows * c->N;
    c->steps = 0;
    *c->status_host = 0;
    if ((e = cudaMemset(c->flags, 0, 3 * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemset(c->fresh[0], 1, (size_t)c->S)) != cudaSuccess ||
        (e = cudaMemset(c->fresh[1], 1, (size_t)c->S)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess)
        return cuda_fail(c, e, "dmsgm_set_band reset");
    return DMSGM_OK;
}

int dmsgm_get_buffers(const dmsgm_ctx* c, dmsgm_buffers* out) {
    if (!c || !out) return DMSGM_EINVAL;
    out->state[0] = c->state[0];
    out->state[1] = c->state[1];
    out->flags = c->flags;
    out->parity = c->cur;
    out->steps = c->steps;
    out->row_bytes = (size_t)tiles_x_of(c) * kTileFloats * sizeof(float);
    out->stream_bytes = stream_floats(c) * sizeof(float);
    return DMSGM_OK;
}

int dmsgm_attach_peer(dmsgm_ctx* c, int side, const dmsgm_buffers* p) {
    if (!c) return DMSGM_EINVAL;
    int rc = band_side_ok(c, side);
    if (rc) return rc;
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_attach_peer sync");
    destroy_graphs(c);
    detach(c, side);
    if (!p) return DMSGM_OK;
    if (!p->state[0] || !p->state[1] || !p->flags) return fail(c, DMSGM_EINVAL, "null peer buffer");
    if (p->stream_bytes != stream_floats(c) * sizeof(float))
        return fail(c, DMSGM_EINVAL, "peer state size differs (width/block/height mismatch)");
    if (p->parity != c->cur || p->steps != c->steps)
        return fail(c, DMSGM_ESTATE, "peer is not in lockstep (parity %d/%d, steps %u/%u)", p->parity, c->cur,
                    p->steps, c->steps);
    c->peer_state[side][0] = (float*)p->state[0];
    c->peer_state[side][1] = (float*)p->state[1];
    // the neighbour above listens on its flags[1] ("from below"), the one below on flags[0]
    c->peer_slot[side] = (unsigned*)p->flags + (side == 0 ? 1 : 0);
    return DMSGM_OK;
}

int dmsgm_get_ipc_handles(const dmsgm_ctx* c, void* out, size_t n) {
    if (!c || !out || n < DMSGM_IPC_BYTES) return DMSGM_EINVAL;
    static_assert(3 * sizeof(cudaIpcMemHandle_t) <= DMSGM_IPC_BYTES, "IPC handle size");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h[3];
    cudaError_t e;
    if ((e = cudaIpcGetMemHandle(&h[0], c->state[0])) != cudaSuccess ||
        (e = cudaIpcGetMemHandle(&h[1], c->state[1])) != cudaSuccess ||
        (e = cudaIpcGetMemHandle(&h[2], c->flags)) != cudaSuccess)
        return cuda_fail(const_cast<dmsgm_ctx*>(c), e, "cudaIpcGetMemHandle");
    memset(out, 0, DMSGM_IPC_BYTES);
    memcpy(out, h, sizeof h);
    return DMSGM_OK;
}

int dmsgm_attach_peer_ipc(dmsgm_ctx* c, int side, const void* handles, size_t n) {
    if (!c) return DMSGM_EINVAL;
    if (!handles || n < DMSGM_IPC_BYTES) return fail(c, DMSGM_EINVAL, "need %d bytes of handles", DMSGM_IPC_BYTES);
    int rc = band_side_ok(c, side);
    if (rc) return rc;
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_attach_peer_ipc sync");
    destroy_graphs(c);
    detach(c, side);
    cudaIpcMemHandle_t h[3];
    memcpy(h, handles, sizeof h);
    for (int k = 0; k < 3; ++k) {
        if ((e = cudaIpcOpenMemHandle(&c->ipc_open[side][k], h[k], cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess) {
            detach(c, side);
            return cuda_fail(c, e, "cudaIpcOpenMemHandle");
        }
    }
    c->peer_state[side][0] = (float*)c->ipc_open[side][0];
    c->peer_state[side][1] = (float*)c->ipc_open[side][1];
    c->peer_slot[side] = (unsigned*)c->ipc_open[side][2] + (side == 0 ? 1 : 0);
    return DMSGM_OK;
}

namespace {
int band_sync_common(dmsgm_ctx* c, int signal, int wait, void* stream, const char* what) {
    if (!c) return DMSGM_EINVAL;
    if (!c->band) return fail(c, DMSGM_ESTATE, "%s: dmsgm_set_band first", what);
    DeviceGuard g(c->device);
    if (!g.ok) return fail(c, DMSGM_ECUDA, "cudaSetDevice(%d) failed", c->device);
    if (!has_peers(c)) return DMSGM_OK;   // a lone band: nothing to exchange
    cudaError_t e = launch_sync(c, signal, wait, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, what);
    return DMSGM_OK;
}
}  // namespace

int dmsgm_band_signal(dmsgm_ctx* c, void* s) { return band_sync_common(c, 1, 0, s, "dmsgm_band_signal"); }
int dmsgm_band_wait(dmsgm_ctx* c, void* s) { return band_sync_common(c, 0, 1, s, "dmsgm_band_wait"); }
int dmsgm_band_sync(dmsgm_ctx* c, void* s) { return band_sync_common(c, 1, 1, s, "dmsgm_band_sync"); }

int dmsgm_get_status(dmsgm_ctx* c, unsigned* out) {
    if (!c || !out) return DMSGM_EINVAL;
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "dmsgm_get_status sync");
    *out = *(volatile unsigned*)c->status_host;
    *(volatile unsigned*)c->status_host = 0;
    return DMSGM_OK;
}

int dmsgm_band_halo_needed(int width, int height, int block, const double* H, int count, int row0, int rows,
                           int* out) {
    if (!H || !out || count < 1 || block < 1 || width <= 0 || height <= 0 || width % block || height % block)
        return DMSGM_EINVAL;
    const int N = block, Wb = width / N, Hb = height / N;
    if (row0 < 0 || rows < 1 || row0 + rows > Hb) return DMSGM_EINVAL;
    int need = 0;
    for (int s = 0; s < count; ++s) {
        const double* h = H + 9 * s;
        // S1 as the kernel computes it (R17: fp32 displacement form, explicit fma)
        float gg[9];
        for (int j = 0; j < 9; ++j) gg[j] = (float)((j == 0 || j == 4 || j == 8) ? h[j] - 1.0 : h[j]);
        for (int bj = row0; bj < row0 + rows; ++bj) {
            const float Y = (float)(N * bj) + 0.5f * (float)N;
            const float r7 = fmaf(gg[7], Y, gg[8]), r1 = fmaf(gg[1], Y, gg[2]), r4 = fmaf(gg[4], Y, gg[5]);
            for (int bi = 0; bi < Wb; ++bi) {
                const float X = (float)(N * bi) + 0.5f * (float)N;
                const float e = fmaf(gg[6], X, r7);
                const float w = 1.0f + e;
                if (!(w > 0x1p-100f && w < 0x1p100f)) continue;   // exposed (R5)
                const float px = fmaf(-X, e, fmaf(gg[0], X, r1));
                const float py = fmaf(-Y, e, fmaf(gg[3], X, r4));
                const float rwN = (1.0f / w) * (1.0f / (float)N);
                const float ex = px * rwN, ey = py * rwN;
                if (!(fabsf(ex) < 1048576.0f && fabsf(ey) < 1048576.0f)) continue;
                const float tx = 0.5f + ex, ty = 0.5f + ey;
                const float fxf = floorf(tx), fyf = floorf(ty);
                const float du = (tx - fxf) - 0.5f, dv = (ty - fyf) - 0.5f;
                const int iu = bi + (int)fxf, iv = bj + (int)fyf;
                const int ju = du > 0.0f ? iu + 1 : iu - 1, jv = dv > 0.0f ? iv + 1 : iv - 1;
                const float a = fabsf(du), b = fabsf(dv);
                const float wt[4] = {(1.0f - a) * (1.0f - b), a * (1.0f - b), (1.0f - a) * b, a * b};
                const int cxs[4] = {iu, ju, iu, ju}, cys[4] = {iv, iv, jv, jv};
                for (int k = 0; k < 4; ++k) {
                    if (!(wt[k] > 0.0f) || cxs[k] < 0 || cxs[k] >= Wb || cys[k] < 0 || cys[k] >= Hb) continue;
                    const int d = cys[k] < row0 ? row0 - cys[k] : (cys[k] >= row0 + rows ? cys[k] - (row0 + rows - 1) : 0);
                    if (d > need) need = d;
                }
            }
        }
    }
    *out = need;
    return DMSGM_OK;
}

const char* dmsgm_last_error(const dmsgm_ctx* c) { return c ? c->err : g_create_err; }

void dmsgm_destroy(dmsgm_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    destroy_graphs(c);
    for (int side = 0; side < 2; ++side)
        for (int k = 0; k < 3; ++k)
            if (c->ipc_open[side][k]) cudaIpcCloseMemHandle(c->ipc_open[side][k]);
    if (c->flags) cudaFree(c->flags);
    if (c->pf_buf) cudaFree(c->pf_buf);
    if (c->wf_buf) cudaFree(c->wf_buf);
    if (c->id_H) cudaFree(c->id_H);
    if (c->item_ctr) cudaFree(c->item_ctr);
    if (c->status_host) cudaFreeHost(c->status_host);
    for (int i = 0; i < 2; ++i) {
        if (c->state[i]) cudaFree(c->state[i]);
        if (c->fresh[i]) cudaFree(c->fresh[i]);
    }
    if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
    if (c->pipe_ready) {
        for (int i = 0; i < kPipeStreams; ++i) {
            cudaStreamDestroy(c->pipe[i]);
            cudaEventDestroy(c->ev_done[i]);
        }
        cudaEventDestroy(c->ev_start);
        cudaEventDestroy(c->ev_dev);
    }
    if (c->st_frames) cudaFree(c->st_frames);
    if (c->st_masks) cudaFree(c->st_masks);
    if (c->st_H) cudaFree(c->st_H);
    delete c;
}

}  // extern "C"
