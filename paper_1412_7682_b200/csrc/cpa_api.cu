// cpa_api.cu -- the C ABI of libcpa.so (declared and documented in
// include/cpa.h): context, argument validation, TMA descriptor set-up and the
// launch sequence of the hot path
//   cpa_accumulate: a3 model sums -> a4 trace moments -> a5 cross term
//   cpa_finalize:   a8 Eq. (1) + per-(b,k) max|rho| -> a9 per-byte ranking
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/cpa.h"
#include "kernels.h"
#include "tables.h"

namespace {

thread_local char g_err[512] = "";

cpa_status fail(cpa_status s, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

cpa_status cuda_fail(cudaError_t e, const char *where)
{
    return fail(CPA_E_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CUDA_TRY(expr, where)                        \
    do {                                             \
        cudaError_t e_ = (expr);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)
// calls that synchronise, read back or allocate cannot be part of a captured graph
#define NO_CAPTURE(c)                                                                              \
    do {                                                                                           \
        if ((c)->capturing)                                                                        \
            return fail(CPA_E_INVALID_ARG, "%s: not allowed while capturing a graph", __func__);   \
    } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

using PFN_addr_range = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
PFN_addr_range get_addr_range()
{
    static PFN_addr_range fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_addr_range)p;
    }
    return fn;
}

constexpr int64_t kMaxTraces = 1LL << 23;  // exact-int64 bound of Eq. (1), see DESIGN.md
constexpr int32_t kMaxSamples = 1 << 22;
constexpr int64_t kStageBytes = 256LL << 20;  // bytes per staging chunk (cpa_accumulate_host / unaligned input)
#ifndef OFFSET_ROWS
#define OFFSET_ROWS 1024
#endif
constexpr int64_t kOffsetRows = OFFSET_ROWS;   // float default offsets: mean of this many leading traces
constexpr bool kF32DefaultNT2 = true;          // float cross term: NT = 2 variant by default
#ifndef F32_MAX_UNIT_NT2
#define F32_MAX_UNIT_NT2 24576
#endif
constexpr int64_t kF32MaxUnitNT2 = F32_MAX_UNIT_NT2;  // fp32 TMEM accumulation length bound (precision)
// partial-sum spill (CPA_OPT_SPILL 3): bound on the 32-bit slice buffer.  Off
// by default: at C3 the cross term ran 0.12 ms faster with plain stores, and the
// reduce pass (5 slices + the sum_hw read-modify-write) cost it back
constexpr int64_t kPartMaxBytes = 3LL << 30;
constexpr bool kF32PartialSpill = false;
// int8 W tensor map: no L2 promotion.  With 256-byte promotion every 128-byte
// box row pulled its neighbour (the peer CTA's half or the next tile group) into
// L2 early, and part of it was evicted again before use: ncu DRAM reads per C4
// launch 12.63 GB (256B) vs 11.51 (128B) vs 11.51 (none), time within noise
#ifndef XT_P_PROMOTION
#define XT_P_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_NONE  // float hi / lo plane maps: C3 2.54 -> 2.40 GB, same time
#endif
#ifndef XT_W_PROMOTION
#define XT_W_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_NONE
#endif
constexpr int64_t kBulkSpillMinUnit = 65536;  // CPA_OPT_SPILL auto: bulk reduce from this unit length (traces) on

}  // namespace

struct cpa_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    int32_t M = 0;
    cpa_dtype dtype = CPA_S8;
    cpa_model model = CPA_HD_LAST;
    void *accum = nullptr;
    uint8_t *d_vtab = nullptr;
    double *d_sqrt_dw = nullptr;
    double *d_maxabs = nullptr, *d_peak = nullptr, *d_best_rho = nullptr;
    int32_t *d_argmax = nullptr, *d_rank = nullptr, *d_best = nullptr;
    int *d_counter = nullptr;  // work-unit counter of the cross-term scheduler
    int64_t kchunk = 0;
    int64_t n_since_reset = 0;  // traces accumulated through this context since init / cpa_reset
    bool hw_zero = true;  // sum_hw holds the zeros of cpa_init / cpa_reset (no cross term since)
    int32_t col0 = 0;  // CPA_OPT_COL0: global index of sample 0 (sample-axis sharding)
    int64_t launches = 0;
    // cpa_accumulate_host staging
    void *d_stage[2] = {nullptr, nullptr};
    uint8_t *d_stage_tx[2] = {nullptr, nullptr};
    int64_t stage_bytes = 0, stage_rows = 0;
    void *d_pack = nullptr;  // 16-byte-pitch rows repacked from a linear staging copy
    int64_t pack_bytes = 0;
    int64_t stage_chunk_bytes = kStageBytes;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
    // float path (a6): per-sample offsets and power-of-two scales ([M] scale |
    // [M] 1/scale | range-repair scratch), fp16 hi and e4m3 lo planes, non-finite flag
    float *d_offset = nullptr;
    bool offset_set = false;
    float *d_scale = nullptr;
    bool scale_set = false;
    uint16_t *d_hi = nullptr;
    uint8_t *d_lo = nullptr;
    int64_t plane_rows = 0;
    int *d_nonfinite = nullptr;
    // pinned host block for the one readback a blocking finalize does (N, the
    // non-finite flag, the key) -- see readback()
    struct HostStatus {
        int64_t n_i;
        double n_f;
        int32_t nonfinite, pad;
        int32_t best[32];
        double best_rho[16];
    } *h_status = nullptr;
    uint32_t *d_hist = nullptr;  // a3 byte-pair histogram scratch (16 x 65536)
    // CPA_OPT_CLASS_SUMS (HW_LAST / HW_FIRST, int8 traces): class-sum cross term
    // (classsum.cu); scratch allocated on first use
    int class_sums = 0;
    int fuse_hist = 0;
    int xt_tiles = 0;  // CPA_OPT_XT_TILES: 0 model, 1 NT = 2, 2 NT = 1 overlapped
    int spill = 0;  // CPA_OPT_SPILL: 0 auto, 1 red.add per element, 2 bulk tensor reduce-add, 3 partial stores
    // CUDA-graph capture of the context's stream (cpa_graph_begin / _end / _launch)
    bool capturing = false;
    bool captured_reset = false;  // a cpa_reset was captured before any accumulate
    cudaGraphExec_t graph_exec = nullptr;
    // host bookkeeping of the sums (what the next calls assume about them): a
    // capture changes it without running anything, so cpa_graph_end restores the
    // state from before the capture and keeps the captured end state, which each
    // replay of a graph that begins with a reset then installs
    struct SumState {
        int64_t n_since_reset;
        bool hw_zero, hw32_live;
        int64_t hw32_n;
    };
    SumState sum_state() const { return SumState{n_since_reset, hw_zero, hw32_live, hw32_n}; }
    void set_sum_state(const SumState &x) {
        n_since_reset = x.n_since_reset;
        hw_zero = x.hw_zero;
        hw32_live = x.hw32_live;
        hw32_n = x.hw32_n;
    }
    SumState pre_capture{}, graph_end_state{};
    bool graph_sets_state = false;
    // CPA_OPT_NARROW: the HW field kept in an int32 shadow [4096][M] while it is
    // exact (hw32_n traces in it, N max|H| max|W| < 2^31); hw32_live: the shadow
    // holds HW contributions not yet in the accumulator (flush() adds them)
    int64_t narrow = 0;
    int32_t *d_hw32 = nullptr;
    bool hw32_live = false;
    int64_t hw32_n = 0;
    cudaError_t flush() {
        if (!hw32_live) return cudaSuccess;
        int l = 0;
        cudaError_t e = cpa::launch_widen_hw(d_hw32, (int64_t *)accum, 4096LL * M, num_sms, stream, &l);
        launches += l;
        hw32_live = false;
        hw32_n = 0;
        hw_zero = false;
        return e;
    }
    uint32_t *d_part = nullptr;  // partial-sum spill slices [kc][4096][ld] (32-bit), grown on demand
    int64_t part_bytes = 0;
    // the partial buffer for kc_count slices of part_ld samples (null: over the
    // memory bound or the allocation failed -- the caller falls back to atomics)
    uint32_t *part_buffer(int64_t kc_count, int64_t part_ld) {
        const int64_t need = kc_count * 4096 * part_ld * 4;
        if (need > kPartMaxBytes) return nullptr;
        if (need > part_bytes) {
            if (capturing) return nullptr;  // no allocation inside a capture: the atomic spill
            if (cudaStreamSynchronize(stream) != cudaSuccess) return nullptr;
            cudaFree(d_part);
            d_part = nullptr;
            part_bytes = 0;
            if (cudaMalloc(&d_part, need) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            part_bytes = need;
        }
        return d_part;
    }
    // cpa_set_row_owners: fused multi-GPU combine (key byte b's sum_hw rows go to owners[b])
    int64_t *owners[16] = {};
    bool owners_set = false;
    unsigned long long *d_clk = nullptr;  // xterm clock probe (globaltimer, clock64 at CTA 0's start/end)
    int32_t *d_cs_cnt = nullptr, *d_cs_off = nullptr, *d_cs_cur = nullptr, *d_cs_perm = nullptr, *d_cs_S = nullptr;
    int64_t cs_perm_n = 0, cs_S_words = 0;
    // CPA_OPT_TIMING: CUDA events recorded on `stream` around every launch
    bool timing = false;
    struct Rec { int phase; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t ev() {
        if (pool.empty()) { cudaEvent_t e; cudaEventCreate(&e); return e; }
        cudaEvent_t e = pool.back(); pool.pop_back(); return e;
    }
    // time the launches `fn` issues on the stream as phase `ph`
    template <typename F> cudaError_t timed(int ph, F &&fn) { return timed_on(ph, stream, fn); }
    template <typename F> cudaError_t timed_on(int ph, cudaStream_t st, F &&fn) {
        if (!timing || capturing) return fn();  // replays of a captured graph are not phase-timed
        Rec r{ph, ev(), ev()};
        cudaEventRecord(r.a, st);
        cudaError_t e = fn();
        cudaEventRecord(r.b, st);
        recs.push_back(r);
        return e;
    }
    // a4 on a low-priority side stream, overlapped with the cross term
    int overlap = 3;   // CPA_OPT_OVERLAP mode (0 serial, 1 low-priority after, 2 high-priority before,
                       // 3 fused into the cross-term kernel)
    cudaStream_t side = nullptr, side_hi = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

extern "C" {

size_t cpa_accum_words(int32_t M) { return (size_t)4098 * (size_t)M + 8193; }
size_t cpa_accum_bytes(int32_t M) { return cpa_accum_words(M) * 8; }
size_t cpa_accum_offset(int32_t M, int field)
{
    const size_t m = (size_t)M;
    switch (field) {
    case 0: return 0;
    case 1: return 4096 * m;
    case 2: return 4097 * m;
    case 3: return 4098 * m;
    case 4: return 4098 * m + 4096;
    case 5: return 4098 * m + 8192;
    default: return (size_t)-1;
    }
}

const char *cpa_status_str(cpa_status s)
{
    switch (s) {
    case CPA_OK: return "CPA_OK";
    case CPA_E_INVALID_ARG: return "CPA_E_INVALID_ARG";
    case CPA_E_BAD_STATE: return "CPA_E_BAD_STATE";
    case CPA_E_CUDA: return "CPA_E_CUDA";
    case CPA_E_NO_MEMORY: return "CPA_E_NO_MEMORY";
    case CPA_E_TOO_FEW_TRACES: return "CPA_E_TOO_FEW_TRACES";
    case CPA_E_OVERFLOW: return "CPA_E_OVERFLOW";
    case CPA_E_UNSUPPORTED_DEVICE: return "CPA_E_UNSUPPORTED_DEVICE";
    case CPA_E_NONFINITE: return "CPA_E_NONFINITE";
    }
    return "CPA_E_UNKNOWN";
}

const char *cpa_last_error(void) { return g_err; }

void cpa_aes_expand_key(const uint8_t key[16], uint8_t round_keys[11][16]) { cpa::aes_expand_key(key, round_keys); }
void cpa_aes_invert_key_schedule(const uint8_t rk[16], int round, uint8_t key[16])
{
    cpa::aes_invert_key_schedule(rk, round, key);
}

int64_t cpa_launch_count(const cpa_ctx *ctx) { return ctx ? ctx->launches : -1; }

cpa_status cpa_reset(cpa_ctx *ctx)
{
    if (!ctx) return fail(CPA_E_INVALID_ARG, "null context");
    CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
    CUDA_TRY(cudaMemsetAsync(ctx->accum, 0, cpa_accum_bytes(ctx->M), ctx->stream), "reset accumulator");
    CUDA_TRY(cudaMemsetAsync(ctx->d_nonfinite, 0, sizeof(int), ctx->stream), "reset flag");
    ctx->n_since_reset = 0;
    ctx->hw_zero = true;
    ctx->hw32_live = false;  // the shadow's contents are dropped with the sums
    ctx->hw32_n = 0;
    if (ctx->capturing) ctx->captured_reset = true;
    return CPA_OK;
}

cpa_status cpa_init(cpa_ctx **out, int32_t M, cpa_dtype dtype, cpa_model model, int device, void *stream,
                    void *d_accum)
{
    if (!out) return fail(CPA_E_INVALID_ARG, "out is null");
    *out = nullptr;
    if (M < 1 || M > kMaxSamples) return fail(CPA_E_INVALID_ARG, "M=%d outside [1, %d]", M, kMaxSamples);
    if (dtype != CPA_S8 && dtype != CPA_U8 && dtype != CPA_F32) return fail(CPA_E_INVALID_ARG, "bad dtype %d", (int)dtype);
    if (model != CPA_HD_LAST && model != CPA_HW_LAST && model != CPA_HW_FIRST)
        return fail(CPA_E_INVALID_ARG, "bad model %d", (int)model);
    if (!d_accum || ((uintptr_t)d_accum & 255)) return fail(CPA_E_INVALID_ARG, "d_accum null or not 256-byte aligned");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(CPA_E_INVALID_ARG, "device %d of %d", device, ndev);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(CPA_E_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; libcpa is built for sm_100a only", device,
                    prop.major, prop.minor);
    if (!get_encode()) return fail(CPA_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");

    cpa_ctx *c = new (std::nothrow) cpa_ctx();
    if (!c) return fail(CPA_E_NO_MEMORY, "context allocation");
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->stream = (cudaStream_t)stream;
    c->M = M;
    c->dtype = dtype;
    c->model = model;
    c->accum = d_accum;

    uint8_t vt[65536];
    cpa::build_vtable((int)model, vt);
    cudaError_t e = cudaMalloc(&c->d_vtab, 65536);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_sqrt_dw, 2 * sizeof(double) * M);  // sqrt(dw) | 1/sqrt(dw)
    if (e == cudaSuccess) e = cudaMalloc(&c->d_maxabs, sizeof(double) * 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_peak, sizeof(double) * 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_best_rho, sizeof(double) * 16);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_argmax, sizeof(int32_t) * 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_rank, sizeof(int32_t) * 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_best, sizeof(int32_t) * 32);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_counter, 256);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_nonfinite, 256);
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&c->h_status, sizeof(cpa_ctx::HostStatus), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_hist, sizeof(uint32_t) * 16 * 65536);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_clk, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_clk, 0, 4 * sizeof(unsigned long long), c->stream);
    if (e == cudaSuccess) {
        int lo = 0, hi = 0;  // numerically greatest = lowest priority
        e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->side_hi, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_offset, sizeof(float) * M);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_scale, 2 * sizeof(float) * M + 5 * (size_t)M + 16);
    if (e != cudaSuccess) {
        cpa_destroy(c);
        return fail(CPA_E_NO_MEMORY, "device scratch: %s", cudaGetErrorString(e));
    }
    e = cudaMemcpyAsync(c->d_vtab, vt, 65536, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_accum, 0, cpa_accum_bytes(M), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_offset, 0, sizeof(float) * M, c->stream);  // until set
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_nonfinite, 0, sizeof(int), c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        cpa_destroy(c);
        return cuda_fail(e, "cpa_init upload");
    }
    *out = c;
    return CPA_OK;
}

cpa_status cpa_set_offsets(cpa_ctx *ctx, const float *d_offsets)
{
    if (!ctx) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(ctx);
    if (ctx->dtype != CPA_F32) return fail(CPA_E_INVALID_ARG, "offsets apply to CPA_F32 contexts only");
    CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (d_offsets)
        CUDA_TRY(cudaMemcpyAsync(ctx->d_offset, d_offsets, sizeof(float) * ctx->M, cudaMemcpyDeviceToDevice, ctx->stream),
                 "offsets");
    else
        CUDA_TRY(cudaMemsetAsync(ctx->d_offset, 0, sizeof(float) * ctx->M, ctx->stream), "offsets");
    ctx->offset_set = true;
    ctx->scale_set = false;  // the split scales follow the spread about the offsets
    return CPA_OK;
}

cpa_status cpa_default_offsets(cpa_ctx *ctx, const float *d_traces, int64_t ld, int64_t N, float *d_out)
{
    if (!ctx) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(ctx);
    if (ctx->dtype != CPA_F32) return fail(CPA_E_INVALID_ARG, "offsets apply to CPA_F32 contexts only");
    if (!d_traces || !d_out || N < 1 || ld < ctx->M) return fail(CPA_E_INVALID_ARG, "bad traces / N / ld / out");
    CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
    int launches = 0;
    CUDA_TRY(cpa::launch_mean_rows(d_traces, ld, N < kOffsetRows ? N : kOffsetRows, ctx->M, d_out, ctx->stream,
                                   &launches),
             "default offsets");
    ctx->launches += launches;
    return CPA_OK;
}

cpa_status cpa_get_offsets(cpa_ctx *ctx, float *d_out, int *is_set)
{
    if (!ctx) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(ctx);
    if (ctx->dtype != CPA_F32) return fail(CPA_E_INVALID_ARG, "offsets apply to CPA_F32 contexts only");
    CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (d_out)
        CUDA_TRY(cudaMemcpyAsync(d_out, ctx->d_offset, sizeof(float) * ctx->M, cudaMemcpyDeviceToDevice, ctx->stream),
                 "offsets");
    if (is_set) *is_set = ctx->offset_set ? 1 : 0;
    return CPA_OK;
}

cpa_status cpa_set_option(cpa_ctx *ctx, int option, int64_t value)
{
    if (!ctx) return fail(CPA_E_INVALID_ARG, "null context");
    if (option == CPA_OPT_STAGE_BYTES) {
        if (value < 0) return fail(CPA_E_INVALID_ARG, "STAGE_BYTES=%lld < 0", (long long)value);
        ctx->stage_chunk_bytes = value ? value : kStageBytes;
        return CPA_OK;
    }
    if (option == CPA_OPT_OVERLAP) {
        if (value < 0 || value > 3) return fail(CPA_E_INVALID_ARG, "OVERLAP=%lld outside [0, 3]", (long long)value);
        ctx->overlap = (int)value;
        return CPA_OK;
    }
    if (option == CPA_OPT_COL0) {
        if (value < 0 || value + ctx->M > (int64_t)INT32_MAX)
            return fail(CPA_E_INVALID_ARG, "COL0=%lld: sample indices must fit int32", (long long)value);
        ctx->col0 = (int32_t)value;
        return CPA_OK;
    }
    if (option == CPA_OPT_TIMING) {
        ctx->timing = value != 0;
        return CPA_OK;
    }
    if (option == CPA_OPT_KCHUNK) {
        if (value < 0 || value % 128 || value > (1 << 20))
            return fail(CPA_E_INVALID_ARG, "KCHUNK=%lld must be a multiple of 128 in [0, 2^20]", (long long)value);
        ctx->kchunk = value;
        return CPA_OK;
    }
    if (option == CPA_OPT_XT_TILES) {
        if (value < 0 || value > 2) return fail(CPA_E_INVALID_ARG, "XT_TILES=%lld outside [0, 2]", (long long)value);
        ctx->xt_tiles = (int)value;
        return CPA_OK;
    }
    if (option == CPA_OPT_NARROW) {
        if (value < 0) return fail(CPA_E_INVALID_ARG, "NARROW=%lld < 0", (long long)value);
        if (ctx->dtype == CPA_F32) {  // fp64 sums: nothing to narrow
            ctx->narrow = 0;
            return CPA_OK;
        }
        NO_CAPTURE(ctx);
        CUDA_TRY(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (value == 0) {
            CUDA_TRY(ctx->flush(), "flush narrow sums");
        } else if (ctx->d_hw32 == nullptr) {
            CUDA_TRY(cudaMalloc(&ctx->d_hw32, 4096LL * ctx->M * sizeof(int32_t)), "cudaMalloc narrow sums");
        }
        ctx->narrow = value;
        return CPA_OK;
    }
    if (option == CPA_OPT_SPILL) {
        if (value < 0 || value > 3) return fail(CPA_E_INVALID_ARG, "SPILL=%lld outside [0, 3]", (long long)value);
        ctx->spill = (int)value;
        return CPA_OK;
    }
    if (option == CPA_OPT_FUSE_HIST) {
        if (value < 0 || value > 1) return fail(CPA_E_INVALID_ARG, "FUSE_HIST=%lld outside [0, 1]", (long long)value);
        ctx->fuse_hist = (int)value;
        return CPA_OK;
    }
    if (option == CPA_OPT_CLASS_SUMS) {
        if (value < 0 || value > 1) return fail(CPA_E_INVALID_ARG, "CLASS_SUMS=%lld outside [0, 1]", (long long)value);
        if (value && ctx->owners_set) return fail(CPA_E_INVALID_ARG, "class sums do not support row owners");
        if (value && (ctx->model == CPA_HD_LAST || ctx->dtype == CPA_F32))
            return fail(CPA_E_INVALID_ARG, "class sums need a single-byte model (HW_LAST/HW_FIRST) and int8 traces");
        ctx->class_sums = (int)value;
        return CPA_OK;
    }
    return fail(CPA_E_INVALID_ARG, "unknown option %d", option);
}

// Cross term by class sums (classsum.cu).  The call's traces are taken in
// super-chunks of <= kCsSuper; each is counting-sorted by class per byte in
// chunks of kCsChunk traces (a chunk's rows span < 256 MB: TLB reach), then per
// block of <= kCsCols samples the class sums S of the super-chunk are built
// column tile by column tile (k_cs_sum) and contracted into sum_hw.  Scratch:
// 64 B per super-chunk trace + 16 KB per sample.
#ifndef CS_CHUNK_LOG2
#define CS_CHUNK_LOG2 15
#endif
constexpr int64_t kCsChunk = 1 << CS_CHUNK_LOG2;
constexpr int64_t kCsSuper = 1 << 20;
constexpr int32_t kCsCols = 8192;
static cpa_status accumulate_class_sums(cpa_ctx *c, const void *d_w, int64_t ld, const uint8_t *d_tx, int64_t n,
                                        int *launches)
{
    const int M = c->M;
    const int64_t sup = n < kCsSuper ? n : kCsSuper;
    const int64_t clen = sup < kCsChunk ? sup : kCsChunk;
    const int64_t max_ch = (sup + clen - 1) / clen;
    const int32_t cols = M < kCsCols ? M : kCsCols;
    if (c->cs_perm_n < max_ch * clen) {
        CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
        for (int32_t **p : {&c->d_cs_cnt, &c->d_cs_off, &c->d_cs_cur, &c->d_cs_perm}) {
            cudaFree(*p);
            *p = nullptr;
        }
        c->cs_perm_n = 0;
        cudaError_t e = cudaMalloc(&c->d_cs_cnt, sizeof(int32_t) * 4096);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_cs_cur, sizeof(int32_t) * 4096);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_cs_off, sizeof(int32_t) * 16 * 257 * max_ch);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_cs_perm, sizeof(int32_t) * 16 * max_ch * clen);
        if (e != cudaSuccess) return fail(CPA_E_NO_MEMORY, "class-sum scratch: %s", cudaGetErrorString(e));
        c->cs_perm_n = max_ch * clen;
    }
    if (c->cs_S_words < (int64_t)4096 * cols) {
        CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
        cudaFree(c->d_cs_S);
        c->d_cs_S = nullptr;
        c->cs_S_words = 0;
        cudaError_t e = cudaMalloc(&c->d_cs_S, sizeof(int32_t) * 4096 * cols);
        if (e != cudaSuccess) return fail(CPA_E_NO_MEMORY, "class sums: %s", cudaGetErrorString(e));
        c->cs_S_words = (int64_t)4096 * cols;
    }
    const bool sgn = c->dtype == CPA_S8;
    int64_t *hw = (int64_t *)c->accum;
    CUDA_TRY(c->timed(2, [&] {
                 cudaError_t e = cudaSuccess;
                 for (int64_t s0 = 0; e == cudaSuccess && s0 < n; s0 += sup) {
                     const int64_t sn = (n - s0) < sup ? (n - s0) : sup;
                     // uniform chunks of clen traces (the last one shorter)
                     const int32_t nch = (int32_t)((sn + clen - 1) / clen);
                     for (int32_t ch = 0; e == cudaSuccess && ch < nch; ch++) {
                         const int64_t i0 = s0 + ch * clen;
                         const int64_t m = (s0 + sn - i0) < clen ? (s0 + sn - i0) : clen;
                         e = cpa::launch_cs_sort(d_tx + i0 * 16, m, clen, c->d_cs_cnt, c->d_cs_off + ch * 16 * 257,
                                                 c->d_cs_cur, c->d_cs_perm + (int64_t)ch * 16 * clen, c->num_sms,
                                                 c->stream, launches);
                     }
                     for (int32_t j0 = 0; e == cudaSuccess && j0 < M; j0 += cols) {
                         const int32_t mc = (M - j0) < cols ? (M - j0) : cols;
                         e = cudaMemsetAsync(c->d_cs_S, 0, sizeof(int32_t) * 4096 * mc, c->stream);
                         if (e == cudaSuccess)
                             e = cpa::launch_cs_sum((const uint8_t *)d_w + s0 * ld, ld, nch, clen, j0, mc, sgn,
                                                    c->d_cs_perm, c->d_cs_off, c->d_cs_S, c->num_sms, c->stream,
                                                    launches);
                         if (e == cudaSuccess)
                             e = cpa::launch_cs_contract(c->d_cs_S, M, j0, mc, c->d_vtab, hw, c->stream, launches);
                     }
                 }
                 return e;
             }),
             "class sums");
    return CPA_OK;
}

static cpa_status accumulate_device(cpa_ctx *c, const void *d_w, int64_t ld, const uint8_t *d_tx, int64_t n)
{
    const int M = c->M;
    int launches = 0;
    // a3 for large N: the cross-term kernel counts the byte pairs as it
    // generates H (CPA_OPT_FUSE_HIST), only the contraction runs here
    const bool fhist = c->fuse_hist && !c->class_sums && n >= cpa::kHistMinTraces;
    if (fhist) CUDA_TRY(cpa::launch_hist_clear(c->d_hist, c->stream), "hist clear");
    if (c->dtype == CPA_F32) {
        double *acc = (double *)c->accum;
        if (!fhist)
            CUDA_TRY(c->timed(0, [&] {
                         return cpa::launch_modelsums_f64(d_tx, n, c->d_vtab, c->d_hist, acc + cpa_accum_offset(M, 3),
                                                          acc + cpa_accum_offset(M, 4), acc + cpa_accum_offset(M, 5),
                                                          c->stream, &launches);
                     }),
                     "modelsums");
        // per-sample offsets (centring keeps the hi/lo split and the fp32
        // accumulation accurate; rho is invariant to them [S:285]): unless the
        // caller set them, the mean of the first <= 1024 traces of the first call
        if (!c->offset_set) {
            CUDA_TRY(cpa::launch_mean_rows((const float *)d_w, ld, n < kOffsetRows ? n : kOffsetRows, M, c->d_offset,
                                           c->stream, &launches),
                     "offsets");
            c->offset_set = true;
        }
        // per-sample power-of-two scales of the split (exact; a precision choice,
        // not a change of the sums): from the first <= 64 traces seen
        if (!c->scale_set) {
            CUDA_TRY(cpa::launch_scale_f32((const float *)d_w, ld, n < 64 ? n : 64, M, c->d_offset, c->d_scale,
                                           c->d_scale + M, c->stream, &launches),
                     "split scales");
            c->scale_set = true;
        }
        const int64_t ldh = (M + 7) / 8 * 8;     // fp16 hi plane pitch (16-byte rows for TMA)
        const int64_t ldl = (M + 15) / 16 * 16;  // e4m3 lo plane pitch
        const int64_t max_rows = (1LL << 30) / (ldh * 2);  // <= 1 GiB per fp16 plane
        const int64_t chunk = n < max_rows ? n : max_rows;
        if (c->plane_rows < chunk) {
            if (c->capturing)
                return fail(CPA_E_INVALID_ARG, "the float planes must be allocated before a capture: run the "
                                               "call once outside it");
            CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
            cudaFree(c->d_hi);
            cudaFree(c->d_lo);
            c->d_hi = nullptr;
            c->d_lo = nullptr;
            c->plane_rows = 0;
            if (cudaMalloc(&c->d_hi, chunk * ldh * 2) != cudaSuccess || cudaMalloc(&c->d_lo, chunk * ldl) != cudaSuccess)
                return fail(CPA_E_NO_MEMORY, "hi/lo planes (%lld rows)", (long long)chunk);
            c->plane_rows = chunk;
        }
        for (int64_t i0 = 0; i0 < n; i0 += chunk) {
            const int64_t m = (n - i0) < chunk ? (n - i0) : chunk;
            const float *w = (const float *)d_w + i0 * ld;
            // float cross-term variant (CPA_OPT_XT_TILES): 1 = NT = 2, 2 = NT = 1, 0 = default
            const bool nt2 = c->xt_tiles == 1 || (c->xt_tiles == 0 && kF32DefaultNT2);
            CUDA_TRY(c->timed(1, [&] {
                         return cpa::launch_split_f32(w, ld, m, M, c->d_offset, c->d_scale, c->d_hi, c->d_lo, ldh,
                                                      ldl, acc + cpa_accum_offset(M, 1), acc + cpa_accum_offset(M, 2),
                                                      c->d_nonfinite, (uint8_t *)(c->d_scale + 2 * M), c->stream,
                                                      &launches);
                     }),
                     "split_f32");
            CUtensorMap mh, ml;
            cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)m};
            cuuint32_t estr[2] = {1, 1};
            for (int k = 0; k < 2; k++) {
                // hi: 64 fp16 = the 128-byte swizzle span; lo: 128 e4m3 bytes; x one stage of traces
                cuuint64_t strides[1] = {(cuuint64_t)(k ? ldl : ldh * 2)};
                cuuint32_t box[2] = {k ? 128u : 64u, (cuuint32_t)cpa::xterm_f32_bk(nt2)};
                CUresult r = get_encode()(k ? &ml : &mh,
                                          k ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                                          k ? (void *)c->d_lo : (void *)c->d_hi, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          XT_P_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) return fail(CPA_E_CUDA, "cuTensorMapEncodeTiled (hi/lo) failed (%d)", (int)r);
            }
            const int64_t kmax = nt2 ? kF32MaxUnitNT2 : 4096;
            const int64_t kc = c->kchunk ? (c->kchunk < kmax ? c->kchunk : kmax)
                                         : cpa::xterm_f32_auto_kchunk(M, m, c->num_sms, nt2);
            // fp64 spill by bulk tensor reduce-add (CPA_OPT_SPILL 0 / 2; M even)
            CUtensorMap mhw;
            bool bulk = (M % 2 == 0) && c->spill == 2;  // default: fp64 atomics (measured faster)
            if (bulk) {
                cuuint64_t hdims[2] = {(cuuint64_t)M, 4096};
                cuuint64_t hstr[1] = {(cuuint64_t)M * 8};
                cuuint32_t hbox[2] = {8, 32};
                bulk = get_encode()(&mhw, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, acc, hdims, hstr, hbox, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
            // partial-sum spill (CPA_OPT_SPILL 3): raw fp32 stores per trace
            // chunk, then one reduce pass adds them (x 2^16 / s_j) into sum_hw
            const int64_t part_ld = (M + 7) / 8 * 8;
            const int64_t kcount = (m + kc - 1) / kc;
            uint32_t *part = (!bulk && (c->spill == 3 || (c->spill == 0 && kF32PartialSpill)))
                                 ? c->part_buffer(kcount, part_ld) : nullptr;
            CUDA_TRY(c->timed(2, [&] {
                         return cpa::launch_xterm_f32(mh, ml, bulk ? &mhw : nullptr, d_tx + i0 * 16, c->d_vtab, acc,
                                                      c->d_scale + M, c->d_counter, M, m, kc, c->num_sms, c->stream,
                                                      &launches, fhist ? c->d_hist : nullptr, c->d_clk, nt2, part,
                                                      part_ld);
                     }),
                     "xterm_f32");
            if (part != nullptr)
                CUDA_TRY(c->timed(5, [&] {
                             return cpa::launch_part_reduce_f32(part, (int32_t)kcount, part_ld, M, c->d_scale + M, acc,
                                                                c->stream, &launches);
                         }),
                         "spill reduce");
            c->hw_zero = false;
        }
        if (fhist)
            CUDA_TRY(c->timed(0, [&] {
                         return cpa::launch_hist_contract_f64(c->d_hist, n, c->d_vtab, acc + cpa_accum_offset(M, 3),
                                                              acc + cpa_accum_offset(M, 4),
                                                              acc + cpa_accum_offset(M, 5), c->stream, &launches);
                     }),
                     "hist contract");
        c->launches += launches;
        return CPA_OK;
    }
    int64_t *acc = (int64_t *)c->accum;
    const bool sgn = c->dtype == CPA_S8;
    // CPA_OPT_NARROW: int32 cross-term sums while exact -- N max|H| max|W| < 2^31
    // with max|H| = 8 (every model's V is a Hamming weight / distance of a byte)
    // and max|W| = 128 (s8) / 255 (u8); NARROW > 1 lowers the trace bound (tests)
    const int64_t n32_max = std::min<int64_t>(((1LL << 31) - 1) / (8 * (sgn ? 128 : 255)),
                                              c->narrow > 1 ? c->narrow : INT64_MAX);
    const bool use32 = c->narrow && c->d_hw32 && !c->class_sums && !c->owners_set && c->spill <= 1 &&
                       (c->hw32_live ? c->hw32_n : 0) + n <= n32_max;
    if (c->hw32_live && !use32) CUDA_TRY(c->flush(), "flush narrow sums");
    if (!fhist)
        CUDA_TRY(c->timed(0, [&] {
                     return cpa::launch_modelsums(d_tx, n, c->d_vtab, c->d_hist, acc + cpa_accum_offset(M, 3),
                                                  acc + cpa_accum_offset(M, 4), acc + cpa_accum_offset(M, 5),
                                                  c->stream, &launches);
                 }),
                 "modelsums");
    if (c->class_sums) {  // a4 serialised, then the class-sum cross term
        CUDA_TRY(c->timed(1, [&] {
                     return cpa::launch_moments_i8(d_w, ld, n, M, sgn, acc + cpa_accum_offset(M, 1),
                                                   acc + cpa_accum_offset(M, 2), 0, c->stream, &launches);
                 }),
                 "moments");
        cpa_status st = accumulate_class_sums(c, d_w, ld, d_tx, n, &launches);
        c->hw_zero = false;
        c->launches += launches;
        return st;
    }
    // a4 (HBM-bound) runs concurrently with the tensor-bound cross term:
    //   overlap 1: launched after it on a low-priority side stream (its blocks
    //              fill whatever registers/threads the cross-term CTAs leave);
    //   overlap 2: launched BEFORE it on a high-priority side stream, one block
    //              per SM, so both kernels are co-resident from the start.
    //   overlap 3: no separate pass: the cross-term kernel's epilogue warps sum
    //              the W tiles it loads anyway (no extra HBM traffic).
    // cross-term variant (CPA_OPT_XT_TILES): the NT = 1 overlapped one cannot
    // fuse a4, which then runs serialised before it (mode 0)
    const cpa::XtermI8Plan plan = cpa::xterm_i8_plan(M, n, c->num_sms, c->owners_set, c->xt_tiles);
    const bool fused = c->overlap == 3 && !plan.overlapped;
    const int mode = (c->side && !fused && c->overlap != 3) ? c->overlap : 0;
    cudaStream_t mst = mode == 2 ? c->side_hi : (mode == 1 ? c->side : c->stream);
    if (mode) {
        CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream), "fork");
        CUDA_TRY(cudaStreamWaitEvent(mst, c->ev_fork, 0), "fork");
    }
    auto moments = [&] {
        return c->timed_on(1, mst, [&] {
            return cpa::launch_moments_i8(d_w, ld, n, M, sgn, acc + cpa_accum_offset(M, 1),
                                          acc + cpa_accum_offset(M, 2), mode == 2 ? 1 : 0, mst, &launches);
        });
    };
    if (!fused && mode != 1) CUDA_TRY(moments(), "moments");
    CUtensorMap tmap;
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {128, 128};  // 128 samples (128-byte swizzle span) x 128 traces
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(d_w), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              XT_W_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CPA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    // the epilogue's int64 spill by bulk tensor reduce-add into sum_hw [4096][M]
    // (rows of M int64 must be 16-byte multiples: M even); the fused multi-GPU
    // combine (row owners) keeps its system-scope red.add.  The map is typed
    // UINT64: the TMA reduce-add rejects INT64 at run time (tools/reduce_probe.cu)
    // and two's-complement addition is the same operation on the same bits.
    // auto (CPA_OPT_SPILL 0): bulk for long units, where it measured 0.5% faster
    // (C4); red.add for short ones, where it measured faster (C2 0.109 vs 0.122 ms,
    // W48 1.18 vs 1.20): the spill is bound by the L2/HBM read-modify-write of
    // sum_hw either way, not by the issuing SM
    const int64_t kc = c->kchunk ? c->kchunk : plan.kc_len;
    CUtensorMap tmap_hw;
    bool bulk = !use32 && (M % 2 == 0) && !c->owners_set &&
                (c->spill == 2 || (c->spill == 0 && kc >= kBulkSpillMinUnit));
    if (bulk) {
        cuuint64_t hdims[2] = {(cuuint64_t)M, 4096};
        cuuint64_t hstr[1] = {(cuuint64_t)M * 8};
        cuuint32_t hbox[2] = {8, 32};
        bulk = get_encode()(&tmap_hw, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, acc, hdims, hstr, hbox, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    // partial-sum spill (CPA_OPT_SPILL 3; not with row owners): raw int32 stores
    // per trace chunk, then one exact reduce pass into the int64 sum_hw
    const int64_t part_ld = (M + 7) / 8 * 8;
    const int64_t kcount = (n + kc - 1) / kc;
    uint32_t *part = (!c->owners_set && c->spill == 3) ? c->part_buffer(kcount, part_ld) : nullptr;
    if (part != nullptr) bulk = false;
    // narrow sums: a fresh shadow is first-touch stored by a one-chunk launch,
    // else zeroed first; a live one is added to
    bool first32 = false;
    if (use32 && !c->hw32_live) {
        if (kcount == 1) first32 = true;
        else CUDA_TRY(cudaMemsetAsync(c->d_hw32, 0, 4096LL * M * sizeof(int32_t), c->stream), "zero narrow sums");
    }
    CUDA_TRY(c->timed(2, [&] {
                 cudaError_t e = cpa::launch_xterm_i8(tmap, bulk ? &tmap_hw : nullptr, d_tx, c->d_vtab, acc,
                                                      c->d_counter, M, n, kc, sgn, c->num_sms, c->stream, &launches,
                                                      fused ? acc + cpa_accum_offset(M, 1) : nullptr,
                                                      fused ? acc + cpa_accum_offset(M, 2) : nullptr,
                                                      fhist ? c->d_hist : nullptr, c->owners_set ? c->owners : nullptr,
                                                      c->d_clk, plan.overlapped,
                                                      use32 ? first32 : (part ? false : c->hw_zero), part, part_ld,
                                                      use32 ? c->d_hw32 : nullptr);
                 return e;
             }),
             "xterm_i8");
    if (part != nullptr)
        CUDA_TRY(c->timed(5, [&] {
                     return cpa::launch_part_reduce_i32(part, (int32_t)kcount, part_ld, M, acc, c->stream, &launches);
                 }),
                 "spill reduce");
    if (use32) {
        c->hw32_live = true;
        c->hw32_n += n;
    } else {
        c->hw_zero = false;
    }
    if (!fused && mode == 1) CUDA_TRY(moments(), "moments");
    if (fhist)
        CUDA_TRY(c->timed(0, [&] {
                     return cpa::launch_hist_contract(c->d_hist, n, c->d_vtab, acc + cpa_accum_offset(M, 3),
                                                      acc + cpa_accum_offset(M, 4), acc + cpa_accum_offset(M, 5),
                                                      c->stream, &launches);
                 }),
                 "hist contract");
    if (mode) {
        CUDA_TRY(cudaEventRecord(c->ev_join, mst), "join");
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "join");
    }
    c->launches += launches;
    return CPA_OK;
}

static cpa_status check_accumulate_args(cpa_ctx *c, const void *w, int64_t ld, const uint8_t *tx, int64_t n)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    if (n < 0) return fail(CPA_E_INVALID_ARG, "N=%lld < 0", (long long)n);
    if (n == 0) return CPA_OK;
    if (!w || !tx) return fail(CPA_E_INVALID_ARG, "null traces or texts");
    if (n > kMaxTraces) return fail(CPA_E_OVERFLOW, "N=%lld per call exceeds 2^23", (long long)n);
    if (c->dtype != CPA_F32 && c->n_since_reset + n > kMaxTraces)
        return fail(CPA_E_OVERFLOW, "%lld + %lld traces since the last reset exceed 2^23 (exact-int64 bound of Eq. (1))",
                    (long long)c->n_since_reset, (long long)n);
    if (ld < c->M) return fail(CPA_E_INVALID_ARG, "ld=%lld < M=%d", (long long)ld, c->M);
    return CPA_OK;
}

static cpa_status accumulate_staged(cpa_ctx *c, const void *src, int64_t ld, const uint8_t *tx, int64_t N);

cpa_status cpa_accumulate(cpa_ctx *c, const void *d_traces, int64_t ld, const uint8_t *d_texts, int64_t N)
{
    cpa_status st = check_accumulate_args(c, d_traces, ld, d_texts, N);
    if (st != CPA_OK || N == 0) return st;
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    const int64_t esz = c->dtype == CPA_F32 ? 4 : 1;
    const bool staged = ((uintptr_t)d_traces & 15) || ((ld * esz) & 15) || ((uintptr_t)d_texts & 15);
    if (c->capturing) {
        // a replay must start from the sums the capture assumed (first-touch
        // stores, the N bookkeeping): the graph begins with cpa_reset
        if (!c->captured_reset)
            return fail(CPA_E_INVALID_ARG, "cpa_accumulate in a graph capture needs a captured cpa_reset first");
        if (staged) return fail(CPA_E_INVALID_ARG, "unaligned traces go through staging buffers: not capturable");
        if (c->class_sums) return fail(CPA_E_INVALID_ARG, "the class-sum cross term is not capturable");
    }
    if (staged)
        st = accumulate_staged(c, d_traces, ld, d_texts, N);  // TMA needs 16-byte strides
    else
        st = accumulate_device(c, d_traces, ld, d_texts, N);
    if (st == CPA_OK) c->n_since_reset += N;
    return st;
}

// Stream (host or unaligned device) traces through the library's staging
// buffers, double-buffered so the copy of chunk c+1 overlaps the kernels of
// chunk c (a1).  Contiguous rows (ld == M) go as ONE linear copy per chunk --
// the H2D DMA runs at full PCIe rate only for linear copies -- and, when a row
// is not a 16-byte multiple, a device repack kernel then lays them out at a
// 16-byte pitch for TMA.  Strided rows fall back to a pitched 2D copy.
static cpa_status accumulate_staged(cpa_ctx *c, const void *src, int64_t ld, const uint8_t *tx, int64_t N)
{
    const int64_t esz = c->dtype == CPA_F32 ? 4 : 1;
    const int64_t rb = c->M * esz;              // bytes per trace row
    const int64_t pitch = (rb + 15) / 16 * 16;  // device row pitch
    const bool linear = ld * esz == rb;
    const bool repack = linear && rb != pitch;
    int64_t chunk = c->stage_chunk_bytes / pitch;
    if (chunk < 1) chunk = 1;
    if (chunk > N) chunk = N;
    const int64_t need = chunk * pitch + 64;  // + slack for the repack kernel's word reads
    if (c->stage_bytes < need || c->stage_rows < chunk || (repack && c->pack_bytes < chunk * pitch)) {
        CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
        for (int k = 0; k < 2; k++) {
            cudaFree(c->d_stage[k]);
            cudaFree(c->d_stage_tx[k]);
            c->d_stage[k] = nullptr;
            c->d_stage_tx[k] = nullptr;
        }
        cudaFree(c->d_pack);
        c->d_pack = nullptr;
        c->stage_bytes = c->stage_rows = c->pack_bytes = 0;
        for (int k = 0; k < 2; k++) {
            if (cudaMalloc(&c->d_stage[k], need) != cudaSuccess ||
                cudaMalloc(&c->d_stage_tx[k], chunk * 16) != cudaSuccess)
                return fail(CPA_E_NO_MEMORY, "staging buffers (%lld bytes)", (long long)need);
        }
        if (repack && cudaMalloc(&c->d_pack, chunk * pitch) != cudaSuccess)
            return fail(CPA_E_NO_MEMORY, "repack buffer (%lld bytes)", (long long)(chunk * pitch));
        c->stage_bytes = need;
        c->stage_rows = chunk;
        c->pack_bytes = repack ? chunk * pitch : 0;
        if (!c->copy_stream) {
            CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
            for (int k = 0; k < 2; k++) {
                CUDA_TRY(cudaEventCreateWithFlags(&c->ev_copied[k], cudaEventDisableTiming), "event");
                CUDA_TRY(cudaEventCreateWithFlags(&c->ev_used[k], cudaEventDisableTiming), "event");
            }
        }
    }
    // the copy stream must not overwrite a buffer earlier compute still reads
    CUDA_TRY(cudaEventRecord(c->ev_used[0], c->stream), "event");
    CUDA_TRY(cudaEventRecord(c->ev_used[1], c->stream), "event");
    int k = 0;
    for (int64_t i0 = 0; i0 < N; i0 += chunk, k ^= 1) {
        const int64_t n = (N - i0) < chunk ? (N - i0) : chunk;
        const uint8_t *s = (const uint8_t *)src + i0 * ld * esz;
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev_used[k], 0), "wait");
        if (linear)
            CUDA_TRY(cudaMemcpyAsync(c->d_stage[k], s, n * rb, cudaMemcpyDefault, c->copy_stream), "copy traces");
        else
            CUDA_TRY(cudaMemcpy2DAsync(c->d_stage[k], pitch, s, ld * esz, rb, n, cudaMemcpyDefault, c->copy_stream),
                     "copy traces");
        CUDA_TRY(cudaMemcpyAsync(c->d_stage_tx[k], tx + i0 * 16, n * 16, cudaMemcpyDefault, c->copy_stream),
                 "copy texts");
        CUDA_TRY(cudaEventRecord(c->ev_copied[k], c->copy_stream), "event");
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_copied[k], 0), "wait");
        const void *w = c->d_stage[k];
        if (repack) {
            int launches = 0;
            CUDA_TRY(cpa::launch_repack((const uint8_t *)c->d_stage[k], rb, (uint8_t *)c->d_pack, pitch, n,
                                        c->stream, &launches),
                     "repack");
            c->launches += launches;
            w = c->d_pack;
        }
        cpa_status st = accumulate_device(c, w, pitch / esz, c->d_stage_tx[k], n);
        if (st != CPA_OK) return st;
        CUDA_TRY(cudaEventRecord(c->ev_used[k], c->stream), "event");
    }
    return CPA_OK;
}

cpa_status cpa_accumulate_host(cpa_ctx *c, const void *h_traces, int64_t ld, const uint8_t *h_texts, int64_t N)
{
    if (c && c->capturing) NO_CAPTURE(c);
    cpa_status st = check_accumulate_args(c, h_traces, ld, h_texts, N);
    if (st != CPA_OK || N == 0) return st;
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    st = accumulate_staged(c, h_traces, ld, h_texts, N);
    if (st != CPA_OK) return st;
    c->n_since_reset += N;
    CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
    return CPA_OK;
}

// N from the accumulator, with the preconditions of Eq. (1) [P:69]
// One round trip per blocking call, after its kernels are queued: N (and the
// float path's non-finite flag, and with_key: the Phase-4 key) into pinned host
// memory, one synchronisation, then the checks (Eq. (1) needs N >= 2; the int
// path's int64 intermediates need N <= 2^23 [DESIGN.md]).  The kernels read N on
// the device, so nothing waits for the host before they run; on an error return
// the device outputs are unspecified.  (Checking first cost the step one or two
// extra host round trips with the GPU idle.)
static cpa_status readback(cpa_ctx *c, bool with_key, bool check, int64_t *n_out)
{
    cpa_ctx::HostStatus *h = c->h_status;
    const size_t off = cpa_accum_offset(c->M, 5);
    const bool f32 = c->dtype == CPA_F32;
    CUDA_TRY(cudaMemcpyAsync(f32 ? (void *)&h->n_f : (void *)&h->n_i,
                             f32 ? (const void *)((const double *)c->accum + off) : (const void *)((const int64_t *)c->accum + off),
                             8, cudaMemcpyDeviceToHost, c->stream), "read N");
    if (f32) CUDA_TRY(cudaMemcpyAsync(&h->nonfinite, c->d_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
                      "read flag");
    if (with_key) {
        CUDA_TRY(cudaMemcpyAsync(h->best, c->d_best, sizeof h->best, cudaMemcpyDeviceToHost, c->stream), "D2H best");
        CUDA_TRY(cudaMemcpyAsync(h->best_rho, c->d_best_rho, sizeof h->best_rho, cudaMemcpyDeviceToHost, c->stream),
                 "D2H best rho");
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
    const int64_t n = f32 ? (int64_t)h->n_f : h->n_i;
    if (check) {
        if (n < 2) return fail(CPA_E_TOO_FEW_TRACES, "N=%lld < 2: Eq. (1) undefined", (long long)n);
        if (f32 && h->nonfinite) return fail(CPA_E_NONFINITE, "a float trace sample was NaN or Inf");
        if (!f32 && n > kMaxTraces)
            return fail(CPA_E_OVERFLOW, "N=%lld > 2^23: Eq. (1) intermediates may overflow int64", (long long)n);
    }
    *n_out = n;
    return CPA_OK;
}

// a8 for hypothesis rows [o.h0, o.h1)
static cpa_status phase3(cpa_ctx *c, const cpa::FinalizeOut &o, int *launches)
{
    if (o.h1 <= o.h0) return CPA_OK;
    CUDA_TRY(c->timed(3, [&] {
                 return c->dtype == CPA_F32
                            ? cpa::launch_finalize_f64((const double *)c->accum, c->M, c->d_offset, c->d_sqrt_dw, o,
                                                       c->stream, launches)
                            : cpa::launch_finalize_i8((const int64_t *)c->accum, c->M, c->d_sqrt_dw, o, c->stream,
                                                      launches, c->hw32_live ? c->d_hw32 : nullptr);
             }),
             "finalize");
    return CPA_OK;
}

// a9 on o.maxabs/argmax/peak, then the key D2H
static cpa_status phase4(cpa_ctx *c, const cpa::FinalizeOut &o, int *launches)
{
    CUDA_TRY(c->timed(4, [&] { return cpa::launch_phase4(o, c->stream, launches); }), "phase4");
    return CPA_OK;
}
// the key of the last readback(with_key)
static void fill_result(cpa_ctx *c, int64_t n, cpa_result *res)
{
    if (!res) return;
    const cpa_ctx::HostStatus *h = c->h_status;
    for (int b = 0; b < 16; b++) {
        res->round_key[b] = (uint8_t)h->best[b];
        res->peak_sample[b] = h->best[16 + b];
        res->peak_rho[b] = h->best_rho[b];
    }
    if (c->model == CPA_HW_FIRST)
        std::memcpy(res->master_key, res->round_key, 16);
    else
        cpa::aes_invert_key_schedule(res->round_key, 10, res->master_key);
    res->n_traces = n;
}

static cpa::FinalizeOut outputs(cpa_ctx *c, double *d_rho, double *d_maxabs, int32_t *d_argmax, double *d_peak,
                                int32_t *d_rank)
{
    cpa::FinalizeOut o;
    o.rho = d_rho;
    o.maxabs = d_maxabs ? d_maxabs : c->d_maxabs;
    o.argmax = d_argmax ? d_argmax : c->d_argmax;
    o.peak = d_peak ? d_peak : c->d_peak;
    o.rank = d_rank ? d_rank : c->d_rank;
    o.best = c->d_best;
    o.best_rho = c->d_best_rho;
    o.col0 = c->col0;
    return o;
}

cpa_status cpa_finalize(cpa_ctx *c, double *d_rho, double *d_maxabs, int32_t *d_argmax, int32_t *d_rank,
                        cpa_result *res)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(c);
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cpa::FinalizeOut o = outputs(c, d_rho, d_maxabs, d_argmax, nullptr, d_rank);
    int launches = 0;
    cpa_status st = phase3(c, o, &launches);
    if (st == CPA_OK) st = phase4(c, o, &launches);
    c->launches += launches;
    int64_t n = 0;
    if (st == CPA_OK) st = readback(c, true, true, &n);
    if (st == CPA_OK) fill_result(c, n, res);
    return st;
}

cpa_status cpa_xterm_clock(cpa_ctx *c, double *mhz)
{
    if (!c || !mhz) return fail(CPA_E_INVALID_ARG, "null argument");
    NO_CAPTURE(c);
    unsigned long long v[4];
    CUDA_TRY(cudaMemcpyAsync(v, c->d_clk, sizeof v, cudaMemcpyDeviceToHost, c->stream), "D2H clock probe");
    CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
    *mhz = (v[2] > v[0] && v[3] > v[1]) ? (double)(v[3] - v[1]) / (double)(v[2] - v[0]) * 1e3 : 0.0;
    return CPA_OK;
}

cpa_status cpa_set_row_owners(cpa_ctx *c, void *const owners[16])
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    if (!owners) {
        c->owners_set = false;
        for (auto &o : c->owners) o = nullptr;
        return CPA_OK;
    }
    if (c->dtype == CPA_F32) return fail(CPA_E_INVALID_ARG, "row owners need int8 traces");
    if (c->class_sums) return fail(CPA_E_INVALID_ARG, "row owners do not support class sums");
    for (int b = 0; b < 16; b++) {
        if (owners[b] && ((uintptr_t)owners[b] & 7)) return fail(CPA_E_INVALID_ARG, "owner %d misaligned", b);
        c->owners[b] = (int64_t *)(owners[b] ? owners[b] : c->accum);
    }
    c->owners_set = true;
    return CPA_OK;
}

cpa_status cpa_peer_atomics(int dev, int peer, int *ok)
{
    if (!ok) return fail(CPA_E_INVALID_ARG, "null argument");
    if (dev == peer) {
        *ok = 1;
        return CPA_OK;
    }
    int access = 0, atomics = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&access, dev, peer), "cudaDeviceCanAccessPeer");
    CUDA_TRY(cudaDeviceGetP2PAttribute(&atomics, cudaDevP2PAttrNativeAtomicSupported, dev, peer),
             "cudaDeviceGetP2PAttribute");
    *ok = access && atomics;
    return CPA_OK;
}

cpa_status cpa_ipc_export(const void *d_ptr, uint8_t handle[64], uint64_t *offset)
{
    if (!d_ptr || !handle || !offset) return fail(CPA_E_INVALID_ARG, "null argument");
    PFN_addr_range range = get_addr_range();
    if (!range) return fail(CPA_E_CUDA, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) return fail(CPA_E_INVALID_ARG, "not a device pointer");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)base), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) <= 64, "handle size");
    std::memset(handle, 0, 64);
    std::memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)((CUdeviceptr)d_ptr - base);
    return CPA_OK;
}

cpa_status cpa_ipc_open(const uint8_t handle[64], uint64_t offset, void **d_ptr)
{
    if (!handle || !d_ptr) return fail(CPA_E_INVALID_ARG, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    *d_ptr = (uint8_t *)base + offset;
    return CPA_OK;
}

cpa_status cpa_ipc_close(void *d_base)
{
    CUDA_TRY(cudaIpcCloseMemHandle(d_base), "cudaIpcCloseMemHandle");
    return CPA_OK;
}

cpa_status cpa_finalize_async(cpa_ctx *c, double *d_rho, double *d_maxabs, int32_t *d_argmax, int32_t *d_rank,
                              int32_t *d_best)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    // host-side checks on the traces this context accumulated since its last
    // reset (no device read: the call must not block); a context whose
    // accumulator was filled from outside (none accumulated here) is not checked
    if (c->n_since_reset == 1)
        return fail(CPA_E_TOO_FEW_TRACES, "N=1 < 2: Eq. (1) undefined");
    if (c->dtype != CPA_F32 && c->n_since_reset > kMaxTraces)
        return fail(CPA_E_OVERFLOW, "N=%lld > 2^23", (long long)c->n_since_reset);
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cpa::FinalizeOut o = outputs(c, d_rho, d_maxabs, d_argmax, nullptr, d_rank);
    if (d_best) o.best = d_best;
    int launches = 0;
    cpa_status st = phase3(c, o, &launches);
    if (st == CPA_OK)
        CUDA_TRY(c->timed(4, [&] { return cpa::launch_phase4(o, c->stream, &launches); }), "phase4");
    c->launches += launches;
    return st;
}

cpa_status cpa_finalize_rows(cpa_ctx *c, int32_t h0, int32_t h1, double *d_rho, double *d_maxabs,
                             int32_t *d_argmax, double *d_peak)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(c);
    if (h0 < 0 || h1 > 4096 || h0 > h1) return fail(CPA_E_INVALID_ARG, "rows [%d, %d) outside [0, 4096]", h0, h1);
    if (!d_maxabs || !d_argmax || !d_peak) return fail(CPA_E_INVALID_ARG, "d_maxabs, d_argmax and d_peak are required");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cpa::FinalizeOut o = outputs(c, d_rho, d_maxabs, d_argmax, d_peak, nullptr);
    o.h0 = h0;
    o.h1 = h1;
    int launches = 0;
    cpa_status st = phase3(c, o, &launches);
    c->launches += launches;
    int64_t n = 0;
    if (st == CPA_OK) st = readback(c, false, true, &n);
    return st;
}

cpa_status cpa_select(cpa_ctx *c, int32_t G, double *d_maxabs, int32_t *d_argmax, double *d_peak, int32_t *d_rank,
                      cpa_result *res)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(c);
    if (G < 1 || G > 65536) return fail(CPA_E_INVALID_ARG, "G=%d outside [1, 65536]", G);
    if (!d_maxabs || !d_argmax || !d_peak) return fail(CPA_E_INVALID_ARG, "d_maxabs, d_argmax and d_peak are required");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cpa::FinalizeOut o = outputs(c, nullptr, d_maxabs, d_argmax, d_peak, d_rank);
    int launches = 0;
    if (G > 1)
        CUDA_TRY(c->timed(4, [&] { return cpa::launch_merge_shards(G, d_maxabs, d_argmax, d_peak, c->stream,
                                                                   &launches); }),
                 "merge shards");
    cpa_status st = phase4(c, o, &launches);
    c->launches += launches;
    int64_t n = 0;
    if (st == CPA_OK) st = readback(c, true, false, &n);
    if (st == CPA_OK) fill_result(c, n, res);
    return st;
}

cpa_status cpa_phase_times(cpa_ctx *c, double ms[CPA_NUM_PHASES], int64_t launches[CPA_NUM_PHASES])
{
    if (!c || !ms) return fail(CPA_E_INVALID_ARG, "null argument");
    NO_CAPTURE(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
    for (int p = 0; p < CPA_NUM_PHASES; p++) {
        ms[p] = 0.0;
        if (launches) launches[p] = 0;
    }
    for (auto &r : c->recs) {
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b), "cudaEventElapsedTime");
        ms[r.phase] += t;
        if (launches) launches[r.phase]++;
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    return CPA_OK;
}

cpa_status cpa_flush(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    CUDA_TRY(c->flush(), "flush narrow sums");
    return CPA_OK;
}

cpa_status cpa_sync(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    NO_CAPTURE(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream), "sync");
    return CPA_OK;
}

// CUDA-graph capture of the context's stream: the calls made between
// cpa_graph_begin and cpa_graph_end (cpa_reset, cpa_accumulate on aligned device
// buffers, cpa_finalize_async) are recorded instead of run, and cpa_graph_launch
// replays them as one graph launch -- no per-kernel host launch cost, no host
// work between the steps of a repeated attack of a fixed shape.
cpa_status cpa_graph_begin(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    if (c->capturing) return fail(CPA_E_INVALID_ARG, "already capturing");
    if (c->stream == nullptr)
        return fail(CPA_E_INVALID_ARG, "graph capture needs a context stream other than the legacy default stream");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    c->capturing = true;
    c->captured_reset = false;
    c->pre_capture = c->sum_state();
    return CPA_OK;
}

cpa_status cpa_graph_end(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    if (!c->capturing) return fail(CPA_E_INVALID_ARG, "not capturing");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    c->graph_end_state = c->sum_state();
    c->graph_sets_state = c->captured_reset;
    c->set_sum_state(c->pre_capture);  // nothing has run yet
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    if (c->graph_exec) {
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
    }
    e = cudaGraphInstantiate(&c->graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        c->graph_exec = nullptr;
        return cuda_fail(e, "cudaGraphInstantiate");
    }
    return CPA_OK;
}

cpa_status cpa_graph_launch(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    if (c->capturing || !c->graph_exec) return fail(CPA_E_INVALID_ARG, "no captured graph");
    CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    CUDA_TRY(cudaGraphLaunch(c->graph_exec, c->stream), "cudaGraphLaunch");
    if (c->graph_sets_state) c->set_sum_state(c->graph_end_state);
    return CPA_OK;
}

cpa_status cpa_destroy(cpa_ctx *c)
{
    if (!c) return fail(CPA_E_INVALID_ARG, "null context");
    cudaSetDevice(c->device);
    if (c->capturing) {  // abandon an unfinished capture
        cudaGraph_t g = nullptr;
        if (cudaStreamEndCapture(c->stream, &g) == cudaSuccess && g) cudaGraphDestroy(g);
        cudaGetLastError();
    }
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    cudaFree(c->d_vtab);
    cudaFree(c->d_sqrt_dw);
    cudaFree(c->d_maxabs);
    cudaFree(c->d_peak);
    cudaFree(c->d_best_rho);
    cudaFree(c->d_argmax);
    cudaFree(c->d_rank);
    cudaFree(c->d_best);
    cudaFree(c->d_counter);
    for (int k = 0; k < 2; k++) {
        cudaFree(c->d_stage[k]);
        cudaFree(c->d_stage_tx[k]);
        if (c->ev_copied[k]) cudaEventDestroy(c->ev_copied[k]);
        if (c->ev_used[k]) cudaEventDestroy(c->ev_used[k]);
    }
    cudaFree(c->d_pack);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->side_hi) {
        cudaStreamSynchronize(c->side_hi);
        cudaStreamDestroy(c->side_hi);
    }
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    cudaFree(c->d_offset);
    cudaFree(c->d_scale);
    cudaFree(c->d_part);
    cudaFree(c->d_hw32);
    cudaFree(c->d_hi);
    cudaFree(c->d_lo);
    cudaFree(c->d_nonfinite);
    cudaFreeHost(c->h_status);
    cudaFree(c->d_hist);
    cudaFree(c->d_clk);
    cudaFree(c->d_cs_cnt);
    cudaFree(c->d_cs_off);
    cudaFree(c->d_cs_cur);
    cudaFree(c->d_cs_perm);
    cudaFree(c->d_cs_S);
    for (auto &r : c->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    delete c;
    return CPA_OK;
}

}  // extern "C"
