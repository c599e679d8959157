/*
 * cpa.h -- C ABI of libcpa.so, the B200 (sm_100a) Correlation Power Analysis
 * engine for AES-128 following Gamaarachchi, Ragel & Jayasinghe,
 * "Accelerating Correlation Power Analysis Using GPUs" (arXiv:1412.7682).
 * [P:n] = line n of the paper text, [S:n] = line n of SPEC.md.
 *
 * Problem statement [P:65-67]: N power traces of M sample points W[i][j] and
 * the N matching ciphertexts (plaintexts for the first-round model) in; the
 * correlation of every (key byte b, sub-key guess k, sample j) by Eq. (1)
 * [P:69] and the round key (Phase 4, [P:85-87]) out.
 *
 * Hypothesis index h = 256*b + k (b = 0..15 key byte, k = 0..255 guess).
 *
 * Conventions for every function:
 *   - Returns cpa_status; CPA_OK = 0.  No C++ exception crosses the ABI.
 *   - Pointers named d_* are CUDA device pointers on the context's device,
 *     h_* are host pointers.  The caller owns every buffer it passes; a
 *     buffer passed to an asynchronous call must stay alive and unmodified
 *     until the next synchronising call (cpa_finalize, cpa_sync, cpa_destroy).
 *   - The library owns only its context, its lookup tables and its scratch.
 *   - Argument errors are reported synchronously; CUDA launch/runtime errors
 *     map to CPA_E_CUDA with detail in cpa_last_error().
 *   - Not thread-safe per context; distinct contexts are independent.
 */
#ifndef CPA_H
#define CPA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CPA_API __attribute__((visibility("default")))
#else
#define CPA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cpa_ctx cpa_ctx; /* opaque; one per GPU / rank */

typedef enum {
    CPA_OK = 0,
    CPA_E_INVALID_ARG = 1,        /* bad size, null pointer, misalignment */
    CPA_E_BAD_STATE = 2,          /* e.g. call on a destroyed context */
    CPA_E_CUDA = 3,               /* CUDA error, see cpa_last_error() */
    CPA_E_NO_MEMORY = 4,          /* device scratch allocation failed */
    CPA_E_TOO_FEW_TRACES = 5,     /* N < 2 at finalize: Eq. (1) undefined [S:268] */
    CPA_E_OVERFLOW = 6,           /* N beyond the exact-int64 bound (2^23 traces) */
    CPA_E_UNSUPPORTED_DEVICE = 7, /* not a compute-capability 10.0 (sm_100a) GPU */
    CPA_E_NONFINITE = 8           /* CPA_F32: a trace sample was NaN/Inf [S:140, S:176];
                                     sticky, reported by cpa_finalize */
} cpa_status;

typedef enum {
    CPA_S8 = 0,  /* signed 8-bit ADC samples (exact int path) */
    CPA_U8 = 1,  /* unsigned 8-bit ADC samples (exact int path) */
    CPA_F32 = 2  /* float32 samples (fp16 hi + e4m3 lo tensor-core path, fp64 sums) */
} cpa_dtype;

/* Selection function H [P:67, P:75] (the paper never writes it out; see
 * DESIGN.md "Readings"):                                                    */
typedef enum {
    CPA_HD_LAST = 0,  /* HW(InvS(c[b] ^ k) ^ c[SR(b)]), last round, ciphertexts [S:85] */
    CPA_HW_LAST = 1,  /* HW(InvS(c[b] ^ k)), last round, ciphertexts */
    CPA_HW_FIRST = 2  /* HW(S(p[b] ^ k)), first round, plaintexts [P:63] */
} cpa_model;

/* ---- packed accumulator ----------------------------------------------------
 * The Phase 1/2 sums [P:75, P:79] live in ONE caller-owned device buffer of
 * cpa_accum_words(M) 8-byte words, so that a multi-GPU run combines partial
 * sums with a single all-reduce(SUM) of that buffer between the last
 * cpa_accumulate and cpa_finalize (traces shard over GPUs, [P:230]).
 * Word layout (offsets in words):
 *   [0, 4096*M)            sum_i H_i W_ij   as [h][j]  (j fastest)
 *   [4096*M, +M)           sum_i W_ij
 *   [4097*M, +M)           sum_i W_ij^2
 *   [4098*M, +4096)        sum_i H_i
 *   [4098*M+4096, +4096)   sum_i H_i^2
 *   [4098*M+8192]          N (trace count)
 * Word type: int64 for CPA_S8/CPA_U8 (exact, order-independent); double for
 * CPA_F32 (all words, including N and the H sums, which stay exact < 2^53).
 */
CPA_API size_t cpa_accum_words(int32_t M);
CPA_API size_t cpa_accum_bytes(int32_t M);
CPA_API size_t cpa_accum_offset(int32_t M, int field); /* field: 0 HW,1 W,2 W2,3 H,4 H2,5 N */

/* Create a context for M samples per trace on CUDA device `device`.
 * stream: cudaStream_t (NULL = legacy default) all work is ordered on.
 * d_accum: caller-owned, cpa_accum_bytes(M) bytes, 256-byte aligned; it is
 * zeroed (asynchronously) here.  1 <= M <= 1<<22.                          */
CPA_API cpa_status cpa_init(cpa_ctx **out, int32_t M, cpa_dtype dtype, cpa_model model,
                    int device, void *stream, void *d_accum);

/* Add N traces to the sums (Phases 1-2, [P:73-79]); asynchronous.
 * d_traces: N rows of M samples, row stride ld ELEMENTS (ld >= M).  Fast path
 *   (read in place by TMA): base 16-byte aligned and ld*sizeof(elem) a
 *   multiple of 16; otherwise the rows are first copied (pitched D2D copy)
 *   into the library's aligned staging buffers.
 * d_texts: N x 16 bytes (ciphertexts; plaintexts for CPA_HW_FIRST), byte b =
 *   AES state byte b (column-major FIPS-197 order [S:107]).
 * N = 0 is a no-op.  Sums are exact (int path), so any chunking or ordering of
 * the traces gives bit-identical results.                                    */
CPA_API cpa_status cpa_accumulate(cpa_ctx *ctx, const void *d_traces, int64_t ld,
                          const uint8_t *d_texts, int64_t N);

/* Same, from HOST buffers: the library streams them through its own device
 * staging buffers (H2D copies overlapped with compute; contiguous rows, ld == M,
 * travel as one linear copy per chunk, which is what reaches full PCIe rate).  Synchronous: returns
 * after the last copy was consumed, so the host buffers may be reused.  Host
 * buffers should be pinned (cudaHostAlloc / cudaHostRegister) for speed.     */
CPA_API cpa_status cpa_accumulate_host(cpa_ctx *ctx, const void *h_traces, int64_t ld,
                               const uint8_t *h_texts, int64_t N);

typedef struct {
    uint8_t round_key[16];   /* Phase 4: best sub-key per byte [P:87] */
    uint8_t master_key[16];  /* key schedule inverted from round 10 [P:63]
                                (= round_key for CPA_HW_FIRST) */
    int32_t peak_sample[16]; /* sample j of max |rho| for the best sub-key */
    double peak_rho[16];     /* signed rho at that sample */
    int64_t n_traces;        /* N the result was computed from */
} cpa_result;

/* Phase 3 + 4 [P:81-87] from the (possibly all-reduced) accumulator; blocks
 * until done.  rho is Eq. (1) [P:69] in fp64 from the exact integer sums,
 * 0 where a variance term is 0 [S:293], clamped to [-1, 1] [S:246].
 * Optional device outputs (NULL to skip):
 *   d_rho     [4096][M] double   (h-major, j fastest)
 *   d_maxabs  [4096]    double   max_j |rho| per hypothesis [S:292]
 *   d_argmax  [4096]    int32    lowest j attaining it [S:298]
 *   d_rank    [4096]    int32    rank of k within byte b (1 = best; ties to
 *                                lower k [S:261, S:298])
 * res (host, may be NULL) receives the recovered key.  The checks on N (and
 * the float non-finite flag) are made after the kernels, from the one readback
 * the call does: on CPA_E_TOO_FEW_TRACES / CPA_E_OVERFLOW / CPA_E_NONFINITE the
 * device outputs are unspecified and res is not written.                     */
CPA_API cpa_status cpa_finalize(cpa_ctx *ctx, double *d_rho, double *d_maxabs,
                        int32_t *d_argmax, int32_t *d_rank, cpa_result *res);

/* Phase 3 + 4 enqueued on the context's stream WITHOUT blocking: streamed
 * checkpoints (the key-rank curve of config C5), where a synchronous finalize
 * after every chunk would leave the GPU idle while the host waits and then
 * launches the next chunk.  Same kernels and arithmetic as cpa_finalize (bit
 * for bit); results land in device memory in stream order, so a later
 * cpa_accumulate on the same stream may run before the caller reads them.
 *   d_rho, d_maxabs, d_argmax, d_rank: as cpa_finalize (NULL = internal
 *             scratch for maxabs/argmax/rank);
 *   d_best    optional [32] int32: best sub-key per byte [0..15] and its peak
 *             sample [16..31].
 * Checks without blocking: CPA_E_TOO_FEW_TRACES / CPA_E_OVERFLOW from the
 * traces this context accumulated since its last reset (N = 1, or > 2^23 for
 * int traces; cpa_accumulate also refuses a running total past 2^23); not
 * checked when none were accumulated here (an externally combined
 * accumulator).  The non-finite flag (f32) is only reported by the blocking
 * calls (cpa_finalize, cpa_finalize_rows): end a stream with one of them.   */
CPA_API cpa_status cpa_finalize_async(cpa_ctx *ctx, double *d_rho, double *d_maxabs, int32_t *d_argmax,
                                      int32_t *d_rank, int32_t *d_best);

/* ---- CUDA-graph replay of a fixed-shape step ------------------------------
 * cpa_graph_begin starts capturing the context's stream (stream capture, thread-
 * local mode; the context's stream must not be the legacy default stream):
 * the calls made until cpa_graph_end are recorded instead of run, and
 * cpa_graph_launch then replays them on the context's stream as ONE graph
 * launch, asynchronously (no per-kernel launch cost, no host work between the
 * kernels of a step).  Capturable: cpa_reset, cpa_accumulate on 16-byte aligned
 * device buffers (not with class sums), cpa_finalize_async; a captured
 * cpa_accumulate needs a captured cpa_reset before it (a replay starts from
 * zeroed sums), and the buffers it allocates on first use (float planes) must
 * already exist -- run the step once outside the capture first.  Calls that
 * synchronise, read back or allocate (cpa_finalize, cpa_finalize_rows,
 * cpa_select, cpa_accumulate_host, cpa_sync, cpa_phase_times, the offset calls)
 * return CPA_E_INVALID_ARG while capturing.  The host's record of the sums
 * (traces since reset, first-touch and CPA_OPT_NARROW shadow state) is left as
 * before the capture by cpa_graph_end and set to the graph's end state by each
 * replay of a graph that begins with cpa_reset; replays update nothing else on
 * the host (launch count, phase times: CPA_OPT_TIMING events are not
 * captured); the pointers and sizes are those of the capture.
 * cpa_graph_end replaces a previous graph; cpa_destroy frees it.            */
CPA_API cpa_status cpa_graph_begin(cpa_ctx *ctx);
CPA_API cpa_status cpa_graph_end(cpa_ctx *ctx);
CPA_API cpa_status cpa_graph_launch(cpa_ctx *ctx);

/* ---- fused multi-GPU combine ([P:230]) -----------------------
 * cpa_set_row_owners: the cross-term kernel adds its int64 partial sum_hw of key
 * byte b (hypothesis rows [256 b, 256 b + 256)) straight into the packed
 * accumulator owners[b] -- typically a peer GPU's, mapped with cpa_ipc_open and
 * reached over NVLink with system-scope atomics -- instead of into this
 * context's own accumulator.  The reduce-scatter of the rows then happens
 * inside the kernel's epilogue, overlapped with the MMAs; only the small fields
 * (sum_w, sum_w2, sum_h, sum_h2, N), which stay in this context's accumulator,
 * still need an all-reduce.  owners[b] NULL = this context's accumulator;
 * owners NULL = off.  int8 traces and the tensor-core path only
 * (CPA_E_INVALID_ARG otherwise).  The caller zeroes every owner accumulator and
 * synchronises the ranks before the first cpa_accumulate, and after the last
 * one before an owner reads its rows (cpa_finalize_rows).  Exact: integer
 * atomics are order-independent, results are bit-identical to one GPU.        */
CPA_API cpa_status cpa_set_row_owners(cpa_ctx *ctx, void *const owners[16]);

/* CUDA IPC of a device buffer (e.g. a torch-allocated accumulator inside a
 * larger allocation): cpa_ipc_export writes a 64-byte handle of the allocation
 * containing d_ptr and the byte offset of d_ptr in it; cpa_ipc_open maps it in
 * another process (same or peer GPU, peer access enabled) and returns the
 * pointer at that offset; cpa_ipc_close unmaps the BASE (pointer - offset).   */
CPA_API cpa_status cpa_ipc_export(const void *d_ptr, uint8_t handle[64], uint64_t *offset);
/* *ok = 1 when device `dev` can access `peer`'s memory with native atomics
 * (peer access + cudaDevP2PAttrNativeAtomicSupported; always 1 for dev == peer):
 * the precondition of routing rows to a peer with cpa_set_row_owners.       */
CPA_API cpa_status cpa_peer_atomics(int dev, int peer, int *ok);
CPA_API cpa_status cpa_ipc_open(const uint8_t handle[64], uint64_t offset, void **d_ptr);
CPA_API cpa_status cpa_ipc_close(void *d_base);

/* ---- sharded Phase 3/4 (multi-GPU) ---------------------------
 * Two ways to split the work of Phase 3 [P:81-83] over G ranks:
 *  (rows)    trace-sharded accumulation; ONE reduce-scatter of the sum_hw rows
 *            (rank r receives hypothesis rows [4096 r/G, 4096 (r+1)/G)) plus an
 *            all-reduce of the small fields (sum_w, sum_w2, sum_h, sum_h2, N);
 *            each rank runs cpa_finalize_rows on its rows; the per-hypothesis
 *            maxima are all-gathered and cpa_select(G = 1) ranks them.
 *  (columns) sample-axis sharding for wide traces: rank r accumulates ALL
 *            traces over its own sample columns (CPA_OPT_COL0 = its first
 *            column), so no sums are exchanged; cpa_finalize_rows(0, 4096) on
 *            every rank, an all-gather of the maxima into [G][4096], then
 *            cpa_select(G) merges them and ranks.
 *
 * cpa_finalize_rows: Eq. (1) [P:69] and max|rho| over this context's samples
 * (Phase 3) for hypotheses h in [h0, h1) only, from the accumulator (whose
 * sum_hw rows [h0, h1) and small fields must hold the combined sums).  Blocks
 * until done.  Same arithmetic as cpa_finalize, bit for bit.
 *   d_rho     optional [h1-h0][M] double (row h at (h-h0)*M)
 *   d_maxabs  [4096] double, d_argmax [4096] int32, d_peak [4096] double
 *             (signed rho at the argmax): only entries h0..h1-1 are written;
 *             argmax is the GLOBAL sample index (local j + CPA_OPT_COL0).
 * Errors as cpa_finalize; CPA_E_INVALID_ARG for a bad row range or a NULL
 * maxabs/argmax/peak.                                                        */
CPA_API cpa_status cpa_finalize_rows(cpa_ctx *ctx, int32_t h0, int32_t h1, double *d_rho,
                                     double *d_maxabs, int32_t *d_argmax, double *d_peak);

/* cpa_select: Phase 4 [P:85-87] from per-hypothesis maxima.  Inputs are G
 * stacked shards, d_maxabs/d_peak [G][4096] double and d_argmax [G][4096]
 * int32 (global sample indices).  For G > 1 the shards are first merged IN
 * PLACE into shard 0 (largest max|rho|; ties to the lowest sample index
 * [S:298]).  Then, as in cpa_finalize: d_rank [4096] (optional) receives the
 * rank of k within byte b, and res (host, optional) the key, peak samples,
 * signed peak rho and N (read from this context's accumulator).  Blocks.     */
CPA_API cpa_status cpa_select(cpa_ctx *ctx, int32_t G, double *d_maxabs, int32_t *d_argmax,
                              double *d_peak, int32_t *d_rank, cpa_result *res);

/* CPA_F32 only: per-sample offsets o_j (device pointer, M floats; NULL = 0)
 * subtracted from every sample before the fp16 hi / e4m3 lo split.  rho is invariant
 * to per-sample offsets [S:285]; centring keeps the split and the fp32 tensor-
 * core accumulation accurate.  Default: the mean of the first <= 1024 traces
 * of the first cpa_accumulate call (cpa_default_offsets).  Multi-GPU: every rank must use the same offsets (the
 * accumulated sums are of the offset samples; a caller combining ranks sets
 * them explicitly, e.g. rank 0's cpa_default_offsets broadcast to every rank).  The
 * finalize also reads them: SPEC's degenerate-column rule compares dw with the
 * RAW second moment [S:293], rebuilt from the centred sums and o_j.  Setting offsets also re-derives
 * the split's per-sample power-of-two scales (from the next accumulate's first
 * <= 64 traces; a precision choice that never changes the sums' meaning).   */
CPA_API cpa_status cpa_set_offsets(cpa_ctx *ctx, const float *d_offsets);
/* CPA_F32 only: copy the offsets in force (M floats; 0 until set) to d_out
 * (device, may be NULL; asynchronous on the context's stream) and report in
 * *is_set (may be NULL) whether they were set -- by cpa_set_offsets or by the
 * first cpa_accumulate.  Lets a multi-GPU caller verify that every rank's sums
 * are centred on the same offsets before it adds them (paper_1412_7682_b200.
 * multigpu.check_same_offsets).  CPA_E_INVALID_ARG for an int context.       */
CPA_API cpa_status cpa_get_offsets(cpa_ctx *ctx, float *d_out, int *is_set);
/* CPA_F32 only: write the offsets the library would choose by default for the
 * device traces d_traces (N rows, stride ld elements) -- the per-sample mean of
 * the first min(N, 1024) rows -- to d_out (device, M floats), asynchronously on
 * the context's stream, without changing the context.  A multi-GPU caller runs
 * it on one rank and broadcasts the result to every rank's cpa_set_offsets.  */
CPA_API cpa_status cpa_default_offsets(cpa_ctx *ctx, const float *d_traces, int64_t ld, int64_t N,
                                       float *d_out);

CPA_API cpa_status cpa_reset(cpa_ctx *ctx);    /* zero the accumulator and the
                                                  non-finite flag (async) */
/* After cpa_init / cpa_reset the library knows sum_hw is zero: the first
 * int8 cpa_accumulate whose work units each cover all of its traces (one trace
 * chunk) STORES its sums instead of adding them (half the HBM traffic of the
 * spill).  So the caller must not write the sum_hw field between cpa_init /
 * cpa_reset and the next cpa_accumulate (contexts with row owners -- which
 * receive peer adds -- never store).                                        */
CPA_API cpa_status cpa_sync(cpa_ctx *ctx);     /* wait for all queued work */
CPA_API cpa_status cpa_destroy(cpa_ctx *ctx);  /* frees the context (not d_accum) */

/* Tuning / test knobs.
 *   CPA_OPT_KCHUNK: traces per split-K work unit of the cross-term kernel
 *                   (multiple of 128, <= 2^20; 0 = automatic).
 *   CPA_OPT_TIMING: nonzero = record CUDA events on the context's stream
 *                   around every kernel launch (read with cpa_phase_times).
 *   CPA_OPT_OVERLAP: how the trace-moment pass (a4) runs next to the cross
 *                   term (int8 traces): 0 = serialised on the context's
 *                   stream; 1 = launched after it on a low-priority side
 *                   stream; 2 = launched before it on a high-priority side
 *                   stream, one block per SM, co-resident with the cross-term
 *                   CTAs; 3 (default) = fused: the cross-term kernel sums the
 *                   W tiles it stages anyway (no separate pass, no extra HBM
 *                   reads).  All modes give identical (exact) sums.
 *   CPA_OPT_STAGE_BYTES: bytes of trace rows per staging chunk of
 *                   cpa_accumulate_host / unaligned cpa_accumulate
 *                   (0 = default 256 MiB; at least one row per chunk).
 *   CPA_OPT_COL0:   global index of this context's sample 0 (sample-axis
 *                   sharding); added to every reported sample index
 *                   (argmax, peak_sample).  Default 0.
 *   CPA_OPT_CLASS_SUMS: 1 = compute the cross term sum H*W by class sums
 *                   (SURVEY 8f NEXT-4): for HW_LAST / HW_FIRST, H depends on
 *                   one text byte x, so sum_i H W_ij = sum_x f(x ^ k) S_b[x][j]
 *                   with S_b[x][j] the sum of W_ij over the traces whose byte b
 *                   is x [P:63, P:79].  Exact (bit-identical to 0).  Needs a
 *                   single-byte model and s8/u8 traces, else
 *                   CPA_E_INVALID_ARG.  Allocates 64 B per trace (<= 2^17
 *                   traces per chunk) + 16 KB per sample (<= 8192 samples per
 *                   block) of scratch on first use.  Default 0 (tensor cores).
 *   CPA_OPT_FUSE_HIST: 1 = for calls of >= 65536 traces the cross-term kernel
 *                   counts the (c_b, c_SR(b)) byte pairs that a3's sum H,
 *                   sum H^2 are contracted from [P:75] as it generates H (no
 *                   separate histogram pass); 0 (default) = separate pass
 *                   (the fused counting cost the cross term what the pass
 *                   cost).  Same exact sums either way.
 *   CPA_OPT_XT_TILES: int8 cross-term variant: 0 (default) = 1; 1 = two
 *                   256-sample tiles per work unit
 *                   (one generated H tile feeds both; a4 fused per OVERLAP;
 *                   the unit's spill waits for its MMAs); 2 = one tile per
 *                   unit with double-buffered TMEM accumulators (the spill
 *                   overlaps the next unit's MMAs: short units, i.e. wide or
 *                   few traces; a4 then runs as a separate pass; measured
 *                   slower on B200).  Same exact sums either way.
 *                   Float traces (CPA_F32): 0 (default) = 1 = two sample tiles
 *                   per unit from one generated H tile, single-buffered fp32
 *                   accumulators spilled every <= 24576 traces; 2 = one tile,
 *                   double-buffered, every <= 4096 traces (measured slower,
 *                   DESIGN.md).  Both within the float tolerance.
 *   CPA_OPT_SPILL:  how the cross term adds each work unit's 32-bit TMEM
 *                   accumulators into sum_hw: 1 = one red.global.add per
 *                   element; 2 = bulk tensor reduce-add
 *                   (cp.reduce.async.bulk.tensor: the TMA unit adds 32 x 8
 *                   int64 / fp64 boxes; needs M even and no row owners, else
 *                   1); 3 = partial sums: each unit STORES its raw int32 /
 *                   fp32 accumulators into its trace chunk's slice of a
 *                   scratch buffer (4096 x 4 B per sample per chunk, <= 3 GiB,
 *                   allocated on first use; else 1), then one pass adds the
 *                   slices into sum_hw (no row owners).  0 (default): int8 =
 *                   2 for work units of >= 65536 traces, else 1; float = 1
 *                   (measured).  Exact (int8) / within the float
 *                   tolerance (float) either way.
 *   CPA_OPT_NARROW: int8 traces. 1 = keep the cross-term field sum_hw in a
 *                   context-owned int32 shadow (4096 x M x 4 bytes, allocated
 *                   by this call; not capturable) while it is exact: while the
 *                   traces in it satisfy N * 8 * max|W| < 2^31 (max|W| = 128
 *                   s8 / 255 u8: N <= 2097151 / 1052688; max|H| = 8 for every
 *                   model).  The cross term then stores / adds 32-bit words
 *                   and cpa_finalize* read the shadow: half the sum_hw bytes in
 *                   both.  The ACCUMULATOR's HW field is stale while the shadow
 *                   is live: cpa_flush adds the shadow into it (call it before
 *                   reading, combining or exporting the accumulator); an
 *                   accumulate that would pass the bound, or uses class sums,
 *                   row owners or CPA_OPT_SPILL 2 / 3, flushes first and goes on
 *                   in int64; cpa_reset drops the shadow.  A value > 1 also
 *                   caps the shadow at that many traces (tests).  0 (default):
 *                   off (flushes a live shadow).  Ignored for float traces.
 *                   Results are bit-identical either way.                     */
enum { CPA_OPT_KCHUNK = 1, CPA_OPT_TIMING = 2, CPA_OPT_OVERLAP = 3, CPA_OPT_STAGE_BYTES = 4,
       CPA_OPT_COL0 = 5, CPA_OPT_CLASS_SUMS = 6, CPA_OPT_FUSE_HIST = 7, CPA_OPT_XT_TILES = 8,
       CPA_OPT_SPILL = 9, CPA_OPT_NARROW = 10 };

/* CPA_OPT_NARROW: add a live int32 shadow of sum_hw into the accumulator's HW
 * field (one kernel on the context's stream, asynchronous; capturable) so the
 * accumulator holds every sum.  No-op without a live shadow.                 */
CPA_API cpa_status cpa_flush(cpa_ctx *ctx);
CPA_API cpa_status cpa_set_option(cpa_ctx *ctx, int option, int64_t value);

/* Per-phase device time (ms) and launch count since the last call, from the
 * CPA_OPT_TIMING events; synchronises the stream.  Phases:
 *   0 model sums (a3)  1 trace moments (a4)  2 cross term (a5/a6)
 *   3 Eq. (1) finalize (a8)  4 phase-4 ranking (a9)
 *   5 partial-sum reduce of the cross term (CPA_OPT_SPILL 3)                */
enum { CPA_NUM_PHASES = 6 };
CPA_API cpa_status cpa_phase_times(cpa_ctx *ctx, double ms[CPA_NUM_PHASES],
                                   int64_t launches[CPA_NUM_PHASES]);

/* Average SM clock (MHz) of the last cross-term launch, from the
 * clock64 and %globaltimer readings its first CTA takes at its start and end
 * (0 if none ran).  Synchronises the stream.  The roofline's issue-rate
 * ceiling at the clock the power cap actually left the kernel.             */
CPA_API cpa_status cpa_xterm_clock(cpa_ctx *ctx, double *mhz);

/* Kernel launches issued by this context since creation (for bench
 * accounting).                                                              */
CPA_API int64_t cpa_launch_count(const cpa_ctx *ctx);

CPA_API const char *cpa_status_str(cpa_status s);
CPA_API const char *cpa_last_error(void); /* thread-local detail of the last error */

/* ---- host helpers (pure, no GPU) ---------------------------------------- */
CPA_API void cpa_aes_expand_key(const uint8_t key[16], uint8_t round_keys[11][16]);
/* master key whose expansion has `rk` as round key `round` (1..10) [P:63] */
CPA_API void cpa_aes_invert_key_schedule(const uint8_t rk[16], int round, uint8_t key[16]);

#ifdef __cplusplus
}
#endif
#endif /* CPA_H */
