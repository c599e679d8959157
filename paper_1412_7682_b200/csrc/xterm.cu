// xterm.cu -- the dominant Phase-2 term [P:79]:
//     sum_hw[h][j] = sum_i H_i(h) * W[i][j]      (h = 256 b + k, 4096 rows)
// as a 4096 x N . N x M contraction on the sm_100a tensor cores.  One kernel
// template, two instantiations:
//   I8  (a5): W int8 (s8/u8), tcgen05.mma kind::i8, exact int32 accumulation in
//        TMEM, spilled to int64 with red.add (bit-exact for any schedule);
//   F32 (a6): W float32 pre-split (k_split_f32) into an fp16 hi plane and an e4m3
//        lo plane (per-sample power-of-two scale s_j): per 64-trace stage 4
//        kind::f16 MMAs (H 2^-16 . hi, K = 16; the fp16 bits of H 2^-16 are H << 8)
//        and 2 kind::f8f6f4 MMAs (H 2^-16 . lo, K = 32; the e5m2 code of H 2^-16
//        is the byte H, lo is e4m3) into ONE fp32 TMEM
//        accumulator over <= 4096 traces per work unit -- 3/4 of the tensor time
//        of two 16-bit MMAs -- spilled to fp64 x 1/s_j with atomicAdd [P:201-217].
//
// The paper computed this serially per (k, b, j) thread [P:121]; here a CTA
// PAIR (cluster of 2, tcgen05 cta_group::2) owns one key byte b (M = 256
// sub-keys, 128 per CTA) and NT = 2 N tiles of 256 samples (I8; F32: one):
//   * A = H (128 sub-keys x BK traces per CTA, MN-major, 128B swizzle) is
//     GENERATED in shared memory from the ciphertext bytes: H[k] = V[c_s][c_b^k]
//     with V[y][x] = HW(InvS[x] ^ y) (nibble-packed 32 KB table in smem), see the
//     generator section.  One A tile feeds NT accumulators, so the generation
//     cost per MAC halves (KB=2, NT=1 -- two key bytes sharing one W tile -- was
//     measured 1.3 ms slower at C4: generation costs issue slots, TMA does not).
//   * B = W (MN-major = the caller's trace-major layout, no transpose): each CTA
//     TMA-loads HALF of each N=256 tile.
//   * Per 128-trace stage: 4 K steps x NT MMAs, one tcgen05.commit per ring
//     (a commit costs ~45 clk of tensor-pipe time, tools/mma_bench); A ring 3 x
//     16 KB, W ring 4 x 32 KB.
//   * Work unit = (byte, trace chunk, N tile group), byte fastest, handed out IN
//     ORDER by a global atomic counter (leader CTA) so the units in flight share
//     a few W blocks in L2 (W streams from HBM about once).
//   * Fused a4 (moments_pass): the epilogue warps, idle during the mainloop,
//     sum W and W^2 over 1/16 of the rows of every W stage they see.
// Warp roles (512 threads per CTA): w0 scheduler (leader) + W TMA producer,
// w1 MMA issuer (leader), w2 TMEM owner, w3
// ciphertext producer, w4-7 epilogue (TMEM lanes 32*(w%4)...) + fused moments,
// w8-15 H generators (8: measured ~1% faster than 16 once NT = 2 halved the generation).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

// XT_EXP (profiling builds only, tools/xt_exp.sh; results are NOT valid):
//   bit 0: W loads re-read the first 8192 traces (L2-resident W)
//   bit 1: generators skip the H generation (barrier traffic only)
//   bit 2: the epilogue skips its global atomics (TMEM reads only)
//   bit 4: no W loads (the leader's producer arrives without tx bytes)
//   bit 32: F32 skips the e4m3 lo MMAs; bit 64: F32 skips the fp16 hi MMAs
#ifndef XT_EXP
#define XT_EXP 0
#endif
#ifndef XT_KB_I8
#define XT_KB_I8 1
#endif
#ifndef XT_NT_I8
#define XT_NT_I8 2
#endif
#ifndef XT_A_STAGES_I8
#define XT_A_STAGES_I8 3
#endif
#ifndef XT_B_STAGES_I8
#define XT_B_STAGES_I8 4
#endif
#ifndef XT_BK_F32
#define XT_BK_F32 64
#endif
#ifndef XT_A_STAGES_F32
#define XT_A_STAGES_F32 4  // (4, 3): C3 cross term 5.00 vs 5.12 ms for (3, 4), 5.25 for (2, 5)
#endif
#ifndef XT_B_STAGES_F32
#define XT_B_STAGES_F32 3
#endif

namespace cpa {
namespace {

// Kernel variants: V_I8 (NT = 2 sample tiles per unit, one accumulator set, fused
// a4), V_F32 (a6), V_I8O (int8 with NT = 1 and double-buffered accumulators: the
// epilogue overlaps the next unit's MMAs; for short units, where the spill of a
// unit would otherwise stall the tensor pipe -- wide traces, few traces).
// V_F32N (a6 with NT = 2): one generated H tile feeds two sample tiles (half the
// generator stores and V reads per MMA, the smem port being what bounds V_F32),
// single-buffered accumulators (the epilogue is exposed; units of <= 24576 traces,
// 32 traces per stage, one ring: one commit frees a stage's H and W slots).
constexpr int V_I8 = 0, V_F32 = 1, V_I8O = 2, V_F32N = 3;
#ifndef XT_UNI_F32N
#define XT_UNI_F32N 1
#endif
#ifndef XT_BK_F32N
#define XT_BK_F32N 32
#endif
#ifndef XT_A_STAGES_F32N
#define XT_A_STAGES_F32N 4
#endif
#ifndef XT_B_STAGES_F32N
#define XT_B_STAGES_F32N 4
#endif
template <int V>
struct Cfg {
    static constexpr bool F32 = V == V_F32 || V == V_F32N;
    static constexpr int ESZ = F32 ? 2 : 1;         // bytes per operand element
    static constexpr int KMMA = F32 ? 16 : 32;      // K per MMA instruction
    static constexpr int KB = F32 ? 1 : XT_KB_I8;   // key bytes per unit (A tiles sharing one W tile)
    static constexpr int NT = V == V_I8 ? XT_NT_I8 : (V == V_F32N ? 2 : 1);  // N=256 sample tiles per unit
    static constexpr int NBUF = (V == V_I8 || V == V_F32N) ? 1 : 2;           // TMEM accumulator buffers
    static constexpr int NACC = KB * NT;            // N=256 accumulators per unit
    static constexpr int BK = V == V_F32N ? XT_BK_F32N : (F32 ? XT_BK_F32 : 128);  // traces per pipeline stage
    static constexpr int BOX_X = 128 / ESZ;         // samples per TMA box (128-byte swizzle span)
    static constexpr int BH_BYTES = BK * 128 * ESZ; // one CTA's half (128 samples) of one N tile: W (I8) / hi (F32)
    static constexpr int BL_BYTES = F32 ? BK * 128 : 0;  // F32: the same half of the e4m3 lo plane
    static constexpr int A_BYTES = BK * 128 * ESZ;  // 128 keys x BK traces: H (I8) / fp16(H) (F32)
    static constexpr int A8_BYTES = F32 ? BK * 128 : 0;  // F32: the e5m2 tile of H 2^-16 (= the bytes H)
    static constexpr int A_ATOM = BK * 128;         // bytes between 128-byte MN groups (A and B)
    static constexpr int A_STAGE = KB * A_BYTES + A8_BYTES;        // generated H tiles of one stage
    static constexpr int B_STAGE = NT * (BH_BYTES + BL_BYTES);     // TMA-loaded W tiles of one stage
    // separate rings: W (TMA, long latency) runs deeper than H (generated on chip)
    static constexpr int A_STAGES = V == V_F32N ? XT_A_STAGES_F32N : (F32 ? XT_A_STAGES_F32 : XT_A_STAGES_I8);
    static constexpr int B_STAGES = V == V_F32N ? XT_B_STAGES_F32N : (F32 ? XT_B_STAGES_F32 : XT_B_STAGES_I8);
    // one ring (V_F32N): the H and W slots of a stage are freed by ONE commit (a
    // tcgen05.commit costs tensor-pipe time; 6 MMAs per stage are too few to hide two)
    static constexpr bool UNI = V == V_F32N && XT_UNI_F32N;
};

constexpr int BMC = 128;          // sub-keys per CTA (pair MMA M = 256)
constexpr int BN = 256;           // samples per accumulator (MMA N)
#ifndef XT_VLDS64
#define XT_VLDS64 1
#endif
#ifndef XT_PREFETCH
#define XT_PREFETCH 0
#endif
constexpr int PREFETCH_STAGES = XT_PREFETCH;  // >0: W boxes prefetched into L2 this many stages ahead
constexpr int TX_STAGES = 4;      // ciphertext ring, prefetched ahead of the stages
constexpr int SCHED_Q = 4;        // depth of the unit-id ring
// V[y][x] = HW(InvS[x] ^ y) is 0..8: stored as nibbles, V[y][2i] | V[y][2i+1] << 4
// (32 KB; the freed 32 KB deepens the W ring)
constexpr int V_BYTES = 32768;
constexpr int EPI_WARPS = 4;
#ifndef XT_GEN_WARPS
#define XT_GEN_WARPS 8
#endif
constexpr int GEN_WARPS = XT_GEN_WARPS;       // every generator warp works on every stage, so
                                              // each waits every phase of every slot in order
                                              // (mbarrier parity waits are 1-bit)
// readers of the unit-id ring: leader = MMA + text producer + epilogue + generators,
// peer = W producer + text producer + epilogue + generators
constexpr int RING_CONSUMERS = 2 * (2 + EPI_WARPS + GEN_WARPS);
#ifndef XT_ST32_ROWS2
#define XT_ST32_ROWS2 1  // narrow first-touch spill: 2 rows x 64 B per warp-wide store
#endif
constexpr int TB_LD = 9;                      // epilogue transpose row stride (words, odd)
// epilogue staging (union): the red.add path's transpose buffer, or the bulk
// path's int64 boxes (per epilogue warp one 32 rows x 8 samples box, 64-byte
// swizzled, 2 KB; the TMA reduce reads it while the warp loads the next columns)
constexpr int RB_BYTES = 32 * 8 * 8;
constexpr int TB_BYTES = (EPI_WARPS * RB_BYTES > EPI_WARPS * 32 * TB_LD * 4) ? EPI_WARPS * RB_BYTES
                                                                             : EPI_WARPS * 32 * TB_LD * 4;
constexpr int MAX_RING = 8;                   // barrier slots reserved per ring
constexpr int SMEM_V = 0;
constexpr int SMEM_A = SMEM_V + V_BYTES;      // A ring, then the B ring (per-config sizes)
constexpr int NUM_BARS = 4 * MAX_RING + 2 * TX_STAGES + 4 + 2 * SCHED_Q + 2 * MAX_RING;
constexpr int THREADS = 32 * (8 + GEN_WARPS);
constexpr uint32_t TMEM_COLS = 512;
template <int V>
__host__ __device__ constexpr int smem_b() { return SMEM_A + Cfg<V>::A_STAGES * Cfg<V>::A_STAGE; }
// per-variant shared-memory layout: [V table | A ring, B ring | epilogue staging |
// ciphertext ring | barriers | unit-id ring, TMEM slot]
template <int V>
struct Lay {
    using C = Cfg<V>;
    static constexpr int RINGS = (C::A_STAGES * C::A_STAGE + C::B_STAGES * C::B_STAGE + 1023) / 1024 * 1024;
    static constexpr int TXB = C::BK * 16;         // ciphertext rows of one stage
    static constexpr int TB = SMEM_A + RINGS;      // 1 KB aligned (64-byte-swizzled TMA boxes)
    static constexpr int TX = TB + TB_BYTES;
    static constexpr int BAR = TX + TX_STAGES * TXB;
    static constexpr int SCHED = BAR + NUM_BARS * 8;
    static constexpr int ALLOC = SCHED + SCHED_Q * 4 + 16;
};
template <int V>
constexpr bool cfg_ok()
{
    using C = Cfg<V>;
    return C::A_STAGES <= MAX_RING && (!C::UNI || C::A_STAGES == C::B_STAGES) && C::B_STAGES <= MAX_RING &&
           C::NACC * C::NBUF * BN == (int)TMEM_COLS && Lay<V>::TB % 1024 == 0 && Lay<V>::ALLOC <= 232448;
}
static_assert(cfg_ok<V_I8>() && cfg_ok<V_F32>() && cfg_ok<V_I8O>() && cfg_ok<V_F32N>(),
              "rings, barriers, TMEM columns, shared memory");

struct Params {
    const uint8_t *texts;    // N x 16
    const uint8_t *vtab;     // 256 x 256 (global copy of V)
    void *hw;                // sum_hw [4096][M]: int64 (I8) or double (F32)
    // fused multi-GPU combine (I8; all null = off): key byte b's rows go to the
    // packed accumulator owners[b] (a peer GPU's, mapped over NVLink), with
    // system-scope atomics, instead of to hw -- the reduce-scatter happens
    // inside the epilogue, overlapped with the MMAs
    int64_t *owners[16];
    // clock probe (null = off): CTA 0 records (globaltimer ns, clock64) at its
    // start and end, so the host can derive the SM clock the kernel ran at
    unsigned long long *clk;
    int *unit_counter;       // zeroed before the launch
    int32_t M;
    int32_t n_tiles;         // tiles of NT*256 samples
    int32_t groups;          // key-byte groups (16 / KB)
    int32_t kc_count;
    int32_t units;
    // tail split (one trace chunk per tile): units [0, full_units) are whole
    // tiles; the remaining tiles are cut into pieces of tail_len traces, ordered
    // piece-major, so the last wave is filled by short units instead of leaving
    // pairs idle (full_units == units: no tail split; see tail_split)
    int32_t full_units;
    int64_t tail_len;
    int64_t N;
    int64_t kc_len;
    uint32_t idesc;
    uint32_t idesc8;         // F32: kind::f8f6f4 (e4m3) descriptor of the lo MMAs
    const float *inv_scale;  // F32: [M] 1 / s_j, applied at the fp64 spill
    // fused a4 (I8 only; null = off): the epilogue warps add sum W, sum W^2 of
    // 1/8 of the rows of every W tile they stage (moments_pass)
    int64_t *sum_w;
    int64_t *sum_w2;
    int32_t w_signed;
    // int8 spill by bulk tensor reduce-add (tmap_hw valid; else red.add.u64)
    int32_t bulk_spill;
    // first touch: sum_hw is known zero and every (row, sample) belongs to ONE
    // work unit of this launch (one trace chunk), so the spill stores instead of
    // adding: half the HBM traffic of a read-modify-write of sum_hw
    int32_t store_hw;
    // fused a3 histogram (null = off): the leader's generators of the units of
    // N tile group 0 count each trace's (c_b, c_SR(b)) pair of their key byte
    // (k_hist_contract turns the counts into sum H, sum H^2 afterwards)
    uint32_t *hist;
    // partial-sum spill (null = off): each unit STORES its raw 32-bit
    // accumulators (int32 / fp32 bits) into its trace chunk's slice
    // part[kc][4096][part_ld] -- plain stores, no read-modify-write of sum_hw in
    // the exposed epilogue; launch_part_reduce adds the slices into sum_hw after
    uint32_t *part;
    int64_t part_ld;
    // narrow sums (CPA_OPT_NARROW): hw is an int32 [4096][M] array (the host
    // guarantees N max|H| max|W| < 2^31, so the int32 sums are exact); first
    // touch stores / red.add.u32 of half the bytes
    int32_t hw32;
};

template <int V>
__device__ __forceinline__ void unit_coords(const Params &p, int u, int &b, int &n_tile, int64_t &t0, int64_t &t1)
{
    if (u >= p.full_units) {  // tail piece: (tile, piece), tiles fastest within a piece
        const int tail_tiles = p.groups * p.n_tiles - p.full_units;
        const int v = u - p.full_units, tile = p.full_units + v % tail_tiles;
        b = (tile % p.groups) * Cfg<V>::KB;
        n_tile = tile / p.groups;
        t0 = (int64_t)(v / tail_tiles) * p.tail_len;
        t1 = t0 + p.tail_len;
        if (t1 > p.N) t1 = p.N;
        return;
    }
    // b = first key byte of the unit's group (bytes b .. b+KB-1)
    b = (u % p.groups) * Cfg<V>::KB;
    const int r = u / p.groups;
    const int kc = r % p.kc_count;
    n_tile = r / p.kc_count;
    t0 = (int64_t)kc * p.kc_len;
    t1 = t0 + p.kc_len;
    if (t1 > p.N) t1 = p.N;
}

__device__ __forceinline__ int shiftrows_src(int b) { return (b & 3) + 4 * (((b >> 2) + (b & 3)) & 3); }

// The fp16 value H 2^-16 for two bytes H0 (byte sel0) and H1 of w, H in 0..8: its
// bit pattern is H << 8 (0x0100..0x0300 are the subnormals m 2^-24 with m = 256 H,
// 0x0400 = 2^-14, 0x0500..0x0700 = (1 + m/1024) 2^-14, 0x0800 = 2^-13: all H 2^-16),
// so one PRMT places H0, H1 in bytes 1 and 3 -- no conversion arithmetic.
__device__ __forceinline__ uint32_t f16x2_h16_of_bytes(uint32_t w, uint32_t sel)
{
    return __byte_perm(w, 0u, sel);
}

// Fused a4 [P:79]: sum W_ij and sum W_ij^2, read from the W ring while the MMAs
// consume it.  Each W tile (trace chunk x NT*256 samples) is staged by the units
// of all G = 16 / KB key-byte groups; the unit of group g sums rows
// g*128/G .. (g+1)*128/G - 1 of every 128-trace stage over its CTA's NT x 128
// samples, so every (trace, sample) is counted exactly once and the work is
// spread evenly over all units (KB * NT == 2: 4 warps x 32 lanes x 4 rows x 4
// samples = 128/G rows x NT*128 samples).  Thread (warp q, lane) owns samples
// 4 lane .. 4 lane + 3 of N tile q % NT, rows 4 (q / NT) .. + 3 of the group's
// slice: 4 LDS.32 (one 128-byte row per warp instruction, conflict-free), a 4x4
// byte transpose (8 PRMT) puts the 4 traces of one sample in a word, and IDP4A
// adds 4 values (x 1) or 4 squares (x itself) per instruction.  Per-thread sums
// are exact in 32 bits (a unit of <= 2^20 traces gives a thread <= 2^15 rows:
// |sum W| <= 2^22, sum W^2 <= 65025 * 2^15 < 2^31); they are added to the int64
// sums with atomics (exact, order-independent).  TMA zero fill (rows >= N,
// samples >= M) adds nothing.
template <bool SIGNED>
__device__ __forceinline__ uint32_t dp4(uint32_t a, uint32_t b, uint32_t c)
{
    if constexpr (SIGNED) return (uint32_t)__dp4a((int)a, (int)b, (int)c);
    else return __dp4a(a, b, c);
}
template <bool SIGNED>
__device__ __forceinline__ void moments_pass(const Params &p, uint32_t bring, uint32_t eit, uint32_t nst, bool leader,
                                             int g, int q, int lane, int j0, uint32_t bfull0, uint32_t mready0,
                                             uint32_t mdone0)
{
    using C = Cfg<V_I8>;
    static_assert(C::KB * C::NT == 2 && C::BL_BYTES == 0 && C::ESZ == 1 && C::BK == 128, "moments_pass thread map");
    constexpr int BS = C::B_STAGES;
    uint32_t s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    const int n = q % C::NT;
    const int row0 = (C::BK * C::KB / 16) * g + 4 * (q / C::NT);
    const uint32_t off0 = n * C::BH_BYTES + row0 * 128 + (lane & 3) * 4;
    for (uint32_t k = 0; k < nst; k++) {
        const uint32_t git = eit + k;
        const int s = (int)(git % BS);
        const uint32_t ph = (git / BS) & 1;
        // CTA-scope waits and a release.cta remote relay, as the MMA issuer's: the
        // cluster-scope forms compile to CCTL.IVALL / MEMBAR.ALL.GPU per stage,
        // which made this warp the pipeline's bottleneck (27 vs 19.5 ms at C4).
        // The TMA engine has written this CTA's half before it completes the tx
        // on the leader's barrier, and shared memory has no cache to go stale.
        if (leader) {
            mbar_wait(bfull0 + 8 * s, ph);  // both halves landed
            if (q == 0 && lane == 0) mbar_arrive_remote(mapa_shared(mready0 + 8 * s, 1));
        } else {
            mbar_wait(mready0 + 8 * s, ph);  // relayed by the leader
        }
        const uint32_t tile = bring + s * C::B_STAGE + off0;
        uint32_t x[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const uint32_t a = tile + r * 128 + ((((uint32_t)lane >> 2) ^ (uint32_t)((row0 + r) & 7)) << 4);
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x[r]) : "r"(a));
        }
        const uint32_t t0 = __byte_perm(x[0], x[1], 0x5140), t1 = __byte_perm(x[0], x[1], 0x7362);
        const uint32_t t2 = __byte_perm(x[2], x[3], 0x5140), t3 = __byte_perm(x[2], x[3], 0x7362);
        const uint32_t y[4] = {__byte_perm(t0, t2, 0x5410), __byte_perm(t0, t2, 0x7632),
                               __byte_perm(t1, t3, 0x5410), __byte_perm(t1, t3, 0x7632)};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            s1[e] = dp4<SIGNED>(y[e], 0x01010101u, s1[e]);
            s2[e] = dp4<SIGNED>(y[e], y[e], s2[e]);
        }
        __syncwarp();  // every lane's loads have returned (their values are consumed above)
        if (lane == 0) mbar_arrive(mdone0 + 8 * s);  // this warp is done with slot s
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const int j = j0 + n * BN + 4 * lane + e;
        if (j < p.M) {
            const int64_t a1 = SIGNED ? (int64_t)(int32_t)s1[e] : (int64_t)s1[e];
            atomicAdd((unsigned long long *)p.sum_w + j, (unsigned long long)a1);
            atomicAdd((unsigned long long *)p.sum_w2 + j, (unsigned long long)s2[e]);
        }
    }
}

template <int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
k_xterm(const __grid_constant__ CUtensorMap tmap_b0, const __grid_constant__ CUtensorMap tmap_b1,
        const __grid_constant__ CUtensorMap tmap_hw, const Params p)
{
    using C = Cfg<V>;
    constexpr bool F32 = C::F32;
    extern __shared__ __align__(1024) uint8_t smem[];  // keeps shared provenance (LDS/STS)
    const uint32_t sbase = smem_u32(smem);
    if (threadIdx.x == 0 && (sbase & 1023)) __trap();  // 128B-swizzle atoms need 1 KB alignment
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the pair's MMAs)
    const bool leader = rank == 0;

    constexpr int AS = C::A_STAGES, BS = C::B_STAGES;
    auto afull_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * s; };                  // leader's is used
    auto aempty_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * (MAX_RING + s); };    // both CTAs
    auto bfull_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * (2 * MAX_RING + s); }; // leader's is used
    auto bempty_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * (3 * MAX_RING + s); };// both CTAs
    auto txfull_bar = [&](int x) { return sbase + Lay<V>::BAR + 8 * (4 * MAX_RING + x); };
    auto txempty_bar = [&](int x) { return sbase + Lay<V>::BAR + 8 * (4 * MAX_RING + TX_STAGES + x); };
    constexpr int BAR_T = 4 * MAX_RING + 2 * TX_STAGES, BAR_S = BAR_T + 4;
    auto tfull_bar = [&](int a) { return sbase + Lay<V>::BAR + 8 * (BAR_T + a); };      // both (multicast)
    auto tempty_bar = [&](int a) { return sbase + Lay<V>::BAR + 8 * (BAR_T + 2 + a); }; // leader's
    auto sfull_bar = [&](int q) { return sbase + Lay<V>::BAR + 8 * (BAR_S + q); };        // both CTAs
    auto sempty_bar = [&](int q) { return sbase + Lay<V>::BAR + 8 * (BAR_S + SCHED_Q + q); };  // leader's
    constexpr int BAR_M = BAR_S + 2 * SCHED_Q;
    // fused moments: W slot s landed (peer: relayed by the leader's epilogue), and
    // this CTA's epilogue warps are done reading it (gates the W producer's refill)
    auto mready_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * (BAR_M + s); };             // peer's
    auto mdone_bar = [&](int s) { return sbase + Lay<V>::BAR + 8 * (BAR_M + MAX_RING + s); };   // both CTAs
    volatile int *sched = (volatile int *)(smem + Lay<V>::SCHED);
    uint32_t *tmem_slot = (uint32_t *)(smem + Lay<V>::SCHED + SCHED_Q * 4);
    auto to_leader = [&](uint32_t a) { return mapa_shared(a, 0); };

    // consumers: the t-th unit of this pair (-1 = done).  Called either by a
    // whole warp (one arrival per warp) or by a single thread (solo = true).
    auto next_unit = [&](uint32_t t, bool solo) {
        const int q = t % SCHED_Q;
        mbar_wait_cluster(sfull_bar(q), (t / SCHED_Q) & 1);
        const int u = sched[q];
        if (!solo) __syncwarp();
        if (solo || lane == 0) mbar_arrive_cluster(to_leader(sempty_bar(q)));
        return u;
    };

    // ---- setup: V table to smem, barriers, TMEM (pair allocation) ----
    {
        // pack the 64 KB byte table into nibbles: 16 bytes in -> 8 bytes out
        const uint4 *src = (const uint4 *)p.vtab;
        uint2 *dst = (uint2 *)(smem + SMEM_V);
        for (int i = threadIdx.x; i < V_BYTES / 8; i += THREADS) {
            const uint4 v = src[i];
            auto pack = [](uint32_t a, uint32_t b) {  // 8 bytes (values < 16) -> 8 nibbles
                const uint32_t e = __byte_perm(a, b, 0x6420), o = __byte_perm(a, b, 0x7531);
                return e | (o << 4);
            };
            dst[i] = make_uint2(pack(v.x, v.y), pack(v.z, v.w));
        }
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmap_b0);
        if (F32) tma_prefetch(&tmap_b1);
        for (int s = 0; s < AS; s++) {
            mbar_init(afull_bar(s), 2 * GEN_WARPS);  // both CTAs' generator warps
            mbar_init(aempty_bar(s), 1);             // multicast tcgen05.commit
        }
        for (int s = 0; s < BS; s++) {
            mbar_init(bfull_bar(s), 1);   // leader's W producer: arrive + tx of both CTAs' loads
            mbar_init(bempty_bar(s), 1);  // multicast tcgen05.commit
            mbar_init(mready_bar(s), 1);  // the leader's epilogue relay
            mbar_init(mdone_bar(s), EPI_WARPS);
        }
        for (int x = 0; x < TX_STAGES; x++) {
            mbar_init(txfull_bar(x), 1);            // ciphertext rows landed
            mbar_init(txempty_bar(x), GEN_WARPS);   // rows consumed by the generators
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), 2 * EPI_WARPS);  // both CTAs' epilogues
        }
        for (int q = 0; q < SCHED_Q; q++) {
            mbar_init(sfull_bar(q), 1);
            mbar_init(sempty_bar(q), RING_CONSUMERS);
        }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();  // peer barriers initialised before any remote arrive; both CTAs
                         // past their launch prologue before the pair TMEM allocation
    if (warp == 2) tmem_alloc_pair<TMEM_COLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (p.clk != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        p.clk[0] = globaltimer_ns();
        p.clk[1] = clock64();
    }

    if (warp == 0) {
        // ================= scheduler (leader) + W TMA producer (both) =================
        if (lane == 0) {
            const uint32_t peer_sched = mapa_shared(smem_u32((const void *)sched), 1);
            uint32_t it = 0;
            uint32_t mpend = 0, mph = 0;  // slots holding a moments stage not yet released, their mdone parities
            for (uint32_t t = 0;; t++) {
                int u;
                if (leader) {
                    u = atomicAdd(p.unit_counter, 1);
                    if (u >= p.units) u = -1;
                    const int q = t % SCHED_Q;
                    // acquire.cluster: pairs with the consumers' release.cluster arrivals
                    // (both CTAs' reads of slot q happen before it is overwritten)
                    mbar_wait_cluster(sempty_bar(q), ((t / SCHED_Q) & 1) ^ 1);
                    sched[q] = u;
                    st_cluster_u32(peer_sched + 4 * q, (uint32_t)u);
                    mbar_arrive(sfull_bar(q));                       // release: ids visible to waiters
                    mbar_arrive_cluster(mapa_shared(sfull_bar(q), 1));
                } else {
                    u = next_unit(t, true);
                }
                if (u < 0) break;
                int b, nt;
                int64_t t0, t1;
                unit_coords<V>(p, u, b, nt, t0, t1);
                const int x0 = nt * (C::NT * BN) + (int)rank * (BN / 2);  // this CTA's half of N tile 0
                const bool mom = !F32 && p.sum_w != nullptr;
                for (int64_t tb = t0; tb < t1; tb += C::BK, it++) {
                    const int s = it % BS;
                    mbar_wait(C::UNI ? aempty_bar(s) : bempty_bar(s), ((it / BS) & 1) ^ 1);
                    if ((mpend >> s) & 1u) {  // the epilogue's moment pass over the old contents
                        mbar_wait(mdone_bar(s), (mph >> s) & 1u);
                        mph ^= 1u << s;
                        mpend &= ~(1u << s);
                    }
                    if (mom) mpend |= 1u << s;
                    // the leader's arrival carries the tx bytes of BOTH CTAs' loads; the
                    // peer's loads only complete tx on it (they cannot land in an earlier
                    // phase: the peer waited for this slot's commit, which follows it)
                    const uint32_t lbar = to_leader(bfull_bar(s));
                    if (XT_EXP & 16) {
                        if (leader) mbar_arrive(bfull_bar(s));
                        continue;
                    }
                    if (leader) mbar_arrive_expect_tx(bfull_bar(s), 2 * C::B_STAGE);
                    uint32_t bdst = sbase + smem_b<V>() + s * C::B_STAGE;
                    const int32_t trow = (XT_EXP & 1) ? (int32_t)(tb & 8191) : (int32_t)tb;
#pragma unroll
                    for (int n = 0; n < C::NT; n++) {
#pragma unroll
                        for (int at = 0; at < C::ESZ; at++) {  // 128-byte MN atoms of this half
                            tma_load_2d_pair(bdst, &tmap_b0, x0 + n * BN + at * C::BOX_X, trow, lbar);
                            bdst += C::A_ATOM;
                            // the load latency (L2 miss -> HBM) exceeds the ring's
                            // slack: pull the box PREFETCH_STAGES ahead into L2
                            const int64_t tp = tb + PREFETCH_STAGES * C::BK;
                            if (PREFETCH_STAGES > 0 && tp < t1)
                                tma_prefetch_2d(&tmap_b0, x0 + n * BN + at * C::BOX_X, (int32_t)tp);
                        }
                        if constexpr (F32) {  // the e4m3 lo half: one 128-byte atom
                            tma_load_2d_pair(bdst, &tmap_b1, x0 + n * BN, trow, lbar);
                            bdst += C::BL_BYTES;
                        }
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ================= ciphertext producer (feeds this CTA's generators) =================
        if (lane == 0) {
            uint32_t it = 0;
            for (uint32_t t = 0;; t++) {
                const int u = next_unit(t, true);
                if (u < 0) break;
                int b, nt;
                int64_t t0, t1;
                unit_coords<V>(p, u, b, nt, t0, t1);
                for (int64_t tb = t0; tb < t1; tb += C::BK, it++) {
                    const int x = it % TX_STAGES;
                    mbar_wait(txempty_bar(x), ((it / TX_STAGES) & 1) ^ 1);
                    const int rows = (int)((t1 - tb) < C::BK ? (t1 - tb) : C::BK);
                    mbar_arrive_expect_tx(txfull_bar(x), rows * 16);
                    bulk_load(sbase + Lay<V>::TX + x * Lay<V>::TXB, p.texts + tb * 16, rows * 16, txfull_bar(x));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ================= MMA issuer (one thread of the leader) =================
            // Lean issue loop: descriptors are precomputed and advanced by adding
            // 16-byte units to their start-address field; the full barrier is waited
            // on at CTA scope (tools/pair_bench: 65% -> 100% of the pair MMA rate).
            const uint64_t adesc0 = smem_desc_sw128(sbase + SMEM_A, C::A_ATOM, 1024);
            const uint64_t bdesc0 = smem_desc_sw128(sbase + smem_b<V>(), C::A_ATOM, 1024);
            uint32_t sa = 0, pa = 0, sb = 0, pb = 0;
            for (uint32_t t = 0;; t++) {
                const int u = next_unit(t, true);
                if (u < 0) break;
                int b, nt;
                int64_t t0, t1;
                unit_coords<V>(p, u, b, nt, t0, t1);
                const uint32_t acc = t % C::NBUF;
                mbar_wait_cluster(tempty_bar(acc), ((t / C::NBUF) & 1) ^ 1);  // both epilogues drained it
                tc_fence_after();
                const uint32_t dbase = tmem_base + acc * (C::NACC * BN);
                uint32_t accum = 0;
                for (int64_t tb = t0; tb < t1; tb += C::BK) {
                    mbar_wait(bfull_bar(sb), pb);
                    mbar_wait(afull_bar(sa), pa);
                    tc_fence_after();
                    const uint64_t ad = adesc0 + (uint64_t)((sa * C::A_STAGE) >> 4);
                    const uint64_t bdd = bdesc0 + (uint64_t)((sb * C::B_STAGE) >> 4);
#pragma unroll
                    for (int kk = 0; kk < C::BK / C::KMMA; kk++) {
                        // K step = KMMA rows of 128 bytes in every MN atom
                        const uint64_t adk = ad + (uint64_t)((kk * C::KMMA * 128) >> 4);
                        const uint64_t bdk = bdd + (uint64_t)((kk * C::KMMA * 128) >> 4);
#pragma unroll
                        for (int n = 0; n < C::NT; n++)
#pragma unroll
                            for (int kb = 0; kb < C::KB; kb++) {
                                const uint64_t a = adk + (uint64_t)((kb * C::A_BYTES) >> 4);
                                const uint64_t bd = bdk + (uint64_t)((n * (C::BH_BYTES + C::BL_BYTES)) >> 4);
                                const uint32_t d = dbase + (kb * C::NT + n) * BN;
                                if (F32) {
                                    if (!(XT_EXP & 64)) mma_f16_pair(d, a, bd, p.idesc, accum);
                                }
                                else mma_i8_pair(d, a, bd, p.idesc, accum);
                            }
                        accum = 1;
                    }
                    if constexpr (F32) {
                        // lo: (H 2^-16, e5m2) . (lo, e4m3), K = 32 rows of 128 bytes per MMA,
                        // into the same accumulator as tile n's hi MMAs
                        static_assert(C::KB == 1, "F32 lo MMAs: one key byte per unit");
                        const uint64_t a8 = ad + (uint64_t)(C::A_BYTES >> 4);
#pragma unroll
                        for (int n = 0; n < C::NT; n++) {
                            const uint64_t b8 = bdd + (uint64_t)((n * (C::BH_BYTES + C::BL_BYTES) + C::BH_BYTES) >> 4);
#pragma unroll
                            for (int k8 = 0; k8 < ((XT_EXP & 32) ? 0 : C::BK / 32); k8++)
                                mma_f8_pair(dbase + n * BN, a8 + (uint64_t)((k8 * 32 * 128) >> 4),
                                            b8 + (uint64_t)((k8 * 32 * 128) >> 4), p.idesc8, 1u);
                        }
                    }
                    mma_commit_pair(aempty_bar(sa), 0x3);  // frees the slots in both CTAs when done
                    if constexpr (!C::UNI) mma_commit_pair(bempty_bar(sb), 0x3);
                    if (++sa == AS) {
                        sa = 0;
                        pa ^= 1;
                    }
                    if (++sb == BS) {
                        sb = 0;
                        pb ^= 1;
                    }
                }
                mma_commit_pair(tfull_bar(acc), 0x3);    // accumulators ready for both epilogues
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ================= epilogue: TMEM -> int64 / fp64 global (atomic add) =================
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        uint32_t *tbuf = (uint32_t *)(smem + Lay<V>::TB) + q * 32 * TB_LD;
        const int rsub = lane >> 3, csub = lane & 7;
        uint32_t eit = 0;     // W ring stage counter (same sequence as the producer's)
        for (uint32_t t = 0;; t++) {
            const int u = next_unit(t, false);
            if (u < 0) break;
            int b, nt;
            int64_t t0, t1;
            unit_coords<V>(p, u, b, nt, t0, t1);
            const uint32_t nst = (uint32_t)((t1 - t0 + C::BK - 1) / C::BK);
            if constexpr (V == V_I8) {
                if (p.sum_w != nullptr) {
                    const int j0 = nt * (C::NT * BN) + (int)rank * (BN / 2);  // this CTA's half of N tile 0
                    if (p.w_signed) moments_pass<true>(p, sbase + smem_b<V>(), eit, nst, leader, b / C::KB, q, lane,
                                                       j0, bfull_bar(0), mready_bar(0), mdone_bar(0));
                    else moments_pass<false>(p, sbase + smem_b<V>(), eit, nst, leader, b / C::KB, q, lane, j0,
                                             bfull_bar(0), mready_bar(0), mdone_bar(0));
                }
            }
            eit += nst;
            const uint32_t acc = t % C::NBUF;
            mbar_wait(tfull_bar(acc), (t / C::NBUF) & 1);  // multicast commit: CTA-scope wait
            tc_fence_after();
            constexpr int CPB = C::NT * BN / 8;  // 8-column groups per key byte
            constexpr int NC = C::NACC * BN / 8;
            const uint32_t tcol = tmem_base + ((uint32_t)(q * 32) << 16) + acc * (C::NACC * BN);
            int64_t *const own = F32 ? nullptr : p.owners[b];  // KB == 1 for the owner routing
            uint32_t v[8];
            tmem_ld_32x32b_x8(tcol, v);
            tmem_ld_wait(v);
            if (p.part != nullptr) {
                // lane = accumulator row: its 8 samples (32 bytes, one sector) per
                // column group straight to the unit's chunk slice; the TMEM load of
                // the next group is in flight during the stores
                static_assert(C::KB == 1, "partial spill: one key byte per unit");
                const int kc = (u / p.groups) % p.kc_count;
                uint32_t *prow = p.part + ((int64_t)kc * 4096 + b * 256 + (int)rank * BMC + q * 32 + lane) * p.part_ld;
#pragma unroll 1
                for (int c = 0; c < NC; c++) {
                    uint32_t vn[8];
                    if (c + 1 < NC) tmem_ld_32x32b_x8(tcol + (c + 1) * 8, vn);
                    const int j = nt * (C::NT * BN) + c * 8;
                    if (!(XT_EXP & 4) && j < p.part_ld) {
                        uint32_t *dst = prow + j;
                        asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(v[0]), "r"(v[1]),
                                     "r"(v[2]), "r"(v[3]) : "memory");
                        asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4), "r"(v[4]), "r"(v[5]),
                                     "r"(v[6]), "r"(v[7]) : "memory");
                    }
                    if (c + 1 < NC) {
                        tmem_ld_wait(vn);
#pragma unroll
                        for (int x = 0; x < 8; x++) v[x] = vn[x];
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(to_leader(tempty_bar(acc)));
                continue;
            }
            // first touch: the unit is the only writer of its cells (a whole tile)
            const bool store_u = p.store_hw && u < p.full_units;
            if (p.bulk_spill && own == nullptr && !store_u) {
                // lane = accumulator row: its 8 samples as int64 (I8) or as fp64 times
                // 2^16 / s_j (F32) into the warp's box (64 B per row, 16-byte chunks
                // XOR-swizzled by (row >> 1) & 3 -- the TMA 64B swizzle, conflict-free
                // STS.128), then ONE bulk tensor reduce-add of the 32 x 8 box into sum_hw
                // by the TMA unit (exact int64 adds / fp64 adds).  The box is rewritten
                // only after the previous reduce has read it.
                const uint32_t box = sbase + Lay<V>::TB + q * RB_BYTES;
                const uint32_t rowb = box + lane * 64;
                const uint32_t swz = ((uint32_t)lane >> 1) & 3;
#pragma unroll 1
                for (int c = 0; c < NC; c++) {
                    const int kb = c / CPB, cc = c % CPB;
                    const int hrow0 = (b + kb) * 256 + (int)rank * BMC + q * 32;
                    uint32_t vn[8];
                    if (c + 1 < NC) tmem_ld_32x32b_x8(tcol + (c + 1) * 8, vn);
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
                    const int j = nt * (C::NT * BN) + cc * 8;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        uint64_t a0, a1;
                        if constexpr (F32) {  // same values as the atomic path: fp32 acc x 2^16 / s_j in fp64
                            const int j0 = j + 2 * k < p.M ? j + 2 * k : p.M - 1;
                            const int j1 = j + 2 * k + 1 < p.M ? j + 2 * k + 1 : p.M - 1;
                            a0 = (uint64_t)__double_as_longlong((double)__uint_as_float(v[2 * k]) *
                                                                (double)p.inv_scale[j0]);
                            a1 = (uint64_t)__double_as_longlong((double)__uint_as_float(v[2 * k + 1]) *
                                                                (double)p.inv_scale[j1]);
                        } else {
                            a0 = (uint64_t)(int64_t)(int32_t)v[2 * k];
                            a1 = (uint64_t)(int64_t)(int32_t)v[2 * k + 1];
                        }
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowb + ((k ^ swz) << 4)),
                                     "r"((uint32_t)a0), "r"((uint32_t)(a0 >> 32)), "r"((uint32_t)a1),
                                     "r"((uint32_t)(a1 >> 32))
                                     : "memory");
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && !(XT_EXP & 4) && j < p.M) {
                        tma_reduce_add_2d(&tmap_hw, j, hrow0, box);
                        bulk_commit();
                    }
                    if (c + 1 < NC) {
                        tmem_ld_wait(vn);
#pragma unroll
                        for (int x = 0; x < 8; x++) v[x] = vn[x];
                    }
                }
                if (lane == 0) bulk_wait_read<0>();  // box free; the adds complete asynchronously
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(to_leader(tempty_bar(acc)));
                continue;
            }
            if (!F32 && own == nullptr && p.hw32 && store_u && XT_ST32_ROWS2) {
                // narrow first touch, two column groups at a time: 32 rows x 16 samples
                // staged in the warp's bulk box (word (r, c) at r*16 + (c ^ ((r >> 1) & 15)):
                // conflict-free both ways), then each warp-wide store covers 2 rows x 64 B
                static_assert(NC % 2 == 0 && CPB % 2 == 0, "column groups in pairs");
                uint32_t *sb = (uint32_t *)(smem + Lay<V>::TB + q * RB_BYTES);
                const int rl = lane >> 4, cl = lane & 15;
                uint32_t v2[8];
                tmem_ld_32x32b_x8(tcol + 8, v2);
                tmem_ld_wait(v2);
#pragma unroll 1
                for (int c = 0; c < NC; c += 2) {
                    const int cc = c % CPB;
                    const int hrow0 = (b + c / CPB) * 256 + (int)rank * BMC + q * 32;
                    uint32_t vn[8], vn2[8];
                    if (c + 2 < NC) {
                        tmem_ld_32x32b_x8(tcol + (c + 2) * 8, vn);
                        tmem_ld_32x32b_x8(tcol + (c + 3) * 8, vn2);
                    }
                    const int sw = (lane >> 1) & 15;
#pragma unroll
                    for (int x = 0; x < 8; x++) {
                        sb[lane * 16 + (x ^ sw)] = v[x];
                        sb[lane * 16 + ((x + 8) ^ sw)] = v2[x];
                    }
                    __syncwarp();
                    const int jc = nt * (C::NT * BN) + cc * 8 + cl;
                    if (!(XT_EXP & 4) && jc < p.M) {
#pragma unroll
                        for (int i = 0; i < 16; i++) {
                            const int row = 2 * i + rl;
                            ((uint32_t *)p.hw)[(int64_t)(hrow0 + row) * p.M + jc] = sb[row * 16 + (cl ^ i)];
                        }
                    }
                    __syncwarp();
                    if (c + 2 < NC) {
                        tmem_ld_wait(vn);
                        tmem_ld_wait(vn2);
#pragma unroll
                        for (int x = 0; x < 8; x++) {
                            v[x] = vn[x];
                            v2[x] = vn2[x];
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(to_leader(tempty_bar(acc)));
                continue;
            }
            // 8 columns at a time through a small transpose buffer: each warp-wide
            // atomic covers 4 rows x 8 consecutive samples = 8 full 32-byte sectors.
            // The TMEM load of the next 8 columns is in flight during the atomics.
#pragma unroll 1
            for (int c = 0; c < NC; c++) {
                const int kb = c / CPB, cc = c % CPB;
                const int hrow0 = (b + kb) * 256 + (int)rank * BMC + q * 32;
                uint32_t vn[8];
                if (c + 1 < NC) tmem_ld_32x32b_x8(tcol + (c + 1) * 8, vn);
#pragma unroll
                for (int x = 0; x < 8; x++) tbuf[lane * TB_LD + x] = v[x];
                __syncwarp();
                const int j = nt * (C::NT * BN) + cc * 8 + csub;  // accumulator column = sample
                if (!(XT_EXP & 4) && j < p.M) {
                    const int64_t off = (int64_t)(hrow0 + rsub) * p.M + j;
                    const double inv = F32 ? (double)p.inv_scale[j] : 1.0;
                    // one unswitched loop per output kind (the kind is uniform per unit)
                    auto put = [&](auto op) {
#pragma unroll
                        for (int rr = 0; rr < 8; rr++)
                            op(off + (int64_t)(4 * rr) * p.M, tbuf[(4 * rr + rsub) * TB_LD + csub]);
                    };
                    if (F32) {
                        put([&](int64_t o, uint32_t bits) {
                            atomicAdd((double *)p.hw + o, (double)__uint_as_float(bits) * inv);
                        });
                    } else if (own != nullptr) {  // peer (or own) accumulator of the row owner
                        put([&](int64_t o, uint32_t bits) {
                            atomicAdd_system((unsigned long long *)own + o, (unsigned long long)(long long)(int32_t)bits);
                        });
                    } else if (p.hw32) {          // narrow sums: 32-bit words
                        if (store_u) put([&](int64_t o, uint32_t bits) { ((uint32_t *)p.hw)[o] = bits; });
                        else put([&](int64_t o, uint32_t bits) { atomicAdd((unsigned int *)p.hw + o, bits); });
                    } else if (store_u) {         // first touch (store_hw): no read-modify-write
                        put([&](int64_t o, uint32_t bits) { ((long long *)p.hw)[o] = (long long)(int32_t)bits; });
                    } else {
                        put([&](int64_t o, uint32_t bits) {
                            atomicAdd((unsigned long long *)p.hw + o, (unsigned long long)(long long)(int32_t)bits);
                        });
                    }
                }
                __syncwarp();
                if (c + 1 < NC) {
                    tmem_ld_wait(vn);
#pragma unroll
                    for (int x = 0; x < 8; x++) v[x] = vn[x];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(to_leader(tempty_bar(acc)));
        }
    } else if (warp >= 8) {
        // ================= hypothesis generators (H tile, MN-major, swizzled) =================
        // A quarter-warp (8 lanes) builds one trace row of one key byte: lane =
        // 16-key chunk.  Warp g owns rows g*ROWS .. g*ROWS+ROWS-1 of every stage.
        // Keys 16c .. 16c+15 need V[c_s][(16c + j) ^ c_b], j = 0..15: the 16
        // nibbles of packed chunk c ^ (c_b >> 4) in the order j ^ (c_b & 15).
        // Per (row, key byte) this is reduced once (lanes 0..ROWS*KB-1) to a
        // descriptor {chunk address with the 8-nibble-half swap (c_b & 8) folded
        // in, PRMT selector for c_b & 7} and broadcast with a shuffle; one chunk
        // costs SHFL + LOP + 2 LDS.32 + 6 (nibble split) + 4 PRMT + STS.128.
        // Rows past the end of the data get (valid) stale-text hypotheses: their
        // W rows are TMA zero fill, so they add nothing.
        const int g = warp - 8;
        const int ql = lane & 7;           // chunk within the 128-key row
        const int sub = lane >> 3;         // row within a group of 4
        const uint8_t *vs = smem + SMEM_V;
        constexpr int ROWS = C::BK / GEN_WARPS;
        constexpr int PASSES = ROWS / 4;
        static_assert(ROWS * C::KB <= 32 && ROWS % 4 == 0, "descriptor lanes");
        uint32_t it = 0;
        for (uint32_t t = 0;; t++) {
            const int u = next_unit(t, false);
            if (u < 0) break;
            int b, nt;
            int64_t t0, t1;
            unit_coords<V>(p, u, b, nt, t0, t1);
            // this lane's descriptor slot: row ROWS*g + lane%ROWS, key byte b + lane/ROWS
            const int drow = ROWS * g + lane % ROWS, dkb = lane / ROWS;
            const int dsrc = shiftrows_src(b + dkb);
            for (int64_t tb = t0; tb < t1; tb += C::BK, it++) {
                const int s = it % AS;
                const uint32_t ph = (it / AS) & 1;
                const int x = it % TX_STAGES;
                mbar_wait(txfull_bar(x), (it / TX_STAGES) & 1);
                const uint8_t *tx = smem + Lay<V>::TX + x * Lay<V>::TXB;
                uint32_t desc = 0;
                if (lane < ROWS * C::KB) {
                    const uint32_t cb = tx[drow * 16 + b + dkb], cs = tx[drow * 16 + dsrc];
                    if (p.hist != nullptr && nt == 0 && leader && tb + drow < t1)  // each (trace, byte) once
                        atomicAdd(p.hist + (((uint32_t)(b + dkb) << 16) | (cb << 8) | cs), 1u);
                    const uint32_t hi = cb >> 4, lo = cb & 15;
                    // output byte jj of an even word takes nibble m = jj ^ (lo & 7) of its
                    // 8-nibble group: even m from the low-nibble word (PRMT 0-3), odd from
                    // the high-nibble word (PRMT 4-7), byte m >> 1
                    uint32_t sel_e = 0;
#pragma unroll
                    for (int jj = 0; jj < 4; jj++) {
                        const uint32_t m = (uint32_t)jj ^ (lo & 7);
                        sel_e |= (((m & 1) << 2) | (m >> 1)) << (4 * jj);
                    }
                    desc = (cs * 128 + (((rank * 8) ^ hi) << 3) + ((lo & 8) ? 4u : 0u)) | (sel_e << 16);
                }
                mbar_wait(aempty_bar(s), ph ^ 1);  // A slot free
#pragma unroll
                for (int kb = 0; kb < C::KB; kb++)  // the unit's key bytes b, b+1, ...
#pragma unroll
                for (int pass = 0; pass < ((XT_EXP & 2) ? 0 : PASSES); pass++) {
                    uint8_t *abase = smem + SMEM_A + s * C::A_STAGE + kb * C::A_BYTES;
                    const int rl = 4 * pass + sub;
                    const int row = ROWS * g + rl;
                    const uint32_t d = __shfl_sync(0xffffffffu, desc, kb * ROWS + rl);
#if XT_VLDS64
                    // one LDS.64 per chunk (a quarter-warp reads one 64-byte half row):
                    // fewer bank conflicts between the quarter-warps than 2 x LDS.32
                    const uint32_t a0 = (d & 0xfff8u) ^ ((uint32_t)ql << 3);
                    const uint2 w2 = *(const uint2 *)(vs + a0);
                    const bool sw = (d & 4u) != 0;
                    const uint32_t wa = sw ? w2.y : w2.x;  // nibbles j ^ lo, j < 8
                    const uint32_t wb = sw ? w2.x : w2.y;  // j >= 8
#else
                    const uint32_t a0 = (d & 0xffffu) ^ ((uint32_t)ql << 3);
                    const uint32_t wa = *(const uint32_t *)(vs + a0);         // nibbles j ^ lo, j < 8
                    const uint32_t wb = *(const uint32_t *)(vs + (a0 ^ 4u));  // j >= 8
#endif
                    const uint32_t la = wa & 0x0F0F0F0Fu, ha = (wa >> 4) & 0x0F0F0F0Fu;
                    const uint32_t lb = wb & 0x0F0F0F0Fu, hb = (wb >> 4) & 0x0F0F0F0Fu;
                    const uint32_t sel_e = d >> 16, sel_o = sel_e ^ 0x2222u;
                    uint4 outv;
                    outv.x = __byte_perm(la, ha, sel_e);
                    outv.y = __byte_perm(la, ha, sel_o);
                    outv.z = __byte_perm(lb, hb, sel_e);
                    outv.w = __byte_perm(lb, hb, sel_o);
                    if (!F32) {
                        *(uint4 *)(abase + row * 128 + ((ql ^ (row & 7)) << 4)) = outv;  // 128B swizzle
                    } else {
                        // 16 keys -> 32 bytes of fp16: keys 16ql.. live in MN atom ql/4,
                        // 16-byte chunks 2(ql%4) and 2(ql%4)+1 of the row (swizzled)
                        const uint4 lo4 = make_uint4(f16x2_h16_of_bytes(outv.x, 0x1404), f16x2_h16_of_bytes(outv.x, 0x3424),
                                                     f16x2_h16_of_bytes(outv.y, 0x1404), f16x2_h16_of_bytes(outv.y, 0x3424));
                        const uint4 hi4 = make_uint4(f16x2_h16_of_bytes(outv.z, 0x1404), f16x2_h16_of_bytes(outv.z, 0x3424),
                                                     f16x2_h16_of_bytes(outv.w, 0x1404), f16x2_h16_of_bytes(outv.w, 0x3424));
                        uint8_t *rowp = abase + (ql >> 2) * C::A_ATOM + row * 128;
                        const int c0i = 2 * (ql & 3);
                        *(uint4 *)(rowp + (((c0i) ^ (row & 7)) << 4)) = lo4;
                        *(uint4 *)(rowp + (((c0i + 1) ^ (row & 7)) << 4)) = hi4;
                        // and the e5m2 tile of H 2^-16: the same bytes as the I8 tile
                        *(uint4 *)(abase + C::A_BYTES + row * 128 + ((ql ^ (row & 7)) << 4)) = outv;
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(afull_bar(s));
                    else mbar_arrive_remote(to_leader(afull_bar(s)));
                    mbar_arrive(txempty_bar(x));
                }
            }
        }
    }

    if (warp >= 4 && warp < 8 && lane == 0) bulk_wait<0>();  // every bulk reduce-add has landed
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer's MMAs / remote arrivals are done with our smem and TMEM
    if (p.clk != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        p.clk[2] = globaltimer_ns();
        p.clk[3] = clock64();
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    }
}

// Tail split (one trace chunk per tile, more tiles than CTA pairs, not a whole
// number of waves): the last, partial wave of whole tiles leaves pairs idle (C5:
// 640 tiles on 74 pairs = 8.65 waves, run as 9).  Keep whole tiles for the full
// waves (rounded down to whole tile groups, so a W tile stays shared by its 16
// key bytes) and cut the remaining tiles into S pieces; S is chosen by simulating
// the in-order, earliest-free-pair schedule with each unit paying its epilogue
// (modelled as ~25k clk against 1024 clk per stage).
#ifndef XT_TAIL_SPLIT
#define XT_TAIL_SPLIT 1
#endif
void tail_split(Params &p, int pairs, int bk)
{
    const int T = p.units;
    if (pairs < 1 || T <= pairs || T % pairs == 0) return;
    // short units (W48: 63 stages, C2: 16) measured SLOWER split (W48 cross term
    // 1.155 vs 1.103 ms, C2 0.101 vs 0.081): their pieces lose the first-touch
    // stores and pay a whole epilogue for a few stages.  Long units only.
    if (p.store_hw || (p.N + bk - 1) / bk < 256) return;
    const int F = (T / pairs) * pairs / p.groups * p.groups;
    const int R = T - F;
    const int64_t stages = (p.N + bk - 1) / bk;
    const double epi = 25000.0 / (1024.0 * (double)stages);  // per unit, in whole-tile lengths
    auto makespan = [&](int S, int64_t len) {
        const int pieces = (int)((p.N + len - 1) / len);
        std::vector<double> busy((size_t)pairs, 0.0);
        auto take = [&](double w) {
            size_t k = 0;
            for (size_t i = 1; i < busy.size(); i++)
                if (busy[i] < busy[k]) k = i;
            busy[k] += w + epi;
        };
        for (int u = 0; u < F; u++) take(1.0);
        for (int q = 0; q < pieces; q++) {
            const double w = (double)std::min(len, p.N - (int64_t)q * len) / (double)p.N;
            for (int t = 0; t < R; t++) take(w);
        }
        (void)S;
        double m = 0.0;
        for (double x : busy) m = x > m ? x : m;
        return m;
    };
    double best = makespan(1, p.N);
    int best_s = 1;
    int64_t best_len = p.N;
    for (int S = 2; S <= 4; S++) {
        const int64_t len = (stages + S - 1) / S * bk;
        if (len >= p.N) break;
        const double m = makespan(S, len);
        if (m < best * 0.995) {
            best = m;
            best_s = S;
            best_len = len;
        }
    }
    if (best_s == 1) return;
    p.full_units = F;
    p.tail_len = best_len;
    p.units = F + R * (int)((p.N + best_len - 1) / best_len);
}

template <int V>
cudaError_t launch(const CUtensorMap &m0, const CUtensorMap &m1, const CUtensorMap *mhw, const uint8_t *d_texts,
                   const uint8_t *d_vtab,
                   void *d_hw, int *d_counter, int32_t M, int64_t N, int64_t kc_len, uint32_t idesc, int num_sms,
                   cudaStream_t stream, int *launches, int64_t *d_sum_w = nullptr, int64_t *d_sum_w2 = nullptr,
                   bool w_signed = true, uint32_t *d_hist = nullptr, int64_t *const *owners = nullptr,
                   unsigned long long *d_clk = nullptr, uint32_t idesc8 = 0, const float *d_inv_scale = nullptr,
                   bool store_hw = false, uint32_t *d_part = nullptr, int64_t part_ld = 0,
                   int32_t *d_hw32 = nullptr)
{
    using Cf = Cfg<V>;
    Params p;
    p.texts = d_texts;
    p.vtab = d_vtab;
    p.hw = d_hw;
    p.unit_counter = d_counter;
    p.M = M;
    p.N = N;
    p.n_tiles = (M + Cf::NT * BN - 1) / (Cf::NT * BN);
    p.groups = 16 / Cf::KB;
    p.kc_len = kc_len;
    p.kc_count = (int32_t)((N + kc_len - 1) / kc_len);
    p.units = p.groups * p.n_tiles * p.kc_count;
    p.idesc = idesc;
    p.idesc8 = idesc8;
    p.inv_scale = d_inv_scale;
    p.sum_w = d_sum_w;
    p.sum_w2 = d_sum_w2;
    p.w_signed = w_signed ? 1 : 0;
    p.hist = d_hist;
    for (int b = 0; b < 16; b++) p.owners[b] = owners ? owners[b] : nullptr;
    p.clk = d_clk;
    p.part = d_part;
    p.part_ld = part_ld;
    if (d_part != nullptr && (part_ld % 8 != 0 || part_ld < M || Cf::KB != 1 || owners != nullptr))
        return cudaErrorInvalidValue;
    p.hw32 = d_hw32 != nullptr;
    if (p.hw32) {
        if (Cf::F32 || mhw != nullptr || d_part != nullptr || owners != nullptr) return cudaErrorInvalidValue;
        p.hw = d_hw32;
    }
    p.bulk_spill = mhw != nullptr;
    p.store_hw = store_hw && p.kc_count == 1 && owners == nullptr && !Cf::F32;
    p.full_units = p.units;
    p.tail_len = 0;
    if (XT_TAIL_SPLIT && p.kc_count == 1 && d_part == nullptr) tail_split(p, num_sms / 2, Cf::BK);
    static std::atomic<unsigned long long> attr_set{0};
    cudaError_t e = smem_attr_once((const void *)k_xterm<V>, Lay<V>::ALLOC, attr_set);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(d_counter, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    const int pairs = (p.units < num_sms / 2 ? p.units : num_sms / 2);
    k_xterm<V><<<2 * pairs, THREADS, Lay<V>::ALLOC, stream>>>(m0, m1, mhw ? *mhw : m0, p);
    if (launches) (*launches)++;
    return cudaGetLastError();
}

// Split-K length: whole stages, chosen to balance the units over the CTA pairs
// while keeping each unit long enough that its epilogue is a small fraction
// (model: ~25k clk per epilogue, 1024 clk per stage; with a double-buffered
// accumulator (F32) the epilogue overlaps the next unit).  max_len bounds the
// int32 exactness (I8: |H W| <= 8 * 255 -> 2^20 traces) or the fp32 rounding
// (F32: 4096 traces).  epi_clk: the epilogue's cost; 3x when it adds the rows
// into a peer GPU's accumulator over NVLink (fused multi-GPU combine), which
// also favours fewer, longer units (less partial-sum traffic per rank).
int64_t auto_kchunk(int32_t M, int64_t N, int num_sms, int kb, int nt, int bk, int64_t max_len, bool overlapped,
                    double epi_clk = 25000.0)
{
    const int64_t tiles = (16LL / kb) * ((M + nt * BN - 1) / (nt * BN));
    const int64_t pairs = num_sms / 2;
    int64_t best_len = 0;
    double best = -1.0;
    for (int64_t kc = 1; kc <= 4096; kc++) {
        int64_t len = (N + kc - 1) / kc;
        len = (len + bk - 1) / bk * bk;
        if (len > max_len) continue;
        const int64_t kcount = (N + len - 1) / len;
        const int64_t units = tiles * kcount;
        const int64_t waves = (units + pairs - 1) / pairs;
        const double stage_clk = (double)((len + bk - 1) / bk) * 1024.0;
        const double epi = overlapped ? 0.0 : epi_clk;
        const double eff = (double)units / (double)(waves * pairs) * stage_clk / (stage_clk + epi);
        if (eff > best + 1e-3) {
            best = eff;
            best_len = len;
        }
        if (len <= bk) break;
    }
    if (best_len == 0) best_len = max_len;
    return best_len;
}

}  // namespace

int xterm_smem_bytes() { return Lay<V_I8>::ALLOC; }
int xterm_f32_bk(bool nt2) { return nt2 ? Cfg<V_F32N>::BK : Cfg<V_F32>::BK; }

int64_t xterm_i8_auto_kchunk(int32_t M, int64_t N, int num_sms, bool remote_epilogue)
{
    return auto_kchunk(M, N, num_sms, Cfg<V_I8>::KB, Cfg<V_I8>::NT, Cfg<V_I8>::BK, 1 << 20, false,
                       remote_epilogue ? 75000.0 : 25000.0);
}

int64_t xterm_f32_auto_kchunk(int32_t M, int64_t N, int num_sms, bool nt2)
{
    // fp32 TMEM accumulation, spilled to fp64 per unit: <= 4096 traces (NT = 1,
    // epilogue overlapped) or <= 24576 (NT = 2: the exposed epilogue amortised
    // over 4x the traces; with mean-centred samples the fp32 partial sums stay
    // small: max |drho| 2.4e-5 at full C3, tools/f32_unit_precision.py)
#ifndef F32_MAX_UNIT_NT2
#define F32_MAX_UNIT_NT2 24576
#endif
    if (nt2) return auto_kchunk(M, N, num_sms, 1, Cfg<V_F32N>::NT, Cfg<V_F32N>::BK, F32_MAX_UNIT_NT2, false);
    return auto_kchunk(M, N, num_sms, Cfg<V_F32>::KB, Cfg<V_F32>::NT, Cfg<V_F32>::BK, 4096, true);
}

XtermI8Plan xterm_i8_plan(int32_t M, int64_t N, int num_sms, bool remote_epilogue, int force)
{
    // NT = 1 with the overlapped spill measured SLOWER everywhere it was meant to
    // help (W48 cross term 1.75 vs 1.18 ms, C2 0.148 vs 0.110, C4 27.8 vs 18.3 ms:
    // generating an A tile per 4 MMAs instead of 8 starves the tensor pipe), so
    // the default is NT = 2; variant 2 stays an exact, tested option.
    XtermI8Plan pl;
    pl.overlapped = force == 2;
    pl.kc_len = pl.overlapped
                    ? auto_kchunk(M, N, num_sms, Cfg<V_I8O>::KB, Cfg<V_I8O>::NT, Cfg<V_I8O>::BK, 1 << 20, true)
                    : xterm_i8_auto_kchunk(M, N, num_sms, remote_epilogue);
    return pl;
}

cudaError_t launch_xterm_i8(const CUtensorMap &tmap_w, const CUtensorMap *tmap_hw, const uint8_t *d_texts,
                            const uint8_t *d_vtab, int64_t *d_hw, int *d_counter, int32_t M, int64_t N, int64_t kc_len,
                            bool w_signed, int num_sms, cudaStream_t stream, int *launches, int64_t *d_sum_w,
                            int64_t *d_sum_w2, uint32_t *d_hist, int64_t *const *owners, unsigned long long *d_clk,
                            bool overlapped, bool hw_zero, uint32_t *d_part, int64_t part_ld, int32_t *d_hw32)
{
    static_assert(Cfg<V_I8>::KB == 1 && Cfg<V_I8O>::KB == 1, "owner routing assumes one key byte per unit");
    if (overlapped) {
        if (d_sum_w != nullptr) return cudaErrorInvalidValue;  // a4 is fused into the NT = 2 variant only
        return launch<V_I8O>(tmap_w, tmap_w, tmap_hw, d_texts, d_vtab, d_hw, d_counter, M, N, kc_len,
                             idesc_i8(2 * BMC, BN, w_signed), num_sms, stream, launches, nullptr, nullptr, w_signed,
                             d_hist, owners, d_clk, 0, nullptr, hw_zero, d_part, part_ld, d_hw32);
    }
    return launch<V_I8>(tmap_w, tmap_w, tmap_hw, d_texts, d_vtab, d_hw, d_counter, M, N, kc_len,
                        idesc_i8(2 * BMC, BN, w_signed), num_sms, stream, launches, d_sum_w, d_sum_w2, w_signed,
                        d_hist, owners, d_clk, 0, nullptr, hw_zero, d_part, part_ld, d_hw32);
}

cudaError_t launch_xterm_f32(const CUtensorMap &tmap_hi, const CUtensorMap &tmap_lo, const CUtensorMap *tmap_hw,
                             const uint8_t *d_texts,
                             const uint8_t *d_vtab, double *d_hw, const float *d_inv_scale, int *d_counter, int32_t M,
                             int64_t N, int64_t kc_len, int num_sms, cudaStream_t stream, int *launches,
                             uint32_t *d_hist, unsigned long long *d_clk, bool nt2, uint32_t *d_part,
                             int64_t part_ld)
{
    if (nt2)
        return launch<V_F32N>(tmap_hi, tmap_lo, tmap_hw, d_texts, d_vtab, d_hw, d_counter, M, N, kc_len,
                              idesc_f16(2 * BMC, BN), num_sms, stream, launches, nullptr, nullptr, true, d_hist, nullptr,
                              d_clk, idesc_e5m2_e4m3(2 * BMC, BN), d_inv_scale, false, d_part, part_ld);
    return launch<V_F32>(tmap_hi, tmap_lo, tmap_hw, d_texts, d_vtab, d_hw, d_counter, M, N, kc_len,
                         idesc_f16(2 * BMC, BN),
                        num_sms, stream, launches, nullptr, nullptr, true, d_hist, nullptr, d_clk,
                        idesc_e5m2_e4m3(2 * BMC, BN), d_inv_scale, false, d_part, part_ld);
}

}  // namespace cpa
