// ring_litmus.cu -- litmus test for the two shared-memory hand-offs of k_xterm
// that compute-sanitizer racecheck reports as "potential WAR hazards"
// (profiles/sanitize_r02.txt), with the product's own PTX wrappers (ptx.cuh):
//
//  A. ciphertext ring (xterm.cu warp 3 -> generator warps): a single producer
//     thread refills slot x with cp.async.bulk (async proxy) after waiting on
//     txempty[x]; 8 consumer warps read the slot with generic loads, __syncwarp,
//     and lane 0 arrives on txempty[x] (mbarrier.arrive: release, CTA scope).
//  B. unit-id ring (xterm.cu scheduler -> next_unit): the pair leader writes id
//     t into its own slot q and the peer CTA's slot with st.shared::cluster,
//     arrives on both sfull[q]; every consumer warp of both CTAs waits on its
//     sfull[q] (acquire.cluster), reads the id, and arrives on the LEADER's
//     sempty[q] (release.cluster); the leader waits on sempty[q] before the
//     next write to slot q.
//
// Every value a consumer reads is checked against the one the protocol
// guarantees (A: the iteration number stamped in the source row; B: t).  A
// refill that overtook a read (the hazard racecheck reports) would be seen as a
// stale or future value.  Millions of hand-offs per run on every SM pair.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/ring_litmus tools/ring_litmus.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ptx_tools.cuh"

using namespace cpa;

constexpr int SLOTS = 4, ROW = 256, CONS_WARPS = 8, Q = 4;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (2 + CONS_WARPS), 1)
k_litmus(const uint32_t *src, int iters, unsigned long long *bad, unsigned long long *seen)
{
    __shared__ __align__(128) uint32_t ring[SLOTS][ROW / 4];
    __shared__ __align__(8) uint64_t full[SLOTS], empty[SLOTS], sfull[Q], sempty[Q];
    __shared__ volatile int sched[Q];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SLOTS; s++) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), CONS_WARPS);
        }
        for (int q = 0; q < Q; q++) {
            mbar_init(smem_u32(&sfull[q]), 1);
            mbar_init(smem_u32(&sempty[q]), 2 * CONS_WARPS);  // consumer warps of both CTAs
        }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();
    unsigned long long nbad = 0, nseen = 0;
    if (warp == 0 && lane == 0) {
        // A: producer (both CTAs, own ring)
        for (int it = 0; it < iters; it++) {
            const int s = it % SLOTS;
            mbar_wait(smem_u32(&empty[s]), ((it / SLOTS) & 1) ^ 1);
            mbar_arrive_expect_tx(smem_u32(&full[s]), ROW);
            bulk_load(smem_u32(&ring[s][0]), src + (size_t)(it % 1024) * (ROW / 4), ROW, smem_u32(&full[s]));
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // B: scheduler (leader)
        const uint32_t peer = mapa_shared(smem_u32((const void *)sched), 1);
        for (int t = 0; t < iters; t++) {
            const int q = t % Q;
            mbar_wait_cluster(smem_u32(&sempty[q]), ((t / Q) & 1) ^ 1);
            sched[q] = t;
            st_cluster_u32(peer + 4 * q, (uint32_t)t);
            mbar_arrive(smem_u32(&sfull[q]));
            mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[q]), 1));
        }
    } else if (warp >= 2) {
        for (int it = 0; it < iters; it++) {
            // B: consumer of the unit-id ring (whole warp, one arrival per warp)
            const int q = it % Q;
            mbar_wait_cluster(smem_u32(&sfull[q]), (it / Q) & 1);
            const int u = sched[q];
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&sempty[q]), 0));
            nbad += (u != it);
            // A: consumer of the bulk-copied ring
            const int s = it % SLOTS;
            mbar_wait(smem_u32(&full[s]), (it / SLOTS) & 1);
            const uint32_t v0 = ring[s][lane], v1 = ring[s][32 + lane];
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
            const uint32_t want = (uint32_t)(it % 1024);
            nbad += (v0 != want) + (v1 != want);
            nseen += 3;
        }
    }
    if (nbad) atomicAdd(bad, nbad);
    if (nseen) atomicAdd(seen, nseen);
    __syncthreads();
    cluster_sync_all();
}

int main(int argc, char **argv)
{
    const int iters = argc > 1 ? atoi(argv[1]) : 200000;
    uint32_t *src;
    cudaMalloc(&src, 1024 * ROW);
    uint32_t h[1024 * ROW / 4];
    for (int r = 0; r < 1024; r++)
        for (int k = 0; k < ROW / 4; k++) h[r * (ROW / 4) + k] = (uint32_t)r;  // row r stamped with r
    cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
    unsigned long long *d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    k_litmus<<<sms / 2 * 2, 32 * (2 + CONS_WARPS)>>>(src, iters, d, d + 1);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long r[2];
    cudaMemcpy(r, d, 16, cudaMemcpyDeviceToHost);
    printf("ring litmus: %d CTA pairs x %d iterations: %llu reads checked, %llu wrong (%s)\n", sms / 2, iters, r[1],
           r[0], cudaGetErrorString(e));
    return (e != cudaSuccess || r[0] != 0) ? 1 : 0;
}
