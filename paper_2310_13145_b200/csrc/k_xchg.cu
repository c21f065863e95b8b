// k_xchg.cu -- device-initiated exchange of the time cut (NEXT-4(c)): the
// sender's blocks store its send buffer straight into the receivers' buffers (peer memory: over
// NVLink / NVSwitch between GPUs, CUDA IPC mappings; plain device pointers inside a one-GPU loopback
// group), the last of them publishes the iteration's epoch in every receiver's flag with a
// system-scope release, and the receiver's blocks spin on their sources' flags with acquire loads
// before the unpack kernel runs.  No NCCL call and no host round trip on the exchange path.
//
//   phase 1: the DP stage costs [G][Tmax][4] to every rank (an all-gather: slot = sender)
//   phase 2: p, phat of the first owned period [G][2] to the previous rank
//   phase 3: the boundary values [G][12] to the next rank
//
// Epochs: inner_total + 1 of the iteration (the same on every rank), so flags never need resetting.
// Each rank sends before it waits, so ranks on different GPUs cannot deadlock.  On ONE GPU the
// ranks of a loopback group are emulated by ONE cooperative launch over all of them (its blocks are
// co-resident), never by separate launches that wait on one another.
#include <algorithm>

#include "ucac_dev.cuh"

namespace ucac {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// rank d.rank's share of one exchange, executed by `nb` blocks (this one is block `b`)
__device__ void xchg_rank(const Dev &d, int phase, int b, int nb) {
    if (d.st->done) return;
    const unsigned long long epoch = (unsigned long long)d.st->inner_total + 1;
    const int r = d.rank, n = d.nranks;
    const bool has_prev = d.own0 > 0, has_next = d.own1 < d.T;
    // ---- send: which buffer, how much, to whom
    const double *src = phase == 1 ? d.tc_stage_send : (phase == 2 ? d.tc2_send : d.tc3_send);
    const size_t cnt = phase == 1 ? (size_t)d.G * d.Tmax * 4 : (size_t)d.G * (phase == 2 ? 2 : 12);
    int q0 = 0, q1 = n;                                   // phase 1: every rank (itself included)
    if (phase == 2) { q0 = has_prev ? r - 1 : 0; q1 = has_prev ? r : 0; }
    if (phase == 3) { q0 = has_next ? r + 1 : 0; q1 = has_next ? r + 2 : 0; }
    for (int q = q0; q < q1; q++) {
        double *dst = (phase == 1 ? d.peer_stage_recv[q] : (phase == 2 ? d.peer_tc2_recv[q] : d.peer_tc3_recv[q])) +
                      (size_t)r * cnt;
        for (size_t k = (size_t)b * blockDim.x + threadIdx.x; k < cnt; k += (size_t)nb * blockDim.x) dst[k] = src[k];
    }
    // ---- the last block of this rank to finish sending publishes the epoch to the receivers
    __shared__ bool last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(d.xarrive + phase - 1, 1u) == (unsigned)nb - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence_system();
        d.xarrive[phase - 1] = 0;
        for (int q = q0; q < q1; q++) st_release_sys(d.peer_flags[q] + (phase - 1) * UCAC_MAX_P2P + r, epoch);
    }
    // ---- wait for this rank's sources (thread 0 of every block spins; the unpack launch follows)
    int s0 = 0, s1 = n;                                   // phase 1: every rank
    if (phase == 2) { s0 = has_next ? r + 1 : 0; s1 = has_next ? r + 2 : 0; }
    if (phase == 3) { s0 = has_prev ? r - 1 : 0; s1 = has_prev ? r : 0; }
    if (threadIdx.x == 0)
        for (int q = s0; q < s1; q++)
            while (ld_acquire_sys(d.xflags + (phase - 1) * UCAC_MAX_P2P + q) < epoch) __nanosleep(64);
    __syncthreads();
}

constexpr int XB = 128, XBLOCKS = 8;   // blocks per rank: the payloads are KBs to a few MB

__global__ void __launch_bounds__(XB) k_xchg(Dev d, int phase) { xchg_rank(d, phase, blockIdx.x, gridDim.x); }

// one-GPU emulation of a group: XBLOCKS blocks per rank in ONE cooperative launch
__global__ void __launch_bounds__(XB) k_xchg_group(const Dev *devs, int phase) {
    const int r = blockIdx.x / XBLOCKS;
    xchg_rank(devs[r], phase, blockIdx.x % XBLOCKS, XBLOCKS);
}

}  // namespace

void launch_xchg(const Dev &d, int phase, cudaStream_t s) { k_xchg<<<XBLOCKS, XB, 0, s>>>(d, phase); }

cudaError_t launch_xchg_group(const Dev *devs_host, int n, int phase, cudaStream_t s, Dev *scratch) {
    cudaError_t e = cudaMemcpyAsync(scratch, devs_host, sizeof(Dev) * n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    const Dev *arg = scratch;
    void *args[] = {(void *)&arg, (void *)&phase};
    return cudaLaunchCooperativeKernel((const void *)k_xchg_group, dim3(XBLOCKS * n), dim3(XB), args, 0, s);
}

}  // namespace ucac
