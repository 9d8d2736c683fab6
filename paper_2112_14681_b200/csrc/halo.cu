// halo.cu — halo exchange of boundary entries between row-block ranks over
// NVLink / NVSwitch peer memory (P:L733-741
// "the neighboring processes first exchange the elements of the solution
// vector on the boundary ... then each MPI rank independently applies the
// local relaxation").
//
// Transport: every rank owns a "mailbox" (one cudaMalloc) = per-source flags
// + two parity copies of its ghost array.  A sending rank's k_halo_put
// gathers the requested entries of its vector and STORES THEM DIRECTLY into
// the neighbour's mailbox (peer pointer: CUDA IPC across processes, plain
// device pointer for ranks sharing a process), then publishes a sequence
// number in the neighbour's flag slot (release at system scope).  The
// receiver's k_halo_wait spins (acquire, bounded by a timeout) until every
// neighbour's flag reached the exchange's sequence number; the kernels that
// read ghosts are ordered after it on the stream.  Interior rows — which
// read no ghost — are launched between put and wait, so the NVLink transfer
// overlaps their HBM-bound work.
//
// Reuse of a parity buffer is safe without an explicit acknowledgement:
// every exchange signals every neighbour in both directions, so when rank p
// starts exchange s it has already observed neighbour q's flag >= s-1, which
// q published after finishing (stream order) every kernel that read parity
// buffer (s-2) & 1 = s & 1.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "nsm_internal.h"
#include "ptx.cuh"

namespace nsm {

namespace {

constexpr int kPutThreads = 256;
constexpr int kPutItems = 4;  // entries per thread per block

using ptx::globaltimer_ns;
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) { ptx::st_release_sys_u64(p, v); }
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) { return ptx::ld_acquire_sys_u64(p); }

__global__ void __launch_bounds__(kPutThreads) k_halo_put(const PutDesc *__restrict__ desc, int npeers,
                                                          const double *__restrict__ src,
                                                          const double *__restrict__ scale, int parity,
                                                          unsigned long long seq, unsigned int *counters) {
    // find this block's peer (few peers: linear scan)
    int q = 0;
    while (q + 1 < npeers && (int)blockIdx.x >= desc[q + 1].block0) ++q;
    const PutDesc D = desc[q];
    const int64_t chunk = (int64_t)blockIdx.x - D.block0;
    const int64_t begin = chunk * (kPutThreads * kPutItems);
    double *dst = D.remote + (int64_t)parity * D.remote_stride;
#pragma unroll
    for (int it = 0; it < kPutItems; ++it) {
        const int64_t e = begin + (int64_t)it * kPutThreads + threadIdx.x;
        if (e < D.count) {
            const int32_t row = __ldg(D.rows + e);
            double v = __ldg(src + row);
            if (scale) v = __ddiv_rn(v, __ldg(scale + row));
            dst[e] = v;  // peer store over NVLink (or local store for a same-GPU rank)
        }
    }
    // last block of this peer publishes the sequence number
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(counters + q, 1u);
        if (done + 1 == (unsigned int)D.nblocks) {
            counters[q] = 0;
            __threadfence_system();
            st_release_sys(D.remote_flag, seq);
        }
    }
}

__global__ void k_halo_wait(const unsigned long long *flags, const int *__restrict__ peers, int npeers,
                            unsigned long long seq, unsigned long long timeout_ns, unsigned int *dist_err) {
    for (int l = threadIdx.x; l < npeers; l += 32) {
        const unsigned long long *f = flags + peers[l];
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_sys(f) < seq) {
            if (globaltimer_ns() - t0 > timeout_ns) {
                atomicOr(dist_err, 1u);  // surfaced by nsm_check as NSM_ERR_DIST
                break;
            }
            __nanosleep(64);
        }
    }
}

}  // namespace

int put_blocks(int64_t count) {
    const int64_t per = (int64_t)kPutThreads * kPutItems;
    return (int)std::max<int64_t>(1, (count + per - 1) / per);
}

cudaError_t launch_halo_put(const PutDesc *desc, int npeers, int total_blocks, const double *src,
                            const double *scale, int parity, unsigned long long seq, unsigned int *counters,
                            cudaStream_t st) {
    if (npeers <= 0) return cudaSuccess;
    k_halo_put<<<total_blocks, kPutThreads, 0, st>>>(desc, npeers, src, scale, parity, seq, counters);
    return cudaGetLastError();
}

cudaError_t launch_halo_wait(const unsigned long long *flags, const int *peers, int npeers, unsigned long long seq,
                             unsigned long long timeout_ns, unsigned int *dist_err, cudaStream_t st) {
    if (npeers <= 0) return cudaSuccess;
    k_halo_wait<<<1, 32, 0, st>>>(flags, peers, npeers, seq, timeout_ns, dist_err);
    return cudaGetLastError();
}

}  // namespace nsm

namespace nsm {
void preload_halo_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_halo_put);
    cudaFuncGetAttributes(&a, k_halo_wait);
}
}  // namespace nsm
