// comm.cu — the cross-rank reduction of the distributed solver layer
// (SURVEY.md §8(f) NEXT-1): Algorithm 1's single "Global synchronization"
// per iteration (step 6; one MPI_AllReduce per iteration,
// P:L299-307) and the restriction onto a replicated coarse level.
//
// A device-side all-reduce over NVLink / NVSwitch peer memory, no NCCL and no
// host round trip: every rank owns a mailbox (one cudaMalloc) = per-source
// flags + two parity copies of nranks slots of `cap` doubles.  k_ar_put
// STORES the rank's m input values into slot `rank` of every rank's mailbox
// (its own included; peer pointers from CUDA IPC across processes, plain
// device pointers for ranks sharing a process) and publishes the operation's
// sequence number in each destination's flag for this source (release, system
// scope).  k_ar_wait_sum waits (acquire, bounded by a timeout) for every
// source's flag and adds the slots in ASCENDING RANK ORDER, so every rank
// computes bit-identical sums — the ranks of a distributed GMRES take the same
// decisions (Givens rotations, stopping test) and run the same number of
// halo exchanges.
//
// Parity buffers need no acknowledgement (the argument of halo.cu): when rank
// p starts operation s it has observed every rank's flag >= s-1, published
// after that rank finished (stream order) the k_ar_wait_sum of s-2, the last
// reader of parity buffer s & 1.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "nsm_internal.h"
#include "ptx.cuh"

using namespace nsm;

namespace {

constexpr int kArThreads = 256;
constexpr int kArItems = 4;          // values per thread per put block
constexpr int64_t kFlagsBytes = 4096;  // flag area (<= 512 ranks), keeps the data 4 KB aligned

struct PeerBox {
    double *data;                    // that rank's data area
    unsigned long long *flags;       // that rank's flags (indexed by source rank)
};

__global__ void __launch_bounds__(kArThreads) k_ar_put(const PeerBox *__restrict__ peers, int rank, int nranks,
                                                       const double *__restrict__ in, int64_t m, int64_t cap,
                                                       int parity, unsigned long long seq,
                                                       unsigned int *__restrict__ counters) {
    const int q = blockIdx.y;  // destination rank
    const PeerBox P = peers[q];
    double *dst = P.data + ((int64_t)parity * nranks + rank) * cap;
    const int64_t begin = (int64_t)blockIdx.x * (kArThreads * kArItems);
#pragma unroll
    for (int it = 0; it < kArItems; ++it) {
        const int64_t j = begin + (int64_t)it * kArThreads + threadIdx.x;
        if (j < m) dst[j] = in[j];  // peer store over NVLink (local store for q == rank / same GPU)
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(counters + q, 1u);
        if (done + 1 == gridDim.x) {  // last block for destination q publishes
            counters[q] = 0;
            __threadfence_system();
            ptx::st_release_sys_u64(P.flags + rank, seq);
        }
    }
}

__global__ void __launch_bounds__(kArThreads) k_ar_wait_sum(const unsigned long long *flags, int nranks,
                                                            const double *data, int64_t m, int64_t cap, int parity,
                                                            unsigned long long seq, unsigned long long timeout_ns,
                                                            unsigned int *err, double *__restrict__ out) {
    __shared__ int failed;
    if (threadIdx.x == 0) failed = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < nranks; q += kArThreads) {
        const uint64_t t0 = ptx::globaltimer_ns();
        while (ptx::ld_acquire_sys_u64(flags + q) < seq) {
            if (ptx::globaltimer_ns() - t0 > timeout_ns) {
                atomicOr(err, 1u);  // surfaced as NSM_ERR_DIST by the host
                failed = 1;
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    __threadfence_system();
    if (failed) return;
    const double *base = data + (int64_t)parity * nranks * cap;
    for (int64_t j = (int64_t)blockIdx.x * kArThreads + threadIdx.x; j < m; j += (int64_t)gridDim.x * kArThreads) {
        double s = base[j];                                   // rank 0
        for (int q = 1; q < nranks; ++q) s = __dadd_rn(s, base[(int64_t)q * cap + j]);  // ascending ranks
        out[j] = s;
    }
}

}  // namespace

struct nsm_comm {
    int device = 0, rank = 0, nranks = 1;
    int64_t cap = 0;
    void *mailbox = nullptr;
    unsigned long long *flags = nullptr;
    double *data = nullptr;
    std::vector<PeerBox> peers;
    std::vector<void *> ipc_base;
    std::vector<bool> connected;
    PeerBox *d_peers = nullptr;
    unsigned int *counters = nullptr;
    unsigned int *err_host = nullptr, *err_dev = nullptr;  // mapped pinned error word
    unsigned long long seq = 0;
    unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
    bool committed = false;
    int64_t ops = 0;
    std::string err;
};

namespace {
thread_local std::string g_comm_err;

nsm_status comm_fail(nsm_comm *c, const std::string &msg, nsm_status st) {
    (c ? c->err : g_comm_err) = msg;
    return st;
}
}  // namespace

// internal (nsm_internal.h): used by nsm_gmres and the distributed V-cycle
nsm_status nsm::comm_allreduce(nsm_comm *c, const double *in, double *out, int64_t m, cudaStream_t s) {
    if (!c->committed) return comm_fail(c, "nsm_comm_allreduce before every rank is connected", NSM_ERR_STATE);
    if (m < 0 || m > c->cap) return comm_fail(c, "nsm_comm_allreduce: m exceeds the capacity", NSM_ERR_ARG);
    if (m == 0) return NSM_OK;
    const unsigned long long seq = ++c->seq;
    const int parity = (int)(seq & 1);
    const unsigned bx = (unsigned)((m + kArThreads * kArItems - 1) / (kArThreads * kArItems));
    k_ar_put<<<dim3(bx, (unsigned)c->nranks), kArThreads, 0, s>>>(c->d_peers, c->rank, c->nranks, in, m, c->cap,
                                                                    parity, seq, c->counters);
    const unsigned gs = (unsigned)std::min<int64_t>(148, (m + kArThreads - 1) / kArThreads);
    k_ar_wait_sum<<<gs, kArThreads, 0, s>>>(c->flags, c->nranks, c->data, m, c->cap, parity, seq, c->timeout_ns,
                                            c->err_dev, out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return comm_fail(c, cudaGetErrorString(e), NSM_ERR_CUDA);
    ++c->ops;
    return NSM_OK;
}

bool nsm::comm_failed(const nsm_comm *c) { return c && *(volatile unsigned int *)c->err_host != 0; }
int nsm::comm_rank(const nsm_comm *c) { return c->rank; }
int nsm::comm_nranks(const nsm_comm *c) { return c->nranks; }
int64_t nsm::comm_capacity(const nsm_comm *c) { return c->cap; }
int nsm::comm_device(const nsm_comm *c) { return c->device; }

extern "C" {

const char *nsm_comm_last_error(const nsm_comm *c) { return c ? c->err.c_str() : g_comm_err.c_str(); }

void nsm_comm_destroy(nsm_comm *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (void *p : c->ipc_base)
        if (p) cudaIpcCloseMemHandle(p);
    cudaFree(c->mailbox);
    cudaFree(c->d_peers);
    cudaFree(c->counters);
    if (c->err_host) cudaFreeHost(c->err_host);
    delete c;
}

nsm_status nsm_comm_create(nsm_comm **out, int rank, int nranks, int64_t capacity, int device) {
    if (!out || nranks < 1 || nranks > 512 || rank < 0 || rank >= nranks || capacity < 1)
        return comm_fail(nullptr, "nsm_comm_create: bad argument", NSM_ERR_ARG);
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return comm_fail(nullptr, "nsm_comm_create: cudaSetDevice failed", NSM_ERR_CUDA);
    nsm_comm *c = new nsm_comm();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    c->cap = (capacity + 31) / 32 * 32;  // 256-byte slots
    c->peers.assign(nranks, PeerBox{nullptr, nullptr});
    c->ipc_base.assign(nranks, nullptr);
    c->connected.assign(nranks, false);
    const size_t bytes = (size_t)kFlagsBytes + 2 * (size_t)nranks * (size_t)c->cap * sizeof(double);
    bool ok = cudaMalloc(&c->mailbox, bytes) == cudaSuccess &&
              cudaMemset(c->mailbox, 0, kFlagsBytes) == cudaSuccess &&
              cudaMalloc(&c->d_peers, nranks * sizeof(PeerBox)) == cudaSuccess &&
              cudaMalloc(&c->counters, nranks * sizeof(unsigned int)) == cudaSuccess &&
              cudaMemset(c->counters, 0, nranks * sizeof(unsigned int)) == cudaSuccess &&
              cudaHostAlloc((void **)&c->err_host, sizeof(unsigned int), cudaHostAllocMapped) == cudaSuccess;
    if (ok) {
        *c->err_host = 0;
        ok = cudaHostGetDevicePointer((void **)&c->err_dev, c->err_host, 0) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        nsm_comm_destroy(c);
        return comm_fail(nullptr, "nsm_comm_create: device allocation failed", NSM_ERR_OOM);
    }
    c->flags = (unsigned long long *)c->mailbox;
    c->data = (double *)((char *)c->mailbox + kFlagsBytes);
    c->peers[rank] = PeerBox{c->data, c->flags};
    c->connected[rank] = true;
    if (nranks == 1) {  // nothing to connect
        if (cudaMemcpy(c->d_peers, c->peers.data(), sizeof(PeerBox), cudaMemcpyHostToDevice) != cudaSuccess) {
            nsm_comm_destroy(c);
            return comm_fail(nullptr, "nsm_comm_create: upload of the peer table failed", NSM_ERR_CUDA);
        }
        c->committed = true;
    }
    // load the kernels now: a lazy module load while a peer's wait spins would stall
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k_ar_put);
    cudaFuncGetAttributes(&a, k_ar_wait_sum);
    preload_solver_kernels();  // nsm_gmres on a distributed operator
    *out = c;
    return NSM_OK;
}

nsm_status nsm_comm_mailbox(nsm_comm *c, void **base, void *ipc_handle) {
    if (!c) return NSM_ERR_ARG;
    if (base) *base = c->mailbox;
    if (ipc_handle) {
        DeviceScope dev(c->device);
        cudaIpcMemHandle_t ih;
        const cudaError_t e = cudaIpcGetMemHandle(&ih, c->mailbox);
        if (e != cudaSuccess) return comm_fail(c, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e), NSM_ERR_CUDA);
        std::memcpy(ipc_handle, &ih, sizeof(ih));
    }
    return NSM_OK;
}

static nsm_status comm_connect(nsm_comm *c, int q, void *peer_base, void *ipc_base) {
    if (!c || q < 0 || q >= c->nranks || q == c->rank || !peer_base) return NSM_ERR_ARG;
    if (c->committed) return comm_fail(c, "nsm_comm_connect after the last rank was connected", NSM_ERR_STATE);
    c->peers[q] = PeerBox{(double *)((char *)peer_base + kFlagsBytes), (unsigned long long *)peer_base};
    c->ipc_base[q] = ipc_base;
    c->connected[q] = true;
    if (std::all_of(c->connected.begin(), c->connected.end(), [](bool v) { return v; })) {
        DeviceScope dev(c->device);
        if (cudaMemcpy(c->d_peers, c->peers.data(), c->nranks * sizeof(PeerBox), cudaMemcpyHostToDevice) != cudaSuccess)
            return comm_fail(c, "nsm_comm_connect: upload of the peer table failed", NSM_ERR_CUDA);
        c->committed = true;
    }
    return NSM_OK;
}

nsm_status nsm_comm_connect(nsm_comm *c, int q, void *peer_base) { return comm_connect(c, q, peer_base, nullptr); }

nsm_status nsm_comm_connect_ipc(nsm_comm *c, int q, const void *ipc_handle) {
    if (!c || !ipc_handle || q < 0 || q >= c->nranks || q == c->rank) return NSM_ERR_ARG;
    DeviceScope dev(c->device);
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, ipc_handle, sizeof(ih));
    void *ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return comm_fail(c, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e), NSM_ERR_CUDA);
    return comm_connect(c, q, ptr, ptr);
}

nsm_status nsm_comm_allreduce(nsm_comm *c, const double *in, double *out, int64_t m, void *stream) {
    if (!c || (m > 0 && (!in || !out))) return NSM_ERR_ARG;
    DeviceScope dev(c->device);
    return comm_allreduce(c, in, out, m, (cudaStream_t)stream);
}

nsm_status nsm_comm_check(nsm_comm *c, void *stream) {
    if (!c) return NSM_ERR_ARG;
    DeviceScope dev(c->device);
    const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return comm_fail(c, cudaGetErrorString(e), NSM_ERR_CUDA);
    if (*(volatile unsigned int *)c->err_host) {
        *(volatile unsigned int *)c->err_host = 0;
        return comm_fail(c, "all-reduce timed out waiting for a rank", NSM_ERR_DIST);
    }
    return NSM_OK;
}

nsm_status nsm_comm_set_timeout(nsm_comm *c, int64_t ms) {
    if (!c || ms <= 0) return NSM_ERR_ARG;
    c->timeout_ns = (unsigned long long)ms * 1000000ull;
    return NSM_OK;
}

nsm_status nsm_comm_stats(const nsm_comm *c, int64_t *allreduces) {
    if (!c || !allreduces) return NSM_ERR_ARG;
    *allreduces = c->ops;
    return NSM_OK;
}

}  // extern "C"
