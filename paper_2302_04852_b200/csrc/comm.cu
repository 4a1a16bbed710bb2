// comm.cu -- the data-parallel dW all_reduce over peer memory (SURVEY §8(f)
// F2; include/sparseprop.h "Data-parallel dW all_reduce over peer memory").
//
// The DP step's only exchange is SUM over ranks of the nnz-length dW buffers
// (the paper's single-CPU runs leave it out, P367).  On one
// NVSwitch node every GPU reaches every peer's memory at full NVLink
// bandwidth, so the sum is one kernel over peer pointers instead of a
// library collective:
//   two-shot, in place: the range is cut into `world` chunks, each chunk into
//   one sub-range per CTA; CTA b of rank r reads sub-range b of chunk r from
//   every rank (16-byte vectors, P2P loads over NVLink), adds them in rank
//   order 0..world-1 and stores the sum into every rank's copy -- so every
//   rank ends with bitwise the same values, and per element the order is
//   fixed (deterministic like the rest of the library).
// Synchronisation is per CTA: before reading, CTA b raises flag (b, r) in
// every peer's signal words ("my dW is complete") and waits for flags (b, q)
// of all q in its own; after storing, the same with a second flag array ("my
// stores into you are done, and I have finished reading you").  A CTA only
// touches sub-range b of each chunk, so waiting for the peers' CTA b covers
// everything it depends on.  Flags carry an epoch (a per-CTA counter in
// device memory incremented by every call), so there is no reset and a
// captured graph replays correctly.  Release / acquire at system scope order
// the data against the flags.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kCommCtas = 8;      // CTAs per call (SMs to reserve while it overlaps compute; NCCL's channel count)
constexpr int kCommThreads = 512;
constexpr uint32_t kCommMagic = 0x5350434dU;  // "SPCM"

struct CommPeers {
    float *data[SP_COMM_MAX_WORLD];
    uint32_t *sig[SP_COMM_MAX_WORLD];  // [2][kCommCtas][SP_COMM_MAX_WORLD] flag words per rank
};

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// flags of phase ph (0: inputs ready, 1: stores done) of CTA b, from rank q
__device__ __forceinline__ uint32_t *flag(uint32_t *sig, int ph, int b, int q) {
    return sig + ((size_t)ph * kCommCtas + b) * SP_COMM_MAX_WORLD + q;
}

// all CTAs b of all ranks meet at phase ph (thread t < world signals rank t
// and then waits for rank t's signal)
__device__ __forceinline__ void cta_barrier(const CommPeers &p, int world, int rank, int ph, uint32_t epoch) {
    __syncthreads();
    const int t = threadIdx.x;
    if (t < world) {
        __threadfence_system();  // this CTA's (and, at ph 0, the earlier kernels') stores before the flag
        st_release_sys(flag(p.sig[t], ph, blockIdx.x, rank), epoch);
        const uint32_t *mine = flag(p.sig[rank], ph, blockIdx.x, t);
        while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCommThreads) p2p_allreduce_kernel(CommPeers p, int world, int rank, int64_t off,
                                                                     int64_t count, uint32_t *epochs, int sync) {
    __shared__ uint32_t ep;
    if (threadIdx.x == 0) {
        ep = epochs[blockIdx.x] + 1;  // this call's epoch (all ranks count calls alike)
        epochs[blockIdx.x] = ep;
    }
    __syncthreads();
    const uint32_t epoch = ep;
    if (sync) cta_barrier(p, world, rank, 0, epoch);
    // the 16-byte aligned body [v0, v0 + 4 * n4) of [off, off + count) in float4
    // units, cut into `world` chunks; chunk `rank` into gridDim.x sub-ranges
    const int64_t v0 = std::min<int64_t>(off + count, (off + 3) & ~(int64_t)3);
    const int64_t n4 = (off + count - v0) / 4, c4 = (n4 + world - 1) / world;
    const int64_t lo4 = std::min<int64_t>(n4, (int64_t)rank * c4), hi4 = std::min<int64_t>(n4, lo4 + c4);
    const int64_t s4 = (hi4 - lo4 + gridDim.x - 1) / gridDim.x;
    const int64_t a4 = lo4 + std::min<int64_t>(hi4 - lo4, (int64_t)blockIdx.x * s4);
    const int64_t b4 = std::min<int64_t>(hi4, a4 + s4);
    for (int64_t i = a4 + threadIdx.x; i < b4; i += blockDim.x) {
        const int64_t e = v0 + 4 * i;
        // (L2-only loads: the values change between calls and come from peers)
        float4 v = __ldcg(reinterpret_cast<const float4 *>(p.data[0] + e));
        for (int q = 1; q < world; ++q) {
            const float4 u = __ldcg(reinterpret_cast<const float4 *>(p.data[q] + e));
            v.x += u.x;
            v.y += u.y;
            v.z += u.z;
            v.w += u.w;
        }
        for (int q = 0; q < world; ++q) *reinterpret_cast<float4 *>(p.data[q] + e) = v;
    }
    // the unaligned head [off, v0) and tail: the last rank's last CTA
    if (rank == world - 1 && blockIdx.x == gridDim.x - 1) {
        const int64_t t0 = v0 + 4 * n4, nh = v0 - off, nt = off + count - t0;
        for (int64_t k = threadIdx.x; k < nh + nt; k += blockDim.x) {
            const int64_t e = k < nh ? off + k : t0 + (k - nh);
            float v = __ldcg(p.data[0] + e);
            for (int q = 1; q < world; ++q) v += __ldcg(p.data[q] + e);
            for (int q = 0; q < world; ++q) p.data[q][e] = v;
        }
    }
    if (sync) cta_barrier(p, world, rank, 1, epoch);
}

}  // namespace
}  // namespace sp

using namespace sp;

struct sp_comm_s {
    uint32_t magic;
    int rank, world;
    int64_t count;
    bool local;               // single-process test communicator (world virtual ranks)
    float *data[SP_COMM_MAX_WORLD];    // device pointers (peers: IPC mappings)
    uint32_t *sig[SP_COMM_MAX_WORLD];
    bool opened[SP_COMM_MAX_WORLD];    // IPC mappings to close
    uint32_t *epochs;          // [kCommCtas] per-CTA call counters (this rank)
    uint32_t *epochs_local[SP_COMM_MAX_WORLD];  // test communicator: one set per virtual rank
};

namespace {
sp_status cfail(sp_status s, const std::string &m) {
    set_error(m);
    return s;
}
constexpr size_t kSigWords = (size_t)2 * kCommCtas * SP_COMM_MAX_WORLD;
bool ok_comm(sp_comm_t c) { return c != nullptr && c->magic == kCommMagic; }

sp_status alloc_rank(sp_comm_t c, int r) {
    if (cudaMalloc((void **)&c->data[r], (size_t)c->count * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void **)&c->sig[r], kSigWords * sizeof(uint32_t)) != cudaSuccess)
        return cfail(SP_ERR_ALLOC, "sp_comm: device allocation failed");
    cudaMemset(c->data[r], 0, (size_t)c->count * sizeof(float));
    cudaMemset(c->sig[r], 0, kSigWords * sizeof(uint32_t));
    return SP_OK;
}
}  // namespace

extern "C" {

int32_t sp_comm_ctas(void) { return kCommCtas; }

sp_status sp_comm_create(int32_t rank, int32_t world, int64_t count, sp_comm_t *out, void *handle_out) {
    if (!out || !handle_out) return cfail(SP_ERR_NULL, "sp_comm_create: NULL argument");
    *out = nullptr;
    if (world < 1 || world > SP_COMM_MAX_WORLD || rank < 0 || rank >= world || count < 1)
        return cfail(SP_ERR_SHAPE, "sp_comm_create: need 1 <= world <= 8, 0 <= rank < world, count >= 1");
    sp_comm_t c = new (std::nothrow) sp_comm_s{};
    if (!c) return cfail(SP_ERR_ALLOC, "sp_comm_create: host allocation failed");
    c->magic = kCommMagic;
    c->rank = rank;
    c->world = world;
    c->count = count;
    sp_status s = alloc_rank(c, rank);
    if (s == SP_OK && cudaMalloc((void **)&c->epochs, kCommCtas * sizeof(uint32_t)) != cudaSuccess)
        s = cfail(SP_ERR_ALLOC, "sp_comm_create: device allocation failed");
    if (s == SP_OK) cudaMemset(c->epochs, 0, kCommCtas * sizeof(uint32_t));
    cudaIpcMemHandle_t h[2];
    if (s == SP_OK && (cudaIpcGetMemHandle(&h[0], c->data[rank]) != cudaSuccess ||
                       cudaIpcGetMemHandle(&h[1], c->sig[rank]) != cudaSuccess))
        s = cfail(SP_ERR_CUDA, "sp_comm_create: cudaIpcGetMemHandle failed");
    if (s == SP_OK && cudaDeviceSynchronize() != cudaSuccess) s = cfail(SP_ERR_CUDA, "sp_comm_create: CUDA error");
    if (s != SP_OK) {
        cudaFree(c->data[rank]);
        cudaFree(c->sig[rank]);
        cudaFree(c->epochs);
        c->magic = 0;
        delete c;
        return s;
    }
    static_assert(2 * sizeof(cudaIpcMemHandle_t) <= SP_COMM_HANDLE_BYTES, "handle record size");
    std::memset(handle_out, 0, SP_COMM_HANDLE_BYTES);
    std::memcpy(handle_out, h, sizeof(h));
    *out = c;
    return SP_OK;
}

sp_status sp_comm_open(sp_comm_t c, const void *handles) {
    if (!ok_comm(c) || c->local) return cfail(SP_ERR_BAD_HANDLE, "sp_comm_open: bad communicator");
    if (!handles) return cfail(SP_ERR_NULL, "sp_comm_open: NULL handles");
    const char *rec = static_cast<const char *>(handles);
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank || c->opened[q]) continue;
        cudaIpcMemHandle_t h[2];
        std::memcpy(h, rec + (size_t)q * SP_COMM_HANDLE_BYTES, sizeof(h));
        void *d = nullptr, *g = nullptr;
        if (cudaIpcOpenMemHandle(&d, h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            return cfail(SP_ERR_CUDA, "sp_comm_open: cudaIpcOpenMemHandle (data) failed for rank " + std::to_string(q));
        if (cudaIpcOpenMemHandle(&g, h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaIpcCloseMemHandle(d);
            return cfail(SP_ERR_CUDA, "sp_comm_open: cudaIpcOpenMemHandle (signals) failed for rank " + std::to_string(q));
        }
        c->data[q] = static_cast<float *>(d);
        c->sig[q] = static_cast<uint32_t *>(g);
        c->opened[q] = true;
    }
    return SP_OK;
}

float *sp_comm_buffer(sp_comm_t c) { return ok_comm(c) ? c->data[c->rank] : nullptr; }

static sp_status launch_allreduce(sp_comm_t c, int rank, int64_t offset, int64_t count, bool sync, uint32_t *epochs,
                                  cudaStream_t st, const char *fn) {
    if (offset < 0 || count < 0 || offset + count > c->count)
        return cfail(SP_ERR_SHAPE, std::string(fn) + ": range outside the buffer");
    if (count == 0) return SP_OK;
    CommPeers p{};
    for (int q = 0; q < c->world; ++q) {
        if (!c->data[q] || !c->sig[q]) return cfail(SP_ERR_BAD_HANDLE, std::string(fn) + ": peers not opened");
        p.data[q] = c->data[q];
        p.sig[q] = c->sig[q];
    }
    count_launches(1);
    p2p_allreduce_kernel<<<kCommCtas, kCommThreads, 0, st>>>(p, c->world, rank, offset, count, epochs, sync ? 1 : 0);
    return check_launch(fn);
}

sp_status sp_comm_allreduce(sp_comm_t c, int64_t offset, int64_t count, sp_stream_t stream) {
    if (!ok_comm(c) || c->local) return cfail(SP_ERR_BAD_HANDLE, "sp_comm_allreduce: bad communicator");
    return launch_allreduce(c, c->rank, offset, count, c->world > 1, c->epochs, static_cast<cudaStream_t>(stream),
                            "sp_comm_allreduce");
}

sp_status sp_comm_destroy(sp_comm_t c) {
    if (!ok_comm(c)) return cfail(SP_ERR_BAD_HANDLE, "sp_comm_destroy: bad communicator");
    cudaDeviceSynchronize();
    for (int q = 0; q < c->world; ++q) {
        if (c->opened[q]) {
            cudaIpcCloseMemHandle(c->data[q]);
            cudaIpcCloseMemHandle(c->sig[q]);
        } else if (c->local || q == c->rank) {
            cudaFree(c->data[q]);
            cudaFree(c->sig[q]);
        }
        if (c->local) cudaFree(c->epochs_local[q]);
    }
    cudaFree(c->epochs);
    c->magic = 0;
    delete c;
    return SP_OK;
}

sp_status sp_comm_create_local(int32_t world, int64_t count, sp_comm_t *out) {
    if (!out) return cfail(SP_ERR_NULL, "sp_comm_create_local: NULL out");
    *out = nullptr;
    if (world < 1 || world > SP_COMM_MAX_WORLD || count < 1)
        return cfail(SP_ERR_SHAPE, "sp_comm_create_local: need 1 <= world <= 8, count >= 1");
    sp_comm_t c = new (std::nothrow) sp_comm_s{};
    if (!c) return cfail(SP_ERR_ALLOC, "sp_comm_create_local: host allocation failed");
    c->magic = kCommMagic;
    c->world = world;
    c->count = count;
    c->local = true;
    for (int r = 0; r < world; ++r) {
        sp_status s = alloc_rank(c, r);
        if (s == SP_OK && cudaMalloc((void **)&c->epochs_local[r], kCommCtas * sizeof(uint32_t)) != cudaSuccess)
            s = cfail(SP_ERR_ALLOC, "sp_comm_create_local: device allocation failed");
        if (s != SP_OK) {
            sp_comm_destroy(c);
            return s;
        }
        cudaMemset(c->epochs_local[r], 0, kCommCtas * sizeof(uint32_t));
    }
    cudaDeviceSynchronize();
    *out = c;
    return SP_OK;
}

float *sp_comm_local_buffer(sp_comm_t c, int32_t rank) {
    return (ok_comm(c) && c->local && rank >= 0 && rank < c->world) ? c->data[rank] : nullptr;
}

sp_status sp_comm_allreduce_as(sp_comm_t c, int32_t rank, int64_t offset, int64_t count, sp_stream_t stream) {
    if (!ok_comm(c) || !c->local) return cfail(SP_ERR_BAD_HANDLE, "sp_comm_allreduce_as: not a local communicator");
    if (rank < 0 || rank >= c->world) return cfail(SP_ERR_SHAPE, "sp_comm_allreduce_as: rank out of range");
    return launch_allreduce(c, rank, offset, count, false, c->epochs_local[rank], static_cast<cudaStream_t>(stream),
                            "sp_comm_allreduce_as");
}

}  // extern "C"
