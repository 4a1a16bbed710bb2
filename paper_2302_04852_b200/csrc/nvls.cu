// nvls.cu -- the data-parallel dW all_reduce through NVLink SHARP (NVLS)
// multicast (include/sparseprop.h "NVLS dW all_reduce").
//
// The DP step's only exchange is SUM over ranks of the nnz-length dW buffers
// (the paper runs one CPU, P367).  comm.cu does it with P2P
// loads of every peer's copy; here every rank's dW buffer is physical memory
// bound to ONE multicast object spanning the ranks' GPUs, so the NVSwitch does
// the reduction: rank r reads each 16-byte vector of its chunk ONCE through
// the multicast address (multimem.ld_reduce.add: the switch returns the sum of
// all ranks' copies) and writes the sum back ONCE (multimem.st: the switch
// stores it into every rank's copy).  Per element each rank moves 2 x 16 bytes
// over NVLink per world ranks instead of 2 x world x 16.
// Synchronisation: per CTA and phase, a flag word in the multicast-bound
// memory, raised on every rank at once by multimem.red.release.add (each rank
// adds 1 to all copies) and polled on the local copy with ld.acquire until it
// reaches world x epoch ("every rank's dW is complete" before the loads, "every
// rank's stores are done" after); the epoch is a per-CTA call counter in
// device memory, so there is no reset and a captured graph replays correctly.
// Every rank ends with the same values (one multicast store); the order of the
// switch's additions is the hardware's (not the fixed rank order of comm.cu).
//
// Setup is collective and follows the driver's multicast protocol: rank 0
// creates the multicast object for `world` devices and exports it as a POSIX
// file descriptor; the other ranks import it (the caller carries the fd
// between processes, e.g. SCM_RIGHTS over a Unix socket); every rank adds its
// device; after a barrier every rank binds its own physical memory and maps
// the multicast range; after a second barrier the buffers are usable.  Driver
// calls go through cudaGetDriverEntryPoint (the library links only cudart).
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <new>
#include <string>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kNvlsCtas = 8;  // CTAs per call (as comm.cu: SMs to leave free while it overlaps compute)
constexpr int kNvlsThreads = 512;
constexpr uint32_t kNvlsMagic = 0x53504e56U;  // "SPNV"
constexpr size_t kSigBytes = 2 * kNvlsCtas * sizeof(uint32_t);

struct Drv {
    CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long);
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*mcGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
    CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*addrFree)(CUdeviceptr, size_t);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
    CUresult (*exportHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
    CUresult (*importHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
    CUresult (*devAttr)(int *, CUdevice_attribute, CUdevice);
    bool ok = false;
};

const Drv &drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        bool all = true;
        auto get = [&](const char *name, auto &fn) {
            void *p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess && p)
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
            else
                all = false;
        };
        get("cuMulticastCreate", d.mcCreate);
        get("cuMulticastAddDevice", d.mcAddDevice);
        get("cuMulticastBindMem", d.mcBindMem);
        get("cuMulticastUnbind", d.mcUnbind);
        get("cuMulticastGetGranularity", d.mcGranularity);
        get("cuMemCreate", d.memCreate);
        get("cuMemRelease", d.memRelease);
        get("cuMemAddressReserve", d.addrReserve);
        get("cuMemAddressFree", d.addrFree);
        get("cuMemMap", d.memMap);
        get("cuMemUnmap", d.memUnmap);
        get("cuMemSetAccess", d.setAccess);
        get("cuMemExportToShareableHandle", d.exportHandle);
        get("cuMemImportFromShareableHandle", d.importHandle);
        get("cuDeviceGetAttribute", d.devAttr);
        d.ok = all;
    });
    return d;
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// all ranks' CTA b meet at phase ph: one multicast add raises the flag on every
// rank; the local copy reaches world * epoch once every rank has added
__device__ __forceinline__ void nvls_barrier(uint32_t *mc_sig, const uint32_t *uc_sig, int world, int ph,
                                             uint32_t epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const int w = ph * kNvlsCtas + blockIdx.x;
        __threadfence_system();  // this CTA's (and, at ph 0, the earlier kernels') stores before the flag
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_sig + w), "r"(1u) : "memory");
        const uint32_t want = (uint32_t)world * epoch;
        while ((int32_t)(ld_acquire_sys_u32(uc_sig + w) - want) < 0) {
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kNvlsThreads) nvls_allreduce_kernel(float *mc, uint32_t *mc_sig,
                                                                      const uint32_t *uc_sig, int world, int rank,
                                                                      int64_t off, int64_t count, uint32_t *epochs) {
    __shared__ uint32_t ep;
    if (threadIdx.x == 0) {
        ep = epochs[blockIdx.x] + 1;  // this call's epoch (all ranks count calls alike)
        epochs[blockIdx.x] = ep;
    }
    __syncthreads();
    const uint32_t epoch = ep;
    nvls_barrier(mc_sig, uc_sig, world, 0, epoch);
    // the 16-byte aligned body of [off, off + count) in float4 units, cut into
    // `world` chunks; chunk `rank` into gridDim.x sub-ranges (as comm.cu)
    const int64_t v0 = std::min<int64_t>(off + count, (off + 3) & ~(int64_t)3);
    const int64_t n4 = (off + count - v0) / 4, c4 = (n4 + world - 1) / world;
    const int64_t lo4 = std::min<int64_t>(n4, (int64_t)rank * c4), hi4 = std::min<int64_t>(n4, lo4 + c4);
    const int64_t s4 = (hi4 - lo4 + gridDim.x - 1) / gridDim.x;
    const int64_t a4 = lo4 + std::min<int64_t>(hi4 - lo4, (int64_t)blockIdx.x * s4);
    const int64_t b4 = std::min<int64_t>(hi4, a4 + s4);
    for (int64_t i = a4 + threadIdx.x; i < b4; i += blockDim.x) {
        float *p = mc + v0 + 4 * i;
        float x, y, z, w;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
                     : "l"(p)
                     : "memory");
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y),
                     "f"(z), "f"(w)
                     : "memory");
    }
    // the unaligned head [off, v0) and tail: the last rank's last CTA, scalar
    if (rank == world - 1 && blockIdx.x == gridDim.x - 1) {
        const int64_t t0 = v0 + 4 * n4, nh = v0 - off, nt = off + count - t0;
        for (int64_t k = threadIdx.x; k < nh + nt; k += blockDim.x) {
            float *p = mc + (k < nh ? off + k : t0 + (k - nh));
            float x;
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(x) : "l"(p) : "memory");
            asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(x) : "memory");
        }
    }
    nvls_barrier(mc_sig, uc_sig, world, 1, epoch);
}

}  // namespace
}  // namespace sp

using namespace sp;

struct sp_nvls_s {
    uint32_t magic;
    int rank, world, device;
    int64_t count;
    size_t bytes;                    // mapped size (granularity multiple): data, then the flag words
    size_t sig_off;                  // byte offset of the flag words
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    bool have_mc = false, have_mem = false, added = false, bound = false;
    CUdeviceptr uc = 0, mcva = 0;    // local (unicast) and multicast mappings
    bool uc_mapped = false, mc_mapped = false;
    uint32_t *epochs = nullptr;      // [kNvlsCtas] per-CTA call counters
};

namespace {
sp_status nfail(sp_status s, const std::string &m) {
    set_error(m);
    return s;
}
bool ok_nvls(sp_nvls_t c) { return c != nullptr && c->magic == kNvlsMagic; }
}  // namespace

extern "C" {

int32_t sp_nvls_supported(void) {
    const Drv &d = drv();
    int dev = 0, v = 0;
    if (!d.ok || cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (d.devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)dev) != CUDA_SUCCESS) return 0;
    return v != 0;
}

sp_status sp_nvls_create(int32_t rank, int32_t world, int64_t count, sp_nvls_t *out, int32_t *fd_out) {
    if (!out || !fd_out) return nfail(SP_ERR_NULL, "sp_nvls_create: NULL argument");
    *out = nullptr;
    *fd_out = -1;
    if (world < 1 || world > SP_COMM_MAX_WORLD || rank < 0 || rank >= world || count < 1)
        return nfail(SP_ERR_SHAPE, "sp_nvls_create: need 1 <= world <= 8, 0 <= rank < world, count >= 1");
    const Drv &d = drv();
    if (!d.ok || !sp_nvls_supported()) return nfail(SP_ERR_CUDA, "sp_nvls_create: no multicast support on this device");
    sp_nvls_t c = new (std::nothrow) sp_nvls_s{};
    if (!c) return nfail(SP_ERR_ALLOC, "sp_nvls_create: host allocation failed");
    c->magic = kNvlsMagic;
    c->rank = rank;
    c->world = world;
    c->count = count;
    cudaGetDevice(&c->device);
    cudaFree(nullptr);  // (a current context for the driver calls)
    c->sig_off = ((size_t)count * sizeof(float) + 255) & ~(size_t)255;
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)world;
    mp.handleTypes = world > 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
    mp.size = c->sig_off + kSigBytes;
    size_t gran = 0;
    if (d.mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) {
        sp_nvls_destroy(c);
        return nfail(SP_ERR_CUDA, "sp_nvls_create: cuMulticastGetGranularity failed");
    }
    c->bytes = (mp.size + gran - 1) / gran * gran;
    mp.size = c->bytes;
    if (rank == 0) {
        const CUresult r = d.mcCreate(&c->mc, &mp);
        if (r != CUDA_SUCCESS) {
            sp_nvls_destroy(c);
            return nfail(SP_ERR_CUDA, "sp_nvls_create: cuMulticastCreate failed (CUresult " + std::to_string((int)r) + ")");
        }
        c->have_mc = true;
        if (world > 1) {
            int fd = -1;
            if (d.exportHandle(&fd, c->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) {
                sp_nvls_destroy(c);
                return nfail(SP_ERR_CUDA, "sp_nvls_create: exporting the multicast handle failed");
            }
            *fd_out = fd;
        }
    }
    // this rank's physical memory (bound to the multicast object by sp_nvls_bind)
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c->device;
    if (d.memCreate(&c->mem, c->bytes, &ap, 0) != CUDA_SUCCESS) {
        sp_nvls_destroy(c);
        return nfail(SP_ERR_ALLOC, "sp_nvls_create: cuMemCreate failed");
    }
    c->have_mem = true;
    if (cudaMalloc((void **)&c->epochs, kNvlsCtas * sizeof(uint32_t)) != cudaSuccess) {
        c->epochs = nullptr;
        sp_nvls_destroy(c);
        return nfail(SP_ERR_ALLOC, "sp_nvls_create: device allocation failed");
    }
    cudaMemset(c->epochs, 0, kNvlsCtas * sizeof(uint32_t));
    *out = c;
    return SP_OK;
}

sp_status sp_nvls_open(sp_nvls_t c, int32_t fd) {
    if (!ok_nvls(c)) return nfail(SP_ERR_BAD_HANDLE, "sp_nvls_open: bad communicator");
    const Drv &d = drv();
    if (!c->have_mc) {
        if (fd < 0) return nfail(SP_ERR_SHAPE, "sp_nvls_open: ranks > 0 need rank 0's multicast fd");
        if (d.importHandle(&c->mc, (void *)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
            return nfail(SP_ERR_CUDA, "sp_nvls_open: importing the multicast handle failed");
        c->have_mc = true;
    }
    if (d.mcAddDevice(c->mc, (CUdevice)c->device) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_open: cuMulticastAddDevice failed");
    c->added = true;
    return SP_OK;
}

sp_status sp_nvls_bind(sp_nvls_t c) {
    if (!ok_nvls(c) || !c->added) return nfail(SP_ERR_BAD_HANDLE, "sp_nvls_bind: communicator not opened");
    const Drv &d = drv();
    if (d.mcBindMem(c->mc, 0, c->mem, 0, c->bytes, 0) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: cuMulticastBindMem failed");
    c->bound = true;
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = c->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.addrReserve(&c->uc, c->bytes, 0, 0, 0) != CUDA_SUCCESS ||
        d.memMap(c->uc, c->bytes, 0, c->mem, 0) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: mapping the local buffer failed");
    c->uc_mapped = true;
    if (d.setAccess(c->uc, c->bytes, &acc, 1) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: cuMemSetAccess (local) failed");
    if (d.addrReserve(&c->mcva, c->bytes, 0, 0, 0) != CUDA_SUCCESS ||
        d.memMap(c->mcva, c->bytes, 0, c->mc, 0) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: mapping the multicast range failed");
    c->mc_mapped = true;
    if (d.setAccess(c->mcva, c->bytes, &acc, 1) != CUDA_SUCCESS)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: cuMemSetAccess (multicast) failed");
    if (cudaMemset((void *)c->uc, 0, c->bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return nfail(SP_ERR_CUDA, "sp_nvls_bind: clearing the buffer failed");
    return SP_OK;
}

float *sp_nvls_buffer(sp_nvls_t c) { return (ok_nvls(c) && c->uc_mapped) ? (float *)c->uc : nullptr; }

sp_status sp_nvls_allreduce(sp_nvls_t c, int64_t offset, int64_t count, sp_stream_t stream) {
    if (!ok_nvls(c) || !c->mc_mapped) return nfail(SP_ERR_BAD_HANDLE, "sp_nvls_allreduce: communicator not bound");
    if (offset < 0 || count < 0 || offset + count > c->count)
        return nfail(SP_ERR_SHAPE, "sp_nvls_allreduce: range outside the buffer");
    if (count == 0) return SP_OK;
    count_launches(1);
    nvls_allreduce_kernel<<<kNvlsCtas, kNvlsThreads, 0, S(stream)>>>(
        (float *)c->mcva, (uint32_t *)(c->mcva + c->sig_off), (const uint32_t *)(c->uc + c->sig_off), c->world,
        c->rank, offset, count, c->epochs);
    return check_launch("sp_nvls_allreduce");
}

int32_t sp_nvls_ctas(void) { return kNvlsCtas; }

sp_status sp_nvls_destroy(sp_nvls_t c) {
    if (!ok_nvls(c)) return nfail(SP_ERR_BAD_HANDLE, "sp_nvls_destroy: bad communicator");
    const Drv &d = drv();
    cudaDeviceSynchronize();
    if (c->mc_mapped) d.memUnmap(c->mcva, c->bytes);
    if (c->mcva) d.addrFree(c->mcva, c->bytes);
    if (c->uc_mapped) d.memUnmap(c->uc, c->bytes);
    if (c->uc) d.addrFree(c->uc, c->bytes);
    if (c->bound) d.mcUnbind(c->mc, (CUdevice)c->device, 0, c->bytes);
    if (c->have_mem) d.memRelease(c->mem);
    if (c->have_mc) d.memRelease(c->mc);
    cudaFree(c->epochs);
    c->magic = 0;
    delete c;
    return SP_OK;
}

}  // extern "C"
