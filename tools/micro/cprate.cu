// cprate.cu -- throughput of tcgen05.cp (shared memory -> TMEM) shapes, issued
// by one thread (or one thread in each of NI warps), measured in SM cycles per
// instruction and bytes of TMEM written per cycle.  One CTA per SM, all SMs.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void *p) {
    return (uint64_t)((su32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)(256 >> 4) << 16) |
           ((uint64_t)1 << 46);
}

template <int SHAPE, int NI>  // 0: 32x128b.warpx4, 1: 128x256b, 2: 128x128b
__global__ void cp_kernel(int reps, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[NI];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = (float)i;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x < NI) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[threadIdx.x])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    long long t0 = clock64();
    if (lane == 0 && warp < NI) {
        unsigned ph = 0;
        for (int r = 0; r < reps; ++r) {
            // 64 instructions, each to its own column range, spread over the issuers
            for (int c = warp; c < 64; c += NI) {
                if (SHAPE == 0)
                    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + 4 * c),
                                 "l"(desc(sm + c * 512))
                                 : "memory");
                else if (SHAPE == 1)
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tbase + 8 * c),
                                 "l"(desc(sm + (c & 15) * 4096))
                                 : "memory");
                else
                    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tbase + 4 * c),
                                 "l"(desc(sm + (c & 31) * 2048))
                                 : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&bar[warp]))
                         : "memory");
            asm volatile(
                "{\n.reg .pred p;\nW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
                    su32(&bar[warp])),
                "r"(ph)
                : "memory");
            ph ^= 1;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

template <int SHAPE, int NI>
void run(const char *name, int tm_bytes_per_instr) {
    long long *cyc;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    auto k = cp_kernel<SHAPE, NI>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int reps = 200;
    k<<<148, 1024, 64 * 1024>>>(reps, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    const double per = m / (reps * 64.0);
    printf("%-28s %s: %6.1f cyc/instr, %7.1f B/cyc TMEM written per SM\n", name, cudaGetErrorString(e), per,
           tm_bytes_per_instr / per);
    cudaFree(cyc);
}

int main() {
    run<0, 1>("32x128b.warpx4, 1 issuer", 2048);
    run<0, 4>("32x128b.warpx4, 4 issuers", 2048);
    run<0, 8>("32x128b.warpx4, 8 issuers", 2048);
    run<0, 16>("32x128b.warpx4, 16 issuers", 2048);
    run<0, 32>("32x128b.warpx4, 32 issuers", 2048);
    run<1, 1>("128x256b, 1 issuer", 4096);
    run<1, 8>("128x256b, 8 issuers", 4096);
    run<1, 32>("128x256b, 32 issuers", 4096);
    run<2, 1>("128x128b, 1 issuer", 2048);
    run<2, 8>("128x128b, 8 issuers", 2048);
    run<2, 32>("128x128b, 32 issuers", 2048);
    return 0;
}
