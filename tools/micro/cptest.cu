// cptest.cu -- check of the tcgen05.cp.32x128b.warpx4 source layout: a
// row-major [8 x 128] fp32 tile in shared memory (512-byte rows) is copied row
// by row into TMEM columns 4c..4c+3 of all four lane quarters; lane 32q+t must
// then hold tile[c][4t..4t+3].  Tries the (LBO, SBO) choices and prints which
// reproduce the tile.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(const void *p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;
}

__global__ void cp_kernel(int lbo, int sbo, int *bad) {
    __shared__ __align__(1024) float tile[8 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) tile[i] = (float)i;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int c = 0; c < 8; ++c) {
            const uint64_t d = desc(tile + c * 128, lbo, sbo);
            asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + 4 * c), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int c = 0; c < 8; ++c) {
        uint32_t r0, r1, r2, r3;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
            : "r"(tq + 4 * c)
            : "memory");
        const float e = (float)(c * 128 + 4 * lane);
        if (__uint_as_float(r0) != e || __uint_as_float(r1) != e + 1 || __uint_as_float(r2) != e + 2 ||
            __uint_as_float(r3) != e + 3)
            atomicAdd(bad, 1);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase) : "memory");
}

int main() {
    int *bad;
    cudaMalloc(&bad, sizeof(int));
    const int opts[4][2] = {{0, 128}, {128, 0}, {128, 128}, {16, 128}};
    for (auto &o : opts) {
        cudaMemset(bad, 0, sizeof(int));
        cp_kernel<<<1, 128>>>(o[0], o[1], bad);
        cudaError_t e = cudaDeviceSynchronize();
        int h = -1;
        cudaMemcpy(&h, bad, sizeof(int), cudaMemcpyDeviceToHost);
        printf("LBO=%3d SBO=%3d: %s, mismatching (thread, row) pairs %d / 1024\n", o[0], o[1], cudaGetErrorString(e), h);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
