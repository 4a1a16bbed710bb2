// tmgather.cu -- microbenchmark: the SpMM inner loop with the gathered
// activation row read from shared memory (LDS.128) vs from tensor memory
// (tcgen05.ld.32x32b.x4 at a warp-uniform column), entries (column, weight)
// broadcast from shared memory in both cases.  Resident data, no pipeline:
// it measures the loop ceiling of each gather source.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmgather tmgather.cu -lcuda
//   ./tmgather            (prints % of FP32 FMA peak at 1965 MHz per mode)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kEnt = 4096;  // entries in shared memory
constexpr int kRows = 64;   // tile rows (columns of W) for the LDS mode

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void fma4(float (&acc)[4], float w, const float (&x)[4]) {
    const float2 ww = make_float2(w, w);
    float2 r0 = __ffma2_rn(ww, make_float2(x[0], x[1]), make_float2(acc[0], acc[1]));
    float2 r1 = __ffma2_rn(ww, make_float2(x[2], x[3]), make_float2(acc[2], acc[3]));
    acc[0] = r0.x; acc[1] = r0.y; acc[2] = r1.x; acc[3] = r1.y;
}

template <int G>  // loads in flight per wait
__device__ __forceinline__ void tm_ldg(const uint32_t (&ta)[G], float (&x)[G][4]) {
    uint32_t r[G][4];
#pragma unroll
    for (int u = 0; u < G; ++u)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]) : "r"(ta[u]) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[u][v] = __uint_as_float(r[u][v]);
}

// MODE 0: LDS gather; 1: TMEM gather (G loads per wait); 2: half LDS, half TMEM
template <int MODE, int G, int NW, int RPW>
__global__ void __launch_bounds__(NW * 32, 1) loop_kernel(int niter, int seglen, float *out) {
    extern __shared__ __align__(128) float smem[];
    __shared__ uint32_t tbase;
    int2 *ent = reinterpret_cast<int2 *>(smem);
    float *tile = smem + 2 * kEnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kEnt; i += NW * 32) {
        uint32_t h = (uint32_t)i * 2654435761u;
        h ^= h >> 13;
        const int c = (int)(h % kRows);
        // LDS: byte offset of tile row c; TMEM: column 4c (2 and 3 modes use both)
        ent[i] = make_int2(c, __float_as_int(1.0f + (float)(h & 7) * 1e-3f));
    }
    for (int i = threadIdx.x; i < kRows * 128; i += NW * 32) tile[i] = (float)(i & 15) * 0.01f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    // fill: warps of quarter q write columns [128*(w/4) ...) of their lanes
    for (int col = (warp >> 2) * 4; col < 512; col += (NW / 4) * 4) {
        uint32_t v = __float_as_uint((float)(col + lane) * 1e-3f);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq + col), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    float acc[RPW][4] = {};
    const char *tb = reinterpret_cast<const char *>(tile + lane * 4);
    int e = (warp * 97) & (kEnt - 1) & ~7;
    for (int it = 0; it < niter; ++it) {
#pragma unroll
        for (int i = 0; i < RPW; ++i)
#pragma unroll 1
          for (int sgi = 0; sgi < seglen; ++sgi) {
            constexpr int NE = G >= 4 ? G : 4;  // entries per step
            int c[NE];
            float w[NE];
#pragma unroll
            for (int p = 0; p < NE; p += 2) {
                const int4 q = *reinterpret_cast<const int4 *>(ent + e + p);
                c[p] = q.x; w[p] = __int_as_float(q.y);
                c[p + 1] = q.z; w[p + 1] = __int_as_float(q.w);
            }
            e = (e + NE) & (kEnt - 1);
            float x[NE][4];
            if constexpr (MODE == 0) {
#pragma unroll
                for (int u = 0; u < NE; ++u) {
                    const float4 t = *reinterpret_cast<const float4 *>(tb + c[u] * 512);
                    x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
                }
            } else if constexpr (MODE == 1) {
#pragma unroll
                for (int u0 = 0; u0 < NE; u0 += G) {
                    uint32_t ta[G];
                    float xx[G][4];
#pragma unroll
                    for (int u = 0; u < G; ++u) ta[u] = tq + (uint32_t)(c[u0 + u] * 4);
                    tm_ldg<G>(ta, xx);
#pragma unroll
                    for (int u = 0; u < G; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) x[u0 + u][v] = xx[u][v];
                }
            } else {  // half and half
                constexpr int H = NE / 2;
                uint32_t ta[H];
                float xx[H][4];
#pragma unroll
                for (int u = 0; u < H; ++u) ta[u] = tq + (uint32_t)(c[u] * 4);
                tm_ldg<H>(ta, xx);
#pragma unroll
                for (int u = 0; u < H; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) x[u][v] = xx[u][v];
#pragma unroll
                for (int u = H; u < NE; ++u) {
                    const float4 t = *reinterpret_cast<const float4 *>(tb + c[u] * 512);
                    x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
                }
            }
#pragma unroll
            for (int u = 0; u < NE; ++u) fma4(acc[i], w[u], x[u]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < RPW; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    out[blockIdx.x * NW * 32 + threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

template <int MODE, int G, int NW, int RPW>
void run(const char *name, float *out, int seglen = 2) {
    const int niter = 1024;
    const size_t smem = 2 * kEnt * sizeof(float) + kRows * 128 * sizeof(float);
    auto k = loop_kernel<MODE, G, NW, RPW>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<148, NW * 32, smem>>>(niter, seglen, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k<<<148, NW * 32, smem>>>(niter, seglen, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    constexpr int NE = G >= 4 ? G : 4;
    const double fma = 148.0 * NW * 32 * (double)niter * seglen * RPW * NE * 4;
    const double peak = 148.0 * 128 * 1.965e9;  // FMA/s
    printf("%-34s %8.1f us  %5.1f %% of FP32 FMA peak\n", name, ms * 1e3, 100.0 * fma / (ms * 1e-3) / peak);
}

int main() {
    float *out;
    CK(cudaMalloc(&out, 148 * 1024 * sizeof(float)));
    run<0, 4, 32, 4>("LDS gather, 32w x 4 rows, 4/grp", out);
    run<0, 8, 16, 8>("LDS gather, 16w x 8 rows, 8/grp", out);
    run<1, 4, 32, 4>("TMEM x4, 32w, 4 per wait", out);
    run<1, 8, 32, 4>("TMEM x4, 32w, 8 per wait", out);
    run<1, 4, 16, 8>("TMEM x4, 16w, 4 per wait", out);
    run<1, 8, 16, 8>("TMEM x4, 16w, 8 per wait", out);
    run<1, 4, 16, 8>("TMEM x4, 16w, 4 per wait, 1 grp/row", out, 1);
    run<1, 4, 32, 4>("TMEM x4, 32w, 4 per wait, 1 grp/row", out, 1);
    run<0, 4, 32, 4>("LDS, 32w, 4/grp, 1 grp/row", out, 1);
    run<2, 8, 32, 4>("half TMEM/half LDS, 32w, 8/grp", out);
    run<2, 8, 16, 8>("half TMEM/half LDS, 16w, 8/grp", out);
    return 0;
}
