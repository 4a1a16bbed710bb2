// step.cu -- elementwise pieces of the data-parallel MLP step (north star
// cfg5): MSE gradient + deterministic loss, and SGD on
// the kept weights.
#include <cuda_runtime.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kMseBlocks = 296;  // 2 x 148 SMs; fixed so the tree is fixed
constexpr int kMseThreads = 256;

// dY = Y - T; per-block partial of 1/2 sum d^2 in fp64, fixed-order tree.
__global__ void __launch_bounds__(kMseThreads)
    mse_kernel(const float *__restrict__ Y, const float *__restrict__ T, float *__restrict__ dY,
               int64_t n, double *__restrict__ partial) {
    __shared__ double sh[kMseThreads];
    double s = 0.0;
    const bool v4 = ((n & 3) == 0) && ((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(T) |
                                        reinterpret_cast<uintptr_t>(dY)) & 15) == 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v4) {
        for (int64_t i = tid; i < n / 4; i += stride) {
            const float4 y = __ldg(reinterpret_cast<const float4 *>(Y) + i);
            const float4 t = __ldg(reinterpret_cast<const float4 *>(T) + i);
            const float4 d = make_float4(y.x - t.x, y.y - t.y, y.z - t.z, y.w - t.w);
            reinterpret_cast<float4 *>(dY)[i] = d;
            s += (double)d.x * d.x + (double)d.y * d.y + (double)d.z * d.z + (double)d.w * d.w;
        }
    } else {
        for (int64_t i = tid; i < n; i += stride) {
            const float d = Y[i] - T[i];
            dY[i] = d;
            s += (double)d * d;
        }
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = kMseThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void mse_final_kernel(const double *__restrict__ partial, int nb, float *__restrict__ loss) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nb; ++i) s += partial[i];
        *loss = (float)(0.5 * s);
    }
}

__global__ void sgd_kernel(float *__restrict__ vals, const float *__restrict__ dW, int64_t nnz,
                           float lr) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nnz) vals[j] = fmaf(-lr, dW[j], vals[j]);
}

}  // namespace

int64_t mse_scratch_floats(int64_t) { return 2 * kMseBlocks; }

void launch_mse(const float *Y, const float *T, float *dY, float *loss, float *scratch, int64_t n,
                cudaStream_t st) {
    double *partial = reinterpret_cast<double *>(scratch);
    count_launches(2);
    mse_kernel<<<kMseBlocks, kMseThreads, 0, st>>>(Y, T, dY, n, partial);
    mse_final_kernel<<<1, 32, 0, st>>>(partial, kMseBlocks, loss);
}

void launch_sgd(float *vals, const float *dW, int64_t nnz, float lr, cudaStream_t st) {
    if (nnz > 0) count_launches(1);
    if (nnz > 0) sgd_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(vals, dW, nnz, lr);
}

}  // namespace sp
