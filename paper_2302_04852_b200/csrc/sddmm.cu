// sddmm.cu -- weight-gradient SDDMM (K4, sp_linear_bwd_weight), SURVEY §8(a)
// row a-4:  dW[j] = sum_b dY[r_j][b] * X[c_j][b]  for every nonzero j (CSR
// order), Eq. (2) (P146-P148) restricted to the mask (P151, P173).
//
// Design: a CTA owns a block of RB = NW*RPW rows and a batch
// range split (blockIdx.x); it walks that range in slices of BT = 32*VEC.
// Per slice, each warp holds dY[r][slice] of its RPW rows in registers and
// streams X[:, slice] through shared memory in column blocks (coalesced
// 16-byte loads).  Per nonzero, each lane accumulates a VEC-long partial dot
// into one of 32 register accumulators; every 32 nonzeros a warp
// transpose-reduce (31 shuffles) leaves lane t with the slice sum of nonzero
// t, which lane t adds into the split's partial buffer (one owner per
// element, fixed order).  A final fixed-order pass sums the splits.  No
// atomics: bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

template <int VEC, int RPW, int NW>
__global__ void __launch_bounds__(NW * 32)
    sddmm_tiled_kernel(int64_t R, int64_t C, int64_t B, int KC, int64_t split_len,
                       const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                       const float *__restrict__ X, const float *__restrict__ dY,
                       float *__restrict__ part, int64_t nnz) {
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) float tile[];  // [KC][BT]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.y * (NW * RPW);
    const int64_t s_lo = (int64_t)blockIdx.x * split_len;
    const int64_t s_hi = std::min<int64_t>(B, s_lo + split_len);
    float *P = part + (int64_t)blockIdx.x * nnz;
    const bool vec4 = (B & 3) == 0;

    int beg[RPW], end[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        beg[i] = r < R ? __ldg(row_ptr + r) : 0;
        end[i] = r < R ? __ldg(row_ptr + r + 1) : 0;
    }

    bool first = true;
    for (int64_t b0 = s_lo; b0 < s_hi; b0 += BT) {
        // dY[r][b0 + lane*VEC ..] for this warp's rows, zero past the range.
        float dy[RPW][VEC];
        const int64_t bl = b0 + lane * VEC;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int64_t r = r0 + warp + (int64_t)i * NW;
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                dy[i][v] = (r < R && bl + v < s_hi) ? __ldg(dY + r * B + bl + v) : 0.f;
        }
        int cur[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) cur[i] = beg[i];

        for (int64_t kb0 = 0; kb0 < C; kb0 += KC) {
            const int nk = (int)std::min<int64_t>(KC, C - kb0);
            const int kb1 = (int)(kb0 + nk);
            const int ckb0 = (int)kb0;
            __syncthreads();
            // X[kb0.., b0..b0+BT); columns >= B are zero-filled (columns in
            // [s_hi, B) never occur: splits are whole slices).
            stage_tile<BT, NT>(tile, X, kb0, nk, B, b0, vec4);
            __syncthreads();
            const float *tl = tile + lane * VEC;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                while (cur[i] < end[i]) {
                    const int k = cur[i] + lane;
                    const int c = k < end[i] ? __ldg(col_idx + k) : INT_MAX;
                    const int n = __popc(__ballot_sync(kFull, c < kb1));
                    if (n == 0) break;
                    float acc[32];
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        acc[t] = 0.f;
                        const int ct = __shfl_sync(kFull, c, t);
                        if (t < n) {
                            float x[VEC];
                            lds_vec<VEC>(tl + (ct - ckb0) * BT, x);
#pragma unroll
                            for (int v = 0; v < VEC; ++v) acc[t] = fmaf(dy[i][v], x[v], acc[t]);
                        }
                    }
                    const float s = transpose_reduce32(acc, lane);
                    if (lane < n) {
                        float *p = P + cur[i] + lane;
                        *p = first ? s : *p + s;
                    }
                    cur[i] += n;
                    if (n < 32) break;
                }
            }
        }
        first = false;
    }
}

// dW[j] = sum_s part[s][j], s ascending.
__global__ void split_reduce_kernel(int64_t nnz, int nsplit, const float *__restrict__ part,
                                    float *__restrict__ dW) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnz) return;
    float s = part[j];
    for (int i = 1; i < nsplit; ++i) s += part[(int64_t)i * nnz + j];
    dW[j] = s;
}

constexpr int kNumSMs = 148;
constexpr int kTileBudget = 64 * 1024;

template <int VEC, int RPW, int NW>
sp_status launch_cfg(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                     cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    const int64_t R = w->R, C = w->C, nnz = w->nnz;
    const int64_t slices = (B + BT - 1) / BT;
    const int64_t rblocks = (R + NW * RPW - 1) / (NW * RPW);
    // batch splits: enough CTAs for ~2 per SM, each split a whole number of slices
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(slices, (2 * kNumSMs + rblocks - 1) / rblocks));
    const int64_t spl = (slices + nsplit - 1) / nsplit;  // slices per split
    nsplit = (slices + spl - 1) / spl;
    int KC = (int)std::min<int64_t>(kTileBudget / (BT * 4), C);
    KC = std::max(KC, 1);
    const size_t smem = (size_t)KC * BT * sizeof(float);
    float *part = dW;
    if (nsplit > 1) {
        if (cudaMallocAsync((void **)&part, (size_t)(nsplit * nnz) * sizeof(float), st) != cudaSuccess) {
            set_error("sp_linear_bwd_weight: scratch allocation failed");
            return SP_ERR_ALLOC;
        }
    }
    auto kern = sddmm_tiled_kernel<VEC, RPW, NW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)nsplit, (unsigned)rblocks);
    count_launches(nsplit > 1 ? 2 : 1);
    kern<<<grid, NW * 32, smem, st>>>(R, C, B, KC, spl * BT, w->row_ptr, w->col_idx, X, dY, part,
                                      nnz);
    if (nsplit > 1) {
        split_reduce_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, (int)nsplit, part, dW);
        cudaFreeAsync(part, st);
    }
    return SP_OK;
}

}  // namespace

sp_status launch_sddmm(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                       cudaStream_t st) {
    if (w->nnz == 0) return SP_OK;
    if (B <= 32) return launch_cfg<1, 4, 8>(w, X, dY, dW, B, st);
    if (B <= 64 || (B & 3) != 0) return launch_cfg<2, 4, 8>(w, X, dY, dW, B, st);
    return launch_cfg<4, 4, 8>(w, X, dY, dW, B, st);
}

}  // namespace sp
