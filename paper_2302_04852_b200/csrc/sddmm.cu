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

struct SddmmArgs {
    int64_t nrow, F, B;
    int KC, nkb, spl;  // column block, #column blocks, slices per split
    const int32_t *ptr, *idx;
    const float *regop;   // [nrow x B]: operand kept in registers (one row per warp row)
    const float *smemop;  // [F x B]: operand staged through shared memory
    float *part;          // [nsplit x nnz] slice-split partials (slot order of ptr/idx)
    int64_t nnz;
};

// v2: grid.x = row blocks (fastest), grid.y = batch splits.  Orientation:
//   CSR (TRANS=false): rows r, regop = dY, smemop = X, slot j (CSR order)
//   CSC (TRANS=true):  rows c, regop = X,  smemop = dY, slot k (CSC order),
// whichever stages the smaller feature dimension (fewer L2 re-reads).  The
// (slice, column block) tiles are double-buffered with cp.async.  Per row, a
// 32-entry index window persists across the column blocks of a slice; each
// segment's partial dots go to 32 register accumulators and one warp
// transpose-reduce, and lane t adds the slice sum into part[split][slot t].
template <int VEC, int RPW, int NW>
__global__ void __launch_bounds__(NW * 32, 1) sddmm_tiled_kernel(const SddmmArgs a) {
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) float smem[];  // [2][KC][BT]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * (NW * RPW);
    const int64_t B = a.B;
    const int64_t s_lo = (int64_t)blockIdx.y * a.spl * BT;
    const int nsl = (int)std::min<int64_t>(a.spl, (B - s_lo + BT - 1) / BT);  // slices in this split
    const int ntile = nsl * a.nkb;
    float *P = a.part + (int64_t)blockIdx.y * a.nnz;
    const bool vec4 = (B & 3) == 0;
    const size_t tile_sz = (size_t)a.KC * BT;

    auto stage = [&](int q, int buf) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        const int64_t k0 = (int64_t)kb * a.KC;
        stage_any<BT, NT>(smem + buf * tile_sz, a.smemop, k0, (int)std::min<int64_t>(a.KC, a.F - k0), B,
                          s_lo + (int64_t)s * BT, vec4);
    };
    stage(0, 0);
    cp_async_commit();

    int beg[RPW], end[RPW], cur[RPW], cw[RPW], co[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        beg[i] = r < a.nrow ? __ldg(a.ptr + r) : 0;
        end[i] = r < a.nrow ? __ldg(a.ptr + r + 1) : 0;
    }
    float rv[RPW][VEC];

    for (int q = 0; q < ntile; ++q) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        const int64_t b0 = s_lo + (int64_t)s * BT;
        if (kb == 0) {
            // new slice: this warp's register-operand rows and fresh windows
            const int64_t bl = b0 + lane * VEC;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = r0 + warp + (int64_t)i * NW;
                const float *src = a.regop + r * B + bl;
                if (r < a.nrow && vec4 && VEC == 4 && bl + 4 <= B) {
                    const float4 t = __ldg(reinterpret_cast<const float4 *>(src));
                    rv[i][0] = t.x;
                    if constexpr (VEC == 4) {
                        rv[i][1] = t.y;
                        rv[i][2] = t.z;
                        rv[i][3] = t.w;
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) rv[i][v] = (r < a.nrow && bl + v < B) ? __ldg(src + v) : 0.f;
                }
                cur[i] = beg[i];
                const int k = beg[i] + lane;
                cw[i] = k < end[i] ? __ldg(a.idx + k) : INT_MAX;
                co[i] = k < end[i] ? cw[i] * (BT * 4) : 0;
            }
        }
        if (q + 1 < ntile) {
            stage(q + 1, (q + 1) & 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int64_t kb0 = (int64_t)kb * a.KC;
        const int kb1 = (int)std::min<int64_t>(kb0 + a.KC, a.F);
        const char *base = reinterpret_cast<const char *>(smem + (q & 1) * tile_sz + lane * VEC) -
                           (size_t)kb0 * BT * 4;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            while (cur[i] < end[i]) {
                // window base wb = cur rounded so that the window holds cur
                const int wb = beg[i] + ((cur[i] - beg[i]) & ~31);
                const int t0 = cur[i] - wb;
                if (t0 == 0 && cur[i] != beg[i]) {  // crossed into a new window
                    const int k = wb + lane;
                    cw[i] = k < end[i] ? __ldg(a.idx + k) : INT_MAX;
                    co[i] = k < end[i] ? cw[i] * (BT * 4) : 0;
                }
                const int L = __popc(__ballot_sync(kFull, cw[i] < kb1));
                if (L <= t0) break;
                // entries t0..L-1 -> acc[u], u = t - t0 (static index), 8 at a time
                float acc[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u] = 0.f;
                const int n = L - t0;
#pragma unroll
                for (int g = 0; g < 32; g += 8) {
                    if (g >= n) break;
                    int off[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int o = __shfl_sync(kFull, co[i], t0 + g + u);  // wraps mod 32
                        off[u] = (g + u < n) ? o : (int)((size_t)kb0 * BT * 4);
                    }
                    float xv[8][VEC];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        lds_vec<VEC>(reinterpret_cast<const float *>(base + off[u]), xv[u]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        float d = 0.f;
#pragma unroll
                        for (int v = 0; v < VEC; ++v) d = fmaf(rv[i][v], xv[u][v], d);
                        acc[g + u] = (g + u < n) ? d : 0.f;
                    }
                }
                const float sum = transpose_reduce32(acc, lane);
                if (lane < n) {
                    float *p = P + cur[i] + lane;
                    *p = (s == 0) ? sum : *p + sum;
                }
                cur[i] = wb + L;
                if (L < 32) break;
            }
        }
        __syncthreads();
    }
}

// dW[perm ? perm[k] : k] = sum_s part[s][k], s ascending.
__global__ void split_reduce_kernel(int64_t nnz, int nsplit, const float *__restrict__ part,
                                    const int32_t *__restrict__ perm, float *__restrict__ dW) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    float s = part[k];
    for (int i = 1; i < nsplit; ++i) s += part[(int64_t)i * nnz + k];
    dW[perm ? perm[k] : k] = s;
}

constexpr int kNumSMs = 148;
constexpr int kSmemBudget = 192 * 1024;

template <int VEC, int RPW, int NW>
sp_status launch_cfg(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                     cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    const bool trans = w->C > w->R;  // stage the smaller feature dimension
    const int64_t nrow = trans ? w->C : w->R, F = trans ? w->R : w->C, nnz = w->nnz;
    const int64_t slices = (B + BT - 1) / BT;
    const int64_t rblocks = (nrow + NW * RPW - 1) / (NW * RPW);
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(slices, (2 * kNumSMs + rblocks - 1) / rblocks));
    const int64_t spl = (slices + nsplit - 1) / nsplit;
    nsplit = (slices + spl - 1) / spl;
    int KC = (int)std::min<int64_t>(kSmemBudget / (2 * BT * 4), F);
    KC = std::max(KC, 1);
    const int nkb = (int)((F + KC - 1) / KC);
    KC = (int)((F + nkb - 1) / nkb);
    const size_t smem = (size_t)2 * KC * BT * sizeof(float);
    const bool direct = nsplit == 1 && !trans;
    float *part = dW;
    if (!direct) {
        if (cudaMallocAsync((void **)&part, (size_t)(nsplit * nnz) * sizeof(float), st) != cudaSuccess) {
            set_error("sp_linear_bwd_weight: scratch allocation failed");
            return SP_ERR_ALLOC;
        }
    }
    SddmmArgs a{nrow, F, B, KC, nkb, (int)spl, trans ? w->col_ptr : w->row_ptr,
                trans ? w->row_idx : w->col_idx, trans ? X : dY, trans ? dY : X, part, nnz};
    auto kern = sddmm_tiled_kernel<VEC, RPW, NW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    count_launches(direct ? 1 : 2);
    kern<<<dim3((unsigned)rblocks, (unsigned)nsplit), NW * 32, smem, st>>>(a);
    if (!direct) {
        split_reduce_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, (int)nsplit, part,
                                                                           trans ? w->perm : nullptr, dW);
        cudaFreeAsync(part, st);
    }
    return SP_OK;
}

}  // namespace

sp_status launch_sddmm(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                       cudaStream_t st) {
    if (w->nnz == 0) return SP_OK;
    if (B <= 32) return launch_cfg<1, 8, 16>(w, X, dY, dW, B, st);
    if (B <= 64 || (B & 3) != 0) return launch_cfg<2, 8, 16>(w, X, dY, dW, B, st);
    return launch_cfg<4, 8, 16>(w, X, dY, dW, B, st);
}

}  // namespace sp
