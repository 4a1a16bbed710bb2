// spmm.cu -- forward SpMM (K2, sp_linear_fwd) and CSC-driven input-gradient
// SpMM (K3, sp_linear_bwd_input).  SURVEY §8(a) rows a-2, a-3.
//
//   out[r][b] = epi( sum_{k in [ptr[r], ptr[r+1])} val(k) * in[idx[k]][b] )
//   forward (P141):  ptr=row_ptr, idx=col_idx, val(k)=vals[k]
//   dX (Eq. 1):      ptr=col_ptr, idx=row_idx, val(k)=vals[perm[k]]
//
// Design: one CTA owns a batch slice of BT = 32*VEC columns
// and a block of RB = NW*RPW rows.  The dense operand `in` is streamed
// through shared memory in column blocks of KC rows (the "activation tile
// staged in shared memory" of the north star), coalesced 16-byte loads along
// the batch.  Each warp owns RPW interleaved rows and keeps their VEC-wide
// accumulators in registers across column blocks; per nonzero every lane
// does VEC FMAs against tile[c][lane*VEC ..] (batch-contiguous vector LDS).
// Each output element is produced by exactly one lane, so there are no
// atomics and the summation order (k ascending) is fixed: bitwise
// reproducible and independent of B and of the launch shape along B.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

template <int VEC, int RPW, int NW, bool CSC, int EPI>
__global__ void __launch_bounds__(NW * 32)
    spmm_tiled_kernel(int64_t rows, int64_t inner, int64_t B, int KC,
                      const int32_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                      const int32_t *__restrict__ perm, const float *__restrict__ vals,
                      const float *__restrict__ in, float *__restrict__ out,
                      const float *__restrict__ gate) {
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) float tile[];  // [KC][BT]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * BT;
    const int64_t r0 = (int64_t)blockIdx.y * (NW * RPW);
    const bool vec4 = (B & 3) == 0;

    float acc[RPW][VEC];
    int cur[RPW], end[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        cur[i] = r < rows ? __ldg(ptr + r) : 0;
        end[i] = r < rows ? __ldg(ptr + r + 1) : 0;
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;
    }

    for (int64_t kb0 = 0; kb0 < inner; kb0 += KC) {
        const int nk = (int)std::min<int64_t>(KC, inner - kb0);
        const int kb1 = (int)(kb0 + nk);
        __syncthreads();  // previous tile fully consumed
        stage_tile<BT, NT>(tile, in, kb0, nk, B, b0, vec4);
        __syncthreads();
        const float *tl = tile + lane * VEC;
        const int ckb0 = (int)kb0;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            // Row i's segment inside this column block, 32 entries at a time:
            // lanes load (index, value) coalesced, then broadcast by shuffle.
            while (cur[i] < end[i]) {
                const int k = cur[i] + lane;
                int c = INT_MAX;
                float w = 0.f;
                if (k < end[i]) {
                    c = __ldg(idx + k);
                    w = CSC ? __ldg(vals + __ldg(perm + k)) : __ldg(vals + k);
                }
                const unsigned bal = __ballot_sync(kFull, c < kb1);
                const int n = __popc(bal);  // columns ascending: a prefix
                if (n == 0) break;
#pragma unroll 4
                for (int t = 0; t < n; ++t) {
                    const int ct = __shfl_sync(kFull, c, t);
                    const float wt = __shfl_sync(kFull, w, t);
                    float x[VEC];
                    lds_vec<VEC>(tl + (ct - ckb0) * BT, x);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(wt, x[v], acc[i][v]);
                }
                cur[i] += n;
                if (n < 32) break;
            }
        }
    }

    // Epilogue: ReLU / ReLU' gate fused; each element written once.
    const int64_t bl = b0 + lane * VEC;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        if (r >= rows) continue;
        float o[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            float a = acc[i][v];
            if (EPI == EPI_RELU) a = fmaxf(a, 0.f);
            if (EPI == EPI_GATE) {
                const int64_t b = bl + v;
                const float g = b < B ? __ldg(gate + r * B + b) : 0.f;
                a = g > 0.f ? a : 0.f;
            }
            o[v] = a;
        }
        float *dst = out + r * B + bl;
        if (vec4 && VEC > 1 && bl + VEC <= B) {
            if constexpr (VEC == 2) *reinterpret_cast<float2 *>(dst) = make_float2(o[0], o[1]);
            if constexpr (VEC == 4)
                *reinterpret_cast<float4 *>(dst) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (bl + v < B) dst[v] = o[v];
        }
    }
}

constexpr int kNumSMs = 148;
constexpr int kTileBudget = 96 * 1024;  // bytes of smem tile per CTA

template <int VEC, int RPW, int NW, bool CSC>
void launch_cfg(int64_t rows, int64_t inner, int64_t B, const int32_t *ptr, const int32_t *idx,
                const int32_t *perm, const float *vals, const float *in, float *out,
                const float *gate, int epi, cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    int KC = (int)std::min<int64_t>(kTileBudget / (BT * 4), inner);
    KC = std::max(KC, 1);
    const size_t smem = (size_t)KC * BT * sizeof(float);
    dim3 grid((unsigned)((B + BT - 1) / BT), (unsigned)((rows + NW * RPW - 1) / (NW * RPW)));
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        kern<<<grid, NW * 32, smem, st>>>(rows, inner, B, KC, ptr, idx, perm, vals, in, out, gate);
    };
    if (epi == EPI_RELU)
        launch(spmm_tiled_kernel<VEC, RPW, NW, CSC, EPI_RELU>);
    else if (epi == EPI_GATE)
        launch(spmm_tiled_kernel<VEC, RPW, NW, CSC, EPI_GATE>);
    else
        launch(spmm_tiled_kernel<VEC, RPW, NW, CSC, EPI_NONE>);
}

template <int VEC, bool CSC>
void launch_vec(int64_t rows, int64_t inner, int64_t B, const int32_t *ptr, const int32_t *idx,
                const int32_t *perm, const float *vals, const float *in, float *out,
                const float *gate, int epi, cudaStream_t st) {
    // Largest row block (fewest re-reads of `in` through L2) that still
    // gives >= 2 CTAs per SM.
    constexpr int NW = 8;
    const int64_t slices = (B + 32 * VEC - 1) / (32 * VEC);
    auto ctas = [&](int rpw) { return slices * ((rows + NW * rpw - 1) / (NW * rpw)); };
    if (ctas(16) >= 2 * kNumSMs)
        launch_cfg<VEC, 16, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else if (ctas(8) >= 2 * kNumSMs)
        launch_cfg<VEC, 8, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else if (ctas(4) >= 2 * kNumSMs)
        launch_cfg<VEC, 4, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else
        launch_cfg<VEC, 2, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
}

}  // namespace

void launch_spmm(int64_t rows, int64_t inner, int64_t B, const int32_t *ptr, const int32_t *idx,
                 const int32_t *perm, const float *vals, const float *in, float *out,
                 const float *gate, int epi, int max_seg, cudaStream_t st) {
    (void)max_seg;
    const bool csc = perm != nullptr;
    if (B <= 32) {
        if (csc) launch_vec<1, true>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
        else launch_vec<1, false>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    } else if (B <= 64 || (B & 3) != 0) {
        if (csc) launch_vec<2, true>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
        else launch_vec<2, false>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    } else {
        if (csc) launch_vec<4, true>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
        else launch_vec<4, false>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    }
}

}  // namespace sp
