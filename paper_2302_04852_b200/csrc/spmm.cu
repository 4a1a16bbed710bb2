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

struct SpmmArgs {
    int64_t rows, inner, B;
    int KC, nkb;
    const int32_t *ptr, *idx, *perm;
    const float *vals, *in;
    float *out;
    const float *gate;
};

// v2: grid.x = row blocks (fastest, so the CTAs sharing one batch slice of
// `in` run together and hit L2), grid.y = batch slices.  `in` column blocks
// are double-buffered in shared memory with cp.async (LDGSTS).  Each warp keeps,
// per owned row, a 32-entry window of (index, value) in registers (one lane per
// entry, loaded coalesced) that persists across column blocks; entries are
// broadcast with shuffles.
template <int VEC, int RPW, int NW, bool CSC, int EPI>
__global__ void __launch_bounds__(NW * 32, 1) spmm_tiled_kernel(const SpmmArgs a) {
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    extern __shared__ __align__(16) float smem[];  // [2][KC][BT]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * (NW * RPW);
    const int64_t b0 = (int64_t)blockIdx.y * BT;
    const int64_t B = a.B;
    const bool vec4 = (B & 3) == 0;
    const size_t tile_sz = (size_t)a.KC * BT;
    (void)tile_sz;

    // kick off the first tile before touching the index structure
    stage_any<BT, NT>(smem, a.in, 0, (int)std::min<int64_t>(a.KC, a.inner), B, b0, vec4);
    cp_async_commit();

    // Per owned row: cursor, end, window base, and this lane's window entry
    // (smem byte offset of its column relative to column 0, and its value).
    float acc[RPW][VEC];
    int cur[RPW], end[RPW], wb[RPW], cw[RPW], co[RPW];
    float ww[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        cur[i] = r < a.rows ? __ldg(a.ptr + r) : 0;
        end[i] = r < a.rows ? __ldg(a.ptr + r + 1) : 0;
        wb[i] = cur[i];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;
    }
    auto load_window = [&](int i) {
        const int k = wb[i] + lane;
        const bool ok = k < end[i];
        cw[i] = ok ? __ldg(a.idx + k) : INT_MAX;
        ww[i] = ok ? (CSC ? __ldg(a.vals + __ldg(a.perm + k)) : __ldg(a.vals + k)) : 0.f;
        co[i] = ok ? cw[i] * (BT * 4) : 0;
    };
#pragma unroll
    for (int i = 0; i < RPW; ++i) load_window(i);

    for (int kb = 0; kb < a.nkb; ++kb) {
        const int64_t kb0 = (int64_t)kb * a.KC;
        if (kb + 1 < a.nkb) {
            const int64_t n0 = kb0 + a.KC;
            stage_any<BT, NT>(smem + ((kb + 1) & 1) * tile_sz, a.in, n0, (int)std::min<int64_t>(a.KC, a.inner - n0),
                              B, b0, vec4);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int kb1 = (int)std::min<int64_t>(kb0 + a.KC, a.inner);
        // byte base such that base + c*BT*4 addresses tile row (c - kb0), this lane's VEC
        const char *base = reinterpret_cast<const char *>(smem + (kb & 1) * tile_sz + lane * VEC) -
                           (size_t)kb0 * BT * 4;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            while (cur[i] < end[i]) {
                int t0 = cur[i] - wb[i];
                if (t0 >= 32) {  // window exhausted: reload (warp-uniform)
                    wb[i] = cur[i];
                    t0 = 0;
                    load_window(i);
                }
                const int L = __popc(__ballot_sync(kFull, cw[i] < kb1));  // ascending: a prefix
                if (L <= t0) break;
                // entries t0 .. L-1, 8 at a time: shuffles, then 8 independent
                // LDS, then the FMAs (entries past L get weight 0, offset 0).
                for (int g = t0; g < L; g += 8) {
                    int off[8];
                    float w[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int t = g + u;
                        const int o = __shfl_sync(kFull, co[i], t);  // lane index wraps mod 32
                        const float x = __shfl_sync(kFull, ww[i], t);
                        off[u] = t < L ? o : (int)((size_t)kb0 * BT * 4);
                        w[u] = t < L ? x : 0.f;
                    }
                    float xv[8][VEC];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        lds_vec<VEC>(reinterpret_cast<const float *>(base + off[u]), xv[u]);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(w[u], xv[u][v], acc[i][v]);
                }
                cur[i] = wb[i] + L;
                if (L < 32) break;  // column block (or row) ended inside the window
            }
        }
        __syncthreads();  // everyone done with this buffer before it is refilled
    }

    // Epilogue: ReLU / ReLU' gate fused; each element written once.
    const int64_t bl = b0 + lane * VEC;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + (int64_t)i * NW;
        if (r >= a.rows) continue;
        float o[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            float x = acc[i][v];
            if (EPI == EPI_RELU) x = fmaxf(x, 0.f);
            if (EPI == EPI_GATE) {
                const int64_t b = bl + v;
                const float g = b < B ? __ldg(a.gate + r * B + b) : 0.f;
                x = g > 0.f ? x : 0.f;
            }
            o[v] = x;
        }
        float *dst = a.out + r * B + bl;
        if (vec4 && VEC > 1 && bl + VEC <= B) {
            if constexpr (VEC == 2) *reinterpret_cast<float2 *>(dst) = make_float2(o[0], o[1]);
            if constexpr (VEC == 4) *reinterpret_cast<float4 *>(dst) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (bl + v < B) dst[v] = o[v];
        }
    }
}

constexpr int kNumSMs = 148;
constexpr int kSmemBudget = 192 * 1024;  // two tile buffers per CTA, 1 CTA / SM

template <int VEC, int RPW, int NW, bool CSC>
void launch_cfg(int64_t rows, int64_t inner, int64_t B, const int32_t *ptr, const int32_t *idx,
                const int32_t *perm, const float *vals, const float *in, float *out,
                const float *gate, int epi, cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    int KC = (int)std::min<int64_t>(kSmemBudget / (2 * BT * 4), inner);
    KC = std::max(KC, 1);
    // balance the column blocks (same count, smallest equal size)
    const int nkb = (int)((inner + KC - 1) / KC);
    KC = (int)((inner + nkb - 1) / nkb);
    const size_t smem = (size_t)2 * KC * BT * sizeof(float);
    SpmmArgs a{rows, inner, B, KC, nkb, ptr, idx, perm, vals, in, out, gate};
    dim3 grid((unsigned)((rows + NW * RPW - 1) / (NW * RPW)), (unsigned)((B + BT - 1) / BT));
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        kern<<<grid, NW * 32, smem, st>>>(a);
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
    // Largest row block (fewest L2 re-reads of `in`) that still fills the
    // 148 SMs with >= 2 waves of CTAs.
    constexpr int NW = 16;
    const int64_t slices = (B + 32 * VEC - 1) / (32 * VEC);
    auto ctas = [&](int rpw) { return slices * ((rows + NW * rpw - 1) / (NW * rpw)); };
    if (ctas(8) >= 2 * kNumSMs)
        launch_cfg<VEC, 8, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else if (ctas(4) >= 2 * kNumSMs)
        launch_cfg<VEC, 4, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else if (ctas(2) >= kNumSMs)
        launch_cfg<VEC, 2, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
    else
        launch_cfg<VEC, 1, NW, CSC>(rows, inner, B, ptr, idx, perm, vals, in, out, gate, epi, st);
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
