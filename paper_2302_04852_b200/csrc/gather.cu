// gather.cu -- direct-gather kernels for the very sparse / small regime.
//
// The tiled kernels stage the dense operand through shared memory once per
// row block: (R / RB) * C * B floats cross L2 -> SM per product.  Gathering
// each nonzero's activation row straight from L2 costs nnz * B floats instead,
// which is less whenever the expected number of nonzeros a row block has in
// one column, RB * d, is below ~1 (e.g. 4096^2 at 99 %, B = 256).  These
// kernels serve that regime: no shared-memory tile, lanes over the batch,
// (index, value) pairs loaded coalesced per 32 and broadcast by shuffles,
// VEC-wide __ldg of the activation row per nonzero.  Same per-element order
// as the tiled kernels' definition (entries ascending), no atomics.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <climits>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

template <int VEC>
__device__ __forceinline__ void ldg_vec4(const float *p, float (&v)[VEC], bool vec, int nvalid) {
    if (vec && nvalid == VEC) {
        if constexpr (VEC == 4) {
            const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
            v[0] = t.x;
            v[1] = t.y;
            v[2] = t.z;
            v[3] = t.w;
        } else if constexpr (VEC == 2) {
            const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
            v[0] = t.x;
            v[1] = t.y;
        } else {
            v[0] = __ldg(p);
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[i] = i < nvalid ? __ldg(p + i) : 0.f;
    }
}

// out[r][b] = epi(sum_k val(k) * in[idx[k]][b]); warp per (row, 32*VEC slice)
template <int VEC, int EPI>
__global__ void __launch_bounds__(256)
    spmm_gather_kernel(int64_t rows, int64_t B, const int32_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                       const int32_t *__restrict__ perm, const float *__restrict__ vals,
                       const float *__restrict__ in, float *__restrict__ out, const float *__restrict__ gate) {
    const int lane = threadIdx.x & 31;
    const int64_t nsl = (B + 32 * VEC - 1) / (32 * VEC);
    const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t r = wid / nsl;
    if (r >= rows) return;
    const int64_t bl = (wid - r * nsl) * 32 * VEC + lane * VEC;
    const int nvalid = (int)std::max<int64_t>(0, std::min<int64_t>(VEC, B - bl));
    const bool vec = (B % VEC) == 0;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    const int beg = __ldg(ptr + r), end = __ldg(ptr + r + 1);
    for (int j0 = beg; j0 < end; j0 += 32) {
        const int j = j0 + lane;
        const int cl = j < end ? __ldg(idx + j) : 0;
        const float wl = j < end ? __ldg(vals + (perm ? __ldg(perm + j) : j)) : 0.f;
        const int n = min(32, end - j0);
#ifndef SP_GATHER_U4
        // GU entries in flight per warp: all their row loads issue before the FMAs
        // (the L2 latency, not its bandwidth, bounds a per-entry load chain;
        // cfg4 99 %: 4 -> 8 in flight, fwd 38 -> 31 us)
#ifndef SP_GATHER_GU
#define SP_GATHER_GU 8
#endif
        constexpr int GU = SP_GATHER_GU;
        int t = 0;
        for (; t + GU <= n; t += GU) {
            float x[GU][VEC];
            float w[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int c = __shfl_sync(kFull, cl, t + u);
                w[u] = __shfl_sync(kFull, wl, t + u);
                ldg_vec4<VEC>(in + (int64_t)c * B + bl, x[u], vec, nvalid);
            }
#pragma unroll
            for (int u = 0; u < GU; ++u) fma_bcast<VEC>(acc, w[u], x[u]);
        }
        for (; t < n; ++t) {
#else
#pragma unroll 4
        for (int t = 0; t < n; ++t) {
#endif
            const int c = __shfl_sync(kFull, cl, t);
            const float w = __shfl_sync(kFull, wl, t);
            float x[VEC];
            ldg_vec4<VEC>(in + (int64_t)c * B + bl, x, vec, nvalid);
            fma_bcast<VEC>(acc, w, x);
        }
    }
    if (nvalid == 0) return;
    float *dst = out + r * B + bl;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
        if (v >= nvalid) break;
        float o = acc[v];
        if (EPI == EPI_RELU) o = fmaxf(o, 0.f);
        if (EPI == EPI_GATE) o = __ldg(gate + r * B + bl + v) > 0.f ? o : 0.f;
        dst[v] = o;
    }
}

// dW[j] = sum_b dY[row(j)][b] * X[col_idx[j]][b]; warp per chunk of <= 32
// consecutive nonzeros of one row (work list chunk_ptr: balanced for skewed
// rows), looping over the whole batch; one transpose-reduce at the end.
template <int VEC>
__global__ void __launch_bounds__(256)
    sddmm_gather_kernel(int64_t R, int64_t B, const int32_t *__restrict__ chunk_ptr,
                        const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ col_idx,
                        const float *__restrict__ X, const float *__restrict__ dY, float *__restrict__ dW) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (wid >= __ldg(chunk_ptr + R)) return;
    int64_t lo = 0, hi = R;  // row r with chunk_ptr[r] <= wid < chunk_ptr[r+1]
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(chunk_ptr + mid) <= wid) lo = mid;
        else hi = mid;
    }
    const int64_t r = lo;
    const int j0 = __ldg(row_ptr + r) + (int)(wid - __ldg(chunk_ptr + r)) * 32;
    const int end = __ldg(row_ptr + r + 1);
    const int n = min(32, end - j0);
    const int cl = lane < n ? __ldg(col_idx + j0 + lane) : 0;
    const bool vec = (B % VEC) == 0;
    float acc[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) acc[u] = 0.f;
    for (int64_t b0 = 0; b0 < B; b0 += 32 * VEC) {
        const int64_t bl = b0 + lane * VEC;
        const int nvalid = (int)std::max<int64_t>(0, std::min<int64_t>(VEC, B - bl));
        float dy[VEC];
        ldg_vec4<VEC>(dY + r * B + bl, dy, vec, nvalid);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int c = __shfl_sync(kFull, cl, u);
            if (u < n) {
                float x[VEC];
                ldg_vec4<VEC>(X + (int64_t)c * B + bl, x, vec, nvalid);
                acc[u] += dot_vec<VEC>(dy, x);
            }
        }
    }
    const float s = transpose_reduce32(acc, lane);
    if (lane < n) dW[j0 + lane] = s;
}

}  // namespace

// Gather path wins when staging would move more bytes than gathering:
// nrb * inner (tile rows streamed per batch column) > nnz (rows gathered).
bool gather_preferred(const sp_weight_s *w, int orient, int64_t B, bool chunked) {
    // the gather SpMM walks a whole row per warp: skewed rows (Zipf) would
    // serialise the tail, so only balanced structures take it (the SDDMM's
    // 32-nonzero chunks are balanced by construction)
    const int64_t rows = orient == 0 ? w->R : w->C;
    const int64_t mx = orient == 0 ? w->max_row_nnz : w->max_col_nnz;
    if (!chunked && (double)mx > 4.0 * (double)w->nnz / (double)rows + 64.0) return false;
    // tiny products (well under one wave of tiles) are latency bound: one pass
    // straight from L2 beats staging tiles
    if ((double)w->nnz * (double)B < 4.0e6) return true;
    const sp_tiling &t = w->til[orient][1];  // the smallest tiling the tiled path would fall back to
    const sp_tiling &t0 = w->til[orient][0];
    const int64_t slices = (B + 127) / 128;
    const sp_tiling &tt = (int64_t)t0.nrb * slices >= 2 * num_sms() ? t0 : t;
    return (double)tt.nrb * (double)tt.inner > 1.25 * (double)w->nnz;
}

void launch_spmm_gather(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out,
                        const float *gate, int epi, cudaStream_t st) {
    const int64_t rows = orient == 0 ? w->R : w->C;
    const int32_t *ptr = orient == 0 ? w->row_ptr : w->col_ptr;
    const int32_t *idx = orient == 0 ? w->col_idx : w->row_idx;
    const int32_t *perm = orient == 0 ? nullptr : w->perm;
    auto go = [&](auto kern, int vec) {
        const int64_t nsl = (B + 32 * vec - 1) / (32 * vec);
        const int64_t warps = rows * nsl;
        count_launches(1);
        note_path("spmm_gather");
        kern<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(rows, B, ptr, idx, perm, w->vals, in, out, gate);
    };
    const int vec = B >= 128 ? 4 : B >= 64 ? 2 : 1;
    if (vec == 4) {
        if (epi == EPI_RELU) go(spmm_gather_kernel<4, EPI_RELU>, 4);
        else if (epi == EPI_GATE) go(spmm_gather_kernel<4, EPI_GATE>, 4);
        else go(spmm_gather_kernel<4, EPI_NONE>, 4);
    } else if (vec == 2) {
        if (epi == EPI_RELU) go(spmm_gather_kernel<2, EPI_RELU>, 2);
        else if (epi == EPI_GATE) go(spmm_gather_kernel<2, EPI_GATE>, 2);
        else go(spmm_gather_kernel<2, EPI_NONE>, 2);
    } else {
        if (epi == EPI_RELU) go(spmm_gather_kernel<1, EPI_RELU>, 1);
        else if (epi == EPI_GATE) go(spmm_gather_kernel<1, EPI_GATE>, 1);
        else go(spmm_gather_kernel<1, EPI_NONE>, 1);
    }
}

void launch_sddmm_gather(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                         cudaStream_t st) {
    const int64_t warps = w->nnz / 32 + w->R;  // >= number of chunks
    auto go = [&](auto kern) {
        count_launches(1);
        note_path("sddmm_gather");
        kern<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(w->R, B, w->chunk_ptr, w->row_ptr, w->col_idx, X, dY, dW);
    };
    if (B >= 128) go(sddmm_gather_kernel<4>);
    else if (B >= 64) go(sddmm_gather_kernel<2>);
    else go(sddmm_gather_kernel<1>);
}

}  // namespace sp
