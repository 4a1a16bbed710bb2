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

// ---- position gather kernels (gather tilings) ---------------------------------
// The same per-thread row gather, driven by a gather tiling (til_g: one column
// block spanning the inner dimension): a warp per position (row, or part row of
// a skewed CSR row), its entries (inner index * kTilRowBytes, weight) loaded
// coalesced per 32 and broadcast by shuffles -- the CSC weights come straight
// from the tiling instead of vals[perm[k]] -- GU row loads in flight per lane.
//   MODE 0  SpMM: out[row] = epi(sum_e w_e * gin[idx_e])   (fwd: CSR tiling; dX: CSC;
//           part rows store raw sums, split_rows_reduce adds them)
//   MODE 1  fused backward on the CSC tiling: dX[i] = gate(sum_e w_e * dY[j_e]) and
//           dW[vidx_e] = <X[i], dY[j_e]> from the same gathered dY rows (Alg. 1, P173-P220)
//   MODE 2  dW alone on the CSR tiling: dW[vidx_e] = <dY[i], X[j_e]>
// MODE 0 takes 128 batch columns per warp (grid.y = slices); MODE 1 / 2 take the
// whole batch (NS = B / 128 <= 4 slices per lane) so that each entry's dot product
// is complete in its warp: one transposed shuffle reduction per GU entries.  Per
// element the sums run over entries in tiling order (ascending inner index).
// (A first version fetched the rows with 1-D bulk copies into per-warp shared-
// memory rings: ~3.8 TB/s whatever the row size, 1.5-2.3x slower than these
// register loads.)
struct PgArgs {
    int64_t B, npos;
    const int32_t *seg;
    const int2 *ent;
    const int32_t *vidx;
    const int32_t *rowmap, *split;  // split: part slot per position (nullptr: none)
    const float *gin;               // gathered operand, rows indexed by ent.x / kTilRowBytes
    const float *rin;               // MODE 1 / 2: the position's row operand (X / dY)
    const float *gate;              // EPI_GATE ReLU' gate rows
    float *out;                     // MODE 0: Y or dX; MODE 1: dX
    float *dW;
    float *vpart;                   // MODE 0 part rows' raw sums [nparts x B]
    int epi;
};

// transposed reduction of N per-lane values over the warp: lane l ends with the
// 32-lane sum of value (l >> (5 - log2 N)) & (N - 1)
template <int N>
__device__ __forceinline__ float pg_reduce(float (&p)[N], int lane) {
#pragma unroll
    for (int o = 16, n = N; o >= 1; o >>= 1) {
        if (n > 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < N / 2; ++i) {
                if (i < n / 2) {
                    const float send = up ? p[i] : p[i + n / 2], keep = up ? p[i + n / 2] : p[i];
                    p[i] = keep + __shfl_xor_sync(kFull, send, o);
                }
            }
            n >>= 1;
        } else {
            p[0] += __shfl_xor_sync(kFull, p[0], o);
        }
    }
    return p[0];
}

template <int NS, int MODE>
__global__ void __launch_bounds__(256) gather_pos_kernel(const PgArgs a) {
    constexpr int GU = 8 / NS, LG = __builtin_ctz(GU);
    constexpr bool DW = MODE != 0, ACC = MODE != 2;
    const int lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    pdl_wait();     // (launched as a programmatic dependent of the previous kernel)
    pdl_trigger();  // (a split-row reduction may follow as a programmatic dependent)
    if (p >= a.npos) return;
    const int r = __ldg(a.rowmap + p);
    if (r < 0) return;  // an unused position (no entries)
    const int64_t c0 = (int64_t)blockIdx.y * 128 * NS;
    bool cv[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) cv[s] = c0 + s * 128 + lane * 4 < a.B;  // (B % 4 == 0)
    float acc[NS][4], xr[NS][4];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[s][v] = xr[s][v] = 0.f;
    if constexpr (DW) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if (cv[s]) {
                const float4 t = __ldg(reinterpret_cast<const float4 *>(a.rin + (int64_t)r * a.B + c0 + s * 128 + lane * 4));
                xr[s][0] = t.x, xr[s][1] = t.y, xr[s][2] = t.z, xr[s][3] = t.w;
            }
    }
    const int e0 = __ldg(a.seg + p), e1 = __ldg(a.seg + p + 1);
    for (int ch = e0; ch < e1; ch += 32) {
        const int n = min(32, e1 - ch);
        const int2 el = lane < n ? __ldg(a.ent + ch + lane) : make_int2(-kTilRowBytes, 0);
        const int vl = (DW && lane < n) ? __ldg(a.vidx + ch + lane) : -1;
        for (int t = 0; t < n; t += GU) {
            float y[GU][NS][4], w[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {  // GU rows in flight before any FMA
                const int off = __shfl_sync(kFull, el.x, (t + u) & 31);
                w[u] = __shfl_sync(kFull, __int_as_float(el.y), (t + u) & 31);
                const bool ok = t + u < n && off >= 0;
                const float *row = a.gin + (int64_t)(ok ? off / kTilRowBytes : 0) * a.B + c0 + lane * 4;
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok && cv[s]) q = __ldg(reinterpret_cast<const float4 *>(row + s * 128));
                    y[u][s][0] = q.x, y[u][s][1] = q.y, y[u][s][2] = q.z, y[u][s][3] = q.w;
                }
            }
            float pd[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                pd[u] = 0.f;
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    if constexpr (ACC) fma_bcast<4>(acc[s], w[u], y[u][s]);
                    if constexpr (DW) pd[u] += dot_vec<4>(xr[s], y[u][s]);
                }
            }
            if constexpr (DW) {
                const float v = pg_reduce<GU>(pd, lane);
                const int u = (lane >> (5 - LG)) & (GU - 1);
                const int slot = __shfl_sync(kFull, vl, (t + u) & 31);
                if ((lane & ((32 >> LG) - 1)) == 0 && t + u < n && slot >= 0) a.dW[slot] = v;
            }
        }
    }
    if constexpr (ACC) {
        const int ps = a.split != nullptr ? __ldg(a.split + p) : -1;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (!cv[s]) continue;
            const int64_t col = c0 + s * 128 + lane * 4;
            float o[4] = {acc[s][0], acc[s][1], acc[s][2], acc[s][3]};
            if (ps >= 0) {  // a part row: raw sums (split_rows_reduce applies the epilogue)
                *reinterpret_cast<float4 *>(a.vpart + (int64_t)ps * a.B + col) = make_float4(o[0], o[1], o[2], o[3]);
                continue;
            }
            if (a.epi == EPI_RELU) {
#pragma unroll
                for (int v = 0; v < 4; ++v) o[v] = fmaxf(o[v], 0.f);
            } else if (a.epi == EPI_GATE) {
                const float4 g = __ldg(reinterpret_cast<const float4 *>(a.gate + (int64_t)r * a.B + col));
                o[0] = g.x > 0.f ? o[0] : 0.f;
                o[1] = g.y > 0.f ? o[1] : 0.f;
                o[2] = g.z > 0.f ? o[2] : 0.f;
                o[3] = g.w > 0.f ? o[3] : 0.f;
            }
            *reinterpret_cast<float4 *>(a.out + (int64_t)r * a.B + col) = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
}

}  // namespace

// Position-gather launch (MODE as gather_pos_kernel).  false: no gather tiling,
// B % 4 != 0, (MODE 0) B < 128 (the plain gather's narrower lanes serve those),
// or (MODE 1 / 2) more than 512 batch columns.
bool launch_gather_pos(const sp_weight_s *w, int orient, int mode, int64_t B, const float *gin, const float *rin,
                       const float *gate, int epi, float *out, float *dW, cudaStream_t st) {
#ifdef SP_NO_GATHER_POS
    return false;
#endif
    const sp_tiling &t = w->til_g[orient];
    if (t.ent == nullptr || (B & 3) != 0 || (mode == 0 && B < 128)) return false;
    const int64_t npos = (int64_t)t.nrb * t.RB;
    // MODE 0: a warp per (position, 128-column slice) while that fits one wave of
    // 64 warps per SM, else 256 columns per warp (e.g. Zipf part rows at 99 %: 1.2
    // waves of 128-column warps)
#ifndef SP_GPOS_NS0_WAVE
#define SP_GPOS_NS0_WAVE 64
#endif
    const int NS = mode == 0 ? ((B > 128 && npos * ((B + 127) / 128) > (int64_t)SP_GPOS_NS0_WAVE * num_sms()) ? 2 : 1)
                             : B <= 128 ? 1 : B <= 256 ? 2 : 4;
    if (mode != 0 && B > 128 * NS) return false;
    float *vpart = nullptr;
    const bool parts = mode == 0 && t.psplit_rows();
    if (parts && scratch_alloc((void **)&vpart, (size_t)t.nparts * B * sizeof(float), st) != cudaSuccess) return false;
    refresh_if_stale(w, t, st);
    PgArgs a{B, npos, t.seg, t.ent, t.vidx, t.rowmap, parts ? t.split : nullptr, gin, rin, gate, out, dW, vpart, epi};
    const dim3 grid((unsigned)((npos + 7) / 8), mode == 0 ? (unsigned)((B + 128 * NS - 1) / (128 * NS)) : 1u);
    if (mode == 0) {
        if (NS == 1) launch_pdl(gather_pos_kernel<1, 0>, grid, dim3(256), 0, st, a);
        else launch_pdl(gather_pos_kernel<2, 0>, grid, dim3(256), 0, st, a);
    }
    else if (mode == 1) {
        if (NS == 1) launch_pdl(gather_pos_kernel<1, 1>, grid, dim3(256), 0, st, a);
        else if (NS == 2) launch_pdl(gather_pos_kernel<2, 1>, grid, dim3(256), 0, st, a);
        else launch_pdl(gather_pos_kernel<4, 1>, grid, dim3(256), 0, st, a);
    } else {
        if (NS == 1) launch_pdl(gather_pos_kernel<1, 2>, grid, dim3(256), 0, st, a);
        else if (NS == 2) launch_pdl(gather_pos_kernel<2, 2>, grid, dim3(256), 0, st, a);
        else launch_pdl(gather_pos_kernel<4, 2>, grid, dim3(256), 0, st, a);
    }
    note_path(mode == 0 ? "spmm_gather_pos" : mode == 1 ? "bwd_gather_pos" : "sddmm_gather_pos");
    count_launches(1);
    if (parts) {
        launch_split_rows_reduce(t, vpart, B, out, gate, epi, st);
        scratch_free(vpart, st);
    }
    return true;
}

// Gather path wins when staging would move more bytes than gathering:
// nrb * inner (tile rows streamed per batch column) > nnz (rows gathered).
bool gather_preferred(const sp_weight_s *w, int orient, int64_t B, bool chunked) {
    // the gather SpMM walks a whole row per warp: skewed rows (Zipf) would
    // serialise the tail, so only balanced structures take it (the SDDMM's
    // 32-nonzero chunks are balanced by construction)
    const int64_t rows = orient == 0 ? w->R : w->C;
    const int64_t mx = orient == 0 ? w->max_row_nnz : w->max_col_nnz;
    // (the position gather walks skewed CSR rows as balanced part rows)
    const bool split_g = orient == 0 && w->til_g[0].ent != nullptr && w->til_g[0].psplit_rows() && B >= 128 &&
                         (B & 3) == 0;  // (launch_gather_pos's conditions)
    if (!chunked && !split_g && (double)mx > 4.0 * (double)w->nnz / (double)rows + 64.0) return false;
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
