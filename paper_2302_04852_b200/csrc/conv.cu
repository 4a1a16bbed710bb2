// conv.cu -- sparse-filter 2-D convolution, stride 1, CHWN (batch-last)
// layout (the paper's SparseConv layout, P293).  SURVEY §8(a) rows a-5..a-7.
//
// The filter [OC][IC][KH][KW] is the handle's R = OC x C = IC*KH*KW CSR
// (column (ic, x, y) = (ic*KH + x)*KW + y), so row oc lists exactly the
// stored taps of output channel oc in the paper's (oc, ic, x, y) order
// (P251).  Implicit im2col: each stored tap is visited directly; pruned taps
// cost nothing (P248).
//
//  fwd   (Eq. 3, P224):  warp per (oc, p, q-chunk), lanes over batch, VEC
//        batch elements per lane, QC output columns in registers.
//  dX    (Eq. 4, P231):  warp per (ic, m, n-chunk), gather over the CSC
//        column of every tap (x, y): no atomics.
//  dW    (Eq. 5, P240):  warp per (oc, 32 consecutive taps); dot products over
//        (p, q, b) with a warp transpose-reduce at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

struct Geo {
    int B, IC, H, W, OC, KH, KW, pad, OH, OW;
};

template <int VEC>
__device__ __forceinline__ void ldg_vec(const float *p, float (&v)[VEC], bool vec_ok, int nvalid) {
    if (vec_ok && nvalid == VEC) {
        if constexpr (VEC == 1) v[0] = __ldg(p);
        if constexpr (VEC == 2) {
            float2 t = __ldg(reinterpret_cast<const float2 *>(p));
            v[0] = t.x;
            v[1] = t.y;
        }
        if constexpr (VEC == 4) {
            float4 t = __ldg(reinterpret_cast<const float4 *>(p));
            v[0] = t.x;
            v[1] = t.y;
            v[2] = t.z;
            v[3] = t.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = e < nvalid ? __ldg(p + e) : 0.f;
    }
}

template <int VEC>
__device__ __forceinline__ void stg_vec(float *p, const float (&v)[VEC], bool vec_ok, int nvalid) {
    if (vec_ok && nvalid == VEC) {
        if constexpr (VEC == 1) *p = v[0];
        if constexpr (VEC == 2) *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
        if constexpr (VEC == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            if (e < nvalid) p[e] = v[e];
    }
}

// ---------------------------------------------------------------- forward
template <int VEC, int QC>
__global__ void __launch_bounds__(256)
    conv_fwd_kernel(Geo g, int nqc, const int32_t *__restrict__ row_ptr,
                    const int32_t *__restrict__ col_idx, const float *__restrict__ vals,
                    const float *__restrict__ X, float *__restrict__ Y) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nbc = (g.B + 32 * VEC - 1) / (32 * VEC);
    // warp -> (oc, p, q-chunk, b-chunk), b-chunk fastest
    int64_t t = wid;
    const int bc = (int)(t % nbc);
    t /= nbc;
    const int qc = (int)(t % nqc);
    t /= nqc;
    const int p = (int)(t % g.OH);
    const int oc = (int)(t / g.OH);
    if (oc >= g.OC) return;
    const int q0 = qc * QC;
    const int b = bc * 32 * VEC + lane * VEC;
    const int nvalid = min(VEC, max(0, g.B - b));
    const bool vec_ok = (g.B % VEC) == 0;
    const int KK = g.KH * g.KW;

    float acc[QC][VEC];
#pragma unroll
    for (int q = 0; q < QC; ++q)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[q][v] = 0.f;

    const int beg = __ldg(row_ptr + oc), end = __ldg(row_ptr + oc + 1);
    for (int j0 = beg; j0 < end; j0 += 32) {
        const int j = j0 + lane;
        const int cl = j < end ? __ldg(col_idx + j) : 0;
        const float wl = j < end ? __ldg(vals + j) : 0.f;
        const int n = min(32, end - j0);
        for (int s = 0; s < n; ++s) {
            const int c = __shfl_sync(kFull, cl, s);
            const float w = __shfl_sync(kFull, wl, s);
            const int ic = c / KK, rem = c - ic * KK;
            const int x = rem / g.KW, y = rem - x * g.KW;
            const int ih = p + x - g.pad;
            if (ih < 0 || ih >= g.H) continue;
            const float *src = X + ((int64_t)ic * g.H + ih) * g.W * g.B;
#pragma unroll
            for (int q = 0; q < QC; ++q) {
                const int iw = q0 + q + y - g.pad;
                if (q0 + q < g.OW && iw >= 0 && iw < g.W) {
                    float xv[VEC];
                    ldg_vec<VEC>(src + (int64_t)iw * g.B + b, xv, vec_ok, nvalid);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[q][v] = fmaf(w, xv[v], acc[q][v]);
                }
            }
        }
    }
    if (nvalid <= 0) return;
#pragma unroll
    for (int q = 0; q < QC; ++q) {
        if (q0 + q >= g.OW) break;
        stg_vec<VEC>(Y + (((int64_t)oc * g.OH + p) * g.OW + q0 + q) * g.B + b, acc[q], vec_ok, nvalid);
    }
}

// ---------------------------------------------------------------- dX
template <int VEC, int QC>
__global__ void __launch_bounds__(256)
    conv_dx_kernel(Geo g, int nqc, const int32_t *__restrict__ col_ptr,
                   const int32_t *__restrict__ row_idx, const int32_t *__restrict__ perm,
                   const float *__restrict__ vals, const float *__restrict__ dY,
                   float *__restrict__ dX) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nbc = (g.B + 32 * VEC - 1) / (32 * VEC);
    int64_t t = wid;
    const int bc = (int)(t % nbc);
    t /= nbc;
    const int qc = (int)(t % nqc);
    t /= nqc;
    const int m = (int)(t % g.H);
    const int ic = (int)(t / g.H);
    if (ic >= g.IC) return;
    const int n0 = qc * QC;
    const int b = bc * 32 * VEC + lane * VEC;
    const int nvalid = min(VEC, max(0, g.B - b));
    const bool vec_ok = (g.B % VEC) == 0;

    float acc[QC][VEC];
#pragma unroll
    for (int q = 0; q < QC; ++q)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[q][v] = 0.f;

    for (int x = 0; x < g.KH; ++x) {
        const int p = m + g.pad - x;
        if (p < 0 || p >= g.OH) continue;
        for (int y = 0; y < g.KW; ++y) {
            const int col = (ic * g.KH + x) * g.KW + y;
            const int beg = __ldg(col_ptr + col), end = __ldg(col_ptr + col + 1);
            for (int k0 = beg; k0 < end; k0 += 32) {
                const int k = k0 + lane;
                const int ocl = k < end ? __ldg(row_idx + k) : 0;
                const float wl = k < end ? __ldg(vals + __ldg(perm + k)) : 0.f;
                const int cnt = min(32, end - k0);
                for (int s = 0; s < cnt; ++s) {
                    const int oc = __shfl_sync(kFull, ocl, s);
                    const float w = __shfl_sync(kFull, wl, s);
                    const float *src = dY + ((int64_t)oc * g.OH + p) * g.OW * g.B;
#pragma unroll
                    for (int q = 0; q < QC; ++q) {
                        const int oq = n0 + q + g.pad - y;
                        if (n0 + q < g.W && oq >= 0 && oq < g.OW) {
                            float dv[VEC];
                            ldg_vec<VEC>(src + (int64_t)oq * g.B + b, dv, vec_ok, nvalid);
#pragma unroll
                            for (int v = 0; v < VEC; ++v) acc[q][v] = fmaf(w, dv[v], acc[q][v]);
                        }
                    }
                }
            }
        }
    }
    if (nvalid <= 0) return;
#pragma unroll
    for (int q = 0; q < QC; ++q) {
        if (n0 + q >= g.W) break;
        stg_vec<VEC>(dX + (((int64_t)ic * g.H + m) * g.W + n0 + q) * g.B + b, acc[q], vec_ok, nvalid);
    }
}

// ---------------------------------------------------------------- dW
template <int VEC>
__global__ void __launch_bounds__(256)
    conv_dw_kernel(Geo g, int groups_per_row, const int32_t *__restrict__ row_ptr,
                   const int32_t *__restrict__ col_idx, const float *__restrict__ X,
                   const float *__restrict__ dY, float *__restrict__ dW) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int oc = (int)(wid / groups_per_row);
    const int grp = (int)(wid % groups_per_row);
    if (oc >= g.OC) return;
    const int beg = __ldg(row_ptr + oc) + grp * 32, end = __ldg(row_ptr + oc + 1);
    if (beg >= end) return;
    const int n = min(32, end - beg);
    const int KK = g.KH * g.KW;
    const int c = lane < n ? __ldg(col_idx + beg + lane) : 0;
    const int ic_l = c / KK, rem = c - ic_l * KK;
    const int x_l = rem / g.KW, y_l = rem - (rem / g.KW) * g.KW;
    const bool vec_ok = (g.B % VEC) == 0;

    float acc[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) acc[t] = 0.f;

    for (int p = 0; p < g.OH; ++p) {
        for (int q = 0; q < g.OW; ++q) {
            const float *dsrc = dY + (((int64_t)oc * g.OH + p) * g.OW + q) * g.B;
            for (int b0 = 0; b0 < g.B; b0 += 32 * VEC) {
                const int b = b0 + lane * VEC;
                const int nvalid = min(VEC, max(0, g.B - b));
                float dv[VEC];
                ldg_vec<VEC>(dsrc + b, dv, vec_ok, nvalid);
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const int ic = __shfl_sync(kFull, ic_l, t);
                    const int ih = p + __shfl_sync(kFull, x_l, t) - g.pad;
                    const int iw = q + __shfl_sync(kFull, y_l, t) - g.pad;
                    if (t < n && ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) {
                        float xv[VEC];
                        ldg_vec<VEC>(X + (((int64_t)ic * g.H + ih) * g.W + iw) * g.B + b, xv,
                                     vec_ok, nvalid);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[t] = fmaf(dv[v], xv[v], acc[t]);
                    }
                }
            }
        }
    }
    const float s = transpose_reduce32(acc, lane);
    if (lane < n) dW[beg + lane] = s;
}

// dst[c][i][j][b] = src[c][i - top][j - left][b] (zero outside), B % 4 == 0
__global__ void pad_kernel(int64_t Cc, int Hs, int Ws, int Hd, int Wd, int top, int left, int64_t B4,
                           const float4 *__restrict__ src, float4 *__restrict__ dst) {
    const int64_t total = Cc * Hd * Wd * B4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i % B4;
        int64_t t = i / B4;
        const int j = (int)(t % Wd);
        t /= Wd;
        const int h = (int)(t % Hd);
        const int64_t c = t / Hd;
        const int hs = h - top, ws = j - left;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hs >= 0 && hs < Hs && ws >= 0 && ws < Ws) v = __ldg(src + ((c * Hs + hs) * Ws + ws) * B4 + b);
        dst[i] = v;
    }
}

void launch_pad(int64_t Cc, int Hs, int Ws, int Hd, int Wd, int top, int left, int64_t B, const float *src, float *dst,
                cudaStream_t st) {
    count_launches(1);
    pad_kernel<<<148 * 8, 256, 0, st>>>(Cc, Hs, Ws, Hd, Wd, top, left, B / 4, reinterpret_cast<const float4 *>(src),
                                        reinterpret_cast<float4 *>(dst));
}

// The tap-tiled path applies (handle built by sp_weight_create_conv, B % 4 == 0,
// pad <= K - 1 so the transposed conv's padding is non-negative).
bool tap_path(const sp_weight_s *w, const Geo &g) {
    return w->tapdev != nullptr && w->conv_kh == g.KH && w->conv_kw == g.KW && g.KH * g.KW <= kMaxTaps &&
           (g.B & 3) == 0 && g.pad <= g.KH - 1 && g.pad <= g.KW - 1;
}

Geo mk(const sp_conv_geom &c) {
    Geo g;
    g.B = c.B;
    g.IC = c.C_in;
    g.H = c.H;
    g.W = c.W;
    g.OC = c.C_out;
    g.KH = c.KH;
    g.KW = c.KW;
    g.pad = c.pad;
    g.OH = c.H + 2 * c.pad - c.KH + 1;
    g.OW = c.W + 2 * c.pad - c.KW + 1;
    return g;
}

constexpr int QC = 8;

// tap offsets of the exact-column path: fwd reads X at (p + x - pad, q + y - pad),
// dX (transposed conv, Eq. 4) reads dY at (m + pad - x, n + pad - y)
void conv_taps_offsets(const Geo &g, bool transposed, ConvCols &cc) {
    for (int x = 0; x < g.KH; ++x)
        for (int y = 0; y < g.KW; ++y) {
            const int t = x * g.KW + y;
            cc.dp[t] = (int8_t)(transposed ? g.pad - x : x - g.pad);
            cc.dq[t] = (int8_t)(transposed ? g.pad - y : y - g.pad);
        }
}

}  // namespace

bool conv_cols(int64_t B, int Po, int Qo, int64_t R, ConvCols *cc) {
    if ((B & 3) != 0 || B < 4) return false;
    ConvCols c{};
    if (B <= 128) {
        if (128 % B != 0) return false;
        c.bsh = __builtin_ctzll((unsigned long long)B);
        c.nq = (int)(128 / B);
        c.bpr = 1;
        c.spr = (Qo + c.nq - 1) / c.nq;
    } else {
        if (B % 128 != 0) return false;
        c.bsh = 7;
        c.nq = 1;
        c.bpr = (int)(B / 128);
        c.spr = Qo * c.bpr;
    }
    c.Po = Po;
    c.Qo = Qo;
    c.B = B;
    c.rowlen = (int64_t)Po * Qo * B;
    c.imgstride = 0;
    c.nslice = (int64_t)Po * c.spr;
    (void)R;
    *cc = c;
    return true;
}

bool conv_cols_nchw(int64_t B, int Po, int Qo, int64_t R, ConvCols *cc) {
    if ((Qo & 3) != 0 || B < 1) return false;
    // np x nq = 128 with nq a power of two >= 4: the tile shape wasting the
    // fewest lanes on the partial last row / column tiles of the image
    ConvCols c{};
    int64_t best = -1;
    for (int nq = 4; nq <= 128; nq *= 2) {
        const int np = 128 / nq;
        const int64_t cols = (int64_t)((Qo + nq - 1) / nq) * nq * ((Po + np - 1) / np) * np;
        if (best < 0 || cols < best) {
            best = cols;
            c.nq = nq;
            c.np = np;
        }
    }
    c.nchw = 1;
    c.qsh = __builtin_ctz((unsigned)c.nq);
    c.nqt = (Qo + c.nq - 1) / c.nq;
    c.npt = (Po + c.np - 1) / c.np;
    c.Po = Po;
    c.Qo = Qo;
    c.B = B;
    c.rowlen = (int64_t)Po * Qo;
    c.imgstride = R * Po * Qo;
    c.nslice = B * c.nqt * c.npt;
    *cc = c;
    return true;
}

void launch_conv_fwd(const sp_weight_s *w, const sp_conv_geom &cg, const float *X, float *Y,
                     cudaStream_t st) {
    const Geo g = mk(cg);
    ConvCols cc;
    if (tap_path(w, g) && conv_cols(g.B, g.OH, g.OW, g.OC, &cc)) {
        // Y[oc][p][q] = sum_taps W_xy . X[p + x - pad][q + y - pad]  (Eq. 3 by taps;
        // exact output positions, the halo zero-filled by the tensor map)
        conv_taps_offsets(g, false, cc);
        launch_refresh_taps(w, 0, g.KH * g.KW, st);
        if (launch_conv_spmm_sk(w, 0, cc, X, g.H, g.W, Y, g.KH * g.KW, st)) return;
    }
    if (tap_path(w, g)) {
        // fallback (batch sizes the exact slicing cannot cut): padded copy and
        // virtual columns, Y[oc] = sum_taps W_xy . shift_{(x*Wp + y)*B}(X_pad)
        const int Hp = g.H + 2 * g.pad, Wp = g.W + 2 * g.pad;
        const int64_t Lp = (int64_t)Hp * Wp * g.B;
        float *Xp = nullptr;
        if (scratch_alloc((void **)&Xp, (size_t)(g.IC * Lp) * sizeof(float), st) == cudaSuccess) {
            launch_pad(g.IC, g.H, g.W, Hp, Wp, g.pad, g.pad, g.B, X, Xp, st);
            int sh[kMaxTaps];
            for (int x = 0; x < g.KH; ++x)
                for (int y = 0; y < g.KW; ++y) sh[x * g.KW + y] = (x * Wp + y) * g.B;
            launch_refresh_taps(w, 0, g.KH * g.KW, st);
            const bool ok = launch_conv_spmm(w, 0, g.B, Xp, Lp, Y, sh, g.KH * g.KW, Wp, g.OH, g.OW, st);
            scratch_free(Xp, st);
            if (ok) return;
        }
    }
    const int nqc = (g.OW + QC - 1) / QC;
    auto go = [&](auto kern, int vec) {
        const int64_t nbc = (g.B + 32 * vec - 1) / (32 * vec);
        const int64_t warps = (int64_t)g.OC * g.OH * nqc * nbc;
        count_launches(1);
        note_path("conv_fwd_direct");
        kern<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(g, nqc, w->row_ptr, w->col_idx, w->vals, X, Y);
    };
    if (g.B <= 32) go(conv_fwd_kernel<1, QC>, 1);
    else if (g.B <= 64 || (g.B & 3)) go(conv_fwd_kernel<2, QC>, 2);
    else go(conv_fwd_kernel<4, QC>, 4);
}

void launch_conv_bwd_input(const sp_weight_s *w, const sp_conv_geom &cg, const float *dY, float *dX,
                           cudaStream_t st) {
    const Geo g = mk(cg);
    ConvCols cc;
    if (tap_path(w, g) && conv_cols(g.B, g.H, g.W, g.IC, &cc)) {
        // transposed conv by taps (Eq. 4): dX[ic][m][n] = sum_taps W_xy^T . dY[m + pad - x][n + pad - y]
        conv_taps_offsets(g, true, cc);
        launch_refresh_taps(w, 1, g.KH * g.KW, st);
        if (launch_conv_spmm_sk(w, 1, cc, dY, g.OH, g.OW, dX, g.KH * g.KW, st)) return;
    }
    if (tap_path(w, g)) {
        // fallback: transposed conv by taps on dY padded by K-1-pad, shifts (K-1-x, K-1-y)
        const int ph = g.KH - 1 - g.pad, pw = g.KW - 1 - g.pad;
        const int Hq = g.OH + 2 * ph, Wq = g.OW + 2 * pw;
        const int64_t Lq = (int64_t)Hq * Wq * g.B;
        float *Dp = nullptr;
        if (scratch_alloc((void **)&Dp, (size_t)(g.OC * Lq) * sizeof(float), st) == cudaSuccess) {
            launch_pad(g.OC, g.OH, g.OW, Hq, Wq, ph, pw, g.B, dY, Dp, st);
            int sh[kMaxTaps];
            for (int x = 0; x < g.KH; ++x)
                for (int y = 0; y < g.KW; ++y) sh[x * g.KW + y] = ((g.KH - 1 - x) * Wq + (g.KW - 1 - y)) * g.B;
            launch_refresh_taps(w, 1, g.KH * g.KW, st);
            const bool ok = launch_conv_spmm(w, 1, g.B, Dp, Lq, dX, sh, g.KH * g.KW, Wq, g.H, g.W, st);
            scratch_free(Dp, st);
            if (ok) return;
        }
    }
    const int nqc = (g.W + QC - 1) / QC;
    auto go = [&](auto kern, int vec) {
        const int64_t nbc = (g.B + 32 * vec - 1) / (32 * vec);
        const int64_t warps = (int64_t)g.IC * g.H * nqc * nbc;
        count_launches(1);
        note_path("conv_dx_direct");
        kern<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(g, nqc, w->col_ptr, w->row_idx, w->perm,
                                                          w->vals, dY, dX);
    };
    if (g.B <= 32) go(conv_dx_kernel<1, QC>, 1);
    else if (g.B <= 64 || (g.B & 3)) go(conv_dx_kernel<2, QC>, 2);
    else go(conv_dx_kernel<4, QC>, 4);
}

// Both conv backward products in one pass (Alg. 2's single pass by taps) on
// the exact dX positions; false when it does not apply (the caller falls back
// to the separate products).
static bool conv_bwd_sk(const sp_weight_s *w, const Geo &g, const float *X, const float *dY, float *dX, float *dW,
                        cudaStream_t st) {
    ConvCols cc;
    if (!tap_path(w, g) || !conv_cols(g.B, g.H, g.W, g.IC, &cc)) return false;
    conv_taps_offsets(g, true, cc);
    return launch_conv_bwd_sk(w, cc, dY, g.OH, g.OW, X, dX, dW, g.KH * g.KW, st);
}

sp_status launch_conv_bwd(const sp_weight_s *w, const sp_conv_geom &cg, const float *X, const float *dY, float *dX,
                          float *dW, cudaStream_t st) {
    const Geo g = mk(cg);
    if (w->nnz > 0 && conv_bwd_sk(w, g, X, dY, dX, dW, st)) return SP_OK;
    launch_conv_bwd_input(w, cg, dY, dX, st);
    return launch_conv_bwd_weight(w, cg, X, dY, dW, st);
}

sp_status launch_conv_bwd_weight(const sp_weight_s *w, const sp_conv_geom &cg, const float *X,
                                 const float *dY, float *dW, cudaStream_t st) {
    const Geo g = mk(cg);
    if (w->nnz == 0) return SP_OK;
    if (tap_path(w, g)) {
        // dW_xy = SDDMM over the virtual output space (Eq. 5 by taps): dY laid
        // out with row width Wp (zeros for q >= OW) against shifted X_pad
        const int Hp = g.H + 2 * g.pad, Wp = g.W + 2 * g.pad;
        const int64_t Lp = (int64_t)Hp * Wp * g.B, Lv = (int64_t)g.OH * Wp * g.B;
        float *Xp = nullptr, *Dv = nullptr;
        if (scratch_alloc((void **)&Xp, (size_t)(g.IC * Lp) * sizeof(float), st) == cudaSuccess &&
            scratch_alloc((void **)&Dv, (size_t)(g.OC * Lv) * sizeof(float), st) == cudaSuccess) {
            launch_pad(g.IC, g.H, g.W, Hp, Wp, g.pad, g.pad, g.B, X, Xp, st);
            launch_pad(g.OC, g.OH, g.OW, g.OH, Wp, 0, 0, g.B, dY, Dv, st);
            int sh[kMaxTaps];
            for (int x = 0; x < g.KH; ++x)
                for (int y = 0; y < g.KW; ++y) sh[x * g.KW + y] = (x * Wp + y) * g.B;
            const bool ok = launch_conv_sddmm(w, g.B, Dv, Xp, Lv, Lp, sh, g.KH * g.KW, dW, st);
            scratch_free(Xp, st);
            scratch_free(Dv, st);
            if (ok) return SP_OK;
        } else {
            if (Xp) scratch_free(Xp, st);
        }
    }
    const int gpr = (w->max_row_nnz + 31) / 32;
    const int64_t warps = (int64_t)g.OC * gpr;
    auto go = [&](auto kern) {
        count_launches(1);
        note_path("conv_dw_direct");
        kern<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(g, gpr, w->row_ptr, w->col_idx, X, dY, dW);
    };
    if (g.B <= 32) go(conv_dw_kernel<1>);
    else if (g.B <= 64 || (g.B & 3)) go(conv_dw_kernel<2>);
    else go(conv_dw_kernel<4>);
    return SP_OK;
}


// ---------------------------------------------------------------------------
// NCHW products: the paper's SparseConvOverON (natural B x C x H x W layout,
// vectorised over the output width, P293, P397-P400).  Same tap tilings and
// stream-K kernels as the CHWN path, with NCHW tensor maps: a slice is an
// np x nq spatial tile of one image and lanes run along the output rows.
// A TMA box may start anywhere in its outer dimensions, but its innermost
// start must be 16-byte aligned: here that is the width, so a tap's column
// shift dq must be a multiple of 4 -- in practice 1 x 1 filters with pad 0
// (the ResNet bottleneck convolutions).  Other shapes (wider filters, W or OW
// not a multiple of 4, direct-kernel filters) run the CHWN kernels -- whose
// slices already span (q, b) jointly, i.e. are vectorised over the output
// width when B is small -- on permuted copies.
namespace {

// dst = src permuted between [B][C][HW] (NCHW) and [C][HW][B] (CHWN)
__global__ void permute_kernel(int64_t B, int64_t C, int64_t HW, int to_chwn, const float *__restrict__ src,
                               float *__restrict__ dst) {
    const int64_t total = B * C * HW;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        if (to_chwn) {  // i = (c*HW + s)*B + b  <-  (b*C + c)*HW + s
            const int64_t b = i % B, t = i / B, sp = t % HW, c = t / HW;
            dst[i] = __ldg(src + (b * C + c) * HW + sp);
        } else {  // i = (b*C + c)*HW + s  <-  (c*HW + s)*B + b
            const int64_t sp = i % HW, t = i / HW, c = t % C, b = t / C;
            dst[i] = __ldg(src + (c * HW + sp) * B + b);
        }
    }
}

void launch_permute(int64_t B, int64_t C, int64_t HW, bool to_chwn, const float *src, float *dst, cudaStream_t st) {
    count_launches(1);
    note_path(to_chwn ? "permute_nchw_chwn" : "permute_chwn_nchw");
    permute_kernel<<<(unsigned)(num_sms() * 8), 256, 0, st>>>(B, C, HW, to_chwn ? 1 : 0, src, dst);
}

}  // namespace

sp_status launch_conv_nchw(const sp_weight_s *w, const sp_conv_geom &cg, int op, const float *X, const float *dY,
                           float *out, float *dW, cudaStream_t st) {
    const Geo g = mk(cg);
    const int ntap = g.KH * g.KW;
    ConvCols cc;
    bool aligned = true;  // every tap's width shift a multiple of 4 floats (16 bytes)
    for (int y = 0; y < g.KW; ++y) aligned = aligned && ((y - g.pad) & 3) == 0 && ((g.pad - y) & 3) == 0;
    // the tap path without its batch-vector condition (NCHW slices do not split the batch)
    const bool taps = w->tapdev != nullptr && w->conv_kh == g.KH && w->conv_kw == g.KW && ntap <= kMaxTaps &&
                      g.pad <= g.KH - 1 && g.pad <= g.KW - 1;
    if (taps && aligned && (g.W & 3) == 0 && (g.OW & 3) == 0 && w->nnz > 0) {
        if (op == 0 && conv_cols_nchw(g.B, g.OH, g.OW, g.OC, &cc)) {  // Y = conv(X)
            conv_taps_offsets(g, false, cc);
            launch_refresh_taps(w, 0, ntap, st);
            if (launch_conv_spmm_sk(w, 0, cc, X, g.H, g.W, out, ntap, st)) return SP_OK;
        } else if (op == 1 && conv_cols_nchw(g.B, g.H, g.W, g.IC, &cc)) {  // dX (Eq. 4)
            conv_taps_offsets(g, true, cc);
            launch_refresh_taps(w, 1, ntap, st);
            if (launch_conv_spmm_sk(w, 1, cc, dY, g.OH, g.OW, out, ntap, st)) return SP_OK;
        } else if ((op == 2 || op == 3) && conv_cols_nchw(g.B, g.H, g.W, g.IC, &cc)) {  // dX + dW / dW alone
            conv_taps_offsets(g, true, cc);
            if (launch_conv_bwd_sk(w, cc, dY, g.OH, g.OW, X, op == 2 ? out : nullptr, dW, ntap, st)) return SP_OK;
        }
    }
    // permuted fallback through the CHWN entry points
    const int64_t nx = (int64_t)g.B * g.IC * g.H * g.W, ny = (int64_t)g.B * g.OC * g.OH * g.OW;
    float *xc = nullptr, *yc = nullptr, *oc = nullptr;
    const bool need_x = op != 1, need_y = op != 0;
    const int64_t no = op == 0 ? ny : op == 3 ? 0 : nx;
    if ((need_x && scratch_alloc((void **)&xc, (size_t)nx * sizeof(float), st) != cudaSuccess) ||
        (need_y && scratch_alloc((void **)&yc, (size_t)ny * sizeof(float), st) != cudaSuccess) ||
        (no > 0 && scratch_alloc((void **)&oc, (size_t)no * sizeof(float), st) != cudaSuccess)) {
        if (xc) scratch_free(xc, st);
        if (yc) scratch_free(yc, st);
        set_error("sp_conv2d_*_nchw: scratch allocation failed");
        return SP_ERR_ALLOC;
    }
    if (need_x) launch_permute(g.B, g.IC, (int64_t)g.H * g.W, true, X, xc, st);
    if (need_y) launch_permute(g.B, g.OC, (int64_t)g.OH * g.OW, true, dY, yc, st);
    sp_status s = SP_OK;
    if (op == 0) launch_conv_fwd(w, cg, xc, oc, st);
    else if (op == 1) launch_conv_bwd_input(w, cg, yc, oc, st);
    else if (op == 2) s = launch_conv_bwd(w, cg, xc, yc, oc, dW, st);
    else s = launch_conv_bwd_weight(w, cg, xc, yc, dW, st);
    if (op == 0) launch_permute(g.B, g.OC, (int64_t)g.OH * g.OW, false, oc, out, st);
    else if (op != 3) launch_permute(g.B, g.IC, (int64_t)g.H * g.W, false, oc, out, st);
    if (xc) scratch_free(xc, st);
    if (yc) scratch_free(yc, st);
    if (oc) scratch_free(oc, st);
    return s;
}

}  // namespace sp
