// fused.cu -- fused CSC-driven linear backward: one pass
// over the nonzeros computes both backward products,
//   dX[c][b] = sum_{r in col c} w(r,c) * dY[r][b]      (Eq. 1, P143-P145)
//   dW(r,c)  = sum_b dY[r][b] * X[c][b]                (Eq. 2, P146-P148)
// which is the paper's Algorithm 1 "single pass" (P173, P187-P220: per
// nonzero, one fmadd updates dX and one accumulates the dW dot product) made
// atomic-free by driving it from the CSC copy: every dX row is owned by one
// warp and every dW entry by one lane of one CTA per batch split.
//
// Structure = the CSC tiling of the handle (rows = W columns c, inner = W
// rows r).  A CTA owns a row block of RB columns and a batch split; per slice
// of 128 batch columns it streams dY[r-block][slice] tiles (2-D TMA, double
// buffered) and holds X[c][slice] of its RPW rows in registers.  Per entry
// (r, w) one 16-byte LDS of dY[r][lane*4..] feeds BOTH 4 FMAs into the dX
// accumulator of row c and a 4-term partial dot into one of 32 register
// accumulators (dW), so the shared-memory traffic that bounds the separate
// kernels is paid once for 2x the FLOPs.  dW slice partials are reduced per
// row pair with one warp transpose-reduce and added into the split's partial
// buffer; dX is written (optionally gated by H > 0, the fused ReLU') at the
// end of each slice.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

struct FusedArgs {
    int64_t nrow, F, B;
    int KC, nkb, spl, cap;
    const int32_t *seg;
    const int2 *ent;
    const int32_t *vidx;
    const float *X;   // [nrow x B] register operand (layer input)
    const float *dY;  // [F x B] staged operand (output gradient)
    const float *H;   // [nrow x B] optional ReLU' gate for dX
    float *dX;        // [nrow x B]
    float *part;      // [nsplit x npad] or dW (direct)
    int64_t npad;
    int direct;
    const int32_t *rowmap;  // tiled position -> row of X / dX (-1 unused)
    int64_t nslice;         // stream-K kernel: batch slices of BT columns
    int nrow_blocks;        // stream-K kernel: row blocks of the tiling
    float *dxpart;          // stream-K kernel: [G][2][RB][BT] raw dX parts of cut items
    int *tickets;           // stream-K kernel: [nrow_blocks * nslice], zero on entry
    // stream-K kernel, conv (CONV = true): slices are exact dX positions (cc: rows
    // ic, output H x W); the register operand X [IC][H][W][B] is read at the same
    // positions (row stride xstride = H*W*B); an item's tiles run over (tap t,
    // column block) with taps[t]'s tiling and a 4-D TMA box of dY [OC][OH][OW][B]
    // offset by (dp[t], dq[t]) (halo zero-filled); dW partial index tapbase[t] + entry
    int64_t xstride;
    int ntap;
    const TapDev *taps;
    int64_t tapbase[kMaxTaps];
    ConvCols cc;
    // stream-K kernel: the tiling's group prefix table for this kernel's group
    // size (sp_tiling::gpre), nullptr: walk the earlier tiles' segment bounds
    const int32_t *gpre;
};

template <int RPW, int NW, bool GATE, bool SENT>
__global__ void __launch_bounds__(NW * 32, 1)
    bwd_fused_kernel(const FusedArgs a, const __grid_constant__ CUtensorMap tmap) {
    static_assert(RPW % 2 == 0, "rows are processed in pairs");
    constexpr int VEC = 4;
    constexpr int BT = 32 * VEC;
    constexpr int RB = NW * RPW;
    // [2][zero row + KC rows][BT] floats, then [2][cap+2] int2.  The zero row in
    // front of each tile is what padding entries (offset -one row) read.
    extern __shared__ __align__(128) float smem[];
    __shared__ uint64_t full[2];
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * (a.KC + 1) * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rb = blockIdx.x;
    const int64_t B = a.B;
    const int64_t s_lo = (int64_t)blockIdx.y * a.spl * BT;
    const int nsl = (int)std::min<int64_t>(a.spl, (B - s_lo + BT - 1) / BT);
    const int ntile = nsl * a.nkb;
    float *P = a.part + (a.direct ? 0 : (int64_t)blockIdx.y * a.npad);
    const size_t tile_sz = (size_t)a.KC * BT;  // TMA bytes per tile
    const size_t buf_sz = tile_sz + BT;         // zero row + tile
    const int ebuf = a.cap + 2;
    const int32_t *segw = a.seg + (int64_t)rb * a.nkb * RB + warp * RPW;
    const int64_t r_base = (int64_t)rb * RB + warp * RPW;

    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < BT; i += NW * 32) {
        smem[i] = 0.f;
        smem[buf_sz + i] = 0.f;
    }
    __syncthreads();
    auto entry_range = [&](int kb, int &e0, int &e1) {
        const int64_t tb = ((int64_t)rb * a.nkb + kb) * RB;
        e0 = __ldg(a.seg + tb) & ~1;
        e1 = __ldg(a.seg + tb + RB);
    };
    auto issue = [&](int q, int buf) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        int e0 = 0, e1 = 0;
        if constexpr (SENT) entry_range(kb, e0, e1);
        const unsigned eb = SENT ? (unsigned)(((e1 - e0) * 8 + 15) & ~15) : 0u;
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        tma_load_2d(smem + buf * buf_sz + BT, &tmap, (int)(s_lo + (int64_t)s * BT), kb * a.KC, &full[buf]);
        if (eb) tma_load_1d(ents + buf * ebuf, a.ent + e0, eb, &full[buf]);
    };
    if (threadIdx.x == 0) issue(0, 0);

    float rv[RPW][VEC], dx[RPW][VEC];
    for (int q = 0; q < ntile; ++q) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        const int buf = q & 1;
        const int64_t bl = s_lo + (int64_t)s * BT + lane * VEC;
        if (kb == 0) {  // new slice: X rows into registers, dX accumulators reset
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = __ldg(a.rowmap + r_base + i);
                const float4 t = (r >= 0 && r < a.nrow && bl + 4 <= B)
                                     ? __ldg(reinterpret_cast<const float4 *>(a.X + r * B + bl))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                rv[i][0] = t.x;
                rv[i][1] = t.y;
                rv[i][2] = t.z;
                rv[i][3] = t.w;
#pragma unroll
                for (int v = 0; v < VEC; ++v) dx[i][v] = 0.f;
            }
        }
        const int sg = lane <= RPW ? __ldg(segw + (int64_t)kb * RB + lane) : 0;
        if (q + 1 < ntile && threadIdx.x == 0) issue(q + 1, buf ^ 1);
        mbar_wait(&full[buf], (q >> 1) & 1);
        int ea = 0;
        if constexpr (SENT) {
            int e1;
            entry_range(kb, ea, e1);
        }
        const char *tb = reinterpret_cast<const char *>(smem + buf * buf_sz + BT + lane * VEC);
        const int2 *es = SENT ? ents + buf * ebuf - ea : a.ent;
#pragma unroll
        for (int m = 0; m < RPW; m += 2) {
            int pa = __shfl_sync(kFull, sg, m);
            const int a1 = __shfl_sync(kFull, sg, m + 1);
            int pb = a1;
            const int b1 = __shfl_sync(kFull, sg, m + 2);
            while (pa < a1 || pb < b1) {
                const int na = min(16, a1 - pa), nb = min(16, b1 - pb);  // even
                float acc[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u] = 0.f;
#pragma unroll
                for (int gq = 0; gq < 16; gq += 4) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // h = 0: row m (entries pa..), 1: row m+1 (pb..)
                        if (gq < (h ? nb : na)) {
                            const int e = (h ? pb : pa) + gq;
                            const int4 p01 = ld_entry_pair(SENT ? es + e : a.ent + e, SENT);
                            const int4 p23 = ld_entry_pair(SENT ? es + e + 2 : a.ent + e + 2, SENT);
                            // a second pair past the segment reads the zero row with weight 0
                            const bool h2 = gq + 2 < (h ? nb : na);
                            const int off[4] = {p01.x, p01.z, h2 ? p23.x : -kTilRowBytes, h2 ? p23.z : -kTilRowBytes};
                            const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w),
                                                h2 ? __int_as_float(p23.y) : 0.f, h2 ? __int_as_float(p23.w) : 0.f};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                // padding entries read the zero row (x = 0 exactly, so
                                // non-finite activations cannot leak into other rows)
                                float x[VEC];
                                lds_vec<VEC>(reinterpret_cast<const float *>(tb + off[u]), x);
                                fma_bcast<VEC>(dx[m + h], w[u], x);           // dX  (Eq. 1)
                                acc[16 * h + gq + u] = dot_vec<VEC>(rv[m + h], x);  // dW  (Eq. 2)
                            }
                        }
                    }
                }
                const float sum = transpose_reduce32(acc, lane);
                const int u = lane & 15;
                if (lane < 16 ? u < na : u < nb) {
                    const int e = (lane < 16 ? pa : pb) + u;
                    if (a.direct) {
                        const int v = __ldg(a.vidx + e);
                        if (v >= 0) P[v] = (s == 0) ? sum : P[v] + sum;
                    } else {
                        P[e] = (s == 0) ? sum : P[e] + sum;
                    }
                }
                pa += na;
                pb += nb;
            }
        }
        if (kb == a.nkb - 1) {  // slice done: dX rows (ReLU' gate fused)
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = __ldg(a.rowmap + r_base + i);
                if (r < 0 || r >= a.nrow || bl >= B) continue;
                float o[VEC];
                if (GATE) {
                    const float4 hv = __ldg(reinterpret_cast<const float4 *>(a.H + r * B + bl));
                    o[0] = hv.x > 0.f ? dx[i][0] : 0.f;
                    o[1] = hv.y > 0.f ? dx[i][1] : 0.f;
                    o[2] = hv.z > 0.f ? dx[i][2] : 0.f;
                    o[3] = hv.w > 0.f ? dx[i][3] : 0.f;
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) o[v] = dx[i][v];
                }
                *reinterpret_cast<float4 *>(a.dX + r * B + bl) = make_float4(o[0], o[1], o[2], o[3]);
            }
        }
        __syncthreads();  // buffer free before it is refilled
    }
}

// ---- TMEM variant ----------------------------------------------------------
// Same pass, two changes that cut the per-entry instruction count:
//  * no static slot layout: every row walks its (padded) segment in groups of
//    4 entries, and each group's 4 dW partials are reduced across the warp on
//    the spot (transpose stages xor 16 / xor 8, then xor 4/2/1: 6 SHFL, 6 SEL,
//    6 FADD for 4 entries), so short segments waste nothing in the reduction;
//  * the per-entry dW sums of successive batch slices accumulate in tensor
//    memory instead of a global read-modify-write: group g of the warp's
//    per-slice sequence lands in TMEM column g/8, lane 8*u + g%8 (u = entry in
//    the group), so every column holds 32 entries and one 32x32b access per 8
//    groups updates them.  The sequence is identical in every slice, and at
//    the end the warp replays it to write each total to dW (or its split's
//    partial row).  Warp w owns TMEM lanes 32*(w%4).. and columns
//    (w/4)*128..+128, i.e. at most 4096 padded entries per warp.
__device__ __forceinline__ void tm_st1(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v))
                 : "memory");
}
__device__ __forceinline__ float tm_ld1(uint32_t taddr) {
    uint32_t r;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r)
        : "r"(taddr)
        : "memory");
    return __uint_as_float(r);
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 4 per-lane partials p[u] (entries u of a group) -> lane l holds the warp
// sum for entry (l >> 3) & 3.  Fixed order: bitwise reproducible.
__device__ __forceinline__ float reduce4(const float (&p)[4], int lane) {
    const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
    const float sa = h16 ? p[0] : p[2], sb = h16 ? p[1] : p[3];
    const float ka = h16 ? p[2] : p[0], kb = h16 ? p[3] : p[1];
    const float ra = ka + __shfl_xor_sync(kFull, sa, 16);
    const float rb = kb + __shfl_xor_sync(kFull, sb, 16);
    const float s8 = h8 ? ra : rb, k8 = h8 ? rb : ra;
    float v = k8 + __shfl_xor_sync(kFull, s8, 8);
    v += __shfl_xor_sync(kFull, v, 4);
    v += __shfl_xor_sync(kFull, v, 2);
    v += __shfl_xor_sync(kFull, v, 1);
    return v;
}

// TMEM columns per warp: the NW/4 warps of a lane quarter share its 512 columns
template <int NW>
constexpr int tm_cols() { return 512 / (NW / 4); }

template <int RPW, int NW, bool GATE>
__global__ void __launch_bounds__(NW * 32, 1)
    bwd_fused_tm_kernel(const FusedArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int VEC = 4;
    constexpr int BT = 32 * VEC;
    constexpr int RB = NW * RPW;
    static_assert(NW % 4 == 0, "whole TMEM lane quarters");
    constexpr int kTmCols = tm_cols<NW>();
    extern __shared__ __align__(128) float smem[];
    __shared__ uint64_t full[2];
    __shared__ int released[2];  // warps done with each buffer (the last one refills it)
    __shared__ uint32_t tmem_base;
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * (a.KC + 1) * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rb = blockIdx.x;
    const int64_t B = a.B;
    const int64_t s_lo = (int64_t)blockIdx.y * a.spl * BT;
    const int nsl = (int)std::min<int64_t>(a.spl, (B - s_lo + BT - 1) / BT);
    const int ntile = nsl * a.nkb;
    const size_t tile_sz = (size_t)a.KC * BT;
    const size_t buf_sz = tile_sz + BT;
    const int ebuf = a.cap + 2;
    const int32_t *segw = a.seg + (int64_t)rb * a.nkb * RB + warp * RPW;
    const int64_t r_base = (int64_t)rb * RB + warp * RPW;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        released[0] = 0;
        released[1] = 0;
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < BT; i += NW * 32) {
        smem[i] = 0.f;
        smem[buf_sz + i] = 0.f;
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tcol = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kTmCols);

    auto entry_range = [&](int kb, int &e0, int &e1) {
        const int64_t tb = ((int64_t)rb * a.nkb + kb) * RB;
        e0 = __ldg(a.seg + tb) & ~1;
        e1 = __ldg(a.seg + tb + RB);
    };
    auto issue = [&](int q, int buf) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        int e0, e1;
        entry_range(kb, e0, e1);
        const unsigned eb = (unsigned)(((e1 - e0) * 8 + 15) & ~15);
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        tma_load_2d(smem + buf * buf_sz + BT, &tmap, (int)(s_lo + (int64_t)s * BT), kb * a.KC, &full[buf]);
        if (eb) tma_load_1d(ents + buf * ebuf, a.ent + e0, eb, &full[buf]);
    };
    if (threadIdx.x == 0) {
        if (ntile > 0) issue(0, 0);
        if (ntile > 1) issue(1, 1);
    }

    float rv[RPW][VEC], dx[RPW][VEC];
    float keep = 0.f;
    int cnt = 0;
    // lane l <= RPW: l-th segment bound of this warp's rows in tile q (prefetched one tile ahead)
    auto seg_bounds = [&](int q) -> int {
        const int kb = q % a.nkb;
        return lane <= RPW ? __ldg(segw + (int64_t)kb * RB + lane) : 0;
    };
    int sgn = ntile > 0 ? seg_bounds(0) : 0;
    for (int q = 0; q < ntile; ++q) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        const int buf = q & 1;
        const int64_t bl = s_lo + (int64_t)s * BT + lane * VEC;
        if (kb == 0) {  // new slice: X rows into registers, dX accumulators reset
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = __ldg(a.rowmap + r_base + i);
                const float4 t = (r >= 0 && r < a.nrow && bl + 4 <= B)
                                     ? __ldg(reinterpret_cast<const float4 *>(a.X + r * B + bl))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                rv[i][0] = t.x;
                rv[i][1] = t.y;
                rv[i][2] = t.z;
                rv[i][3] = t.w;
#pragma unroll
                for (int v = 0; v < VEC; ++v) dx[i][v] = 0.f;
            }
            cnt = 0;
        }
        const int sg = sgn;
        if (q + 1 < ntile) sgn = seg_bounds(q + 1);
        mbar_wait(&full[buf], (q >> 1) & 1);
        int ea, e1t;
        entry_range(kb, ea, e1t);
        const char *tb = reinterpret_cast<const char *>(smem + buf * buf_sz + BT + lane * VEC);
        const int2 *es = ents + buf * ebuf - ea;
        auto flush = [&](int col) {
            const uint32_t ta = tcol + (uint32_t)col;
            if (s == 0) {
                tm_st1(ta, keep);
            } else {
                const float old = tm_ld1(ta);
                tm_st1(ta, old + keep);
            }
            keep = 0.f;
        };
#pragma unroll
        for (int m = 0; m < RPW; ++m) {
            const int g0 = __shfl_sync(kFull, sg, m), g1 = __shfl_sync(kFull, sg, m + 1);
            for (int e = g0; e < g1; e += 4) {
                const int4 p01 = ld_entry_pair(es + e, true);
                const int4 p23 = ld_entry_pair(es + e + 2, true);
                const int off[4] = {p01.x, p01.z, p23.x, p23.z};
                const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w), __int_as_float(p23.y),
                                    __int_as_float(p23.w)};
                float p[4] = {0.f, 0.f, 0.f, 0.f};
                // padding entries read the zero row in front of the tile; a second pair
                // past the segment (length 2 mod 4) is skipped
                auto entry = [&](int u) {
                    float x[VEC];
                    lds_vec<VEC>(reinterpret_cast<const float *>(tb + off[u]), x);
                    fma_bcast<VEC>(dx[m], w[u], x);   // dX  (Eq. 1)
                    p[u] = dot_vec<VEC>(rv[m], x);    // dW partial (Eq. 2)
                };
                if (e + 2 < g1) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) entry(u);
                } else {
                    entry(0);
                    entry(1);
                }
                const float v = reduce4(p, lane);
                if ((lane & 7) == (cnt & 7)) keep = v;
                ++cnt;
                if ((cnt & 7) == 0) flush((cnt >> 3) - 1);
            }
        }
        if (kb == a.nkb - 1) {  // slice done: last partial column, dX rows (ReLU' gate fused)
            if (cnt & 7) flush(cnt >> 3);
            tm_wait_st();
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = __ldg(a.rowmap + r_base + i);
                if (r < 0 || r >= a.nrow || bl >= B) continue;
                float o[VEC];
                if (GATE) {
                    const float4 hv = __ldg(reinterpret_cast<const float4 *>(a.H + r * B + bl));
                    o[0] = hv.x > 0.f ? dx[i][0] : 0.f;
                    o[1] = hv.y > 0.f ? dx[i][1] : 0.f;
                    o[2] = hv.z > 0.f ? dx[i][2] : 0.f;
                    o[3] = hv.w > 0.f ? dx[i][3] : 0.f;
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) o[v] = dx[i][v];
                }
                *reinterpret_cast<float4 *>(a.dX + r * B + bl) = make_float4(o[0], o[1], o[2], o[3]);
            }
        }
        // release the buffer; the last warp to finish tile q refills it with tile q+2
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&released[buf], 1) == NW - 1) {
                released[buf] = 0;
                __threadfence_block();
                if (q + 2 < ntile) issue(q + 2, buf);
            }
        }
    }

    // replay one slice's group sequence: TMEM (column, lane) -> entry, write totals
    if (nsl > 0) {
        float *P = a.part + (a.direct ? 0 : (int64_t)blockIdx.y * a.npad);
        int c2 = 0, my_e = -1;
        auto out = [&](int col) {
            const float val = tm_ld1(tcol + (uint32_t)col);
            if (my_e >= 0) {
                if (a.direct) {
                    const int v = __ldg(a.vidx + my_e);
                    if (v >= 0) P[v] = val;
                } else {
                    P[my_e] = val;
                }
            }
            my_e = -1;
        };
        for (int kb = 0; kb < a.nkb; ++kb) {
            const int sg = lane <= RPW ? __ldg(segw + (int64_t)kb * RB + lane) : 0;
            for (int m = 0; m < RPW; ++m) {
                const int g0 = __shfl_sync(kFull, sg, m), g1 = __shfl_sync(kFull, sg, m + 1);
                for (int e = g0; e < g1; e += 4) {
                    const int u = (lane >> 3) & 3;
                    if ((lane & 7) == (c2 & 7)) my_e = u < g1 - e ? e + u : -1;
                    ++c2;
                    if ((c2 & 7) == 0) out((c2 >> 3) - 1);
                }
            }
        }
        if (c2 & 7) out(c2 >> 3);
    }
    tm_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
}

// ---- stream-K schedule ------------------------------------------------------
// The work is the tile sequence (row block rb, batch slice sl, column block kb),
// rb-major, T = nrb * nslice * nkb tiles; CTA c of G runs the contiguous range
// [c*T/G, (c+1)*T/G), so every SM gets the same number of tiles (+-1) instead
// of a whole number of slices.  An item (rb, sl) cut by range boundaries is
// shared by the CTAs whose ranges cover it: each stores its raw dX part, and
// the last to arrive (an integer ticket per item) adds the parts in CTA order,
// gates and stores -- a fixed order, so the result is deterministic.  A job is
// one CTA's run of tiles of one row block: its dW sums (TMEM, as above) go to
// row (c - first CTA of rb) of the partial buffer, summed per entry in fixed
// order by job_reduce_kernel.
__host__ __device__ __forceinline__ int64_t sk_lo(int64_t c, int64_t T, int64_t G) { return c * T / G; }
constexpr int kMaxJobTab = 1024;  // job_reduce_kernel's table of CTA range starts
__host__ __device__ __forceinline__ int64_t sk_cta(int64_t t, int64_t T, int64_t G) {
    int64_t c = t * G / T;
    while (c + 1 < G && sk_lo(c + 1, T, G) <= t) ++c;
    while (c > 0 && sk_lo(c, T, G) > t) --c;
    return c;
}

__device__ __forceinline__ void tm_st4(uint32_t taddr, const float (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(__float_as_uint(v[0])),
                 "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3]))
                 : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r0, r1, r2, r3;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "r"(taddr)
        : "memory");
    v[0] = __uint_as_float(r0);
    v[1] = __uint_as_float(r1);
    v[2] = __uint_as_float(r2);
    v[3] = __uint_as_float(r3);
}
__device__ __forceinline__ void tm_ld4x2(uint32_t ta, float (&v)[4], uint32_t tb, float (&w)[4]) {
    uint32_t r0, r1, r2, r3, q0, q1, q2, q3;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%8];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%9];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(q0), "=r"(q1), "=r"(q2), "=r"(q3)
        : "r"(ta), "r"(tb)
        : "memory");
    v[0] = __uint_as_float(r0);
    v[1] = __uint_as_float(r1);
    v[2] = __uint_as_float(r2);
    v[3] = __uint_as_float(r3);
    w[0] = __uint_as_float(q0);
    w[1] = __uint_as_float(q1);
    w[2] = __uint_as_float(q2);
    w[3] = __uint_as_float(q3);
}

__device__ __forceinline__ void tm_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tm_ld8x2(uint32_t ta, float (&v)[8], uint32_t tb, float (&w)[8]) {
    uint32_t r[8], q[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%16];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%17];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
        : "r"(ta), "r"(tb)
        : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = __uint_as_float(r[i]);
        w[i] = __uint_as_float(q[i]);
    }
}
// Half-warp reduce4: 4 per-lane partials of each half-warp's own 4 entries ->
// lane 16h + l holds the 16-lane sum for entry (l >> 2) & 3 of half h
// (transpose stages xor 8 / xor 4, then xor 2/1: 5 SHFL for 8 entries).
__device__ __forceinline__ float reduce4h(const float (&p)[4], int lane) {
    const bool h8 = (lane & 8) != 0, h4 = (lane & 4) != 0;
    const float sa = h8 ? p[0] : p[2], sb = h8 ? p[1] : p[3];
    const float ka = h8 ? p[2] : p[0], kb = h8 ? p[3] : p[1];
    const float ra = ka + __shfl_xor_sync(kFull, sa, 8);
    const float rb = kb + __shfl_xor_sync(kFull, sb, 8);
    const float s4 = h4 ? ra : rb, k4 = h4 ? rb : ra;
    float v = k4 + __shfl_xor_sync(kFull, s4, 4);
    v += __shfl_xor_sync(kFull, v, 2);
    v += __shfl_xor_sync(kFull, v, 1);
    return v;
}

// TMEM columns of one warp (32 warps: 8 per lane quarter, 64 columns each):
// [0, 4*RPW) the X rows of its RPW rows (the dW register operand), [4*RPW,
// 8*RPW) their dX accumulators, the rest dW sums (8 groups of 4 entries per
// column).  Keeping the per-row state in TMEM (loaded per row segment) frees
// the registers that 32 resident warps need.  RPW = 4 (128-row blocks) for
// linear layers: 32 dW columns (256 groups); RPW = 2 (64-row blocks) for the
// fused conv backward: 48 columns.  DWONLY drops the dX columns.
// TMEM columns per warp: the NW/4 warps of a lane quarter share its 512 columns
template <int NW>
constexpr int sk_cpw() { return (512 / (NW / 4)) & ~7; }
// HALF: half-warp entries (8 columns per row for the X row and the dX accumulator)
template <int RPW, bool DWONLY, bool HALF = false>
constexpr int sk_dw0() { return (DWONLY ? 1 : 2) * RPW * (HALF ? 8 : 4); }
template <int RPW, bool DWONLY, int NW = 32, bool HALF = false>
constexpr int sk_dwcols() { return sk_cpw<NW>() - sk_dw0<RPW, DWONLY, HALF>(); }

#ifdef SP_FUSED_TS
// (measurement build only: tools/dbg/fused_ts.py) per-CTA %globaltimer stamps of
// the last fused launch: [cta][0] entry, [1] first tile ready, [2] main loop done, [3] exit
__device__ unsigned long long g_fused_ts[1024][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FUSED_TS(k) \
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_fused_ts[blockIdx.x][k] = gtimer()
#else
#define FUSED_TS(k)
#endif
template <int RPW, int NW, bool GATE, bool DWONLY, int NBUF, bool CONV, bool HALF = false>
__global__ void __launch_bounds__(NW * 32, 1)
    bwd_fused_sk_kernel(const FusedArgs a, const __grid_constant__ CUtensorMap tmap) {
    FUSED_TS(0);
    constexpr int VEC = 4;
    constexpr int SW = HALF ? 8 : 4;  // TMEM columns per row (X row, dX accumulator)
    constexpr int RV0 = 0, DX0 = SW * RPW, DW0 = sk_dw0<RPW, DWONLY, HALF>(), DWC = sk_dwcols<RPW, DWONLY, NW, HALF>();
    // entry groups: GE entries (4: one per warp quarter-sweep; HALF: 8, 4 per half-warp),
    // 2^GSH groups per TMEM dW column (32 lanes = GE entries x copies)
    constexpr int GE = HALF ? 8 : 4, GL = HALF ? 3 : 2, GSH = HALF ? 2 : 3, GM = (1 << GSH) - 1;
    constexpr int BT = 32 * VEC;
    constexpr int RB = NW * RPW;
    static_assert(NW % 4 == 0 && NW <= 32 && (RPW == 4 || RPW == 2 || RPW == 1), "TMEM column plan: whole lane quarters");
    extern __shared__ __align__(128) float smem[];
    __shared__ uint64_t full[NBUF];
    __shared__ int released[NBUF];  // warps done with each buffer (the last one refills it)
#ifndef SP_FUSED_EA_LDG
    __shared__ int tile_ea[NBUF];   // first (staged) entry of the tile in each buffer, set by its issuer
#endif
    __shared__ uint32_t tmem_base;
    __shared__ int last_flag;
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)NBUF * (a.KC + 1) * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tpi = CONV ? a.ntap * a.nkb : a.nkb;  // tiles per item
    const int64_t T = (int64_t)a.nrow_blocks * a.nslice * tpi, G = gridDim.x;
    const int t0 = (int)sk_lo(blockIdx.x, T, G);  // T < 2^31 (checked by the launcher)
    const int first_item = t0 / tpi;
    const int ntile = (int)sk_lo(blockIdx.x + 1, T, G) - t0;
    const int nsl = (int)a.nslice;
    const size_t tile_sz = (size_t)a.KC * BT;
    const size_t buf_sz = tile_sz + BT;
    const int ebuf = a.cap + 2;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            released[b] = 0;
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < NBUF * BT; i += NW * 32) smem[(i / BT) * buf_sz + i % BT] = 0.f;  // zero rows
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const uint32_t tcol = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * sk_cpw<NW>());

    struct Tile {
        int rb, sl, r;  // r: tile within the item (tap * nkb + kb for conv)
    };
    auto tap_of = [&](int r) { return CONV ? r / a.nkb : 0; };
    auto kb_of = [&](int r) { return CONV ? r - (r / a.nkb) * a.nkb : r; };
    auto seg_of = [&](int r) -> const int32_t * { return CONV ? a.taps[tap_of(r)].seg : a.seg; };
    auto tile_of = [&](int q) -> Tile {  // 32-bit: used for the first tile and the refills
        const int t = t0 + q, it = t / tpi;
        Tile id;
        id.r = t - it * tpi;
        id.rb = it / nsl;
        id.sl = it - id.rb * nsl;
        return id;
    };
    auto next_tile = [&](Tile id) -> Tile {
        if (++id.r == tpi) {
            id.r = 0;
            if (++id.sl == nsl) {
                id.sl = 0;
                ++id.rb;
            }
        }
        return id;
    };
    auto entry_range = [&](const Tile &id, int &e0, int &e1) {
        const int64_t tb = ((int64_t)id.rb * a.nkb + kb_of(id.r)) * RB;
        const int32_t *sgp = seg_of(id.r);
        e0 = __ldg(sgp + tb) & ~1;
        e1 = __ldg(sgp + tb + RB);
    };
    auto issue = [&](int q, int buf) {
        const Tile id = tile_of(q);
        int e0, e1;
        entry_range(id, e0, e1);
        const unsigned eb = (unsigned)(((e1 - e0) * 8 + 15) & ~15);
        const int2 *ent = CONV ? a.taps[tap_of(id.r)].ent : a.ent;
#ifndef SP_FUSED_EA_LDG
        tile_ea[buf] = e0;  // published to the consumers by the arrive below (release)
#endif
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        if constexpr (CONV) {
            int c[4];
            cc_coords(a.cc, id.sl, tap_of(id.r), kb_of(id.r) * a.KC, c);
            tma_load_4d(smem + buf * buf_sz + BT, &tmap, c[0], c[1], c[2], c[3], &full[buf]);
        } else {
            tma_load_2d(smem + buf * buf_sz + BT, &tmap, id.sl * BT, kb_of(id.r) * a.KC, &full[buf]);
        }
        if (eb) tma_load_1d(ents + buf * ebuf, ent + e0, eb, &full[buf]);
    };
    pdl_wait();  // (launched as a programmatic dependent: the prologue above overlapped the previous kernel)
    if (threadIdx.x == 0)
        for (int b = 0; b < NBUF && b < ntile; ++b) issue(b, b);
    // the job reduction that follows (programmatic dependent launch) may start its
    // CTAs -- and their job search -- on SMs this one-wave grid frees; it waits for
    // this grid's completion before reading the partial rows
    pdl_trigger();
    // this warp's segment bounds of (rb, tile r): lane l <= RPW holds the l-th
    auto segw_of = [&](int rb, int r) -> const int32_t * {
        return seg_of(r) + ((int64_t)rb * a.nkb + kb_of(r)) * RB + warp * RPW;
    };
    auto seg_bounds = [&](const Tile &id) -> int {
        return lane <= RPW ? __ldg(segw_of(id.rb, id.r) + lane) : 0;
    };

    // tile r of an item is touched by the job running item-local tiles
    // [ja, ja + len) of its row block (ra = ja % tpi)
    auto touched = [&](int r, int ra, int len) -> bool {
        int d = r - ra;
        if (d < 0) d += tpi;
        return len >= tpi || d < len;
    };
    // write this job's dW sums (row block rb, local tiles [ja, ja + len)); tiles the
    // job never touched are skipped (job_reduce_kernel skips them too)
    auto dump = [&](int rb, int ja, int len) {
        const int64_t job = blockIdx.x - sk_cta((int64_t)rb * a.nslice * tpi, T, G);
        float *P = a.part + job * a.npad;
        int c2 = 0, my_e = -1;
        const int ra = ja % tpi;
        auto out = [&](int col) {
            const float val = tm_ld1(tcol + DW0 + (uint32_t)col);
            if (my_e >= 0) P[my_e] = val;
            my_e = -1;
        };
        // the groups of touched tile r (c2 = its first group's index in the item)
        auto walk = [&](int r) {
            const int sg = lane <= RPW ? __ldg(segw_of(rb, r) + lane) : 0;
            const int64_t base = CONV ? a.tapbase[tap_of(r)] : 0;
            for (int m = 0; m < RPW; ++m) {
                const int g0 = __shfl_sync(kFull, sg, m), g1 = __shfl_sync(kFull, sg, m + 1);
                for (int e = g0; e < g1; e += GE) {
                    const int u = HALF ? (lane >> 2) & 3 : (lane >> 3) & 3;
                    const int idx = HALF ? 2 * u + (lane >> 4) : u;  // entry in the group
                    if ((lane & GM) == (c2 & GM)) my_e = idx < g1 - e ? (int)(base + e + idx) : -1;
                    ++c2;
                    if ((c2 & GM) == 0) out((c2 >> GSH) - 1);
                }
            }
        };
        if (a.gpre != nullptr) {
            // only the touched tiles: one or two (cyclic) runs of consecutive tiles,
            // each starting at its first group's column from the prefix table
            const int32_t *gp = a.gpre + ((int64_t)rb * NW + warp) * (tpi + 1);
            const int n1 = len >= tpi ? tpi - ra : min(len, tpi - ra);
            const int n2 = len >= tpi ? ra : len - n1;
            c2 = __ldg(gp + ra);
            for (int r = ra; r < ra + n1; ++r) walk(r);
            if (c2 & GM) out(c2 >> GSH);
            if (n2 > 0) {
                c2 = __ldg(gp);
                for (int r = 0; r < n2; ++r) walk(r);
            }
        } else {
        for (int r = 0; r < tpi; ++r) {
            if (!touched(r, ra, len)) {  // advance the slot sequence past this tile
                const int sg = lane <= RPW ? __ldg(segw_of(rb, r) + lane) : 0;
                int gs = 0;
#pragma unroll
                for (int m = 0; m < RPW; ++m)
                    gs += (__shfl_sync(kFull, sg, m + 1) - __shfl_sync(kFull, sg, m) + GE - 1) >> GL;
                if ((c2 & GM) != 0 && ((c2 + gs) >> GSH) != (c2 >> GSH)) out(c2 >> GSH);
                c2 += gs;
                continue;
            }
            walk(r);
        }
        }
        if (c2 & GM) out(c2 >> GSH);
    };

    float keep = 0.f;
    int cnt = 0, cur_rb = -1, job_a = 0;  // job_a: first item-local tile of the current job in its row block
    bool whole = true;  // current item started at its first tile in this CTA
    Tile nid = tile_of(0);
    int sgn = ntile > 0 ? seg_bounds(nid) : 0;
    for (int q = 0; q < ntile; ++q) {
        const Tile id = nid;
        const int buf = q % NBUF;
        const int64_t r_base = (int64_t)id.rb * RB + warp * RPW;
        const int64_t bl = (int64_t)id.sl * BT + lane * VEC;
        if (id.rb != cur_rb) {  // new job: clear the dW sums
            if (cur_rb >= 0) dump(cur_rb, job_a, t0 + q - job_a - (int)((int64_t)cur_rb * a.nslice * tpi));
            job_a = t0 + q - (int)((int64_t)id.rb * a.nslice * tpi);
            for (int c = 0; c < DWC; ++c) tm_st1(tcol + DW0 + (uint32_t)c, 0.f);
            cur_rb = id.rb;
        }
        if (q == 0 || id.r == 0) {  // new item: X rows to TMEM, dX accumulators cleared
            const float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + r_base + i) : r_base + i;
                // HALF: lane 16h + j holds batch columns 4j.. and 64 + 4j.. of the slice
                const int64_t bx = HALF ? (int64_t)id.sl * BT + (lane & 15) * VEC : bl;
#pragma unroll
                for (int hh = 0; hh < (HALF ? 2 : 1); ++hh) {
                    const int64_t bc = bx + hh * 64;
                    // conv: the slice's exact positions (-1 past the row: zero)
                    const int64_t xo = CONV ? cc_off(a.cc, id.sl, (int)(bc - (int64_t)id.sl * BT)) : bc;
                    const float4 t = (r >= 0 && r < a.nrow && xo >= 0 && (CONV || bc + 4 <= a.xstride))
                                         ? __ldg(reinterpret_cast<const float4 *>(a.X + r * a.xstride + xo))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float tv[4] = {t.x, t.y, t.z, t.w};
                    tm_st4(tcol + RV0 + SW * i + 4 * hh, tv);
                    if constexpr (!DWONLY) tm_st4(tcol + DX0 + SW * i + 4 * hh, z);
                }
            }
            whole = id.r == 0;
            // group index of this tile's first group in the slice sequence
            cnt = 0;
            if (a.gpre != nullptr)
                cnt = __ldg(a.gpre + ((int64_t)id.rb * NW + warp) * (tpi + 1) + id.r);
            else
            for (int k = 0; k < id.r; ++k) {  // groups of 4 per row segment (a last group may hold 2)
                const int32_t *sw = segw_of(id.rb, k);
#pragma unroll
                for (int i = 0; i < RPW; ++i) cnt += (__ldg(sw + i + 1) - __ldg(sw + i) + GE - 1) >> GL;
            }
        }
        tm_wait_st();  // TMEM stores of earlier tiles land before this tile reads them back
        const int sg = sgn;
        nid = next_tile(id);
        if (q + 1 < ntile) sgn = seg_bounds(nid);
        mbar_wait(&full[buf], (q / NBUF) & 1);
        if (q == 0) FUSED_TS(1);
        // the tile's first staged entry: from its issuer through shared memory (cfg5
        // fused backward -1.5 %, cfg3 -2 us)
        int ea, e1t;
#ifndef SP_FUSED_EA_LDG
        ea = tile_ea[buf];
#else
        entry_range(id, ea, e1t);
#endif
        const char *tb = reinterpret_cast<const char *>(smem + buf * buf_sz + BT + lane * VEC);
        const int2 *es = ents + buf * ebuf - ea;
        auto flush = [&](int col) {
            const uint32_t ta = tcol + DW0 + (uint32_t)col;
            const float old = tm_ld1(ta);
            tm_st1(ta, old + keep);
            keep = 0.f;
        };
        if constexpr (HALF) {
            // half-warp h takes entries h, 2+h, 4+h, 6+h of each group of 8 (segments
            // have even length, so a group's valid entries are warp-uniform); lane
            // 16h + j covers batch columns 4j.. and 64 + 4j.. (two 16-byte loads per entry)
            // 32-bit shared-window bases, pinned in registers (an opaque mov: the
            // compiler would otherwise rematerialize them from %tid in every group)
            uint32_t tbs, ess;
            const int lane_p = (int)pin_u32((uint32_t)lane);  // lane bits for the reduction, pinned
            asm volatile("mov.u32 %0, %1;" : "=r"(tbs) : "r"(smem_u32(smem + buf * buf_sz + BT + (lane & 15) * VEC)));
            asm volatile("mov.u32 %0, %1;" : "=r"(ess) : "r"(smem_u32(ents + buf * ebuf) + (uint32_t)((lane >> 4) - ea) * 8u));
#pragma unroll 1
            for (int m = 0; m < RPW; ++m) {
                const int g0 = __shfl_sync(kFull, sg, m), g1 = __shfl_sync(kFull, sg, m + 1);
                if (g0 == g1) continue;
                float rv[8], dx[8];
                if constexpr (DWONLY)
                    tm_ld8(tcol + RV0 + 8 * m, rv);
                else
                    tm_ld8x2(tcol + RV0 + 8 * m, rv, tcol + DX0 + 8 * m, dx);
                for (int e = g0; e < g1; e += 8) {
                    float p[4] = {0.f, 0.f, 0.f, 0.f};
                    auto entry = [&](int u) {
                        int qx, qy;
                        asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(qx), "=r"(qy) : "r"(ess + (uint32_t)(e + 2 * u) * 8u));
                        const int2 q = make_int2(qx, qy);
                        float x[8];
                        const uint32_t ta = tbs + (uint32_t)q.x;
                        asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%8];\n"
                            "ld.shared.v4.f32 {%4, %5, %6, %7}, [%8+256];"
                            : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                            : "r"(ta));
                        if constexpr (!DWONLY) fma_bcast<8>(dx, __int_as_float(q.y), x);  // dX  (Eq. 1 / Eq. 4)
                        p[u] = dot_vec<8>(rv, x);  // dW partial (Eq. 2 / Eq. 5)
                    };
                    const int rem = g1 - e;  // even
                    if (rem >= 8) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) entry(u);
                    } else {  // a short group: entries 0 .. rem/2 - 1 of each half
                        entry(0);
                        if (rem > 2) entry(1);
                        if (rem > 4) entry(2);
                    }
                    const float v = reduce4h(p, lane_p);
                    if ((lane_p & GM) == (cnt & GM)) keep = v;
                    ++cnt;
                    if ((cnt & GM) == 0) flush((cnt >> GSH) - 1);
                }
                if constexpr (!DWONLY) tm_st8(tcol + DX0 + 8 * m, dx);
            }
        } else {
        const uint32_t tbs = pin_u32(smem_u32(tb));  // 32-bit shared-window base, pinned (see pin_u32)
#pragma unroll 1
        for (int m = 0; m < RPW; ++m) {
            const int g0 = __shfl_sync(kFull, sg, m), g1 = __shfl_sync(kFull, sg, m + 1);
            if (g0 == g1) continue;
            float rv[VEC], dx[VEC];
            if constexpr (DWONLY)
                tm_ld4(tcol + RV0 + 4 * m, rv);
            else
                tm_ld4x2(tcol + RV0 + 4 * m, rv, tcol + DX0 + 4 * m, dx);
            for (int e = g0; e < g1; e += 4) {
                const int4 p01 = ld_entry_pair(es + e, true);
                const int4 p23 = ld_entry_pair(es + e + 2, true);
                const int off[4] = {p01.x, p01.z, p23.x, p23.z};
                const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w), __int_as_float(p23.y),
                                    __int_as_float(p23.w)};
                float p[4] = {0.f, 0.f, 0.f, 0.f};
                // padding entries read the zero row in front of the tile; a second pair
                // past the segment (length 2 mod 4) is skipped
                auto entry = [&](int u) {
                    float x[VEC];
                    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                        : "r"(tbs + (uint32_t)off[u]));
                    if constexpr (!DWONLY) fma_bcast<VEC>(dx, w[u], x);   // dX  (Eq. 1 / Eq. 4)
                    p[u] = dot_vec<VEC>(rv, x);    // dW partial (Eq. 2 / Eq. 5)
                };
                if (e + 2 < g1) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) entry(u);
                } else {
                    entry(0);
                    entry(1);
                }
                const float v = reduce4(p, lane);
                if ((lane & GM) == (cnt & GM)) keep = v;
                ++cnt;
                if ((cnt & GM) == 0) flush((cnt >> GSH) - 1);
            }
            if constexpr (!DWONLY) tm_st4(tcol + DX0 + 4 * m, dx);
        }
        }
        const bool item_end = id.r == tpi - 1 || q == ntile - 1;
        if (item_end && DWONLY) {  // item done here: partial column
            if (cnt & GM) flush(cnt >> GSH);
            tm_wait_st();
        } else if (item_end) {  // item done here: partial column, dX rows
            if (cnt & GM) flush(cnt >> GSH);
            tm_wait_st();
            // dX row i of this item, batch columns bl..bl+3 (HALF: the two half-warp
            // partial sums added, low half to lanes 0-15, high half to 16-31)
            auto load_dx = [&](int i, float (&o)[VEC]) {
                if constexpr (HALF) {
                    float lo[4], hi[4];
                    tm_ld4x2(tcol + DX0 + 8 * i, lo, tcol + DX0 + 8 * i + 4, hi);
                    const bool h = (lane & 16) != 0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) o[v] = (h ? hi[v] : lo[v]) + __shfl_xor_sync(kFull, h ? lo[v] : hi[v], 16);
                } else {
                    tm_ld4(tcol + DX0 + 4 * i, o);
                }
            };
            // (ReLU' gate and) store of dX rows (rb, warp*RPW + i), columns bl..bl+3
            auto store = [&](int i, float (&o)[VEC]) {
                if constexpr (CONV) {  // exact positions (tap tilings: identity rows)
                    const int64_t r = r_base + i;
                    if (r >= a.nrow) return;
                    const int64_t off = cc_off(a.cc, (int)(bl / BT), (int)(bl % BT));
                    if (off < 0) return;
                    *reinterpret_cast<float4 *>(a.dX + r * a.xstride + off) = make_float4(o[0], o[1], o[2], o[3]);
                    return;
                }
                // gate H == X (the DP step's ReLU'): the row's X slice is already in
                // TMEM -- lane 16h + j holds columns 4j.. (h = 0) and 64 + 4j.. (h = 1),
                // exactly the 4 columns this lane stores (loaded before any divergence)
                float hx[4] = {0.f, 0.f, 0.f, 0.f};
                const bool gate_tm = HALF && GATE && a.H == a.X;
                if constexpr (HALF && GATE) {
                    if (gate_tm) {
                        float rv8[8];
                        tm_ld8(tcol + RV0 + 8 * i, rv8);
                        const bool h = (lane & 16) != 0;
#pragma unroll
                        for (int v = 0; v < 4; ++v) hx[v] = h ? rv8[4 + v] : rv8[v];
                    }
                }
                const int64_t r = __ldg(a.rowmap + r_base + i);
                if (r < 0 || r >= a.nrow || bl >= a.B) return;
                if (GATE) {
                    if (!gate_tm) {
                        const float4 hv = __ldg(reinterpret_cast<const float4 *>(a.H + r * a.B + bl));
                        hx[0] = hv.x, hx[1] = hv.y, hx[2] = hv.z, hx[3] = hv.w;
                    }
                    o[0] = hx[0] > 0.f ? o[0] : 0.f;
                    o[1] = hx[1] > 0.f ? o[1] : 0.f;
                    o[2] = hx[2] > 0.f ? o[2] : 0.f;
                    o[3] = hx[3] > 0.f ? o[3] : 0.f;
                }
                *reinterpret_cast<float4 *>(a.dX + r * a.B + bl) = make_float4(o[0], o[1], o[2], o[3]);
            };
            if (whole && id.r == tpi - 1) {  // the whole item ran here
#pragma unroll 1
                for (int i = 0; i < RPW; ++i) {
                    float o[VEC];
                    load_dx(i, o);
                    store(i, o);
                }
            } else {
                // cut item: store the raw part; the last CTA of the item to arrive sums the
                // parts in CTA order (deterministic), gates and stores
                const int item = id.rb * nsl + id.sl;
                const int slot = item == first_item ? 0 : 1;
                float *mine = a.dxpart + ((int64_t)(blockIdx.x * 2 + slot) * RB + warp * RPW) * BT + lane * VEC;
#pragma unroll 1
                for (int i = 0; i < RPW; ++i) {
                    float o[VEC];
                    load_dx(i, o);
                    *reinterpret_cast<float4 *>(mine + i * BT) = make_float4(o[0], o[1], o[2], o[3]);
                }
                __threadfence();
                __syncthreads();
                const int64_t c0 = sk_cta((int64_t)item * tpi, T, G);
                const int64_t c1 = sk_cta((int64_t)item * tpi + tpi - 1, T, G);
                if (threadIdx.x == 0) {
                    const int old = atomicAdd(a.tickets + item, 1);
                    last_flag = old == (int)(c1 - c0);
                }
                __syncthreads();
                if (last_flag) {
                    __threadfence();
                    float sum[RPW][VEC];
#pragma unroll
                    for (int i = 0; i < RPW; ++i)
#pragma unroll
                        for (int v = 0; v < VEC; ++v) sum[i][v] = 0.f;
                    for (int64_t c = c0; c <= c1; ++c) {
                        const int sc = item == (int)(sk_lo(c, T, G) / tpi) ? 0 : 1;
                        const float *pp = a.dxpart + ((c * 2 + sc) * RB + warp * RPW) * BT + lane * VEC;
#pragma unroll
                        for (int i = 0; i < RPW; ++i) {
                            const float4 t = __ldcg(reinterpret_cast<const float4 *>(pp + i * BT));
                            sum[i][0] += t.x;
                            sum[i][1] += t.y;
                            sum[i][2] += t.z;
                            sum[i][3] += t.w;
                        }
                    }
#pragma unroll
                    for (int i = 0; i < RPW; ++i) store(i, sum[i]);
                }
            }
        }
        // release the buffer; the last warp to finish tile q refills it with tile q+NBUF
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const int prev = atomicAdd(&released[buf], 1);
            if (prev == NW - 1) {
                released[buf] = 0;
                __threadfence_block();
                if (q + NBUF < ntile) issue(q + NBUF, buf);
            }
        }
    }
    tm_wait_st();
    FUSED_TS(2);
    if (cur_rb >= 0) dump(cur_rb, job_a, t0 + ntile - job_a - (int)((int64_t)cur_rb * a.nslice * tpi));
    tm_fence_before();
    __syncthreads();
    FUSED_TS(3);
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
}

// dW[vidx[e]] = sum over the jobs of e's row block that touched e's tile of
// part[job][base + e] (fixed order).  grid (tap * nrb * nkb + rb * nkb + kb,
// chunk of 256 entries): warp 0 finds the jobs that touched the tile (one lane
// per candidate CTA), then each entry sums their rows in job order.  Linear
// layers: ntap = 1, taps = nullptr (seg / vidx of the tiling, base 0).
struct JobReduceArgs {
    int64_t npad, nslice, G;
    int nrb, nkb, RB, ntap;
    const int32_t *seg, *vidx;  // linear
    const TapDev *taps;         // conv
    int64_t tapbase[kMaxTaps];
    const float *part;
    float *dW;
    int64_t chunk;  // entries per CTA (grid.y chunks per tile)
};
__global__ void __launch_bounds__(256) job_reduce_kernel(const JobReduceArgs a) {
    __shared__ int rows[kMaxJobTab];  // part rows (job indices) that touched this tile, ascending
    __shared__ int nrows;
    const int tpb = a.nrb * a.nkb;
    const int tap = blockIdx.x / tpb, tile = blockIdx.x - tap * tpb, rb = tile / a.nkb, kb = tile - rb * a.nkb;
    const int32_t *seg = a.taps ? a.taps[tap].seg : a.seg;
    const int32_t *vidx = a.taps ? a.taps[tap].vidx : a.vidx;
    const int64_t base_e = a.taps ? a.tapbase[tap] : 0;
    // blockIdx.y: a chunk of the tile's entries (grid.y > 1 only when the tiles
    // alone would not fill the GPU)
    const int64_t t0e = seg[(int64_t)tile * a.RB], t1e = seg[(int64_t)(tile + 1) * a.RB];
    const int64_t e0 = t0e + (int64_t)blockIdx.y * a.chunk, e1 = min(t1e, e0 + a.chunk);
    if (e0 >= e1) return;
    const int tpi = a.ntap * a.nkb, r = tap * a.nkb + kb;
    const int64_t T = (int64_t)a.nrb * a.nslice * tpi, G = a.G;
    const int64_t base = (int64_t)rb * a.nslice * tpi, end = base + a.nslice * tpi;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t c0 = sk_cta(base, T, G), c1 = sk_cta(end - 1, T, G);
        int n = 0;
        for (int64_t cb = c0; cb <= c1; cb += 32) {
            const int64_t c = cb + lane;
            bool hit = false;
            if (c <= c1) {
                const int64_t ja = std::max(sk_lo(c, T, G), base) - base;
                const int64_t len = std::min(sk_lo(c + 1, T, G), end) - base - ja;
                int64_t d = r - ja % tpi;
                if (d < 0) d += tpi;
                hit = len >= tpi || d < len;
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (hit) rows[n + __popc(m & ((1u << lane) - 1))] = (int)(c - c0);
            n += __popc(m);
        }
        if (lane == 0) nrows = n;
    }
    __syncthreads();
    // launched as a programmatic dependent of the fused kernel: everything above
    // reads only the tiling; the partial rows are complete once the primary is
    pdl_wait();
    // the CTA loops over its entries (the job search above is paid once per
    // CTA: one per tile when the tiles fill the GPU)
    const int n = nrows;
    const int64_t bd = blockDim.x;
    if (n >= 8) {
        // many parts per entry (a conv tile: ~37): one entry per thread, 16 part
        // loads in flight, added in job order
        for (int64_t e = e0 + threadIdx.x; e < e1; e += bd) {
            const int v = vidx[e];
            if (v < 0) continue;
            const float *pe = a.part + base_e + e;
            float s = 0.f;
            int j = 0;
            for (; j + 16 <= n; j += 16) {
                float pv[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) pv[u] = pe[(int64_t)rows[j + u] * a.npad];
#pragma unroll
                for (int u = 0; u < 16; ++u) s += pv[u];
            }
#pragma unroll 4
            for (; j < n; ++j) s += pe[(int64_t)rows[j] * a.npad];
            a.dW[v] = s;
        }
        return;
    }
    // few parts per entry (cfg4 95 %: ~3): EU entries per thread at once, their
    // EU x JB part loads independent; each entry's sum still in job order
    constexpr int EU = 4, JB = 4;
    for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += EU * bd) {
        int v[EU];
        float s[EU];
#pragma unroll
        for (int u = 0; u < EU; ++u) {
            const int64_t e = eb + u * bd;
            v[u] = e < e1 ? __ldg(vidx + e) : -1;  // (-1: padding entry or past the chunk)
            s[u] = 0.f;
        }
        const float *pe = a.part + base_e + eb;
        int j = 0;
        for (; j + JB <= n; j += JB) {
            float pv[JB][EU];
#pragma unroll
            for (int q = 0; q < JB; ++q) {
                const float *pr = pe + (int64_t)rows[j + q] * a.npad;
#pragma unroll
                for (int u = 0; u < EU; ++u) pv[q][u] = v[u] >= 0 ? pr[u * bd] : 0.f;
            }
#pragma unroll
            for (int q = 0; q < JB; ++q)
#pragma unroll
                for (int u = 0; u < EU; ++u) s[u] += pv[q][u];
        }
        for (; j < n; ++j) {
            const float *pr = pe + (int64_t)rows[j] * a.npad;
#pragma unroll
            for (int u = 0; u < EU; ++u) s[u] += v[u] >= 0 ? pr[u * bd] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < EU; ++u)
            if (v[u] >= 0) a.dW[v[u]] = s[u];
    }
}


// job_reduce_kernel as a programmatic dependent of the fused kernel just
// enqueued on `st` (PDL: its launch and job search overlap the fused grid's tail)
void launch_job_reduce(dim3 grid, const JobReduceArgs &ja, cudaStream_t st) {
    launch_pdl(job_reduce_kernel, grid, dim3(256), 0, st, ja);
}

// entries per job_reduce CTA: whole tiles when the tiles alone give >= 4 CTAs
// per SM (the per-CTA job search is paid once per tile), else 256-entry chunks
int64_t jr_chunk(int64_t ntiles, int64_t max_tile) {
    if (max_tile < 1) return 256;
    const int64_t ny = std::max<int64_t>(1, (4LL * num_sms() + ntiles - 1) / ntiles);
    const int64_t c = std::max<int64_t>(256, (max_tile + ny - 1) / ny);
    return (c + 255) / 256 * 256;
}

}  // namespace

// Stream-K launch of the TMEM kernel (fused backward, or dW alone when dX is
// null).  Returns false when it does not apply (ragged B, staged entries do
// not fit, too many entry groups per warp for the TMEM columns).
template <int TRPW, int TNW = 32, bool HALF = false, int NB = 2>
static bool launch_sk_rpw(const sp_weight_s *w, const sp_tiling &t, const float *X, const float *dY, const float *H,
                          float *dX, float *dW, int64_t B, cudaStream_t st) {
    constexpr int BT = 128, RBT = TRPW * TNW;
    const bool dwonly = dX == nullptr;
    const int64_t slices = (B + BT - 1) / BT;
    const int64_t T = (int64_t)t.nrb * slices * t.nkb;
    // tiny problems (a few tiles) go to the separate kernels: the reduce pass would dominate
    if (T >= (1LL << 31) || T < 32) return false;
    const int64_t G = std::min<int64_t>(num_sms(), T);
    // HALF reads entry pairs up to 6 entries past a segment (masked): slack in the staging
    const int cap = (t.max_tile + (HALF ? 8 : 2) + 3) & ~3;
    const size_t smem = NB * ((size_t)(t.KC + 1) * BT * sizeof(float) + (size_t)(cap + 2) * sizeof(int2));
    if (smem > (size_t)(226 * 1024)) return false;
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, dY, t.inner, B, BT, t.KC)) return false;
    int64_t maxjobs = 1;
    for (int64_t rb = 0; rb < t.nrb; ++rb) {
        const int64_t tl = rb * slices * t.nkb;
        maxjobs = std::max<int64_t>(maxjobs, sk_cta(tl + slices * t.nkb - 1, T, G) - sk_cta(tl, T, G) + 1);
    }
    if (maxjobs > kMaxJobTab) return false;
    float *part = nullptr, *dxpart = nullptr;
    int *tickets = nullptr;
    const int64_t nitems = (int64_t)t.nrb * slices;
    if (scratch_alloc((void **)&part, (size_t)(maxjobs * t.npad) * sizeof(float), st) != cudaSuccess) return false;
    if (!dwonly && (scratch_alloc((void **)&dxpart, (size_t)G * 2 * RBT * BT * sizeof(float), st) != cudaSuccess ||
                    scratch_alloc((void **)&tickets, (size_t)nitems * sizeof(int), st) != cudaSuccess)) {
        scratch_free(part, st);
        return false;
    }
    if (!dwonly) launch_zero_i32(tickets, nitems, st);
    refresh_if_stale(w, t, st);  // CSC-tiled weights from vals (through perm)
    FusedArgs a{t.rows, t.inner, B, t.KC, t.nkb, 0, cap, t.seg, t.ent, t.vidx, X, dY, H, dX, part, t.npad,
                0, t.rowmap, slices, t.nrb, dxpart, tickets, B, 1, nullptr, {}, {},
                (t.RPWg == TRPW && t.RB == TRPW * TNW) ? t.gpre[HALF ? 1 : 0] : nullptr};
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_path(dwonly ? "sddmm_sk" : HALF ? "bwd_fused_sk_half" : "bwd_fused_sk");
        launch_pdl(kern, dim3((unsigned)G), dim3(TNW * 32), smem, st, a, tmap);
    };
    if (dwonly) go(bwd_fused_sk_kernel<TRPW, TNW, false, true, NB, false, HALF>);
    else if (H) go(bwd_fused_sk_kernel<TRPW, TNW, true, false, NB, false, HALF>);
    else go(bwd_fused_sk_kernel<TRPW, TNW, false, false, NB, false, HALF>);
    const int64_t ntl = (int64_t)t.nrb * t.nkb, jch = jr_chunk(ntl, t.max_tile);
    JobReduceArgs ja{t.npad, slices, G, t.nrb, t.nkb, RBT, 1, t.seg, t.vidx, nullptr, {}, part, dW, jch};
    launch_job_reduce(dim3((unsigned)ntl, (unsigned)((t.max_tile + jch - 1) / jch)), ja, st);
    count_launches(3);  // refresh, kernel, reduce
    scratch_free(part, st);
    if (!dwonly) {
        scratch_free(dxpart, st);
        scratch_free(tickets, st);
    }
    return true;
}

// Stream-K launch of the TMEM kernel (fused backward, or dW alone when dX is
// null).  The CSC tiling is the largest row block whose per-warp entry groups
// fit the TMEM dW columns: 128 rows (4 per warp), else 64 (2), else 32 (1).
// Returns false when none applies (ragged B, staged entries do not fit, rows
// too long -- e.g. Zipf rows with thousands of entries).
static bool launch_sk(const sp_weight_s *w, const float *X, const float *dY, const float *H, float *dX, float *dW,
                      int64_t B, cudaStream_t st) {
    if ((B & 3) != 0 || w->nnz == 0) return false;
    const bool dw = dX == nullptr;
    auto fits = [&](const sp_tiling &t, int64_t cols) { return t.seg != nullptr && t.max_warp_groups <= cols * 8; };
    auto fits8 = [&](const sp_tiling &t, int64_t cols) { return t.seg != nullptr && t.max_warp_groups8 <= cols * 4; };
    // half-warp entries (8 batch columns per lane): dW alone on 128-row blocks, the
    // fused backward on 64-row blocks (32 warps x 2 rows, else 16 warps x 4 rows)
    if (dw && fits8(w->til[1][0], sk_dwcols<4, true, 32, true>()) && w->til[1][0].RB == 128 &&
        launch_sk_rpw<4, 32, true>(w, w->til[1][0], X, dY, H, dX, dW, B, st))
        return true;
    if (!dw && fits8(w->til_f[0], sk_dwcols<2, false, 32, true>()) &&
        launch_sk_rpw<2, 32, true>(w, w->til_f[0], X, dY, H, dX, dW, B, st))
        return true;
    if (!dw && fits8(w->til_f[2], sk_dwcols<4, false, 16, true>()) &&
        launch_sk_rpw<4, 16, true>(w, w->til_f[2], X, dY, H, dX, dW, B, st))
        return true;
    // whole-warp entries (more dW columns per warp): long rows (e.g. Zipf head rows)
    if (fits(w->til[1][0], dw ? sk_dwcols<4, true>() : sk_dwcols<4, false>()) && w->til[1][0].RB == 128 &&
        launch_sk_rpw<4>(w, w->til[1][0], X, dY, H, dX, dW, B, st))
        return true;
    if (dw) return false;  // dW alone: smaller row blocks lose to the tiled SDDMM (more fill per entry)
    if (fits(w->til_f[0], sk_dwcols<2, false>()) &&
        launch_sk_rpw<2>(w, w->til_f[0], X, dY, H, dX, dW, B, st))
        return true;
    if (fits(w->til_f[1], sk_dwcols<1, false>()) &&
        launch_sk_rpw<1>(w, w->til_f[1], X, dY, H, dX, dW, B, st))
        return true;
    return false;
}

bool launch_sddmm_sk(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B, cudaStream_t st) {
    return launch_sk(w, X, dY, nullptr, nullptr, dW, B, st);
}

// Conv backward by taps through the stream-K TMEM kernel (the paper's Alg. 2
// single pass, P297-P347, made atomic-free by the CSC-of-taps drive): rows ic
// of the 64-row tap tilings (tapf), inner oc; slices are the exact dX positions
// cc (H x W x B per channel); tap t = (x, y) reads dY [OC][OH][OW][B] through a
// 4-D tensor map at (m + pad - x, n + pad - y) (cc.dp / cc.dq; out-of-range rows
// and columns zero-filled: Eq. 4 with its bounds clipped, C6); X [IC][H][W][B] is
// read at the slice's positions.  dX (CHWN, or null for dW alone) and dW at the
// conv handle's CSR slots.
bool launch_conv_bwd_sk(const sp_weight_s *w, const ConvCols &cc, const float *dY, int64_t OH, int64_t OW,
                        const float *X, float *dX, float *dW, int ntap, cudaStream_t st) {
    constexpr int TRPW = 2, TNW = 32, BT = 128, RBF = TRPW * TNW;
    if (w->nnz == 0 || ntap > kMaxTaps) return false;
    const sp_tiling &t0 = w->tapf[0];
    if (t0.RB != RBF || t0.seg == nullptr) return false;
    const bool dwonly = dX == nullptr;
    // half-warp entries (8 batch columns per lane) when the groups of 8 fit the TMEM dW columns
    const bool half = !dwonly && w->tapf_groups8 <= (int64_t)sk_dwcols<TRPW, false, TNW, true>() * 4;
    const int64_t groups_cap = (int64_t)(dwonly ? sk_dwcols<TRPW, true>() : sk_dwcols<TRPW, false>()) * 8;
    if (!half && w->tapf_groups > groups_cap) return false;
    const int64_t slices = cc.nslice;
    const int64_t xrow = cc.rowlen;  // floats between channels of X / dX
    const int64_t T = (int64_t)t0.nrb * slices * ntap * t0.nkb;
    if (T >= (1LL << 31)) return false;
    const int64_t G = std::min<int64_t>(num_sms(), T);
    int mx = 0;
    int64_t tapbase[kMaxTaps] = {}, tot = 0;
    for (int t = 0; t < ntap; ++t) {
        mx = std::max(mx, w->tapf[t].max_tile);
        tapbase[t] = tot;
        tot += w->tapf[t].npad;
    }
    const int cap = (mx + (half ? 8 : 2) + 3) & ~3;  // HALF reads entry pairs past a segment (masked)
    const size_t stage = (size_t)(t0.KC + 1) * BT * sizeof(float) + (size_t)(cap + 2) * sizeof(int2);
#ifdef SP_CONV_NBUF3
    const int nbuf = 3 * stage <= (size_t)(226 * 1024) ? 3 : 2;
#else
    const int nbuf = 2;  // (three buffers when they fit measured 2-4 us slower on cfg3)
#endif
    if (nbuf * stage > (size_t)(226 * 1024)) return false;
    CUtensorMap tmap{};
    if (!make_tmap_conv(&tmap, dY, cc, t0.inner, OH, OW, t0.KC)) return false;
    int64_t maxjobs = 1;
    const int64_t per_rb = slices * ntap * t0.nkb;
    for (int64_t rb = 0; rb < t0.nrb; ++rb)
        maxjobs = std::max<int64_t>(maxjobs, sk_cta(rb * per_rb + per_rb - 1, T, G) - sk_cta(rb * per_rb, T, G) + 1);
    float *part = nullptr, *dxpart = nullptr;
    int *tickets = nullptr;
    const int64_t nitems = (int64_t)t0.nrb * slices;
    if (scratch_alloc((void **)&part, (size_t)(maxjobs * tot) * sizeof(float), st) != cudaSuccess) return false;
    if (!dwonly && (scratch_alloc((void **)&dxpart, (size_t)G * 2 * RBF * BT * sizeof(float), st) != cudaSuccess ||
                    scratch_alloc((void **)&tickets, (size_t)nitems * sizeof(int), st) != cudaSuccess)) {
        scratch_free(part, st);
        return false;
    }
    if (!dwonly) launch_zero_i32(tickets, nitems, st);
    launch_refresh_taps(w, 2, ntap, st);  // fused tap tilings' weights from vals
    FusedArgs a{t0.rows, t0.inner, cc.B, t0.KC, t0.nkb, 0, cap, nullptr, nullptr, nullptr, X, dY, nullptr, dX, part,
                tot, 0, nullptr, slices, t0.nrb, dxpart, tickets, xrow, ntap, w->tapdev + 2 * kMaxTaps, {}, cc, nullptr};
    for (int t = 0; t < ntap; ++t) a.tapbase[t] = tapbase[t];
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nbuf * stage));
        note_path(dwonly ? "conv_sddmm_sk" : "conv_bwd_fused_sk");
        launch_pdl(kern, dim3((unsigned)G), dim3(TNW * 32), (size_t)(nbuf * stage), st, a, tmap);
    };
    if (half) {
        if (nbuf == 3) go(bwd_fused_sk_kernel<TRPW, TNW, false, false, 3, true, true>);
        else go(bwd_fused_sk_kernel<TRPW, TNW, false, false, 2, true, true>);
    } else if (nbuf == 3) {
        if (dwonly) go(bwd_fused_sk_kernel<TRPW, TNW, false, true, 3, true>);
        else go(bwd_fused_sk_kernel<TRPW, TNW, false, false, 3, true>);
    } else {
        if (dwonly) go(bwd_fused_sk_kernel<TRPW, TNW, false, true, 2, true>);
        else go(bwd_fused_sk_kernel<TRPW, TNW, false, false, 2, true>);
    }
    const int64_t ntl = (int64_t)ntap * t0.nrb * t0.nkb, jch = jr_chunk(ntl, mx);
    JobReduceArgs ja{tot, slices, G, t0.nrb, t0.nkb, RBF, ntap, nullptr, nullptr, w->tapdev + 2 * kMaxTaps, {}, part, dW,
                     jch};
    for (int t = 0; t < ntap; ++t) ja.tapbase[t] = tapbase[t];
    launch_job_reduce(dim3((unsigned)ntl, (unsigned)((mx + jch - 1) / jch)), ja, st);
    count_launches(3);  // refresh, kernel, reduce
    scratch_free(part, st);
    if (!dwonly) {
        scratch_free(dxpart, st);
        scratch_free(tickets, st);
    }
    return true;
}

sp_status launch_bwd_fused(const sp_weight_s *w, const float *X, const float *dY, const float *H, float *dX,
                           float *dW, int64_t B, cudaStream_t st) {
    // very sparse: the position-gather kernel (both products from each gathered dY row)
    if (w->nnz > 0 && gather_preferred(w, 1, B) &&
        launch_gather_pos(w, 1, 1, B, dY, X, H, H ? EPI_GATE : EPI_NONE, dX, dW, st))
        return SP_OK;
    // stream-K TMEM kernel (any B % 4 == 0) when the rows fit its TMEM columns
    if (launch_sk(w, X, dY, H, dX, dW, B, st)) return SP_OK;
    // slice-split grids: B % 4 == 0, at least one full slice, the big CSC tiling
    if ((B & 3) != 0 || B < 128 || w->nnz == 0) return SP_ERR_SHAPE;
    constexpr int RPW = 8, NW = 16, BT = 128;
    constexpr int TRPW = 4, TNW = 32;  // TMEM variant: 32 warps x 4 rows (same 128-row blocks)
    const sp_tiling &t = w->til[1][0];
    const int64_t slices = (B + BT - 1) / BT;
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, dY, t.inner, B, BT, t.KC)) return SP_ERR_SHAPE;
    const size_t tiles = (size_t)2 * (t.KC + 1) * BT * sizeof(float);
    const int cap = (t.max_tile + 2 + 3) & ~3;
    const bool sent = tiles + (size_t)2 * (cap + 2) * sizeof(int2) <= (size_t)(226 * 1024);
    const size_t smem = tiles + (sent ? (size_t)2 * (cap + 2) * sizeof(int2) : 0);
    // TMEM variant: staged entries and at most kTmCols*32 padded entries per warp
    const bool tm = sent && t.max_warp_groups <= (int64_t)tm_cols<TNW>() * 8;  // 8 groups per TMEM column
    if ((int64_t)t.nrb * slices < num_sms()) return SP_ERR_SHAPE;  // too little parallelism: use the separate kernels
    int64_t nsplit, spl;
    if (tm) {
        // one wave: the largest per-CTA slice count that keeps nrb * nsplit <= #SMs
        spl = std::max<int64_t>(1, (slices * t.nrb + num_sms() - 1) / num_sms());
        nsplit = (slices + spl - 1) / spl;
        while (nsplit * t.nrb > num_sms()) {
            ++spl;
            nsplit = (slices + spl - 1) / spl;
        }
    } else {
        const int64_t want = 2LL * num_sms() * 4;
        nsplit = std::max<int64_t>(1, std::min<int64_t>(slices, (want + t.nrb - 1) / t.nrb));
        spl = (slices + nsplit - 1) / nsplit;
        nsplit = (slices + spl - 1) / spl;
    }
    const bool direct = nsplit == 1;
    float *part = dW;
    if (!direct) {
        if (scratch_alloc((void **)&part, (size_t)(nsplit * t.npad) * sizeof(float), st) != cudaSuccess) {
            set_error("sp_linear_bwd: scratch allocation failed");
            return SP_ERR_ALLOC;
        }
    }
    refresh_if_stale(w, t, st);  // CSC-tiled weights from vals (through perm)
    FusedArgs a{t.rows, t.inner, B, t.KC, t.nkb, (int)spl, cap, t.seg, t.ent, t.vidx, X, dY, H, dX, part, t.npad,
                direct ? 1 : 0, t.rowmap, slices, t.nrb, nullptr, nullptr, B, 1, nullptr, {}, {}, nullptr};
    auto pick = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_path(tm ? "bwd_fused_tm_split" : "bwd_fused_split");
        kern<<<dim3((unsigned)t.nrb, (unsigned)nsplit), (tm ? TNW : NW) * 32, smem, st>>>(a, tmap);
    };
    count_launches(direct ? 1 : 2);
    if (tm) {
        if (H) pick(bwd_fused_tm_kernel<TRPW, TNW, true>);
        else pick(bwd_fused_tm_kernel<TRPW, TNW, false>);
    } else if (H) {
        if (sent) pick(bwd_fused_kernel<RPW, NW, true, true>);
        else pick(bwd_fused_kernel<RPW, NW, true, false>);
    } else {
        if (sent) pick(bwd_fused_kernel<RPW, NW, false, true>);
        else pick(bwd_fused_kernel<RPW, NW, false, false>);
    }
    if (!direct) {
        launch_split_reduce(t.npad, (int)nsplit, part, t.vidx, dW, st);
        scratch_free(part, st);
    }
    return SP_OK;
}

}  // namespace sp

#ifdef SP_FUSED_TS
extern "C" int sp_debug_fused_ts(unsigned long long *out, int n) {
    return cudaMemcpyFromSymbol(out, sp::g_fused_ts, (size_t)n * 4 * sizeof(unsigned long long)) == cudaSuccess ? 0 : 1;
}
#endif
