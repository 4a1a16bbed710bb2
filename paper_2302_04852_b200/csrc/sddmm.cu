// sddmm.cu -- weight-gradient SDDMM (K4, sp_linear_bwd_weight), SURVEY §8(a)
// row a-4:  dW[j] = sum_b dY[r_j][b] * X[c_j][b]  for every nonzero j (CSR
// order), Eq. (2) (P146-P148) restricted to the mask (P151, P173).
//
// Design.  It uses the handle's tiled structure of one
// orientation, chosen so that the operand staged through shared memory is the
// one with the smaller feature dimension (fewer L2 re-reads):
//   CSR tiling (rows r):    register operand dY[r], staged operand X  [C x B]
//   CSC tiling (rows c):    register operand X[c],  staged operand dY [R x B]
// A CTA owns one row block (RB rows) and a batch split (whole slices of BT =
// 32*VEC columns).  For each (slice, column block) the staged tile [KC x BT] is
// double-buffered with cp.async; each warp holds the register-operand slices
// of its RPW rows.  Rows are handled in pairs: up to 16 entries of each row of
// the pair feed 32 register accumulators (lane-partial dots over VEC batch
// elements), one warp transpose-reduce (31 shuffles) turns them into 32 slice
// sums, and lane t adds its sum into the split's partial buffer (entry order,
// one owner per element).  A final fixed-order pass sums the splits and
// scatters to CSR order through vidx.  No atomics: bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

struct SddmmArgs {
    int64_t nrow, F, B;
    int KC, nkb, spl;        // column block, #column blocks, slices per split
    int cap;                 // entry-buffer capacity when entries are staged
    int tma;                 // 1: TMA staging (tensor map valid), 0: synchronous path
    const int32_t *seg;
    const int2 *ent;
    const int32_t *vidx;
    const float *regop;      // [nrow x B]
    const float *smemop;     // [F x B]
    float *part;             // [nsplit x nnz] in entry order (or dW if direct)
    int64_t nnz;
    int direct;              // single split: write dW[vidx[e]] directly
    const int32_t *rowmap;   // tiled position -> register-operand row (nullptr: identity)
    // conv (CONV=true): grid.z = tap; tap t uses taps[t]'s tiling, reads the
    // padded activation shifted by sh[t] columns, and keeps its partials at
    // part[split*nnz + tapbase[t] + e] (nnz = total padded entries of all taps)
    const TapDev *taps;
    int sh[kMaxTaps];
    int64_t tapbase[kMaxTaps];
};

__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int VEC>
__device__ __forceinline__ float dotv(const float (&a)[VEC], const float *p) {
    float x[VEC];
    lds_vec<VEC>(p, x);
    float d = 0.f;
#pragma unroll
    for (int v = 0; v < VEC; ++v) d = fmaf(a[v], x[v], d);
    return d;
}

template <int VEC, int RPW, int NW, bool SENT, bool CONV>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1)
    sddmm_tiled_kernel(const SddmmArgs a_, const __grid_constant__ CUtensorMap tmap) {
    // conv: select this CTA's tap (grid.z) -- its tiling, shift and partials
    SddmmArgs a = a_;
    int shift = 0;
    if constexpr (CONV) {
        const TapDev td = a_.taps[blockIdx.z];
        a.seg = td.seg;
        a.ent = td.ent;
        a.vidx = td.vidx;
        shift = a_.sh[blockIdx.z];
        a.part = a_.part + a_.tapbase[blockIdx.z];
    }
    static_assert(RPW % 2 == 0, "rows are processed in pairs");
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    constexpr int RB = NW * RPW;
    extern __shared__ __align__(128) float smem[];  // [2][KC][BT] floats, then [2][cap+2] int2
    __shared__ uint64_t full[2];
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * a.KC * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rb = blockIdx.x;
    const int64_t B = a.B;
    const int64_t s_lo = (int64_t)blockIdx.y * a.spl * BT;
    const int nsl = (int)std::min<int64_t>(a.spl, (B - s_lo + BT - 1) / BT);
    const int ntile = nsl * a.nkb;
    float *P = a.part + (a.direct ? 0 : (int64_t)blockIdx.y * a.nnz);
    const bool vec4 = (B & 3) == 0;
    const size_t tile_sz = (size_t)a.KC * BT;
    const int32_t *segw = a.seg + (int64_t)rb * a.nkb * RB + warp * RPW;

    const int ebuf = a.cap + 2;
    const bool tma = a.tma != 0;
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto entry_range = [&](int kb, int &e0, int &e1) {
        const int64_t tb = ((int64_t)rb * a.nkb + kb) * RB;
        e0 = __ldg(a.seg + tb) & ~1;
        e1 = __ldg(a.seg + tb + RB);
    };
    // tile q = (slice q / nkb, column block q % nkb): TMA issue by one thread
    auto issue = [&](int q, int buf) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        int e0 = 0, e1 = 0;
        if constexpr (SENT) entry_range(kb, e0, e1);
        const unsigned eb = SENT ? (unsigned)(((e1 - e0) * 8 + 15) & ~15) : 0u;
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        tma_load_2d(smem + buf * tile_sz, &tmap, (int)(s_lo + (int64_t)s * BT) + shift, kb * a.KC, &full[buf]);
        if (eb) tma_load_1d(ents + buf * ebuf, a.ent + e0, eb, &full[buf]);
    };
    if (tma && threadIdx.x == 0) issue(0, 0);

    float rv[RPW][VEC];
    int sg = 0;
    for (int q = 0; q < ntile; ++q) {
        const int s = q / a.nkb, kb = q - s * a.nkb;
        if (kb == 0) {  // new slice: this warp's register-operand rows
            const int64_t bl = s_lo + (int64_t)s * BT + lane * VEC;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int64_t tpos = (int64_t)rb * RB + warp * RPW + i;
                int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + tpos) : tpos;
                if (r < 0) r = a.nrow;  // unused position: zeros
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
            }
        }
        sg = lane <= RPW ? __ldg(segw + (int64_t)kb * RB + lane) : 0;
        const int buf = q & 1;
        if (q + 1 < ntile) {
            if (tma && threadIdx.x == 0) issue(q + 1, buf ^ 1);
            if constexpr (!SENT) {  // entries of the next column block into L1
                const int kbn = (q + 1) % a.nkb;
                const int sn = lane <= RPW ? __ldg(segw + (int64_t)kbn * RB + lane) : 0;
                const int e0 = __shfl_sync(kFull, sn, 0), e1 = __shfl_sync(kFull, sn, RPW);
                for (int l = (e0 >> 4) + lane; l < ((e1 + 15) >> 4); l += 32)
                    prefetch_l1(a.ent + ((int64_t)l << 4));
            }
        }
        int ea = 0;
        if (tma) {
            mbar_wait(&full[buf], (q >> 1) & 1);
            if constexpr (SENT) {
                int e1;
                entry_range(kb, ea, e1);
            }
        } else {  // ragged B: synchronous staging of this tile
            const int64_t k0 = (int64_t)kb * a.KC;
            stage_tile<BT, NT>(smem + buf * tile_sz, a.smemop, k0, (int)std::min<int64_t>(a.KC, a.F - k0), B,
                               s_lo + (int64_t)s * BT, false);
            if constexpr (SENT) {
                int e1;
                entry_range(kb, ea, e1);
                for (int i = threadIdx.x; i < e1 - ea; i += NT) ents[buf * ebuf + i] = __ldg(a.ent + ea + i);
            }
            __syncthreads();
        }
        constexpr int SH = VEC == 4 ? 0 : VEC == 2 ? 1 : 2;
        const char *tb = reinterpret_cast<const char *>(smem + buf * tile_sz + lane * VEC);
        const int2 *es = SENT ? ents + buf * ebuf - ea : a.ent;
        // dot of the register-operand slice with tile row of entry e (0 for padding)
        auto dot_e = [&](const float(&r)[VEC], int off) -> float {
            // padding entries (offset -1) read tile row 0; their slot is never written
            float x[VEC];
            lds_vec<VEC>(reinterpret_cast<const float *>(tb + (max(off, 0) >> SH)), x);
            return dot_vec<VEC>(r, x);
        };
        // offsets of entries e..e+3; a second pair past the segment (nv == 2) reads row 0
        auto offs4 = [&](int e, int nv, int (&o)[4]) {
            const int4 p01 = ld_entry_pair(SENT ? es + e : a.ent + e, SENT);
            const int4 p23 = ld_entry_pair(SENT ? es + e + 2 : a.ent + e + 2, SENT);
            o[0] = p01.x;
            o[1] = p01.z;
            o[2] = nv > 2 ? p23.x : -1;
            o[3] = nv > 2 ? p23.z : -1;
        };
#pragma unroll
        for (int m = 0; m < RPW; m += 2) {
            int pa = __shfl_sync(kFull, sg, m);
            const int a1 = __shfl_sync(kFull, sg, m + 1);
            int pb = a1;
            const int b1 = __shfl_sync(kFull, sg, m + 2);
            while (pa < a1 || pb < b1) {
                // segments are padded to even lengths: a last group of 2 masks its
                // second pair (those slots are never written)
                const int na = min(16, a1 - pa), nb = min(16, b1 - pb);
                float acc[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) acc[u] = 0.f;
#pragma unroll
                for (int g = 0; g < 16; g += 4) {
                    if (g < na) {
                        int o[4];
                        offs4(pa + g, na - g, o);
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[g + u] = dot_e(rv[m], o[u]);
                    }
                    if (g < nb) {
                        int o[4];
                        offs4(pb + g, nb - g, o);
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[16 + g + u] = dot_e(rv[m + 1], o[u]);
                    }
                }
                const float sum = transpose_reduce32(acc, lane);
                const int u = lane & 15;
                const bool mine = lane < 16 ? u < na : u < nb;
                if (mine) {
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
        __syncthreads();  // buffer free before it is refilled
    }
}

// dW[vidx[e]] = sum_s part[s][e], s ascending.
__global__ void split_reduce_kernel(int64_t nnz, int nsplit, const float *__restrict__ part,
                                    const int32_t *__restrict__ vidx, float *__restrict__ dW) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int v = vidx[e];
    if (v < 0) return;  // padding entry
    float s = part[e];
    for (int i = 1; i < nsplit; ++i) s += part[(int64_t)i * nnz + e];
    dW[v] = s;
}


template <int VEC, int RPW, int NW>
sp_status launch_cfg(const sp_weight_s *w, const sp_tiling &t, const float *regop, const float *smemop,
                     float *dW, int64_t B, int ctas_per_sm, cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    const int64_t nnz = t.npad;  // partials are kept per (padded) entry
    const int64_t slices = (B + BT - 1) / BT;
    const int64_t want = (int64_t)ctas_per_sm * num_sms() * 4;  // >= 4 waves: small tail
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(slices, (want + t.nrb - 1) / t.nrb));
    const int64_t spl = (slices + nsplit - 1) / nsplit;
    nsplit = (slices + spl - 1) / spl;
    const size_t tiles = (size_t)2 * t.KC * BT * sizeof(float);
    const int cap = (t.max_tile + 2 + 3) & ~3;  // keeps both entry buffers 16-byte aligned
    const bool sent = tiles + (size_t)2 * (cap + 2) * sizeof(int2) <= (size_t)(226 * 1024) / (NW == 8 ? 2 : 1);
    const size_t smem = tiles + (sent ? (size_t)2 * (cap + 2) * sizeof(int2) : 0);
    const bool direct = nsplit == 1;
    float *part = dW;
    if (!direct) {
        if (scratch_alloc((void **)&part, (size_t)(nsplit * nnz) * sizeof(float), st) != cudaSuccess) {
            set_error("sp_linear_bwd_weight: scratch allocation failed");
            return SP_ERR_ALLOC;
        }
    }
    CUtensorMap tmap{};
    const bool tma = (B & 3) == 0 && make_tmap_2d(&tmap, smemop, t.inner, B, BT, t.KC);
    SddmmArgs a{t.rows, t.inner, B, t.KC, t.nkb, (int)spl, cap, tma ? 1 : 0, t.seg, t.ent, t.vidx, regop, smemop,
                part, nnz, direct ? 1 : 0, t.rowmap, nullptr, {}, {}};
    count_launches(direct ? 1 : 2);
    {
        auto kern = sent ? sddmm_tiled_kernel<VEC, RPW, NW, true, false> : sddmm_tiled_kernel<VEC, RPW, NW, false, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_path("sddmm_tiled");
        kern<<<dim3((unsigned)t.nrb, (unsigned)nsplit), NW * 32, smem, st>>>(a, tmap);
    }
    if (!direct) {
        split_reduce_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, (int)nsplit, part, t.vidx, dW);
        scratch_free(part, st);
    }
    return SP_OK;
}

template <int VEC>
sp_status launch_vec(const sp_weight_s *w, const sp_tiling &t, int var, const float *regop,
                     const float *smemop, float *dW, int64_t B, cudaStream_t st) {
    if (var == 0) return launch_cfg<VEC, 8, 16>(w, t, regop, smemop, dW, B, 2, st);
    return launch_cfg<VEC, 4, 8>(w, t, regop, smemop, dW, B, 4, st);
}

// conv: dW[vidx_t[e]] = sum_s part[s][tapbase_t + e]  (grid.y = tap)
struct TapBase {
    int64_t v[kMaxTaps];
};
__global__ void conv_split_reduce_kernel(const TapDev *__restrict__ taps, const TapBase tapbase,
                                         int64_t totpad, int nsplit, const float *__restrict__ part,
                                         float *__restrict__ dW) {
    const TapDev t = taps[blockIdx.y];
    const int64_t base = tapbase.v[blockIdx.y];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < t.npad; e += (int64_t)gridDim.x * blockDim.x) {
        const int v = t.vidx[e];
        if (v < 0) continue;
        float s = part[base + e];
        for (int i = 1; i < nsplit; ++i) s += part[(int64_t)i * totpad + base + e];
        dW[v] = s;
    }
}

}  // namespace

bool launch_conv_sddmm(const sp_weight_s *w, int64_t B, const float *dYv, const float *Xp, int64_t Lv, int64_t Lp,
                       const int *sh, int ntap, float *dW, cudaStream_t st) {
    (void)B;
    constexpr int VEC = 4, RPW = 8, NW = 16, BT = 128;
    const sp_tiling &t0 = w->tap[0][0];  // rows oc, inner ic
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, Xp, t0.inner, Lp, BT, t0.KC)) return false;
    int64_t tapbase[kMaxTaps] = {};
    int64_t tot = 0;
    int mx = 0;
    for (int t = 0; t < ntap; ++t) {
        tapbase[t] = tot;
        tot += w->tap[t][0].npad;
        mx = std::max(mx, w->tap[t][0].max_tile);
    }
    const int64_t slices = (Lv + BT - 1) / BT;
    const int64_t want = 2LL * num_sms() * 4;
    const int64_t units = (int64_t)t0.nrb * ntap;
    int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(slices, (want + units - 1) / units));
    const int64_t spl = (slices + nsplit - 1) / nsplit;
    nsplit = (slices + spl - 1) / spl;
    const int cap = (mx + 2 + 3) & ~3;
    const size_t tiles = (size_t)2 * t0.KC * BT * sizeof(float);
    const bool sent = tiles + (size_t)2 * (cap + 2) * sizeof(int2) <= (size_t)(226 * 1024);
    const size_t smem = tiles + (sent ? (size_t)2 * (cap + 2) * sizeof(int2) : 0);
    float *part = nullptr;
    if (scratch_alloc((void **)&part, (size_t)(nsplit * tot) * sizeof(float), st) != cudaSuccess) return false;
    TapBase tbv;
    for (int t = 0; t < kMaxTaps; ++t) tbv.v[t] = tapbase[t];
    SddmmArgs a{t0.rows, t0.inner, Lv, t0.KC, t0.nkb, (int)spl, cap, 1, nullptr, nullptr, nullptr, dYv, Xp,
                part, tot, 0, nullptr, w->tapdev, {}, {}};
    for (int t = 0; t < ntap; ++t) {
        a.sh[t] = sh[t];
        a.tapbase[t] = tapbase[t];
    }
    auto kern = sent ? sddmm_tiled_kernel<VEC, RPW, NW, true, true> : sddmm_tiled_kernel<VEC, RPW, NW, false, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    count_launches(2);
    note_path("conv_sddmm_tiled");
    kern<<<dim3((unsigned)t0.nrb, (unsigned)nsplit, (unsigned)ntap), NW * 32, smem, st>>>(a, tmap);
    conv_split_reduce_kernel<<<dim3(64, ntap), 256, 0, st>>>(w->tapdev, tbv, tot, (int)nsplit, part, dW);
    scratch_free(part, st);
    return true;
}

void launch_split_reduce(int64_t npad, int nsplit, const float *part, const int32_t *vidx, float *dW,
                         cudaStream_t st) {
    split_reduce_kernel<<<(unsigned)((npad + 255) / 256), 256, 0, st>>>(npad, nsplit, part, vidx, dW);
}

sp_status launch_sddmm(const sp_weight_s *w, const float *X, const float *dY, float *dW, int64_t B,
                       cudaStream_t st) {
    if (w->nnz == 0) return SP_OK;
    if (gather_preferred(w, 0, B, true)) {
        if (!launch_gather_pos(w, 0, 2, B, X, dY, nullptr, EPI_NONE, nullptr, dW, st)) launch_sddmm_gather(w, X, dY, dW, B, st);
        return SP_OK;
    }
    // the stream-K TMEM kernel (fused.cu) in its dW-only mode when it applies
    if (launch_sddmm_sk(w, X, dY, dW, B, st)) return SP_OK;
    // stage the smaller feature dimension; the CSC tiling when the CSR one has
    // split (part) rows, which would reload a row's register operand per part
    const int orient = (w->C > w->R || w->til[0][0].psplit_rows()) ? 1 : 0;
    const float *regop = orient ? X : dY;
    const float *smemop = orient ? dY : X;
    const int vec = B <= 32 ? 1 : (B <= 64 || (B & 3)) ? 2 : 4;
    // small problems (few row blocks and slices) use the small tiling
    const int var = (int64_t)w->til[orient][0].nrb * ((B + 32 * vec - 1) / (32 * vec)) < num_sms() ? 1 : 0;
    const sp_tiling &t = w->til[orient][var];
    if (vec == 4) return launch_vec<4>(w, t, var, regop, smemop, dW, B, st);
    if (vec == 2) return launch_vec<2>(w, t, var, regop, smemop, dW, B, st);
    return launch_vec<1>(w, t, var, regop, smemop, dW, B, st);
}

}  // namespace sp
