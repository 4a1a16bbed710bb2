// slab.cu -- batch-slab kernels for the very sparse regime (the gather tilings).
//
// At RB * d < 1 (e.g. 4096^2 at 98-99 %, B = 256) a staged [KC x 128] tile row
// serves less than one entry of its row block, so the position-gather kernels
// (gather.cu) fetch every nonzero's activation row from L2 instead: nnz * B * 4
// bytes cross L2 -> SM per product, and at ~7-9 TB/s that is what bounds them.
// Here the staging is turned the other way: a CTA stages the WHOLE inner
// dimension of a narrow batch slice (the slab, [inner x BS] floats, BS = 8..64
// columns, <= 200 KB) into shared memory once, with cp.async, and then every
// position of its chunk gathers its entries' rows from the slab.  Per product
// the L2 -> SM bytes fall to (CTAs * slab) + (slices * entries * 8) -- for
// cfg4 at 99 % ~62 MB instead of 172 MB -- and the gathers run at the shared-
// memory rate (P173: each gathered value still feeds one FMA per batch column).
//
// Mapping: a warp per position (row) at a time; its lanes are L = BS / 4 column
// lanes (one float4 of the slice each) x E = 32 / L entry lanes: a step takes E
// consecutive entries of the row's segment (one coalesced load, issued a step
// ahead), each entry lane gathers its entry's slab row, and at the row's end the
// entry lanes' partial sums are added by a fixed shuffle tree.  (A first version
// ran P = 32 / L positions per warp in lockstep, each lane group streaming its
// own segment: 16 entry streams per warp missed L1 on nearly every step, and it
// was 1.4x slower than the position-gather kernels.)  Positions are dealt to the
// nchunk CTAs of a slice round-robin (p = q * nchunk + chunk): every chunk gets
// the same mix of long and short rows (positions are in longest-first order).
//   MODE 0  SpMM: out[row(p)][slice] = epi(sum_e w_e * gin[idx_e][slice])
//           (orient 0 fwd, orient 1 dX; Zipf part rows store raw sums to vpart)
//   MODE 1  fused backward (orient 1): dX as MODE 0 from the dY slab, and per
//           entry the slice's share of <X[k], dY[i_e]> (X[k] in registers),
//           reduced over the L column lanes and stored to dwpart[slice][e]
//   MODE 2  dW alone (orient 0): the MODE 1 dot products without dX
// The per-slice dW shares are summed in slice order by split_reduce (one
// dW element = one fixed-order sum: deterministic, no atomics).  Every output
// element of MODE 0 / dX is a fixed-order sum (entry lanes' strided partials,
// then the shuffle tree): deterministic, within the tolerance of the other
// kernels' ascending order.
#include <cuda_runtime.h>

#include <algorithm>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

constexpr int kSlabThreads = 1024;
constexpr size_t kSlabMaxBytes = 200 * 1024;

struct SlabArgs {
    int64_t B, npos, inner, npad;
    int nchunk;
    const int32_t *seg;
    const int2 *ent;
    const int32_t *rowmap, *split;
    const float *gin;   // gathered operand [inner x B]
    const float *rin;   // MODE 1 / 2: the position's own row operand [rows x B]
    const float *gate;  // EPI_GATE rows
    float *out;         // MODE 0: Y or dX; MODE 1: dX
    float *dwpart;      // MODE 1 / 2: [slices x npad]
    float *vpart;       // MODE 0 part rows' raw sums [nparts x B]
    int epi;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

template <int BS, int MODE>
__global__ void __launch_bounds__(kSlabThreads, 1) slab_kernel(const SlabArgs a) {
    constexpr int L = BS / 4, E = 32 / L;  // column lanes (one float4 each), entry lanes
    constexpr int LL = __builtin_ctz(L);
    constexpr int SH = 9 - __builtin_ctz(BS * 4);  // ent.x = inner * kTilRowBytes -> slab byte offset
    static_assert(kTilRowBytes == 512 && BS * 4 <= kTilRowBytes, "slab row offsets are shifted tile offsets");
    constexpr bool DW = MODE != 0, ACC = MODE != 2;
    // entry-lane reduction of the 4 accumulators: transposed over the T top lane
    // bits (16, 8), plain over the rest; NV values per lane remain
    constexpr int T = E >= 4 ? 2 : E == 2 ? 1 : 0, NV = 4 >> T;
    constexpr int PLAIN = T == 0 ? 0 : (((16 >> (T - 1)) - 1) & ~(L - 1));
    extern __shared__ float4 slab[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lq = lane & (L - 1), j = lane >> LL;
    const int64_t c0 = (int64_t)blockIdx.y * BS;
    const int chunk = blockIdx.x;
    pdl_wait();  // (a programmatic dependent of the producer of gin / rin)
    // ---- stage the slab: inner rows x L float4s, zero-filled past B
    {
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(slab);
        const int64_t n4 = a.inner * L;
        for (int64_t i = threadIdx.x; i < n4; i += kSlabThreads) {
            const int64_t row = i >> LL;
            const int64_t col = c0 + (i & (L - 1)) * 4;
            const bool ok = col < a.B;
            cp_async16(sbase + (uint32_t)(i * 16), a.gin + row * a.B + (ok ? col : 0), ok);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    pdl_trigger();  // (every CTA is resident: the reduction that follows may start its prologue)
#ifdef SP_SLAB_STAGE_ONLY
    return;  // measurement build: the staging alone
#endif
    const int64_t col = c0 + lq * 4;
    const bool cv = col < a.B;
    const char *sb = reinterpret_cast<const char *>(slab) + lq * 16;
    const int64_t nq = (a.npos - chunk + a.nchunk - 1) / a.nchunk;  // this chunk's positions
    float *dwp = DW ? a.dwpart + (int64_t)blockIdx.y * a.npad : nullptr;
    // the warp's rows q = warp + 32 k: lane k holds row k's (r, e0, e1) for a batch
    // of 32 rows, and the first entries of the next row are loaded while a row
    // is walked (the per-row chain rowmap -> seg -> entry -> gather was the
    // bound of a version without it: ~3 L2 round trips per 41-entry row)
    const int64_t nrw = nq > warp ? (nq - warp + 31) / 32 : 0;
    int mr = -1, me0 = 0, me1 = 0;
    int2 nxt = make_int2(0, 0);
    for (int64_t k = 0; k < nrw; ++k) {
        const int kk = (int)(k & 31);
        if (kk == 0) {  // metadata of the next 32 rows
            const int64_t qq = warp + 32 * (k + lane);
            mr = -1, me0 = me1 = 0;
            if (k + lane < nrw) {
                const int64_t pp = qq * a.nchunk + chunk;
                mr = __ldg(a.rowmap + pp);
                if (mr >= 0) {
                    me0 = __ldg(a.seg + pp);
                    me1 = __ldg(a.seg + pp + 1);
                }
            }
            const int f0 = __shfl_sync(kFull, me0, 0), f1 = __shfl_sync(kFull, me1, 0);
            nxt = f0 + j < f1 ? __ldg(a.ent + f0 + j) : make_int2(0, 0);
        }
        const int r = __shfl_sync(kFull, mr, kk);
        const int e0 = __shfl_sync(kFull, me0, kk), e1 = __shfl_sync(kFull, me1, kk);
        const int64_t p = (int64_t)(warp + 32 * k) * a.nchunk + chunk;
        int2 en = nxt;
        {  // the next row's first entries (within this metadata batch)
            const int n0 = __shfl_sync(kFull, me0, (kk + 1) & 31), n1 = __shfl_sync(kFull, me1, (kk + 1) & 31);
            nxt = (kk < 31 && n0 + j < n1) ? __ldg(a.ent + n0 + j) : make_int2(0, 0);
        }
        if (r < 0) continue;  // an unused position (warp-uniform)
        float acc[4] = {0.f, 0.f, 0.f, 0.f}, xr[4] = {0.f, 0.f, 0.f, 0.f};
        if (DW && cv) {
            const float4 t = __ldg(reinterpret_cast<const float4 *>(a.rin + (int64_t)r * a.B + col));
            xr[0] = t.x, xr[1] = t.y, xr[2] = t.z, xr[3] = t.w;
        }
        // E consecutive entries per step, one per entry lane (coalesced loads, the
        // next step's entry loaded before this step's gather)
        for (int e = e0; e < e1; e += E) {
            const int2 cur = en;
            en = e + E + j < e1 ? __ldg(a.ent + e + E + j) : make_int2(0, 0);
            const float4 t = *reinterpret_cast<const float4 *>(sb + (max(cur.x, 0) >> SH));
            const float y[4] = {t.x, t.y, t.z, t.w};
            if constexpr (ACC) fma_bcast<4>(acc, __int_as_float(cur.y), y);
            if constexpr (DW) {
                float pd = dot_vec<4>(xr, y);
#pragma unroll
                for (int o = L / 2; o >= 1; o >>= 1) pd += __shfl_xor_sync(kFull, pd, o);
                if (lq == 0 && e + j < e1) dwp[e + j] = pd;
            }
        }
        if constexpr (ACC) {
            // sum the entry lanes' partials (fixed tree: deterministic)
            float v[4] = {acc[0], acc[1], acc[2], acc[3]};
            int n = 4;
#pragma unroll
            for (int o = 16; o >= L; o >>= 1) {
                if (n > 1) {
                    const bool up = (lane & o) != 0;
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        if (i < n / 2) {
                            const float send = up ? v[i] : v[i + n / 2], keep = up ? v[i + n / 2] : v[i];
                            v[i] = keep + __shfl_xor_sync(kFull, send, o);
                        }
                    }
                    n >>= 1;
                } else {
                    v[0] += __shfl_xor_sync(kFull, v[0], o);
                }
            }
            if ((lane & PLAIN) != 0 || !cv) continue;
            const int u0 = T == 2 ? ((lane >> 3) & 2) | ((lane >> 3) & 1) : T == 1 ? ((lane >> 3) & 2) : 0;
            const int ps = (MODE == 0 && a.split != nullptr) ? __ldg(a.split + p) : -1;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int64_t c = col + u0 + i;
                float o = v[i];
                if (ps >= 0) {  // a part row: raw sums (split_rows_reduce applies the epilogue)
                    a.vpart[(int64_t)ps * a.B + c] = o;
                    continue;
                }
                if (a.epi == EPI_RELU) o = fmaxf(o, 0.f);
                else if (a.epi == EPI_GATE) o = __ldg(a.gate + (int64_t)r * a.B + c) > 0.f ? o : 0.f;
                a.out[(int64_t)r * a.B + c] = o;
            }
        }
    }
}

// slab width: the widest of 64 / 32 / 16 / 8 columns whose slab fits, not
// (much) wider than the batch
int slab_width(int64_t inner, int64_t B) {
    for (int bs = 64; bs >= 8; bs >>= 1)
        if ((size_t)inner * bs * sizeof(float) <= kSlabMaxBytes && (bs <= B || bs == 8)) return bs;
    return 0;
}

// chunks per slice: minimise waves x (staging + the CTA's share of the gathers),
// one CTA per SM (the slab takes most of the shared memory)
int slab_chunks(int64_t slices, int64_t inner, int bs, int64_t npad, int64_t npos) {
    const double stage = (double)inner * bs * 4.0 / 64.0;       // cycles at ~64 B/clk/SM from L2
    const double work = (double)slices * npad * bs * 4.0 / 80.0;  // gathered bytes at ~80 B/clk/SM
    int best = 1;
    double bt = 1e300;
    const int64_t maxc = std::max<int64_t>(1, std::min<int64_t>(npos, 64));
    for (int64_t c = 1; c <= maxc; ++c) {
        const int64_t ctas = slices * c;
        const double waves = (double)((ctas + num_sms() - 1) / num_sms());
        const double t = waves * (stage + work / (double)ctas);
        if (t < bt * 0.999) {
            bt = t;
            best = (int)c;
        }
    }
    return best;
}

template <int BS>
void slab_go(const SlabArgs &a, int mode, int64_t slices, cudaStream_t st) {
    const size_t smem = (size_t)a.inner * BS * sizeof(float);
    const dim3 grid((unsigned)a.nchunk, (unsigned)slices);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(kern, grid, dim3(kSlabThreads), smem, st, a);
    };
    if (mode == 0) go(slab_kernel<BS, 0>);
    else if (mode == 1) go(slab_kernel<BS, 1>);
    else go(slab_kernel<BS, 2>);
}

}  // namespace

// Slab launch on a gather tiling (MODE as slab_kernel).  false: no gather
// tiling, B % 4 != 0, B < 8, or no slab width fits the inner dimension.
bool launch_slab(const sp_weight_s *w, int orient, int mode, int64_t B, const float *gin, const float *rin,
                 const float *gate, int epi, float *out, float *dW, cudaStream_t st) {
#ifdef SP_NO_SLAB
    return false;
#endif
    const sp_tiling &t = w->til_g[orient];
    if (t.ent == nullptr || (B & 3) != 0 || B < 8) return false;
    const int bs = slab_width(t.inner, B);
    if (bs == 0) return false;
    const int64_t slices = (B + bs - 1) / bs;
    if (slices > 65535) return false;
    const int64_t npos = (int64_t)t.nrb * t.RB;
    const int nchunk = slab_chunks(slices, t.inner, bs, t.npad, npos);
    float *vpart = nullptr, *dwpart = nullptr;
    const bool parts = mode == 0 && t.psplit_rows();
    if (parts && scratch_alloc((void **)&vpart, (size_t)t.nparts * B * sizeof(float), st) != cudaSuccess) return false;
    if (mode != 0 && scratch_alloc((void **)&dwpart, (size_t)slices * t.npad * sizeof(float), st) != cudaSuccess) {
        if (vpart) scratch_free(vpart, st);
        return false;
    }
    refresh_if_stale(w, t, st);
    SlabArgs a{B, npos, t.inner, t.npad, nchunk, t.seg, t.ent, t.rowmap, parts ? t.split : nullptr,
               gin, rin, gate, out, dwpart, vpart, epi};
    if (bs == 64) slab_go<64>(a, mode, slices, st);
    else if (bs == 32) slab_go<32>(a, mode, slices, st);
    else if (bs == 16) slab_go<16>(a, mode, slices, st);
    else slab_go<8>(a, mode, slices, st);
    note_path(mode == 0 ? "spmm_slab" : mode == 1 ? "bwd_slab" : "sddmm_slab");
    count_launches(1);
    if (parts) {
        launch_split_rows_reduce(t, vpart, B, out, gate, epi, st);
        scratch_free(vpart, st);
    }
    if (mode != 0) {
        launch_split_reduce(t.npad, (int)slices, dwpart, t.vidx, dW, st);
        count_launches(1);
        scratch_free(dwpart, st);
    }
    return true;
}

}  // namespace sp
