// spmm.cu -- forward SpMM (K2, sp_linear_fwd) and CSC-driven input-gradient
// SpMM (K3, sp_linear_bwd_input).  SURVEY §8(a) rows a-2, a-3.
//
//   out[r][b] = epi( sum over the entries (c, w) of row r of w * in[c][b] )
//   forward (P141):  rows of the CSR      (out = Y [R x B],  in = X  [C x B])
//   dX (Eq. 1):      rows of the CSC copy (out = dX [C x B], in = dY [R x B]),
//                    w = vals[perm[k]]  -- gather form, no atomics.
//
// Design: the handle carries a tiled copy of each orientation
// (row blocks of RB rows x column blocks of KC inner columns; entries of one
// (row block, column block, row) segment are contiguous and store the
// block-local column and the value).  A CTA owns one row block and one batch
// slice of BT = 32*VEC columns.  The `in` tile [KC x BT] of each column block
// and the tile's entries arrive by TMA (a 2-D box and a 1-D bulk copy) into
// one of two buffers; the last warp done with a buffer refills it.  Each warp
// owns RPW consecutive tiled rows and keeps their VEC-wide accumulators in
// registers across column blocks.  Per pair of entries: one broadcast 16-byte
// LDS of (column, value) x 2; per entry one vector LDS of tile[column][lane*VEC..]
// and VEC FFMAs (FFMA2).  Ragged B (B % 4 != 0) stages synchronously.  Every output element is
// produced by exactly one lane in a fixed order (entries ascending): no
// atomics, bitwise reproducible, independent of B and of the grid.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

struct SpmmArgs {
    int64_t rows, inner, B;
    int KC, nkb, cap;  // cap: entry-buffer capacity (entries) when staged
    int tma;           // 1: stage with TMA (tensor map valid), 0: synchronous path
    const int32_t *seg;
    const int2 *ent;
    const float *in;
    float *out;
    const float *gate;
    const int32_t *rowmap;  // tiled position -> output row (nullptr: identity)
    const int32_t *psplit;  // tiled position -> part slot of a split row (-1 whole; nullptr: none)
    float *vpart;           // [nparts x B] raw sums of the part rows
    // conv (CONV=true): the tile sequence runs over (tap, column block); tap t
    // uses taps[t]'s tiling and reads the padded input shifted by sh[t]
    // columns; output column n = ((p*Wv) + q)*B + b is stored compactly to
    // out[r][p][q][b] when p < OHv, q < OWv.
    int ntap;
    const TapDev *taps;
    int sh[kMaxTaps];
    int64_t Wv, OHv, OWv;
};

__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Prefetch into L1 the entry lines [e0, e1) (128-byte lines = 16 entries).
__device__ __forceinline__ void prefetch_entries(const int2 *ent, int e0, int e1, int lane) {
    const int l0 = e0 >> 4, l1 = (e1 + 15) >> 4;
    for (int l = l0 + lane; l < l1; l += 32) prefetch_l1(ent + ((int64_t)l << 4));
}

// SENT: the tile's entries are staged in shared memory too (next tile's
// entries arrive with its activation tile); otherwise entries are read with
// warp-uniform global loads (tiles larger than the entry buffer).
// Staging: B % 4 == 0 -> a 2-D TMA box per tile + a 1-D bulk copy of its
// entries, issued by one thread into a double buffer, completion on one
// mbarrier per buffer; otherwise (ragged B) a synchronous per-element path.
template <int VEC, int RPW, int NW, int EPI, bool SENT, bool CONV>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1)
    spmm_tiled_kernel(const SpmmArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int BT = 32 * VEC;
    constexpr int NT = NW * 32;
    constexpr int RB = NW * RPW;
    extern __shared__ __align__(128) float smem[];  // [2][KC][BT] floats, [2][cap+2] int2
    __shared__ uint64_t full[2];
    __shared__ int released[2];  // TMA path: warps done with each buffer (the last one refills it)
    __shared__ int tile_ea[2];   // TMA path: first staged entry of the tile in each buffer, set by its issuer
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * (a.KC + 1) * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rb = blockIdx.x;
    const int64_t b0 = (int64_t)blockIdx.y * BT;
    const int64_t B = a.B;
    const bool vec4 = CONV || a.tma != 0;  // TMA path (B % 4 == 0 and a tensor map)
    const size_t tile_sz = (size_t)a.KC * BT;
    const size_t buf_sz = tile_sz + BT;  // a zero row (what padding entries read) + the tile
    const int ebuf = a.cap + 2;
    const int ntile = CONV ? a.ntap * a.nkb : a.nkb;

    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        released[0] = 0;
        released[1] = 0;
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < BT; i += NT) {  // the zero rows in front of the two tiles
        smem[i] = 0.f;
        smem[buf_sz + i] = 0.f;
    }
    __syncthreads();

    // tile q -> (tap t, column block kb) and its tiling arrays
    auto tap_of = [&](int q) { return CONV ? q / a.nkb : 0; };
    auto kb_of = [&](int q) { return CONV ? q - (q / a.nkb) * a.nkb : q; };
    auto seg_of = [&](int t) -> const int32_t * { return CONV ? a.taps[t].seg : a.seg; };
    auto ent_of = [&](int t) -> const int2 * { return CONV ? a.taps[t].ent : a.ent; };
    auto entry_range = [&](int q, int &e0, int &e1) {
        const int64_t tb = ((int64_t)rb * a.nkb + kb_of(q)) * RB;
        const int32_t *sgp = seg_of(tap_of(q));
        e0 = __ldg(sgp + tb) & ~1;
        e1 = __ldg(sgp + tb + RB);
    };
    // issue tile q into buffer buf (one thread, TMA path)
    auto issue = [&](int q, int buf) {
        const int t = tap_of(q);
        const int64_t k0 = (int64_t)kb_of(q) * a.KC;
        int e0 = 0, e1 = 0;
        if constexpr (SENT) entry_range(q, e0, e1);
        const unsigned eb = SENT ? (unsigned)(((e1 - e0) * 8 + 15) & ~15) : 0u;
        if constexpr (SENT) tile_ea[buf] = e0;  // published to the consumers by the arrive below (release)
        // the box is always KC x BT floats (OOB rows / columns zero-filled)
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        tma_load_2d(smem + buf * buf_sz + BT, &tmap, (int)(b0 + (CONV ? a.sh[t] : 0)), (int)k0, &full[buf]);
        if (eb) tma_load_1d(ents + buf * ebuf, ent_of(t) + e0, eb, &full[buf]);
    };
    pdl_wait();  // (launched as a programmatic dependent: the prologue above overlapped the previous kernel)
    if (vec4 && threadIdx.x == 0) {
        issue(0, 0);
        if (ntile > 1) issue(1, 1);
    }
    pdl_trigger();  // (a split-row reduction may follow as a programmatic dependent)

    // lane l <= RPW holds the l-th segment bound of this warp's rows in tile q
    // (rows rb*RB + warp*RPW + i).
    auto seg_bounds = [&](int q) -> int {
        const int32_t *segw = seg_of(tap_of(q)) + ((int64_t)rb * a.nkb + kb_of(q)) * RB + warp * RPW;
        return lane <= RPW ? __ldg(segw + lane) : 0;
    };
    int sg = seg_bounds(0);
    if constexpr (!SENT) prefetch_entries(ent_of(0), __shfl_sync(kFull, sg, 0), __shfl_sync(kFull, sg, RPW), lane);

    float acc[RPW][VEC];
#pragma unroll
    for (int i = 0; i < RPW; ++i)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;

    for (int q = 0; q < ntile; ++q) {
        const int buf = q & 1;
        const int kb = kb_of(q);
        int sgn = 0;
        if (q + 1 < ntile) {
            sgn = seg_bounds(q + 1);
            if constexpr (!SENT)
                prefetch_entries(ent_of(tap_of(q + 1)), __shfl_sync(kFull, sgn, 0), __shfl_sync(kFull, sgn, RPW),
                                 lane);
        }
        int ea = 0;
        if (vec4) {
            mbar_wait(&full[buf], (q >> 1) & 1);
            if constexpr (SENT) {
#ifndef SP_SPMM_EA_LDG
                ea = tile_ea[buf];  // (a shared-memory read instead of two dependent global ones)
#else
                int e1;
                entry_range(q, ea, e1);
#endif
            }
        } else {  // ragged B: synchronous staging of this tile (never CONV)
            const int64_t k0 = (int64_t)kb * a.KC;
            stage_tile<BT, NT>(smem + buf * buf_sz + BT, a.in, k0, (int)std::min<int64_t>(a.KC, a.inner - k0), B, b0,
                               false);
            if constexpr (SENT) {
                int e1;
                entry_range(q, ea, e1);
                for (int i = threadIdx.x; i < e1 - ea; i += NT) ents[buf * ebuf + i] = __ldg(a.ent + ea + i);
            }
            __syncthreads();
        }
        // tile row byte offsets are stored for 128-float rows; narrower tiles shift
        constexpr int SH = VEC == 4 ? 0 : VEC == 2 ? 1 : 2;
        const char *tb = reinterpret_cast<const char *>(smem + buf * buf_sz + BT + lane * VEC);
        const int2 *gent = ent_of(tap_of(q));
        const int2 *es = SENT ? ents + buf * ebuf - ea : gent;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int s0 = __shfl_sync(kFull, sg, i), s1 = __shfl_sync(kFull, sg, i + 1);
            // segments are padded to even lengths (weight-0 entries); groups of 4
            for (int e = s0; e < s1; e += 4) {
                // 4 entries in two 16-byte broadcast loads; the second pair is masked
                // (no load, weight 0) when it lies past the segment
                const int4 p01 = ld_entry_pair(es + e, SENT);
                const int4 p23 = ld_entry_pair(es + e + 2, SENT);
                const int off[4] = {p01.x, p01.z, p23.x, p23.z};
                const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w), __int_as_float(p23.y),
                                    __int_as_float(p23.w)};
                float x[4][VEC];
                if (e + 2 < s1) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) lds_vec<VEC>(reinterpret_cast<const float *>(tb + (off[u] >> SH)), x[u]);
#pragma unroll
                    for (int u = 0; u < 4; ++u) fma_bcast<VEC>(acc[i], w[u], x[u]);
                } else {  // last pair of the segment
#pragma unroll
                    for (int u = 0; u < 2; ++u) lds_vec<VEC>(reinterpret_cast<const float *>(tb + (off[u] >> SH)), x[u]);
#pragma unroll
                    for (int u = 0; u < 2; ++u) fma_bcast<VEC>(acc[i], w[u], x[u]);
                }
            }
        }
        if (vec4) {  // release the buffer; the last warp done with tile q refills it with tile q+2
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&released[buf], 1) == NW - 1) {
                    released[buf] = 0;
                    __threadfence_block();
                    if (q + 2 < ntile) issue(q + 2, buf);
                }
            }
        } else {
            __syncthreads();  // everyone done with this buffer before it is restaged
        }
        sg = sgn;
    }

    const int64_t bl = b0 + lane * VEC;
    if constexpr (CONV) {
        // compact store of the valid output columns (VEC-aligned groups share (p, q))
        const int64_t pq = bl / B, b = bl - pq * B;
        const int64_t qq = pq % a.Wv, pp = pq / a.Wv;
        if (pp >= a.OHv || qq >= a.OWv) return;
        const int64_t col = (pp * a.OWv + qq) * B + b, rowlen = a.OHv * a.OWv * B;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int64_t r = (int64_t)rb * RB + warp * RPW + i;
            if (r >= a.rows) continue;
            float *dst = a.out + r * rowlen + col;  // (tap tilings keep the identity row order)
            if constexpr (VEC == 4) *reinterpret_cast<float4 *>(dst) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            else
#pragma unroll
                for (int v = 0; v < VEC; ++v) dst[v] = acc[i][v];
        }
        return;
    } else {
    // Epilogue: ReLU / ReLU' gate fused; each element written once.
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t tpos = (int64_t)rb * RB + warp * RPW + i;
        const int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + tpos) : tpos;
        if (r < 0 || r >= a.rows) continue;
        if (a.psplit) {  // a part row: raw sums to its slot (split_reduce applies the epilogue)
            const int sv = __ldg(a.psplit + tpos);
            if (sv >= 0) {
#pragma unroll
                for (int v = 0; v < VEC; ++v)
                    if (bl + v < B) a.vpart[(int64_t)sv * B + bl + v] = acc[i][v];
                continue;
            }
        }
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
        if ((B & 3) == 0 && VEC > 1 && bl + VEC <= B) {
            if constexpr (VEC == 2) *reinterpret_cast<float2 *>(dst) = make_float2(o[0], o[1]);
            if constexpr (VEC == 4) *reinterpret_cast<float4 *>(dst) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (bl + v < B) dst[v] = o[v];
        }
    }
    }  // (not CONV)
}

// The stream-K SpMM (spmm_sk.cu) runs when the per-item grid is short (< 2
// waves of 128-row items) and the items are long (>= 8 column blocks) -- e.g.
// the 768-row cfg5 layer at a per-rank batch of 2048-4096: +10-17%.  Elsewhere
// the per-item grid wins (measured) and keeps every output element's order
// independent of B.
constexpr int kSmemLimit = 226 * 1024;  // per SM, usable by CTAs (minus static mbarriers)

template <int VEC, int RPW, int NW>
void launch_cfg(const sp_tiling &t, int64_t B, const float *in, float *out, const float *gate, int epi,
                cudaStream_t st) {
    constexpr int BT = 32 * VEC;
    const size_t tiles = (size_t)2 * (t.KC + 1) * BT * sizeof(float);
    // stage the entries too when both buffers fit next to the activation tiles
    const int cap = (t.max_tile + 2 + 3) & ~3;  // keeps both entry buffers 16-byte aligned
    const bool sent = tiles + (size_t)2 * (cap + 2) * sizeof(int2) <= (size_t)kSmemLimit / (NW == 8 ? 2 : 1);
    const size_t smem = tiles + (sent ? (size_t)2 * (cap + 2) * sizeof(int2) : 0);
    CUtensorMap tmap{};
    const bool tma = (B & 3) == 0 && make_tmap_2d(&tmap, in, t.inner, B, BT, t.KC);
    float *vpart = nullptr;
    if (t.split && scratch_alloc((void **)&vpart, (size_t)t.nparts * B * sizeof(float), st) != cudaSuccess) return;
    SpmmArgs a{t.rows, t.inner, B, t.KC, t.nkb, cap, tma ? 1 : 0, t.seg, t.ent, in, out, gate, t.rowmap,
               t.split, vpart, 0, nullptr, {}, 0, 0, 0};
    dim3 grid((unsigned)t.nrb, (unsigned)((B + BT - 1) / BT));
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        note_path("spmm_tiled");
        launch_pdl(kern, grid, dim3(NW * 32), smem, st, a, tmap);
        if (vpart) {
            launch_split_rows_reduce(t, vpart, B, out, gate, epi, st);
            scratch_free(vpart, st);
        }
    };
    if (sent) {
        if (epi == EPI_RELU) launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_RELU, true, false>);
        else if (epi == EPI_GATE) launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_GATE, true, false>);
        else launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_NONE, true, false>);
    } else {
        if (epi == EPI_RELU) launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_RELU, false, false>);
        else if (epi == EPI_GATE) launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_GATE, false, false>);
        else launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_NONE, false, false>);
    }
}

// variant 0: RB = 128 = 32 warps x 4 rows, KC = 192 (1 CTA / SM);
// variant 1: RB = 32 = 8 warps x 4 rows, KC = 96 (2 CTAs / SM).
template <int VEC>
void launch_variant(const sp_tiling &t, int v, int64_t B, const float *in, float *out, const float *gate,
                    int epi, cudaStream_t st) {
    if (v == 0) launch_cfg<VEC, 4, 32>(t, B, in, out, gate, epi, st);
    else launch_cfg<VEC, 4, 8>(t, B, in, out, gate, epi, st);
}

template <int VEC>
bool conv_spmm_vec(const sp_weight_s *w, int orient, int64_t B, const float *in, int64_t Lp, float *out,
                   const int *sh, int ntap, int64_t Wv, int64_t OHv, int64_t OWv, cudaStream_t st) {
    constexpr int RPW = 8, NW = 16, BT = 32 * VEC;
    const sp_tiling &t0 = w->tap[0][orient];
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, in, t0.inner, Lp, BT, t0.KC)) return false;
    int mx = 0;
    for (int t = 0; t < ntap; ++t) mx = std::max(mx, w->tap[t][orient].max_tile);
    const int cap = (mx + 2 + 3) & ~3;
    const size_t tiles = (size_t)2 * (t0.KC + 1) * BT * sizeof(float);
    const bool sent = tiles + (size_t)2 * (cap + 2) * sizeof(int2) <= (size_t)kSmemLimit;
    const size_t smem = tiles + (sent ? (size_t)2 * (cap + 2) * sizeof(int2) : 0);
    SpmmArgs a{t0.rows, t0.inner, B, t0.KC, t0.nkb, cap, 1, nullptr, nullptr, nullptr, out, nullptr, nullptr,
               nullptr, nullptr, ntap, w->tapdev + orient * kMaxTaps, {}, Wv, OHv, OWv};
    for (int t = 0; t < ntap; ++t) a.sh[t] = sh[t];
    const int64_t Nv = OHv * Wv * B;
    dim3 grid((unsigned)t0.nrb, (unsigned)((Nv + BT - 1) / BT));
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        count_launches(1);
        note_path("conv_spmm_tiled");
        launch_pdl(kern, grid, dim3(NW * 32), smem, st, a, tmap);
    };
    if (sent) launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_NONE, true, true>);
    else launch(spmm_tiled_kernel<VEC, RPW, NW, EPI_NONE, false, true>);
    return true;
}

}  // namespace

// Conv products as tap-tiled SpMM on a padded copy (see conv.cu; the fallback
// of the exact-column stream-K path for batch sizes it cannot slice): in = padded activation
// [inner x Lp], taps[t] tilings of orientation `orient`, shift sh[t] columns;
// virtual output columns Nv = OHv * Wv * B stored compactly.  Narrower batch
// slices when the grid would not fill two waves.
bool launch_conv_spmm(const sp_weight_s *w, int orient, int64_t B, const float *in, int64_t Lp, float *out,
                      const int *sh, int ntap, int64_t Wv, int64_t OHv, int64_t OWv, cudaStream_t st) {
    const int64_t Nv = OHv * Wv * B;
    if ((int64_t)w->tap[0][orient].nrb * ((Nv + 127) / 128) >= 2 * num_sms())
        return conv_spmm_vec<4>(w, orient, B, in, Lp, out, sh, ntap, Wv, OHv, OWv, st);
    return conv_spmm_vec<2>(w, orient, B, in, Lp, out, sh, ntap, Wv, OHv, OWv, st);
}

void launch_spmm(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out,
                 const float *gate, int epi, cudaStream_t st) {
    if (w->nnz == 0 || gather_preferred(w, orient, B)) {  // staging would move more bytes than gathering
        if (w->nnz == 0) {
            cudaMemsetAsync(out, 0, (size_t)((orient == 0 ? w->R : w->C) * B) * sizeof(float), st);
            return;
        }
        if (!launch_gather_pos(w, orient, 0, B, in, nullptr, gate, epi, out, nullptr, st))
            launch_spmm_gather(w, orient, B, in, out, gate, epi, st);
        return;
    }
    {
        const sp_tiling &t0 = w->til[orient][0];
        const int64_t items = (int64_t)t0.nrb * ((B + 127) / 128);
        if (items < 2 * num_sms() && t0.nkb >= 8 && launch_spmm_sk(w, orient, B, in, out, gate, epi, st)) return;
    }
    // Choose the largest row block and batch vector that still fill the GPU.
    int vec = B <= 32 ? 1 : (B <= 64 || (B & 3)) ? 2 : 4;
    int var = 0;
    auto ctas = [&](int v, int vv) {
        return (int64_t)w->til[orient][v].nrb * ((B + 32 * vv - 1) / (32 * vv));
    };
#ifndef SP_VAR1_BELOW_X10
#define SP_VAR1_BELOW_X10 6  // (was 20: cfg2a fwd 28.7 -> 24.6 us on the 32-warp kernel, 96 CTAs)
#endif
    if (ctas(0, vec) * 10 < SP_VAR1_BELOW_X10 * num_sms()) var = 1;
    while (var == 1 && vec > 1 && ctas(1, vec) < 2 * num_sms()) vec >>= 1;
    // the 32-warp layout takes the split-source kernel: the same entries in the
    // same order (bitwise the shared-memory kernel's result), a third of the
    // gathers from TMEM
    if (var == 0 && vec == 4) {
        // A per-item grid whose last wave is less than half full leaves most SMs
        // idle for a whole item: its items (whole batch slices) go to the
        // stream-K kernel over every SM first, then the split-source grid runs
        // the full waves (768-row cfg5 layer at B = 16384: 768 items = 5.19
        // waves, 372 us; the 738 items of 4.99 waves take 314 us; split: 343-353 us)
        const sp_tiling &t0 = w->til[orient][0];
        const int64_t nsl = (B + 127) / 128, items = (int64_t)t0.nrb * nsl, G = num_sms();
        const int64_t s1 = (items / G) * G / std::max(t0.nrb, 1);  // whole slices within the full waves
#ifndef SP_NO_WAVE_TAIL
#ifndef SP_TAIL_X10
#define SP_TAIL_X10 5  // last wave under half full (70 %: the 768-row layer at B = 8192, 59 % full, 186.4 -> 185.7 us only)
#endif
        if (items > G && items % G > 0 && 10 * (items % G) < SP_TAIL_X10 * G && s1 > 0 && s1 < nsl && t0.split == nullptr &&
            t0.nkb >= 8 &&  // (long items only: on 4-tile items the tail's cut items cost more, 3072-row layer)
            launch_spmm_sk(w, orient, B, in, out, gate, epi, st, s1, nsl)) {
            if (launch_spmm_hyb(w, orient, B, in, out, gate, epi, st, s1)) return;
            // (cannot happen for the shapes that reach here; complete the slices plainly)
            refresh_if_stale(w, w->til[orient][0], st);
            launch_variant<4>(w->til[orient][0], 0, B, in, out, gate, epi, st);
            return;
        }
#endif
        if (launch_spmm_hyb(w, orient, B, in, out, gate, epi, st)) return;
    }
    const sp_tiling &t = w->til[orient][var];
    refresh_if_stale(w, t, st);
    if (vec == 4) launch_variant<4>(t, var, B, in, out, gate, epi, st);
    else if (vec == 2) launch_variant<2>(t, var, B, in, out, gate, epi, st);
    else launch_variant<1>(t, var, B, in, out, gate, epi, st);
}

}  // namespace sp
