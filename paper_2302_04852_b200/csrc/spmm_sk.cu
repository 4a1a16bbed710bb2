// spmm_sk.cu -- stream-K schedule of the tiled SpMM (forward Y = W X, P141;
// CSC-driven dX = W^T dY, Eq. 1): one wave of CTAs, each running an equal
// contiguous range of the tile sequence (row block rb, batch slice sl, column
// block kb), so small or ragged problems (few batch slices, few row blocks)
// still occupy every SM and no CTA pays a pipeline start per item.
//
// An item (rb, sl) whose kb range is cut by range boundaries is finished by
// the last of its CTAs to arrive (per-item ticket): every part stores its raw
// sums, and the last one adds the parts in CTA order -- a fixed order, so the
// result is deterministic -- applies the epilogue (ReLU / ReLU' gate) and
// writes the output.  Tiles are staged exactly as in spmm.cu (2-D TMA box of
// the activation + 1-D bulk copy of the entries, two buffers, the last warp
// done with a buffer refills it).
#include <cuda_runtime.h>

#include <algorithm>

#include "sp_internal.cuh"
#include "tile.cuh"

namespace sp {
namespace {

// The gathers below load slots 0..2 of an entry group (0 of a last pair)
// unpredicated: that is only safe while every segment is padded to an EVEN
// length, so that a segment's last slot is the only one that can be padding.
static_assert(kTilPad == 2 && kTapPad == 2, "only a segment's last slot may be padding");


__host__ __device__ __forceinline__ int64_t lo_of(int64_t c, int64_t T, int64_t G) { return c * T / G; }
__host__ __device__ __forceinline__ int64_t cta_of(int64_t t, int64_t T, int64_t G) {
    int64_t c = t * G / T;
    while (c + 1 < G && lo_of(c + 1, T, G) <= t) ++c;
    while (c > 0 && lo_of(c, T, G) > t) --c;
    return c;
}

struct SkArgs {
    int64_t rows, B, nslice;
    int KC, nkb, nrb, cap;
    const int32_t *seg;
    const int2 *ent;
    float *out;
    const float *gate;
    const int32_t *rowmap;
    const int32_t *psplit;  // tiled position -> part slot of a split row (-1 whole; nullptr: none)
    float *vpart;          // [nparts x B] raw sums of the part rows
    const int32_t *split;  // TMM: tmsplit of the (linear) tiling
    float *part;    // [G][2][RB][BT] raw sums of cut items (slot 0: the CTA's first item, 1: its last)
    int *tickets;   // [nrb * nslice], zero on entry, reset by the finishing CTA
    // conv (CONV = true): an item's tiles run over (tap t, column block); tap t uses
    // taps[t]'s tiling and a 4-D TMA box of the CHWN input at the slice's exact
    // output positions offset by (dp[t], dq[t]) (halo zero-filled by the hardware);
    // column c of slice sl is out[r][p][q][b] (ConvCols)
    int ntap;
    const TapDev *taps;
    ConvCols cc;
    int s0;  // linear: the first batch slice (slice sl of the grid covers columns (s0 + sl) * BT ..)
};

// TMM: the last kHybTC rows of every tile are mirrored in tensor memory and a
// segment's tail (from its tmsplit index) is gathered from there once the copy
// is complete -- the split-source scheme of spmm_hyb.cu (same entries, same
// order: bitwise the same result)
template <int RPW, int NW, int EPI, bool CONV, bool TMM = false>
__global__ void __launch_bounds__(NW * 32, 1)
    spmm_sk_kernel(const SkArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int VEC = 4;
    constexpr int BT = 32 * VEC;
    constexpr int RB = NW * RPW;
    extern __shared__ __align__(128) float smem[];  // [2][KC][BT] floats, [2][cap+2] int2
    __shared__ uint64_t full[2], tfull[2];
    __shared__ int released[2], ticket[2];
    __shared__ int tile_ea[2];  // first staged entry of the tile in each buffer, set by its issuer
    __shared__ int last_flag;
    __shared__ uint32_t tmem_base;
    int2 *ents = reinterpret_cast<int2 *>(smem + (size_t)2 * a.KC * BT);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t B = a.B;
    const int tpi = CONV ? a.ntap * a.nkb : a.nkb;  // tiles per item
    const int64_t T = (int64_t)a.nrb * a.nslice * tpi, G = gridDim.x;
    const int t0 = (int)lo_of(blockIdx.x, T, G);  // T < 2^31 (launcher)
    const int ntile = (int)lo_of(blockIdx.x + 1, T, G) - t0;
    const int nsl = (int)a.nslice;
    const size_t tile_sz = (size_t)a.KC * BT;
    const int ebuf = a.cap + 2;
    const int first_item = t0 / tpi;

    constexpr int kIssue = 8;  // warps issuing a tile's TMEM copies (TMM)
    const int c0 = a.KC - kHybTC;  // first mirrored tile row (TMM)
    if (TMM && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        released[0] = 0;
        released[1] = 0;
        if (TMM) {
            mbar_init(&tfull[0], kIssue);
            mbar_init(&tfull[1], kIssue);
            ticket[0] = 0;
            ticket[1] = 0;
        }
        fence_mbar_init();
    }
    uint32_t tq = 0;
    if constexpr (TMM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
        if (warp < 4) {  // zero columns in front of each TMEM buffer (padding entries read them)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq), "r"(0u) : "memory");
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tq + 256), "r"(0u)
                         : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (TMM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    struct Tile {
        int rb, sl, r;  // r: tile within the item (tap * nkb + kb for conv)
    };
    auto tap_of = [&](const Tile &id) { return CONV ? id.r / a.nkb : 0; };
    auto kb_of = [&](const Tile &id) { return CONV ? id.r - (id.r / a.nkb) * a.nkb : id.r; };
    auto seg_of = [&](const Tile &id) -> const int32_t * { return CONV ? a.taps[tap_of(id)].seg : a.seg; };
    auto ent_of = [&](const Tile &id) -> const int2 * { return CONV ? a.taps[tap_of(id)].ent : a.ent; };
    auto tile_of = [&](int q) -> Tile {
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
        const int64_t tb = ((int64_t)id.rb * a.nkb + kb_of(id)) * RB;
        const int32_t *sgp = seg_of(id);
        e0 = __ldg(sgp + tb) & ~1;
        e1 = __ldg(sgp + tb + RB);
    };
    auto issue = [&](int q, int buf) {
        const Tile id = tile_of(q);
        int e0, e1;
        entry_range(id, e0, e1);
        const unsigned eb = (unsigned)(((e1 - e0) * 8 + 15) & ~15);
        tile_ea[buf] = e0;  // published to the consumers by the arrive below (release)
        mbar_arrive_expect_tx(&full[buf], (unsigned)(tile_sz * sizeof(float)) + eb);
        if constexpr (CONV) {
            int c[4];
            cc_coords(a.cc, id.sl, tap_of(id), kb_of(id) * a.KC, c);
            tma_load_4d(smem + buf * tile_sz, &tmap, c[0], c[1], c[2], c[3], &full[buf]);
        } else {
            tma_load_2d(smem + buf * tile_sz, &tmap, (id.sl + a.s0) * BT, kb_of(id) * a.KC, &full[buf]);
        }
        if (eb) tma_load_1d(ents + buf * ebuf, ent_of(id) + e0, eb, &full[buf]);
    };
    pdl_wait();  // (launched as a programmatic dependent: the prologue above overlapped the previous kernel)
    if (threadIdx.x == 0) {
        if (ntile > 0) issue(0, 0);
        if (ntile > 1) issue(1, 1);
    }
    pdl_trigger();  // (a split-row reduction may follow as a programmatic dependent)
    // lane l <= RPW: the l-th segment bound of this warp's rows; TMM: lanes 8 + i
    // hold row i's tmsplit
    auto split_of = [&](const Tile &id) -> const int32_t * { return CONV ? a.taps[tap_of(id)].split : a.split; };
    auto seg_bounds = [&](const Tile &id) -> int {
        const int64_t sb = ((int64_t)id.rb * a.nkb + kb_of(id)) * RB + warp * RPW;
        if (lane <= RPW) return __ldg(seg_of(id) + sb + lane);
        if (TMM && lane >= 8 && lane < 8 + RPW) return __ldg(split_of(id) + sb + lane - 8);
        return 0;
    };
    // epilogue of rows (rb, lr = warp*RPW + i) for batch columns bl..bl+3
    auto store = [&](int rb, int i, int64_t bl, const float (&v)[VEC]) {
        const int64_t tpos = (int64_t)rb * RB + warp * RPW + i;
        if constexpr (CONV) {  // exact output positions (tap tilings: identity rows)
            if (tpos >= a.rows) return;
            const int64_t off = cc_off(a.cc, (int)(bl / BT), (int)(bl % BT));
            if (off < 0) return;
            float *dst = a.out + tpos * a.cc.rowlen + off;
            *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
            return;
        }
        const int64_t r = a.rowmap ? (int64_t)__ldg(a.rowmap + tpos) : tpos;
        if (r < 0 || r >= a.rows || bl >= B) return;
        if (a.psplit) {  // a part row: raw sums to its slot (split_reduce applies the epilogue)
            const int sv = __ldg(a.psplit + tpos);
            if (sv >= 0) {
                *reinterpret_cast<float4 *>(a.vpart + (int64_t)sv * B + bl) = make_float4(v[0], v[1], v[2], v[3]);
                return;
            }
        }
        float o[VEC];
#pragma unroll
        for (int u = 0; u < VEC; ++u) {
            float x = v[u];
            if (EPI == EPI_RELU) x = fmaxf(x, 0.f);
            if (EPI == EPI_GATE) x = __ldg(a.gate + r * B + bl + u) > 0.f ? x : 0.f;
            o[u] = x;
        }
        *reinterpret_cast<float4 *>(a.out + r * B + bl) = make_float4(o[0], o[1], o[2], o[3]);
    };

    float acc[RPW][VEC];
    int r_first = 0;
    Tile nid = tile_of(0);
    int sgn = ntile > 0 ? seg_bounds(nid) : 0;
    for (int q = 0; q < ntile; ++q) {
        const Tile id = nid;
        const int buf = q & 1;
        if (q == 0 || id.r == 0) {  // new item
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;
            r_first = id.r;
        }
        const int sg = sgn;
        nid = next_tile(id);
        if (q + 1 < ntile) sgn = seg_bounds(nid);
        const unsigned par = (unsigned)(q >> 1) & 1u;
        mbar_wait(&full[buf], par);
        if constexpr (TMM) {  // the first kIssue warps to start the tile copy its last rows into TMEM
            if (lane == 0) {
                const int tk = atomicAdd(&ticket[buf], 1);
                if (tk == NW - 1) ticket[buf] = 0;
                if (tk < kIssue) {
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t dst = tmem_base + (uint32_t)(buf * 256 + 4);
                    const float *src = smem + buf * tile_sz + (size_t)c0 * BT;
                    for (int c = tk; c < kHybTC; c += kIssue) {
                        const uint64_t d = (uint64_t)((smem_u32(src + c * BT) >> 4) & 0x3FFF) |
                                           ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
                        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dst + 4 * c), "l"(d)
                                     : "memory");
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&tfull[buf]))
                                 : "memory");
                }
            }
            __syncwarp();
        }
#ifndef SP_SPMM_EA_LDG
        // (a shared-memory read instead of two dependent global ones: stream-K SpMM
        // -3 to -5 %; the split-source kernel measured slower with it and keeps the loads)
        const int ea = tile_ea[buf];
#else
        int ea, e1t;
        entry_range(id, ea, e1t);
#endif
        // 32-bit shared-window bases pinned in registers (see pin_u32)
        const uint32_t tbs = pin_u32(smem_u32(smem + buf * tile_sz + lane * VEC));
        const uint32_t ess = pin_u32(smem_u32(ents + buf * ebuf) - (uint32_t)ea * 8u);
        // groups of 4 entries (a last lone pair) of [e0, e1) from shared memory
        auto lds_part = [&](float (&ac)[VEC], int e0, int e1) {
            for (int e = e0; e < e1; e += 4) {
                const int4 p01 = lds_entry_pair_s(ess + (uint32_t)e * 8u);
                const int4 p23 = lds_entry_pair_s(ess + (uint32_t)(e + 2) * 8u);
                const int off[4] = {p01.x, p01.z, p23.x, p23.z};
                const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w), __int_as_float(p23.y),
                                    __int_as_float(p23.w)};
                float x[4][VEC];
                if (e + 2 < e1) {
#pragma unroll
                    for (int u = 0; u < 3; ++u) lds_row_s<VEC>(tbs, off[u], x[u]);  // even padding: only the
                    lds_row_or_zero_s<VEC>(tbs, off[3], x[3]);                        // last slot can be padding
#pragma unroll
                    for (int u = 0; u < 4; ++u) fma_bcast<VEC>(ac, w[u], x[u]);
                } else {  // last pair of the segment
                    lds_row_s<VEC>(tbs, off[0], x[0]);
                    lds_row_or_zero_s<VEC>(tbs, off[1], x[1]);
#pragma unroll
                    for (int u = 0; u < 2; ++u) fma_bcast<VEC>(ac, w[u], x[u]);
                }
            }
        };
        if constexpr (!TMM) {
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int s0 = __shfl_sync(kFull, sg, i), s1 = __shfl_sync(kFull, sg, i + 1);
                lds_part(acc[i], s0, s1);
            }
        } else {
            // TMEM column = tb0 + (offset >> 7) in the mirrored rows; padding entries
            // (offset < 0, at a segment's end) select the zero columns
            const uint32_t tcol = tq + (uint32_t)(buf * 256);
            const uint32_t tb0 = pin_u32(tcol + (uint32_t)(4 - 4 * c0));
            // segments (linear and conv tap tilings) are padded to even lengths, so
            // only a segment's last slot can be padding
            auto tcolumn = [&](int off) -> uint32_t { return off >= 0 ? tb0 + (uint32_t)(off >> 7) : tcol; };
            auto tcol_real = [&](int off) -> uint32_t { return tb0 + (uint32_t)(off >> 7); };
            bool tm_ok = false;
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const int s0 = __shfl_sync(kFull, sg, i), s1 = __shfl_sync(kFull, sg, i + 1);
                const int sp = __shfl_sync(kFull, sg, 8 + i);
                lds_part(acc[i], s0, sp);
                if (sp < s1 && !tm_ok) {  // is the TMEM copy of this tile complete yet? (non-blocking)
                    unsigned ok;
                    asm volatile(
                        "{\n.reg .pred P;\nmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}\n"
                        : "=r"(ok)
                        : "r"(smem_u32(&tfull[buf])), "r"(par)
                        : "memory");
                    tm_ok = __shfl_sync(kFull, (int)ok, 0) != 0;
                    if (tm_ok) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                if (!tm_ok) {
                    lds_part(acc[i], sp, s1);
                    continue;
                }
                for (int e = sp; e < s1; e += 4) {
                    const int4 p01 = lds_entry_pair_s(ess + (uint32_t)e * 8u);
                    const int4 p23 = lds_entry_pair_s(ess + (uint32_t)(e + 2) * 8u);
                    uint32_t r[16];
                    if (e + 2 < s1) {
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%16];\n"
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%17];\n"
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%18];\n"
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12, %13, %14, %15}, [%19];\n"
                            "tcgen05.wait::ld.sync.aligned;"
                            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                              "=r"(r[14]), "=r"(r[15])
                            : "r"(tcol_real(p01.x)), "r"(tcol_real(p01.z)), "r"(tcol_real(p23.x)), "r"(tcolumn(p23.z))
                            : "memory");
                        const float w[4] = {__int_as_float(p01.y), __int_as_float(p01.w), __int_as_float(p23.y),
                                            __int_as_float(p23.w)};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float x[VEC] = {__uint_as_float(r[4 * u]), __uint_as_float(r[4 * u + 1]),
                                                  __uint_as_float(r[4 * u + 2]), __uint_as_float(r[4 * u + 3])};
                            fma_bcast<VEC>(acc[i], w[u], x);
                        }
                    } else {
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%8];\n"
                            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%9];\n"
                            "tcgen05.wait::ld.sync.aligned;"
                            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                              "=r"(r[7])
                            : "r"(tcol_real(p01.x)), "r"(tcolumn(p01.z))
                            : "memory");
                        const float w[2] = {__int_as_float(p01.y), __int_as_float(p01.w)};
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const float x[VEC] = {__uint_as_float(r[4 * u]), __uint_as_float(r[4 * u + 1]),
                                                  __uint_as_float(r[4 * u + 2]), __uint_as_float(r[4 * u + 3])};
                            fma_bcast<VEC>(acc[i], w[u], x);
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        }
        // release the buffer; the last warp to finish tile q refills it with tile q+2
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&released[buf], 1) == NW - 1) {
                released[buf] = 0;
                __threadfence_block();
                if (q + 2 < ntile) {
                    if constexpr (TMM) mbar_wait(&tfull[buf], (unsigned)(q >> 1) & 1u);  // the copies read the buffer
                    issue(q + 2, buf);
                }
            }
        }
        if (id.r != tpi - 1 && q != ntile - 1) continue;

        // ---- this CTA's part of item (rb, sl) is done
        const int64_t bl = (int64_t)(id.sl + a.s0) * BT + lane * VEC;
        if (r_first == 0 && id.r == tpi - 1) {  // whole item: store directly
#pragma unroll
            for (int i = 0; i < RPW; ++i) store(id.rb, i, bl, acc[i]);
            continue;
        }
        const int item = id.rb * nsl + id.sl;
        const int slot = item == first_item ? 0 : 1;
        float *mine = a.part + ((int64_t)(blockIdx.x * 2 + slot) * RB + warp * RPW) * BT + lane * VEC;
#pragma unroll
        for (int i = 0; i < RPW; ++i)
            *reinterpret_cast<float4 *>(mine + i * BT) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        __threadfence();
        __syncthreads();
        const int64_t c0 = cta_of((int64_t)item * tpi, T, G), c1 = cta_of((int64_t)item * tpi + tpi - 1, T, G);
        if (threadIdx.x == 0) {
            const int old = atomicAdd(a.tickets + item, 1);
            last_flag = old == (int)(c1 - c0);
            if (last_flag) a.tickets[item] = 0;  // ready for the next launch
        }
        __syncthreads();
        if (!last_flag) continue;
        __threadfence();
        // last part in: sum the parts in CTA order, epilogue, store
        float sum[RPW][VEC];
#pragma unroll
        for (int i = 0; i < RPW; ++i)
#pragma unroll
            for (int v = 0; v < VEC; ++v) sum[i][v] = 0.f;
        for (int64_t c = c0; c <= c1; ++c) {
            const int s = item == (int)(lo_of(c, T, G) / tpi) ? 0 : 1;
            const float *pp = a.part + ((c * 2 + s) * RB + warp * RPW) * BT + lane * VEC;
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
        for (int i = 0; i < RPW; ++i) store(id.rb, i, bl, sum[i]);
    }
    if constexpr (TMM) {  // the copies of the last tiles complete before TMEM is released
        if (threadIdx.x == 0)
            for (int q = ntile > 2 ? ntile - 2 : 0; q < ntile; ++q) mbar_wait(&tfull[q & 1], (unsigned)(q >> 1) & 1u);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

}  // namespace

bool launch_spmm_sk(const sp_weight_s *w, int orient, int64_t B, const float *in, float *out, const float *gate,
                    int epi, cudaStream_t st, int64_t s_begin, int64_t s_end) {
    constexpr int RPW = 4, NW = 32, BT = 128;
    if ((B & 3) != 0 || w->nnz == 0) return false;
    if (s_end < 0) s_end = (B + BT - 1) / BT;
    auto smem_of = [&](const sp_tiling &tt) {
        return (size_t)2 * tt.KC * BT * sizeof(float) + (size_t)2 * (((tt.max_tile + 2 + 3) & ~3) + 2) * sizeof(int2);
    };
    // the 192-column tiling, else (denser masks) the 128-column one, whose
    // staged entries fit beside the two activation tiles
    const sp_tiling *tp = &w->til[orient][0];
    if (smem_of(*tp) > (size_t)(226 * 1024) && w->til_k[orient].ent != nullptr) tp = &w->til_k[orient];
    const sp_tiling &t = *tp;
    if (t.RB != RPW * NW) return false;
    // slices [s_begin, s_end) (a sub-range: the last wave of a per-item grid, see
    // launch_spmm; part rows would need the whole batch in one launch)
    if (s_begin < 0 || s_begin >= s_end || ((s_begin > 0 || s_end < (B + BT - 1) / BT) && t.split)) return false;
    const int64_t nslice = s_end - s_begin;
    const int64_t T = (int64_t)t.nrb * nslice * t.nkb;
    if (T >= (1LL << 31)) return false;
    const int64_t G = std::min<int64_t>(num_sms(), T);
    const int cap = (t.max_tile + 2 + 3) & ~3;
    const size_t smem = smem_of(t);
    if (smem > (size_t)(226 * 1024)) return false;
    CUtensorMap tmap{};
    if (!make_tmap_2d(&tmap, in, t.inner, B, BT, t.KC)) return false;
    const int64_t nitems = (int64_t)t.nrb * nslice;
    float *part = nullptr;
    int *tickets = nullptr;
    if (scratch_alloc((void **)&part, (size_t)G * 2 * 128 * BT * sizeof(float), st) != cudaSuccess ||
        scratch_alloc((void **)&tickets, (size_t)nitems * sizeof(int), st) != cudaSuccess)
        return false;
    launch_zero_i32(tickets, nitems, st);
    refresh_if_stale(w, t, st);
    float *vpart = nullptr;
    if (t.split && scratch_alloc((void **)&vpart, (size_t)t.nparts * B * sizeof(float), st) != cudaSuccess)
        return false;
    SkArgs a{t.rows, B, nslice, t.KC, t.nkb, t.nrb, cap, t.seg, t.ent, out, gate, t.rowmap, t.split, vpart,
             t.tmsplit, part, tickets, 0, nullptr, {}};
    a.s0 = (int)s_begin;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_path(tp == &w->til_k[orient] ? "spmm_sk_k128" : "spmm_sk");
        launch_pdl(kern, dim3((unsigned)G), dim3(NW * 32), smem, st, a, tmap);
    };
    // (the TMEM mirror of the tiles' last rows measured slower on the linear
    // stream-K shapes: 768-row layer, B = 2048 / 4096: 83 -> 87 / 131 -> 143 us)
    if (epi == EPI_RELU) go(spmm_sk_kernel<RPW, NW, EPI_RELU, false>);
    else if (epi == EPI_GATE) go(spmm_sk_kernel<RPW, NW, EPI_GATE, false>);
    else go(spmm_sk_kernel<RPW, NW, EPI_NONE, false>);
    count_launches(1);
    if (vpart) {
        launch_split_rows_reduce(t, vpart, B, out, gate, epi, st);
        scratch_free(vpart, st);
    }
    scratch_free(part, st);
    scratch_free(tickets, st);
    return true;
}

// Conv products (see conv.cu) through the stream-K schedule: `in` is the CHWN
// input [inner][Hi][Wi][B] of the product (fwd: X, dX: dY), taps[t] tilings of
// orientation `orient`, exact output columns cc (Po x Qo x B per row).
bool launch_conv_spmm_sk(const sp_weight_s *w, int orient, const ConvCols &cc, const float *in, int64_t Hi,
                         int64_t Wi, float *out, int ntap, cudaStream_t st) {
    constexpr int RPW = 4, NW = 32, BT = 128;
    const sp_tiling &t0 = w->tap[0][orient];
    if (w->nnz == 0 || t0.RB != RPW * NW) return false;
    const int64_t nslice = cc.nslice;
    const int64_t T = (int64_t)t0.nrb * nslice * ntap * t0.nkb;
    if (T >= (1LL << 31)) return false;
    const int64_t G = std::min<int64_t>(num_sms(), T);
    int mx = 0;
    for (int t = 0; t < ntap; ++t) mx = std::max(mx, w->tap[t][orient].max_tile);
    const int cap = (mx + 2 + 3) & ~3;
    const size_t smem = (size_t)2 * t0.KC * BT * sizeof(float) + (size_t)2 * (cap + 2) * sizeof(int2);
    if (smem > (size_t)(226 * 1024)) return false;
    CUtensorMap tmap{};
    if (!make_tmap_conv(&tmap, in, cc, t0.inner, Hi, Wi, t0.KC)) return false;
    const int64_t nitems = (int64_t)t0.nrb * nslice;
    float *part = nullptr;
    int *tickets = nullptr;
    if (scratch_alloc((void **)&part, (size_t)G * 2 * 128 * BT * sizeof(float), st) != cudaSuccess ||
        scratch_alloc((void **)&tickets, (size_t)nitems * sizeof(int), st) != cudaSuccess)
        return false;
    launch_zero_i32(tickets, nitems, st);
    SkArgs a{t0.rows, cc.B, nslice, t0.KC, t0.nkb, t0.nrb, cap, nullptr, nullptr, out, nullptr, nullptr, nullptr,
             nullptr, nullptr, part, tickets, ntap, w->tapdev + orient * kMaxTaps, cc};
    // conv tap tiles have 128 rows: the TMEM mirror covers half of them (cfg3
    // fwd / dX 206 -> 202 / 201 us)
    bool tmm = t0.KC > kHybTC;
    for (int t = 0; t < ntap; ++t) tmm = tmm && w->tap[t][orient].tmsplit != nullptr && w->tap[t][orient].KC == t0.KC;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        note_path("conv_spmm_sk");
        launch_pdl(kern, dim3((unsigned)G), dim3(NW * 32), smem, st, a, tmap);
    };
    if (tmm) go(spmm_sk_kernel<RPW, NW, EPI_NONE, true, true>);
    else go(spmm_sk_kernel<RPW, NW, EPI_NONE, true>);
    count_launches(1);
    scratch_free(part, st);
    scratch_free(tickets, st);
    return true;
}

}  // namespace sp
