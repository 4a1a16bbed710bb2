// tile.cuh -- shared-memory staging of a dense activation tile and warp
// helpers used by the SpMM and SDDMM kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
    using T = float;
};
template <>
struct VecT<2> {
    using T = float2;
};
template <>
struct VecT<4> {
    using T = float4;
};

template <int VEC>
__device__ __forceinline__ void lds_vec(const float *p, float (&v)[VEC]) {
    if constexpr (VEC == 1) {
        v[0] = *p;
    } else if constexpr (VEC == 2) {
        float2 t = *reinterpret_cast<const float2 *>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    }
}

// Two consecutive (offset, value) entries in one 16-byte load.
__device__ __forceinline__ int4 ld_entry_pair(const int2 *p, bool smem) {
    return smem ? *reinterpret_cast<const int4 *>(p) : __ldg(reinterpret_cast<const int4 *>(p));
}

// Predicated shared loads (no branch: the destination keeps its prior value
// when the predicate is false, so callers pre-zero it).
__device__ __forceinline__ void lds128_pred(float4 &v, const void *p, bool pred) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%5];\n}\n"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
        : "r"((int)pred), "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds64_pred(float2 &v, const void *p, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.shared.v2.f32 {%0, %1}, [%3];\n}\n"
                 : "+f"(v.x), "+f"(v.y)
                 : "r"((int)pred), "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds32_pred(float &v, const void *p, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %1, 0;\n@q ld.shared.f32 %0, [%2];\n}\n"
                 : "+f"(v)
                 : "r"((int)pred), "r"(smem_u32(p)));
}

// VEC-wide load of tile row `off` (bytes from `tb`) or zeros for a padding
// entry (off < 0): the predicated-off load costs no shared-memory bandwidth
// and no branch.
template <int VEC, int SH>
__device__ __forceinline__ void lds_row_or_zero(const char *tb, int off, float (&v)[VEC]) {
    const bool ok = off >= 0;
    const void *p = tb + (ok ? (off >> SH) : 0);
    if constexpr (VEC == 4) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        lds128_pred(t, p, ok);
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    } else if constexpr (VEC == 2) {
        float2 t = make_float2(0.f, 0.f);
        lds64_pred(t, p, ok);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        float t = 0.f;
        lds32_pred(t, p, ok);
        v[0] = t;
    }
}

// The same with a 32-bit shared-window base (callers pin it in a register
// with an opaque mov, so the compiler does not rematerialize it from %tid).
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
    uint32_t r;
    asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ int4 lds_entry_pair_s(uint32_t a) {
    int4 q;
    asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(a));
    return q;
}
// an entry that cannot be padding (not a segment's last slot): plain load
template <int VEC>
__device__ __forceinline__ void lds_row_s(uint32_t tbs, int off, float (&v)[VEC]) {
    static_assert(VEC == 4, "32-bit-address variant: 16-byte rows only");
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(tbs + (uint32_t)off));
}
template <int VEC>
__device__ __forceinline__ void lds_row_or_zero_s(uint32_t tbs, int off, float (&v)[VEC]) {
    static_assert(VEC == 4, "32-bit-address variant: 16-byte rows only");
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    asm("{\n.reg .pred q;\nsetp.ge.s32 q, %4, 0;\n@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%5];\n}\n"
        : "+f"(t.x), "+f"(t.y), "+f"(t.z), "+f"(t.w)
        : "r"(off), "r"(tbs + (uint32_t)(off >= 0 ? off : 0)));
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
}

// Stage rows [k0, k0+nk) x batch columns [b0, b0+BT) of a row-major
// [nrows x B] fp32 activation into smem tile[nk][BT] (row stride BT),
// zero-filling batch columns >= B.  16-byte vector path when B % 4 == 0.
template <int BT, int NT>
__device__ __forceinline__ void stage_tile(float *__restrict__ tile, const float *__restrict__ src,
                                           int64_t k0, int nk, int64_t B, int64_t b0, bool vec4) {
    constexpr int Q = BT / 4;  // float4 chunks per tile row (BT >= 32)
    const int total = nk * Q;
    if (vec4) {
        for (int i = threadIdx.x; i < total; i += NT) {
            const int k = i / Q, q = (i - k * Q) * 4;
            const int64_t b = b0 + q;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b < B) v = __ldg(reinterpret_cast<const float4 *>(src + (k0 + k) * B + b));
            *reinterpret_cast<float4 *>(tile + k * BT + q) = v;
        }
    } else {
        for (int i = threadIdx.x; i < total; i += NT) {
            const int k = i / Q, q = (i - k * Q) * 4;
            const int64_t b = b0 + q;
            const float *s = src + (k0 + k) * B + b;
            float4 v;
            v.x = b + 0 < B ? __ldg(s + 0) : 0.f;
            v.y = b + 1 < B ? __ldg(s + 1) : 0.f;
            v.z = b + 2 < B ? __ldg(s + 2) : 0.f;
            v.w = b + 3 < B ? __ldg(s + 3) : 0.f;
            *reinterpret_cast<float4 *>(tile + k * BT + q) = v;
        }
    }
}

// ---- cp.async (LDGSTS) helpers: 16-byte global->shared copies that bypass
// registers; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Asynchronous version of stage_tile for B % 4 == 0 (16-byte aligned rows):
// issues the copies and returns; the caller commits / waits.
template <int BT, int NT>
__device__ __forceinline__ void stage_tile_async(float *__restrict__ tile, const float *__restrict__ src,
                                                 int64_t k0, int nk, int64_t B, int64_t b0) {
    constexpr int Q = BT / 4;
    const int total = nk * Q;
    for (int i = threadIdx.x; i < total; i += NT) {
        const int k = i / Q, q = (i - k * Q) * 4;
        const int64_t b = b0 + q;
        const bool in = b < B;
        cp_async16(tile + k * BT + q, src + (k0 + k) * B + (in ? b : 0), in ? 16 : 0);
    }
}

// Stage a tile either asynchronously (vec4) or synchronously (ragged B).
template <int BT, int NT>
__device__ __forceinline__ void stage_any(float *tile, const float *src, int64_t k0, int nk, int64_t B,
                                          int64_t b0, bool vec4) {
    if (vec4)
        stage_tile_async<BT, NT>(tile, src, k0, nk, B, b0);
    else
        stage_tile<BT, NT>(tile, src, k0, nk, B, b0, false);
}

// ---- TMA (cp.async.bulk) + mbarrier helpers ------------------------------

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make mbarrier inits visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// plain arrive (count 1) on a CTA mbarrier
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (UBLKCP), completion counted on `bar`.
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 2-D tensor TMA (UTMALDG): box at (batch c0, row c1) of the tensor map into
// dst; out-of-bounds rows / batch columns are zero-filled by the hardware.
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// 4-D tensor TMA: box at (b, q, p, channel) of a CHWN map (make_tmap_conv);
// coordinates outside the tensor (the conv halo) are zero-filled.
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// ConvCols (sp_internal.cuh): the tensor-map coordinates of tap t's tile of
// slice sl (channel block starting at kc): CHWN (b0, q0 + dq, p + dp, kc),
// NCHW (q0 + dq, p0 + dp, kc, b)
__device__ __forceinline__ void cc_coords(const ConvCols &g, int sl, int t, int kc, int (&c)[4]) {
    if (g.nchw) {
        const int per = g.nqt * g.npt, b = sl / per, r = sl - b * per, pt = r / g.nqt;
        c[0] = (r - pt * g.nqt) * g.nq + g.dq[t];
        c[1] = pt * g.np + g.dp[t];
        c[2] = kc;
        c[3] = b;
        return;
    }
    const int p = sl / g.spr, r = sl - p * g.spr;
    int q0, b0;
    if (g.bpr == 1) {
        q0 = r * g.nq;
        b0 = 0;
    } else {
        q0 = r / g.bpr;
        b0 = (r - q0 * g.bpr) * 128;
    }
    c[0] = b0;
    c[1] = q0 + g.dq[t];
    c[2] = p + g.dp[t];
    c[3] = kc;
}
// column c (0..127) of slice sl -> float offset of its output position from the
// start of its channel row (add r * rowlen), or -1 outside the output (a partial
// slice at the edge of a row / image)
__device__ __forceinline__ int64_t cc_off(const ConvCols &g, int sl, int c) {
    if (g.nchw) {
        const int per = g.nqt * g.npt, b = sl / per, r = sl - b * per, pt = r / g.nqt;
        const int p = pt * g.np + (c >> g.qsh), q = (r - pt * g.nqt) * g.nq + (c & (g.nq - 1));
        if (p >= g.Po || q >= g.Qo) return -1;
        return (int64_t)b * g.imgstride + (int64_t)p * g.Qo + q;
    }
    const int p = sl / g.spr, r = sl - p * g.spr;
    int q0, b0;
    if (g.bpr == 1) {
        q0 = r * g.nq;
        b0 = 0;
    } else {
        q0 = r / g.bpr;
        b0 = (r - q0 * g.bpr) * 128;
    }
    const int q = q0 + (c >> g.bsh);
    if (q >= g.Qo) return -1;
    return ((int64_t)p * g.Qo + q) * g.B + b0 + (c & ((1 << g.bsh) - 1));
}

// Issue (from one warp) the TMA copies of rows [k0, k0+nk) x batch columns
// [b0, b0 + min(BT, B-b0)) of a [rows x B] activation (B % 4 == 0) into
// tile[nk][BT], plus optionally `ebytes` of entries, all on `bar`.
template <int BT>
__device__ __forceinline__ void tma_stage_tile(float *tile, const float *src, int64_t k0, int nk, int64_t B,
                                               int64_t b0, uint64_t *bar, void *edst, const void *esrc,
                                               unsigned ebytes, int lane) {
    const int ncol = (int)(B - b0 < BT ? B - b0 : BT);
    const unsigned rb = (unsigned)ncol * 4u;
    if (lane == 0) mbar_arrive_expect_tx(bar, rb * (unsigned)nk + ebytes);
    __syncwarp();
    for (int k = lane; k < nk; k += 32) tma_load_1d(tile + (size_t)k * BT, src + (k0 + k) * B + b0, rb, bar);
    if (lane == 0 && ebytes) tma_load_1d(edst, esrc, ebytes, bar);
}

// ---- packed FP32 math (sm_100 FFMA2 / FMUL2: two lanes per instruction,
// each element rounded exactly like fmaf / fmul) ----------------------------
template <int VEC>
__device__ __forceinline__ void fma_bcast(float (&acc)[VEC], float w, const float (&x)[VEC]) {
    if constexpr (VEC == 1) {
        acc[0] = fmaf(w, x[0], acc[0]);
    } else {
        const float2 ww = make_float2(w, w);
#pragma unroll
        for (int v = 0; v < VEC; v += 2) {
            const float2 r = __ffma2_rn(ww, make_float2(x[v], x[v + 1]), make_float2(acc[v], acc[v + 1]));
            acc[v] = r.x;
            acc[v + 1] = r.y;
        }
    }
}

// sum_v a[v] * x[v] with paired products (order: (a0x0 + a2x2) + (a1x1 + a3x3))
template <int VEC>
__device__ __forceinline__ float dot_vec(const float (&a)[VEC], const float (&x)[VEC]) {
    if constexpr (VEC == 1) {
        return a[0] * x[0];
    } else {
        float2 p = __fmul2_rn(make_float2(a[0], a[1]), make_float2(x[0], x[1]));
#pragma unroll
        for (int v = 2; v < VEC; v += 2)
            p = __ffma2_rn(make_float2(a[v], a[v + 1]), make_float2(x[v], x[v + 1]), p);
        return p.x + p.y;
    }
}

// Warp transpose-reduce of 32 per-lane partials: on return, lane t holds
// sum over lanes of acc[t] (in acc[0]).  31 shuffles for 32 sums.
__device__ __forceinline__ float transpose_reduce32(float (&acc)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const float send = up ? acc[i] : acc[i + s];
            const float keep = up ? acc[i + s] : acc[i];
            acc[i] = keep + __shfl_xor_sync(kFull, send, s);
        }
    }
    return acc[0];
}

}  // namespace sp
