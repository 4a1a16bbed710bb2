// api.cu -- the extern "C" boundary of libsparseprop (include/sparseprop.h).
// Argument validation, handle lifetime, dispatch to the kernels.  No C++
// exception crosses the ABI; every entry point returns sp_status.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <new>
#include <string>

#include "sp_internal.cuh"

namespace sp {

static thread_local std::string g_err;
static thread_local std::string g_path;

void begin_path() { g_path.clear(); }
void note_path(const char *name) {
    if (!g_path.empty()) g_path += '+';
    g_path += name;
}
static std::atomic<unsigned long long> g_launches{0};

void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

void set_error(const std::string &msg) { g_err = msg; }

namespace {
constexpr int kMaxDev = 64;
std::mutex g_dev_mu;
int g_sms[kMaxDev] = {};
cudaMemPool_t g_pool[kMaxDev] = {};
bool g_pool_done[kMaxDev] = {};

int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
}  // namespace

std::atomic<int> g_sm_reserve{0};

int num_sms() {
    const int d = cur_dev();
    int n = 148;
    if (d >= 0 && d < kMaxDev) {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (g_sms[d] == 0) {
            int v = 0;
            g_sms[d] = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) == cudaSuccess && v > 0 ? v : 148;
        }
        n = g_sms[d];
    }
    return std::max(1, n - g_sm_reserve.load());
}

cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st) {
    // under stream capture the allocation becomes a graph memory node (the
    // graph owns it; the library pool is only for eager launches)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
        return cudaMallocAsync(p, bytes, st);
    const int d = cur_dev();
    cudaMemPool_t pool = nullptr;
    if (d >= 0 && d < kMaxDev) {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (!g_pool_done[d]) {
            g_pool_done[d] = true;
            cudaMemPoolProps pp{};
            pp.allocType = cudaMemAllocationTypePinned;
            pp.location.type = cudaMemLocationTypeDevice;
            pp.location.id = d;
            if (cudaMemPoolCreate(&g_pool[d], &pp) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(g_pool[d], cudaMemPoolAttrReleaseThreshold, &thr);
            } else {
                g_pool[d] = nullptr;
                cudaGetLastError();
            }
        }
        pool = g_pool[d];
    }
    if (pool) return cudaMallocFromPoolAsync(p, bytes, pool, st);
    return cudaMallocAsync(p, bytes, st);
}

cudaError_t scratch_free(void *p, cudaStream_t st) { return cudaFreeAsync(p, st); }

sp_status check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return SP_ERR_CUDA;
    }
    return SP_OK;
}

}  // namespace sp

using namespace sp;

namespace {

constexpr int64_t kI32Max = 2147483647LL;

sp_status fail(sp_status s, const std::string &msg) {
    set_error(msg);
    return s;
}

bool ok_handle(sp_weight_t w) { return w != nullptr && w->magic == SP_MAGIC; }

#define SP_CHECK_HANDLE(w, fn) \
    if (!ok_handle(w)) return fail(SP_ERR_BAD_HANDLE, std::string(fn) + ": bad or destroyed handle")

sp_status check_B(int64_t B, int64_t rows_a, int64_t rows_b, const char *fn) {
    if (B < 1) return fail(SP_ERR_SHAPE, std::string(fn) + ": B must be >= 1");
    if (rows_a * B > (int64_t)1 << 40 || rows_b * B > (int64_t)1 << 40)
        return fail(SP_ERR_OVERFLOW, std::string(fn) + ": activation too large");
    return SP_OK;
}

sp_status check_geom(sp_weight_t w, const sp_conv_geom *g, const char *fn) {
    if (!g) return fail(SP_ERR_NULL, std::string(fn) + ": geometry is NULL");
    if (g->B < 1 || g->C_in < 1 || g->H < 1 || g->W < 1 || g->C_out < 1 || g->KH < 1 || g->KW < 1 ||
        g->pad < 0)
        return fail(SP_ERR_SHAPE, std::string(fn) + ": non-positive conv dimension");
    const int64_t OH = (int64_t)g->H + 2 * g->pad - g->KH + 1;
    const int64_t OW = (int64_t)g->W + 2 * g->pad - g->KW + 1;
    if (OH < 1 || OW < 1) return fail(SP_ERR_SHAPE, std::string(fn) + ": empty output");
    if (w->R != g->C_out || w->C != (int64_t)g->C_in * g->KH * g->KW)
        return fail(SP_ERR_SHAPE, std::string(fn) + ": weight handle does not match C_out x C_in*KH*KW");
    const int64_t nx = (int64_t)g->C_in * g->H * g->W * g->B;
    const int64_t ny = (int64_t)g->C_out * OH * OW * g->B;
    if (nx > ((int64_t)1 << 40) || ny > ((int64_t)1 << 40))
        return fail(SP_ERR_OVERFLOW, std::string(fn) + ": activation too large");
    return SP_OK;
}

}  // namespace

extern "C" {

const char *sp_last_error(void) { return g_err.c_str(); }

const char *sp_last_path(void) { return g_path.c_str(); }

uint64_t sp_launch_count(void) { return g_launches.load(); }

sp_status sp_set_sm_reserve(int32_t n) {
    if (n < 0) return fail(SP_ERR_SHAPE, "sp_set_sm_reserve: n must be >= 0");
    sp::g_sm_reserve.store(n);
    return SP_OK;
}

const char *sp_version(void) { return "libsparseprop 0.2 sm_100a fp32 (CUDA cores, TMEM state, deterministic: no atomic output accumulation)"; }

sp_status sp_weight_create(int64_t R, int64_t C, const float *dense, const uint8_t *mask,
                           sp_stream_t stream, sp_weight_t *out) {
    if (!out) return fail(SP_ERR_NULL, "sp_weight_create: out is NULL");
    *out = nullptr;
    if (!dense || !mask) return fail(SP_ERR_NULL, "sp_weight_create: dense or mask is NULL");
    if (R < 1 || C < 1) return fail(SP_ERR_SHAPE, "sp_weight_create: R and C must be >= 1");
    if (R > kI32Max || C > kI32Max)
        return fail(SP_ERR_OVERFLOW, "sp_weight_create: R and C must fit int32");
    sp_weight_s *w = new (std::nothrow) sp_weight_s();
    if (!w) return fail(SP_ERR_ALLOC, "sp_weight_create: host allocation failed");
    w->magic = SP_MAGIC;
    const sp_status s = build_weight(R, C, dense, mask, S(stream), w);
    if (s != SP_OK) {
        cudaDeviceSynchronize();
        free_weight(w);
        w->magic = 0;
        delete w;
        return s;
    }
    *out = w;
    return SP_OK;
}

sp_status sp_weight_create_conv(int32_t C_out, int32_t C_in, int32_t KH, int32_t KW, const float *dense,
                                const uint8_t *mask, sp_stream_t stream, sp_weight_t *out) {
    if (C_out < 1 || C_in < 1 || KH < 1 || KW < 1)
        return fail(SP_ERR_SHAPE, "sp_weight_create_conv: dimensions must be >= 1");
    sp_status s = sp_weight_create(C_out, (int64_t)C_in * KH * KW, dense, mask, stream, out);
    if (s != SP_OK) return s;
    s = build_conv_taps(*out, C_out, C_in, KH, KW, S(stream));
    if (s != SP_OK) {
        sp_weight_destroy(*out, stream);
        *out = nullptr;
        return fail(s, "sp_weight_create_conv: tap tiling build failed");
    }
    return SP_OK;
}

sp_status sp_weight_destroy(sp_weight_t w, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_weight_destroy");
    cudaStreamSynchronize(S(stream));
    cudaDeviceSynchronize();  // work on other streams may still read the handle (as cudaFree would wait)
    free_weight(w);
    w->magic = 0;
    delete w;
    return SP_OK;
}

int64_t sp_weight_nnz(sp_weight_t w) { return ok_handle(w) ? w->nnz : -1; }
int64_t sp_weight_rows(sp_weight_t w) { return ok_handle(w) ? w->R : -1; }
int64_t sp_weight_cols(sp_weight_t w) { return ok_handle(w) ? w->C : -1; }

sp_status sp_weight_vals(sp_weight_t w, float **vals) {
    SP_CHECK_HANDLE(w, "sp_weight_vals");
    if (!vals) return fail(SP_ERR_NULL, "sp_weight_vals: out is NULL");
    *vals = w->vals;
    return SP_OK;
}

sp_status sp_weight_indices(sp_weight_t w, const int32_t **row_ptr, const int32_t **col_idx,
                            const int32_t **col_ptr, const int32_t **row_idx, const int32_t **perm) {
    SP_CHECK_HANDLE(w, "sp_weight_indices");
    if (row_ptr) *row_ptr = w->row_ptr;
    if (col_idx) *col_idx = w->col_idx;
    if (col_ptr) *col_ptr = w->col_ptr;
    if (row_idx) *row_idx = w->row_idx;
    if (perm) *perm = w->perm;
    return SP_OK;
}

sp_status sp_weight_to_dense(sp_weight_t w, const float *nz, float *dense_out, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_weight_to_dense");
    if (!dense_out || (!nz && w->nnz > 0)) return fail(SP_ERR_NULL, "sp_weight_to_dense: NULL buffer");
    launch_to_dense(w, nz, dense_out, S(stream));
    return check_launch("sp_weight_to_dense");
}

sp_status sp_weight_gather(sp_weight_t w, const float *dense, float *nz_out, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_weight_gather");
    if (!dense || (!nz_out && w->nnz > 0)) return fail(SP_ERR_NULL, "sp_weight_gather: NULL buffer");
    launch_gather_dense(w, dense, nz_out, S(stream));
    return check_launch("sp_weight_gather");
}

// ---- B % 4 != 0 (the paper's own B = 902, S75): the float4 / TMA kernels need
// 16-byte aligned activation rows, so from kPadMinB columns on the backward
// products (dW alone, the fused backward) run on zero-padded copies
// [rows x Bp], Bp = B rounded up to 4, and dX is copied back.  The pad columns
// are zeros: they add nothing to dW (each dot product gains +0 terms) and land
// only in the discarded columns of dX, so every kept element is the same sum
// the unpadded kernels would form (within the tolerance: the kernel family,
// hence the order, may differ).  Paper layer 3072 x 768, B = 902: backward
// 403 -> 180 us at 80 %, 182 -> 83 us at 95 %.  The forward and the separate
// dX keep the narrow-lane tail kernels (the copies and the 8-column last slice
// of a padded 904-column batch cost more than they gain: 141 vs 159 us at 80 %).
// Below kPadMinB every product runs the tail kernels on the caller's buffers.
constexpr int64_t kPadMinB = 64;
static bool want_pad(int64_t B) {
#ifdef SP_NO_PAD4
    return false;
#endif
    return (B & 3) != 0 && B >= kPadMinB;
}

__global__ void pad_cols_kernel(const float *__restrict__ src, float *__restrict__ dst, int64_t rows, int64_t B,
                                int64_t Bp) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = rows * Bp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / Bp, c = i - r * Bp;
        dst[i] = c < B ? __ldg(src + r * B + c) : 0.f;
    }
}
__global__ void unpad_cols_kernel(const float *__restrict__ src, float *__restrict__ dst, int64_t rows, int64_t B,
                                  int64_t Bp) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = rows * B;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / B, c = i - r * B;
        dst[i] = __ldg(src + r * Bp + c);
    }
}
static unsigned pad_grid(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8); }

// scratch buffers of the padded operands of one call (freed stream-ordered)
struct PadSet {
    cudaStream_t st;
    float *buf[4] = {nullptr, nullptr, nullptr, nullptr};
    int n = 0;
    bool failed = false;
    explicit PadSet(cudaStream_t s) : st(s) {}
    float *alloc(int64_t floats) {
        void *p = nullptr;
        if (scratch_alloc(&p, (size_t)std::max<int64_t>(floats, 1) * sizeof(float), st) != cudaSuccess) {
            failed = true;
            return nullptr;
        }
        return buf[n++] = static_cast<float *>(p);
    }
    const float *in(const float *src, int64_t rows, int64_t B, int64_t Bp) {
        if (!src) return nullptr;
        float *d = alloc(rows * Bp);
        if (!d) return nullptr;
        launch_pdl(pad_cols_kernel, dim3(pad_grid(rows * Bp)), dim3(256), 0, st, src, d, rows, B, Bp);
        count_launches(1);
        return d;
    }
    void out(const float *src, float *dst, int64_t rows, int64_t B, int64_t Bp) {
        launch_pdl(unpad_cols_kernel, dim3(pad_grid(rows * B)), dim3(256), 0, st, src, dst, rows, B, Bp);
        count_launches(1);
    }
    ~PadSet() {
        for (int i = 0; i < n; ++i) scratch_free(buf[i], st);
    }
};

static sp_status linear_fwd_impl(sp_weight_t w, const float *X, float *Y, int64_t B, int epi,
                                 sp_stream_t stream, const char *fn) {
    SP_CHECK_HANDLE(w, fn);
    begin_path();
    if (!X || !Y) return fail(SP_ERR_NULL, std::string(fn) + ": NULL tensor");
    sp_status s = check_B(B, w->R, w->C, fn);
    if (s != SP_OK) return s;
    launch_spmm(w, 0, B, X, Y, nullptr, epi, S(stream));
    return check_launch(fn);
}

sp_status sp_linear_fwd(sp_weight_t w, const float *X, float *Y, int64_t B, sp_stream_t stream) {
    return linear_fwd_impl(w, X, Y, B, EPI_NONE, stream, "sp_linear_fwd");
}

sp_status sp_linear_fwd_relu(sp_weight_t w, const float *X, float *Y, int64_t B, sp_stream_t stream) {
    return linear_fwd_impl(w, X, Y, B, EPI_RELU, stream, "sp_linear_fwd_relu");
}

static sp_status linear_dx_impl(sp_weight_t w, const float *dY, const float *H, float *dX, int64_t B,
                                int epi, sp_stream_t stream, const char *fn) {
    SP_CHECK_HANDLE(w, fn);
    begin_path();
    if (!dY || !dX || (epi == EPI_GATE && !H)) return fail(SP_ERR_NULL, std::string(fn) + ": NULL tensor");
    sp_status s = check_B(B, w->R, w->C, fn);
    if (s != SP_OK) return s;
    launch_spmm(w, 1, B, dY, dX, H, epi, S(stream));
    return check_launch(fn);
}

sp_status sp_linear_bwd_input(sp_weight_t w, const float *dY, float *dX, int64_t B, sp_stream_t stream) {
    return linear_dx_impl(w, dY, nullptr, dX, B, EPI_NONE, stream, "sp_linear_bwd_input");
}

sp_status sp_linear_bwd_input_relu(sp_weight_t w, const float *dY, const float *H, float *dX, int64_t B,
                                   sp_stream_t stream) {
    return linear_dx_impl(w, dY, H, dX, B, EPI_GATE, stream, "sp_linear_bwd_input_relu");
}

sp_status sp_linear_bwd_weight(sp_weight_t w, const float *X, const float *dY, float *dW, int64_t B,
                               sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_linear_bwd_weight");
    begin_path();
    if (!X || !dY || (!dW && w->nnz > 0)) return fail(SP_ERR_NULL, "sp_linear_bwd_weight: NULL tensor");
    sp_status s = check_B(B, w->R, w->C, "sp_linear_bwd_weight");
    if (s != SP_OK) return s;
    if (want_pad(B) && w->nnz > 0) {
        const int64_t Bp = (B + 3) & ~(int64_t)3;
        PadSet ps(S(stream));
        note_path("pad_b4");
        const float *Xp = ps.in(X, w->C, B, Bp);
        const float *dYp = ps.in(dY, w->R, B, Bp);
        if (ps.failed) return fail(SP_ERR_ALLOC, "sp_linear_bwd_weight: scratch allocation failed");
        s = launch_sddmm(w, Xp, dYp, dW, Bp, S(stream));
        if (s != SP_OK) return s;
        return check_launch("sp_linear_bwd_weight");
    }
    s = launch_sddmm(w, X, dY, dW, B, S(stream));
    if (s != SP_OK) return s;
    return check_launch("sp_linear_bwd_weight");
}

static sp_status linear_bwd_impl(sp_weight_t w, const float *X, const float *dY, const float *H, float *dX,
                                 float *dW, int64_t B, sp_stream_t stream, const char *fn) {
    SP_CHECK_HANDLE(w, fn);
    begin_path();
    if (!X || !dY || !dX || (!dW && w->nnz > 0)) return fail(SP_ERR_NULL, std::string(fn) + ": NULL tensor");
    sp_status s = check_B(B, w->R, w->C, fn);
    if (s != SP_OK) return s;
    if (want_pad(B)) {
        const int64_t Bp = (B + 3) & ~(int64_t)3;
        PadSet ps(S(stream));
        note_path("pad_b4");
        const float *Xp = ps.in(X, w->C, B, Bp);
        const float *dYp = ps.in(dY, w->R, B, Bp);
        const float *Hp = H == X ? Xp : ps.in(H, w->C, B, Bp);  // (the DP step's gate is X itself)
        float *dXp = ps.alloc(w->C * Bp);
        if (ps.failed) return fail(SP_ERR_ALLOC, std::string(fn) + ": scratch allocation failed");
        s = launch_bwd_fused(w, Xp, dYp, Hp, dXp, dW, Bp, S(stream));
        if (s == SP_ERR_SHAPE) {
            launch_spmm(w, 1, Bp, dYp, dXp, Hp, Hp ? EPI_GATE : EPI_NONE, S(stream));
            s = check_launch(fn);
            if (s == SP_OK) s = launch_sddmm(w, Xp, dYp, dW, Bp, S(stream));
        }
        if (s != SP_OK) return s;
        ps.out(dXp, dX, w->C, B, Bp);
        return check_launch(fn);
    }
    s = launch_bwd_fused(w, X, dY, H, dX, dW, B, S(stream));
    if (s == SP_ERR_SHAPE) {  // fused path not applicable: the two separate products
        launch_spmm(w, 1, B, dY, dX, H, H ? EPI_GATE : EPI_NONE, S(stream));
        s = check_launch(fn);
        if (s != SP_OK) return s;
        s = launch_sddmm(w, X, dY, dW, B, S(stream));
    }
    if (s != SP_OK) return s;
    return check_launch(fn);
}

sp_status sp_linear_bwd(sp_weight_t w, const float *X, const float *dY, float *dX, float *dW, int64_t B,
                        sp_stream_t stream) {
    return linear_bwd_impl(w, X, dY, nullptr, dX, dW, B, stream, "sp_linear_bwd");
}

sp_status sp_linear_bwd_relu(sp_weight_t w, const float *X, const float *dY, const float *H, float *dX, float *dW,
                             int64_t B, sp_stream_t stream) {
    if (!H) return fail(SP_ERR_NULL, "sp_linear_bwd_relu: H is NULL");
    return linear_bwd_impl(w, X, dY, H, dX, dW, B, stream, "sp_linear_bwd_relu");
}

sp_status sp_conv2d_fwd(sp_weight_t w, const sp_conv_geom *g, const float *X, float *Y, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_conv2d_fwd");
    begin_path();
    sp_status s = check_geom(w, g, "sp_conv2d_fwd");
    if (s != SP_OK) return s;
    if (!X || !Y) return fail(SP_ERR_NULL, "sp_conv2d_fwd: NULL tensor");
    launch_conv_fwd(w, *g, X, Y, S(stream));
    return check_launch("sp_conv2d_fwd");
}

sp_status sp_conv2d_bwd_input(sp_weight_t w, const sp_conv_geom *g, const float *dY, float *dX,
                              sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_conv2d_bwd_input");
    begin_path();
    sp_status s = check_geom(w, g, "sp_conv2d_bwd_input");
    if (s != SP_OK) return s;
    if (!dY || !dX) return fail(SP_ERR_NULL, "sp_conv2d_bwd_input: NULL tensor");
    launch_conv_bwd_input(w, *g, dY, dX, S(stream));
    return check_launch("sp_conv2d_bwd_input");
}

sp_status sp_conv2d_bwd_weight(sp_weight_t w, const sp_conv_geom *g, const float *X, const float *dY,
                               float *dW, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_conv2d_bwd_weight");
    begin_path();
    sp_status s = check_geom(w, g, "sp_conv2d_bwd_weight");
    if (s != SP_OK) return s;
    if (!X || !dY || (!dW && w->nnz > 0)) return fail(SP_ERR_NULL, "sp_conv2d_bwd_weight: NULL tensor");
    s = launch_conv_bwd_weight(w, *g, X, dY, dW, S(stream));
    if (s != SP_OK) return s;
    return check_launch("sp_conv2d_bwd_weight");
}

sp_status sp_conv2d_bwd(sp_weight_t w, const sp_conv_geom *g, const float *X, const float *dY, float *dX,
                        float *dW, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_conv2d_bwd");
    begin_path();
    sp_status s = check_geom(w, g, "sp_conv2d_bwd");
    if (s != SP_OK) return s;
    if (!X || !dY || !dX || (!dW && w->nnz > 0)) return fail(SP_ERR_NULL, "sp_conv2d_bwd: NULL tensor");
    s = launch_conv_bwd(w, *g, X, dY, dX, dW, S(stream));
    if (s != SP_OK) return s;
    return check_launch("sp_conv2d_bwd");
}

static sp_status conv_nchw_impl(sp_weight_t w, const sp_conv_geom *g, int op, const float *X, const float *dY,
                                float *out, float *dW, sp_stream_t stream, const char *fn) {
    SP_CHECK_HANDLE(w, fn);
    begin_path();
    sp_status s = check_geom(w, g, fn);
    if (s != SP_OK) return s;
    if ((op != 1 && !X) || (op != 0 && !dY) || (op != 3 && !out) || (op >= 2 && !dW && w->nnz > 0))
        return fail(SP_ERR_NULL, std::string(fn) + ": NULL tensor");
    s = launch_conv_nchw(w, *g, op, X, dY, out, dW, S(stream));
    if (s != SP_OK) return s;
    return check_launch(fn);
}

sp_status sp_conv2d_fwd_nchw(sp_weight_t w, const sp_conv_geom *g, const float *X, float *Y, sp_stream_t stream) {
    return conv_nchw_impl(w, g, 0, X, nullptr, Y, nullptr, stream, "sp_conv2d_fwd_nchw");
}

sp_status sp_conv2d_bwd_input_nchw(sp_weight_t w, const sp_conv_geom *g, const float *dY, float *dX,
                                   sp_stream_t stream) {
    return conv_nchw_impl(w, g, 1, nullptr, dY, dX, nullptr, stream, "sp_conv2d_bwd_input_nchw");
}

sp_status sp_conv2d_bwd_nchw(sp_weight_t w, const sp_conv_geom *g, const float *X, const float *dY, float *dX,
                             float *dW, sp_stream_t stream) {
    return conv_nchw_impl(w, g, 2, X, dY, dX, dW, stream, "sp_conv2d_bwd_nchw");
}

sp_status sp_conv2d_bwd_weight_nchw(sp_weight_t w, const sp_conv_geom *g, const float *X, const float *dY, float *dW,
                                    sp_stream_t stream) {
    return conv_nchw_impl(w, g, 3, X, dY, nullptr, dW, stream, "sp_conv2d_bwd_weight_nchw");
}

int64_t sp_mse_scratch_floats(int64_t n) { return mse_scratch_floats(n); }

sp_status sp_mse_grad(const float *Y, const float *T, float *dY, float *loss_out, float *scratch, int64_t n,
                      sp_stream_t stream) {
    if (!Y || !T || !dY || !loss_out || !scratch) return fail(SP_ERR_NULL, "sp_mse_grad: NULL tensor");
    if (n < 1) return fail(SP_ERR_SHAPE, "sp_mse_grad: n must be >= 1");
    if (reinterpret_cast<uintptr_t>(scratch) & 7) return fail(SP_ERR_SHAPE, "sp_mse_grad: scratch must be 8-byte aligned");
    launch_mse(Y, T, dY, loss_out, scratch, n, S(stream));
    return check_launch("sp_mse_grad");
}

sp_status sp_sgd(float *vals, const float *dW, int64_t nnz, float lr, sp_stream_t stream) {
    if ((!vals || !dW) && nnz > 0) return fail(SP_ERR_NULL, "sp_sgd: NULL tensor");
    if (nnz < 0) return fail(SP_ERR_SHAPE, "sp_sgd: nnz < 0");
    launch_sgd(vals, dW, nnz, lr, S(stream));
    return check_launch("sp_sgd");
}

sp_status sp_weight_set_managed(sp_weight_t w, int managed) {
    SP_CHECK_HANDLE(w, "sp_weight_set_managed");
    w->managed = managed ? 1 : 0;
    ++w->version;  // whatever vals hold now: every tiling refreshes at its next use
    return SP_OK;
}

sp_status sp_weight_sgd(sp_weight_t w, const float *dW, float lr, sp_stream_t stream) {
    SP_CHECK_HANDLE(w, "sp_weight_sgd");
    if (!dW && w->nnz > 0) return fail(SP_ERR_NULL, "sp_weight_sgd: NULL dW");
    launch_weight_sgd(w, dW, lr, S(stream));
    return check_launch("sp_weight_sgd");
}

sp_status sp_weights_sgd(const sp_weight_t *Ws, const float *const *dWs, int32_t n, float lr, sp_stream_t stream) {
    if (!Ws || !dWs) return fail(SP_ERR_NULL, "sp_weights_sgd: NULL array");
    if (n < 1 || n > SP_SGD_BATCH_MAX) return fail(SP_ERR_SHAPE, "sp_weights_sgd: need 1 <= n <= SP_SGD_BATCH_MAX");
    for (int i = 0; i < n; ++i) {
        SP_CHECK_HANDLE(Ws[i], "sp_weights_sgd");
        if (!dWs[i] && Ws[i]->nnz > 0) return fail(SP_ERR_NULL, "sp_weights_sgd: NULL dW");
        for (int k = 0; k < i; ++k)
            if (Ws[k] == Ws[i]) return fail(SP_ERR_SHAPE, "sp_weights_sgd: a handle appears twice");
    }
    launch_weights_sgd(Ws, dWs, n, lr, S(stream));
    return check_launch("sp_weights_sgd");
}

}  // extern "C"
