// api.cu -- the C ABI of liboz2.so (declared in include/oz2.h): argument
// checking, handles, workspace, TMA tensor maps and the launch sequence of
// Algorithm 1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/oz2.h"
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace {

Oz2Table g_tabs[OZ2_MAX_MODULI + 1];
bool g_tabs_ok = false;
std::once_flag g_tabs_once;
std::mutex g_mu;
bool g_dev_uploaded[64] = {false};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

void build_tables_once() {
    g_tabs_ok = (oz2_build_tables(g_tabs) == 0);
    for (int N = 2; N <= OZ2_MAX_MODULI && g_tabs_ok; N++) {
        if (g_tabs[N].JB != oz2::crt_bytes(N) || g_tabs[N].WS != oz2::crt_swords(N) ||
            g_tabs[N].WX != oz2::crt_words(N))
            g_tabs_ok = false;                                       // kernels assume these
    }
}

int ensure_device(int dev) {
    std::call_once(g_tabs_once, build_tables_once);
    if (!g_tabs_ok) return OZ2_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= 64) return OZ2_ERR_NO_DEVICE;
    if (!g_encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return OZ2_ERR_CUDA;
        g_encode = (EncodeTiledFn)fn;
    }
    if (!g_dev_uploaded[dev]) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cudaSetDevice(dev) != cudaSuccess) return OZ2_ERR_NO_DEVICE;
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) { cudaSetDevice(cur); return OZ2_ERR_NO_DEVICE; }
        if (prop.major != 10) { cudaSetDevice(cur); return OZ2_ERR_NO_DEVICE; }
        cudaError_t e = cudaMemcpyToSymbol(c_tab, g_tabs, sizeof(g_tabs));
        if (e == cudaSuccess) e = oz2::upload_tables_gemm(g_tabs, sizeof(g_tabs));
        if (e == cudaSuccess) {
            oz2::launch_init_bfrag(0);
            e = cudaStreamSynchronize(0);
        }
        cudaSetDevice(cur);
        if (e != cudaSuccess) return OZ2_ERR_CUDA;
        g_dev_uploaded[dev] = true;
    }
    return OZ2_OK;
}

}  // namespace

namespace oz2 {
int host_T(int N) {
    std::call_once(g_tabs_once, build_tables_once);
    return g_tabs[N].T;
}
int host_L(int N) {
    std::call_once(g_tabs_once, build_tables_once);
    return g_tabs[N].L;
}
}  // namespace oz2

// NVTX ranges (SURVEY section 5 tracing): one per public entry point, named after
// it; free when no tool is attached (nvtx3 is header-only and dormant)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct oz2_context {
    int device;
    int num_sms;
    cudaStream_t stream;
    int mode;
    void* ws_user;
    size_t ws_user_bytes;
    void* ws_own;
    size_t ws_own_bytes;
    int profiling;
    std::vector<cudaEvent_t> events;   // OZ2_NUM_STAGES + 1 per profiled call
    // oz2_dgemm_host pipeline: copy streams and events (created on first use)
    cudaStream_t s_h2d, s_d2h;
    std::vector<cudaEvent_t> pipe_ev;
    // B's conversion runs on s_aux concurrently with A's (fork / join events)
    cudaStream_t s_aux;
    cudaEvent_t ev_fork, ev_join;
    int sm_limit;                      // 0 = all SMs; else the persistent GEMM's SM budget
    // TRMM: the masked triangular operand (handle-owned, grown on demand)
    void* tbuf;
    size_t tbuf_bytes;
    // condition (13) certificates: device words [0] sticky refusal status,
    // [1] beta of oz2_dgemm_scaled, [4..8] partial maxima and the width flag
    // (allocated on first use)
    int* cert;
    int certify;                       // oz2_dgemm_scaled certifies (default 1)
};

namespace {
// SMs the persistent GEMM may use (even: CTA pairs)
inline int gemm_sms(const oz2_context* h) {
    static const int env_limit = [] { const char* v = getenv("OZ2_SM_LIMIT"); return v && *v ? atoi(v) : 0; }();
    const int lim = h->sm_limit > 0 ? h->sm_limit : env_limit;
    const int s = lim > 0 && lim < h->num_sms ? lim : h->num_sms;
    return s & ~1;
}
}  // namespace

namespace {
// stage boundary marker (profiling only): one event per boundary, no sync
inline void mark(oz2_handle_t h) {
    if (!h->profiling) return;
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return;
    cudaEventRecord(ev, h->stream);
    h->events.push_back(ev);
}
void drop_events(oz2_handle_t h) {
    for (cudaEvent_t ev : h->events) cudaEventDestroy(ev);
    h->events.clear();
}
}  // namespace

namespace {

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

struct Layout {
    int64_t ldr;
    size_t off_Ares, off_Bres, off_e, off_f, off_stats, off_scratch, off_sync;
    size_t off_E, off_F, off_pr, off_pc;     // accu line 1: max exponents, row / column maxima of P
    size_t off_R;                            // small problems: uint8 c''_t planes [N][m][n]
    size_t off_tiles;                        // SYRK: the triangle's tile list
    size_t total;
};

Layout layout_for(int64_t m, int64_t n, int64_t k, int N, int num_sms, int64_t stats_cols = -1,
                  bool with_B = true, size_t ntiles = 0) {
    Layout L;
    L.ldr = round_up(k > 0 ? k : 1, 16);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = (size_t)round_up((int64_t)(off + bytes), 256); return o; };
    L.off_Ares = take((size_t)N * (size_t)m * (size_t)L.ldr);
    L.off_Bres = take(with_B ? (size_t)N * (size_t)n * (size_t)L.ldr : 0);
    L.off_e = take(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    L.off_f = take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    L.off_stats = take(oz2::cols_stats_bytes(k, stats_cols >= 0 ? stats_cols : n));
    L.off_scratch = take(oz2::fused_scratch_bytes(m, n, N, num_sms));
    L.off_sync = take(256);
    L.off_E = take(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    L.off_F = take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    L.off_pr = take(sizeof(uint32_t) * (size_t)(m > 0 ? m : 1));
    L.off_pc = take(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    L.off_R = take(oz2::gemm_unit_parallel(m, n, num_sms) ? (size_t)N * (size_t)m * (size_t)n : 0);
    L.off_tiles = take(sizeof(uint32_t) * ntiles);
    L.total = off;
    return L;
}

int check_common(int64_t m, int64_t n, int64_t k, int N) {
    if (m < 0 || n < 0 || k < 0) return OZ2_ERR_INVALID_ARG;
    if (N < 2 || N > OZ2_MAX_MODULI) return OZ2_ERR_NUM_MODULI;
    if (k >= OZ2_MAX_K) return OZ2_ERR_K_TOO_LARGE;
    if (m > INT32_MAX || n > INT32_MAX) return OZ2_ERR_INVALID_ARG;
    return OZ2_OK;
}

int kstar_for(oz2_handle_t h, int N, int64_t k, int* kstar) {
    *kstar = 0;
    if (h->mode == OZ2_MODE_EQ17) {
        int ks = oz2_host_eq17_k(N, k);
        if (ks < 1) return OZ2_ERR_BUDGET;
        *kstar = ks;
    }
    return OZ2_OK;
}

int get_workspace(oz2_handle_t h, size_t bytes, uint8_t** ws) {
    if (h->ws_user) {
        if (h->ws_user_bytes < bytes) return OZ2_ERR_WORKSPACE;
        *ws = (uint8_t*)h->ws_user;
        return OZ2_OK;
    }
    if (h->ws_own_bytes < bytes) {
        if (h->ws_own) {
            cudaStreamSynchronize(h->stream);
            cudaFree(h->ws_own);
            h->ws_own = nullptr;
            h->ws_own_bytes = 0;
        }
        if (cudaMalloc(&h->ws_own, bytes) != cudaSuccess) return OZ2_ERR_CUDA;
        h->ws_own_bytes = bytes;
    }
    *ws = (uint8_t*)h->ws_own;
    return OZ2_OK;
}

// 3-D tensor map over residue planes [N][rows][ldr] (int8), box 128 x box_rows x 1, 128B swizzle
// (pstride > 0: bytes between planes, for a row range of larger planes)
int make_plane_map(CUtensorMap* tm, const int8_t* base, int64_t rows, int64_t k, int64_t ldr, int N,
                   int box_rows, int64_t pstride = 0) {
    cuuint64_t dims[3] = {(cuuint64_t)k, (cuuint64_t)rows, (cuuint64_t)N};
    cuuint64_t strides[2] = {(cuuint64_t)ldr, (cuuint64_t)(pstride > 0 ? pstride : ldr * rows)};
    cuuint32_t box[3] = {(cuuint32_t)oz2::gemm_bk(), (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          oz2::gemm_bk() == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? OZ2_OK : OZ2_ERR_CUDA;
}

inline int cuda_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? OZ2_OK : OZ2_ERR_CUDA;
}

struct DevGuard {
    int prev;
    bool changed;
    explicit DevGuard(int dev) : prev(0), changed(false) {
        cudaGetDevice(&prev);
        if (prev != dev) { cudaSetDevice(dev); changed = true; }
    }
    ~DevGuard() { if (changed) cudaSetDevice(prev); }
};

oz2_handle_t g_default[64] = {nullptr};

int check_op_args(int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                  int64_t ldb, const double* C, int64_t ldc, int N);
int accu_line1(oz2_handle_t h, int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
               const double* B, int64_t ldb, int N, uint8_t* ws, const Layout& L, int32_t* e, int32_t* f);
int certify_into(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                 int64_t ldb, const int32_t* e, const int32_t* f, int N, int32_t* beta);

// a bound |trunc(2^e a)| < 2^xbits of the handle's line-1 rule: FAST ||2^e a||_2 <= 2^T
// (reading R4), EQ17 |2^e a| < 2^k* (reading R5); ACCU (and caller exponents) 64 =
// the residue kernels' widest integers for N
int xbits_rule(oz2_handle_t h, int N, int kstar) {
    if (h->mode == OZ2_MODE_FAST) return oz2::host_T(N) + 1;
    if (h->mode == OZ2_MODE_EQ17) return kstar;
    return 64;
}

int ensure_cert(oz2_handle_t h) {
    if (h->cert) return OZ2_OK;
    if (cudaMalloc(&h->cert, 16 * sizeof(int)) != cudaSuccess) { h->cert = nullptr; return OZ2_ERR_CUDA; }
    if (cudaMemset(h->cert, 0, 16 * sizeof(int)) != cudaSuccess) return OZ2_ERR_CUDA;
    return OZ2_OK;
}

int env_flag(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

int ensure_aux(oz2_handle_t h) {
    if (!h->s_aux && cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking) != cudaSuccess) return OZ2_ERR_CUDA;
    if (!h->ev_fork && cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess) return OZ2_ERR_CUDA;
    if (!h->ev_join && cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) return OZ2_ERR_CUDA;
    return OZ2_OK;
}

}  // namespace

namespace oz2 {
unsigned long long& launch_counter_ref() {
    static unsigned long long n = 0;
    return n;
}
}  // namespace oz2

extern "C" {

int oz2_version(void) { return 200; }

unsigned long long oz2_kernel_launches(void) { return __atomic_load_n(&oz2::launch_counter_ref(), __ATOMIC_RELAXED); }

const char* oz2_strerror(int code) {
    switch (code) {
        case OZ2_OK: return "ok";
        case OZ2_ERR_INVALID_ARG: return "invalid argument";
        case OZ2_ERR_NUM_MODULI: return "num_moduli must be in [2, 20]";
        case OZ2_ERR_K_TOO_LARGE: return "k too large: < 2^20, and < 2^17 for oz2_modmul's int32 products (PAPER.md:457-459)";
        case OZ2_ERR_BUDGET: return "EQ17 mode: Eq. (17) budget k_A < 1 for this (N, k)";
        case OZ2_ERR_CUDA: return "CUDA error";
        case OZ2_ERR_NO_DEVICE: return "no sm_100 CUDA device";
        case OZ2_ERR_WORKSPACE: return "workspace too small";
        case OZ2_ERR_NOT_UNIQUE: return "condition (13) 2 c_max < M not certified for the given exponents (PAPER.md:370-381): C was set to NaN";
        default: return "unknown error";
    }
}

int oz2_tables(int N, int32_t* moduli, int32_t* y, uint32_t* w_words, uint32_t* M_words, int32_t* nbytes,
               int32_t* L, int32_t* T) {
    std::call_once(g_tabs_once, build_tables_once);
    if (!g_tabs_ok) return OZ2_ERR_INVALID_ARG;
    if (N < 2 || N > OZ2_MAX_MODULI) return OZ2_ERR_NUM_MODULI;
    const Oz2Table& t = g_tabs[N];
    for (int i = 0; i < N; i++) {
        if (moduli) moduli[i] = t.m[i];
        if (y) y[i] = t.y[i];
        if (w_words) for (int x = 0; x < OZ2_MAX_WORDS; x++) w_words[OZ2_MAX_WORDS * i + x] = t.w32[i][x];
    }
    if (M_words) for (int x = 0; x < OZ2_MAX_WORDS; x++) M_words[x] = t.M32[x];
    if (nbytes) *nbytes = t.JB;
    if (L) *L = t.L;
    if (T) *T = t.T;
    return OZ2_OK;
}

int oz2_eq17_k(int N, int64_t q) {
    if (N < 2 || N > OZ2_MAX_MODULI) return -2;
    return oz2_host_eq17_k(N, q);
}

int oz2_create(oz2_handle_t* h, int device) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = ensure_device(device);
    if (rc) return rc;
    oz2_context* c = new (std::nothrow) oz2_context();
    if (!c) return OZ2_ERR_INVALID_ARG;
    c->device = device;
    if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        delete c;
        return OZ2_ERR_CUDA;
    }
    c->mode = OZ2_MODE_FAST;
    c->certify = 1;
    *h = c;
    return OZ2_OK;
}

int oz2_destroy(oz2_handle_t h) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    drop_events(h);
    for (cudaEvent_t ev : h->pipe_ev) cudaEventDestroy(ev);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    if (h->s_aux) cudaStreamDestroy(h->s_aux);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->ws_own) cudaFree(h->ws_own);
    if (h->tbuf) cudaFree(h->tbuf);
    if (h->cert) cudaFree(h->cert);
    delete h;
    return OZ2_OK;
}

int oz2_set_stream(oz2_handle_t h, void* stream) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    h->stream = (cudaStream_t)stream;
    return OZ2_OK;
}

int oz2_set_mode(oz2_handle_t h, int mode) {
    if (!h || (mode != OZ2_MODE_FAST && mode != OZ2_MODE_EQ17 && mode != OZ2_MODE_ACCU)) return OZ2_ERR_INVALID_ARG;
    h->mode = mode;
    return OZ2_OK;
}

int oz2_set_workspace(oz2_handle_t h, void* ptr, size_t bytes) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    h->ws_user = ptr;
    h->ws_user_bytes = ptr ? bytes : 0;
    return OZ2_OK;
}

int oz2_set_sm_limit(oz2_handle_t h, int sms) {
    if (!h || sms < 0) return OZ2_ERR_INVALID_ARG;
    h->sm_limit = sms;
    return OZ2_OK;
}

int oz2_set_certify(oz2_handle_t h, int enable) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    h->certify = enable ? 1 : 0;
    return OZ2_OK;
}

int oz2_status(oz2_handle_t h) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    if (!h->cert) return OZ2_OK;
    DevGuard g(h->device);
    int st = 0;
    if (cudaMemcpyAsync(&st, h->cert, sizeof(int), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
        return OZ2_ERR_CUDA;
    if (st && cudaMemsetAsync(h->cert, 0, sizeof(int), h->stream) != cudaSuccess) return OZ2_ERR_CUDA;
    return st ? OZ2_ERR_NOT_UNIQUE : OZ2_OK;
}

int oz2_certify(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                int64_t ldb, const int32_t* e, const int32_t* f, int N, int32_t* beta) {
    NvtxRange nvtx_("oz2_certify");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (!beta || lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1) || (m > 0 && k > 0 && (!A || !e)) ||
        (n > 0 && k > 0 && (!B || !f)))
        return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    return certify_into(h, m, n, k, A, lda, B, ldb, e, f, N, beta);
}

int oz2_set_profiling(oz2_handle_t h, int enable) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    h->profiling = enable ? 1 : 0;
    return OZ2_OK;
}

int oz2_stage_times(oz2_handle_t h, double* ms, int64_t* calls) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    const size_t per = OZ2_NUM_STAGES + 1;
    double acc[OZ2_NUM_STAGES] = {0};
    int64_t nc = (int64_t)(h->events.size() / per);
    int rc = OZ2_OK;
    for (int64_t c = 0; c < nc && rc == OZ2_OK; c++) {
        for (size_t s = 0; s < OZ2_NUM_STAGES; s++) {
            float t = 0.f;
            if (cudaEventSynchronize(h->events[c * per + s + 1]) != cudaSuccess ||
                cudaEventElapsedTime(&t, h->events[c * per + s], h->events[c * per + s + 1]) != cudaSuccess) {
                rc = OZ2_ERR_CUDA;
                break;
            }
            acc[s] += t;
        }
    }
    if (ms) for (int s = 0; s < OZ2_NUM_STAGES; s++) ms[s] = acc[s];
    if (calls) *calls = nc;
    drop_events(h);
    return rc;
}

size_t oz2_workspace_bytes(int64_t m, int64_t n, int64_t k, int N) {
    if (m < 0 || n < 0 || k < 0 || N < 2 || N > OZ2_MAX_MODULI) return 0;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
        cudaGetLastError();
        sms = 160;                                   // conservative (> 148) without a device
    }
    return layout_for(m, n, k, N, sms, std::max(m, n)).total;
}

// ---------------------------------------------------------------------------
// split API
// ---------------------------------------------------------------------------
int oz2_scale_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda, int N, int32_t* e) {
    NvtxRange nvtx_("oz2_scale_rows");
    if (!h || h->mode == OZ2_MODE_ACCU) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, 1, k, N);
    if (rc) return rc;
    if (lda < (k > 0 ? k : 1) || (m > 0 && (!A || !e))) return OZ2_ERR_INVALID_ARG;
    int kstar;
    if ((rc = kstar_for(h, N, k, &kstar))) return rc;
    DevGuard g(h->device);
    oz2::launch_rows(A, m, k, lda, N, 1, h->mode, kstar, e, nullptr, 0, h->stream);
    return cuda_status();
}

int oz2_scale_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb, int N, int32_t* f) {
    NvtxRange nvtx_("oz2_scale_cols");
    if (!h || h->mode == OZ2_MODE_ACCU) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(1, n, k, N);
    if (rc) return rc;
    if (ldb < (n > 0 ? n : 1) || (n > 0 && (!B || !f))) return OZ2_ERR_INVALID_ARG;
    int kstar;
    if ((rc = kstar_for(h, N, k, &kstar))) return rc;
    DevGuard g(h->device);
    uint8_t* ws;
    if ((rc = get_workspace(h, oz2::cols_stats_bytes(k, n), &ws))) return rc;
    oz2::launch_cols_exponents(B, k, n, ldb, N, h->mode, kstar, f, ws, h->stream);
    return cuda_status();
}

int oz2_scale_accu(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   const double* B, int64_t ldb, int N, int32_t* e, int32_t* f) {
    NvtxRange nvtx_("oz2_scale_accu");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    if ((m > 0 && !e) || (n > 0 && !f) || ((m > 0 || n > 0) && k > 0 && (!A || !B))) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    if (k == 0 || m == 0 || n == 0) {                 // no products: zero rows / columns get 0
        if (m > 0) cudaMemsetAsync(e, 0, sizeof(int32_t) * (size_t)m, h->stream);
        if (n > 0) cudaMemsetAsync(f, 0, sizeof(int32_t) * (size_t)n, h->stream);
        return cuda_status();
    }
    Layout L = layout_for(m, n, k, 1, gemm_sms(h));
    uint8_t* ws;
    if ((rc = get_workspace(h, L.total, &ws))) return rc;
    return accu_line1(h, OZ2_OP_N, OZ2_OP_N, m, n, k, A, lda, B, ldb, N, ws, L, e, f);
}

int oz2_trunc_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda, const int32_t* e,
                   double* Ap) {
    if (!h || m < 0 || k < 0 || lda < (k > 0 ? k : 1)) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    oz2::launch_trunc_rows(A, m, k, lda, e, Ap, h->stream);
    return cuda_status();
}

int oz2_trunc_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb, const int32_t* f,
                   double* BpT) {
    if (!h || n < 0 || k < 0 || ldb < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    oz2::launch_trunc_cols(B, k, n, ldb, f, BpT, h->stream);
    return cuda_status();
}

int oz2_residues_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda, const int32_t* e,
                      int N, int8_t* Ares, int64_t ld_res) {
    NvtxRange nvtx_("oz2_residues_rows");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, 1, k, N);
    if (rc) return rc;
    if (lda < (k > 0 ? k : 1) || ld_res < k || ld_res % 16) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    if (k > 0) oz2::launch_rows(A, m, k, lda, N, 2, h->mode, 0, const_cast<int32_t*>(e), Ares, ld_res, h->stream);
    return cuda_status();
}

int oz2_residues_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb, const int32_t* f,
                      int N, int8_t* Bres, int64_t ld_res) {
    NvtxRange nvtx_("oz2_residues_cols");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(1, n, k, N);
    if (rc) return rc;
    if (ldb < (n > 0 ? n : 1) || ld_res < k || ld_res % 16) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    oz2::launch_cols_residues(B, k, n, ldb, f, N, Bres, ld_res, h->stream);
    return cuda_status();
}

int oz2_modmul(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const int8_t* Ares, const int8_t* Bres,
               int64_t ld_res, int N, int32_t* Cprod) {
    NvtxRange nvtx_("oz2_modmul");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (ld_res < k || ld_res % 16) return OZ2_ERR_INVALID_ARG;
    if (k >= (int64_t)1 << 17) return OZ2_ERR_K_TOO_LARGE;     // int32 C'_t exact only below 2^17
    if (m == 0 || n == 0) return OZ2_OK;
    DevGuard g(h->device);
    if (k == 0) {
        return cudaMemsetAsync(Cprod, 0, sizeof(int32_t) * (size_t)N * m * n, h->stream) == cudaSuccess ? OZ2_OK
                                                                                                        : OZ2_ERR_CUDA;
    }
    CUtensorMap tA, tB;
    if ((rc = make_plane_map(&tA, Ares, m, k, ld_res, N, 128))) return rc;
    if ((rc = make_plane_map(&tB, Bres, n, k, ld_res, N, 256 / oz2::gemm_cta_group()))) return rc;
    uint8_t* ws;
    if ((rc = get_workspace(h, 256, &ws))) return rc;
    if (oz2::launch_modmul(&tA, &tB, m, n, k, N, Cprod, (uint32_t*)ws, gemm_sms(h), h->stream)) return OZ2_ERR_CUDA;
    return cuda_status();
}

int oz2_crt(oz2_handle_t h, int64_t m, int64_t n, const int32_t* Cprod, const int32_t* e, const int32_t* f,
            int N, double* C, int64_t ldc, const int32_t* beta) {
    NvtxRange nvtx_("oz2_crt");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, 0, N);
    if (rc) return rc;
    if (ldc < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    if (beta && (rc = ensure_cert(h))) return rc;
    oz2::launch_crt(Cprod, m, n, e, f, N, C, ldc, h->stream);
    if (beta) oz2::launch_refuse(beta, N, C, m, n, ldc, h->cert, h->stream);
    return cuda_status();
}

// ---------------------------------------------------------------------------
// main entry points
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

// Argument checks of the DGEMM surface (row-major): op(A) m x k, op(B) k x n.
int check_op_args(int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                  int64_t ldb, const double* C, int64_t ldc, int N) {
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if ((ta != OZ2_OP_N && ta != OZ2_OP_T) || (tb != OZ2_OP_N && tb != OZ2_OP_T)) return OZ2_ERR_INVALID_ARG;
    const int64_t need_a = ta == OZ2_OP_N ? k : m, need_b = tb == OZ2_OP_N ? n : k;
    if (lda < (need_a > 0 ? need_a : 1) || ldb < (need_b > 0 ? need_b : 1) || ldc < (n > 0 ? n : 1))
        return OZ2_ERR_INVALID_ARG;
    if (m > 0 && n > 0 && (!C || (k > 0 && (!A || !B)))) return OZ2_ERR_INVALID_ARG;
    return OZ2_OK;
}

// Alg. 1 line 1 by the OS II-accu rule (reading R18): e[m], f[n] from op(A),
// op(B).  Uses plane 0 of the residue buffers for the 7-bit approximations
// (overwritten by the residues afterwards).  k < 2^17 (exact int32 bound GEMM).
// OS II-accu line 1 without the last step: E, F, and the row / column maxima
// of the bound P = Ahat Bhat^T in the workspace (L.off_E, off_F, off_pr, off_pc)
int accu_bound(oz2_handle_t h, int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
               const double* B, int64_t ldb, int N, uint8_t* ws, const Layout& L) {
    if (k >= (int64_t)1 << 17) return OZ2_ERR_K_TOO_LARGE;
    uint8_t* Ah = ws + L.off_Ares;
    uint8_t* Bh = ws + L.off_Bres;
    int32_t* E = (int32_t*)(ws + L.off_E);
    int32_t* F = (int32_t*)(ws + L.off_F);
    uint32_t* pr = (uint32_t*)(ws + L.off_pr);
    uint32_t* pc = (uint32_t*)(ws + L.off_pc);
    if (ta == OZ2_OP_N) {
        oz2::launch_rows_hat7(A, m, k, lda, E, Ah, L.ldr, h->stream);
    } else {
        oz2::launch_cols_exponents(A, k, m, lda, N, OZ2_MODE_ACCU, 0, E, ws + L.off_stats, h->stream);
        oz2::launch_cols_hat7(A, k, m, lda, E, Ah, L.ldr, h->stream);
    }
    if (tb == OZ2_OP_N) {
        oz2::launch_cols_exponents(B, k, n, ldb, N, OZ2_MODE_ACCU, 0, F, ws + L.off_stats, h->stream);
        oz2::launch_cols_hat7(B, k, n, ldb, F, Bh, L.ldr, h->stream);
    } else {
        oz2::launch_rows_hat7(B, n, k, ldb, F, Bh, L.ldr, h->stream);
    }
    CUtensorMap tA, tB;
    int rc;
    if ((rc = make_plane_map(&tA, (const int8_t*)Ah, m, k, L.ldr, 1, 128))) return rc;
    if ((rc = make_plane_map(&tB, (const int8_t*)Bh, n, k, L.ldr, 1, 256 / oz2::gemm_cta_group()))) return rc;
    if (oz2::launch_bound_gemm(&tA, &tB, m, n, k, pr, pc, (uint32_t*)(ws + L.off_sync), gemm_sms(h), h->stream))
        return OZ2_ERR_CUDA;
    return cuda_status();
}

int accu_line1(oz2_handle_t h, int ta, int tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
               const double* B, int64_t ldb, int N, uint8_t* ws, const Layout& L, int32_t* e, int32_t* f) {
    int rc = accu_bound(h, ta, tb, m, n, k, A, lda, B, ldb, N, ws, L);
    if (rc) return rc;
    oz2::launch_accu_finalize((int32_t*)(ws + L.off_E), (uint32_t*)(ws + L.off_pr), m, N, e, h->stream);
    oz2::launch_accu_finalize((int32_t*)(ws + L.off_F), (uint32_t*)(ws + L.off_pc), n, N, f, h->stream);
    return cuda_status();
}

// condition (13) certificate of caller exponents into *beta (certify.cu): the
// Cauchy-Schwarz bound, and for k < 2^17 also the OS II-accu bound
int certify_into(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                 int64_t ldb, const int32_t* e, const int32_t* f, int N, int32_t* beta) {
    int rc;
    if ((rc = ensure_cert(h))) return rc;
    Layout L = layout_for(m, n, k, 1, gemm_sms(h), std::max(m, n));
    uint8_t* ws;
    if ((rc = get_workspace(h, L.total, &ws))) return rc;
    oz2::AccuBound ab{(const int32_t*)(ws + L.off_E), (const int32_t*)(ws + L.off_F),
                      (const uint32_t*)(ws + L.off_pr), (const uint32_t*)(ws + L.off_pc)};
    const bool with_p = k > 0 && k < ((int64_t)1 << 17) && m > 0 && n > 0;
    if (with_p && (rc = accu_bound(h, OZ2_OP_N, OZ2_OP_N, m, n, k, A, lda, B, ldb, N, ws, L))) return rc;
    oz2::launch_certify(A, m, k, lda, B, n, ldb, e, f, N, h->cert + 4, ws + L.off_stats, beta, with_p ? &ab : nullptr,
                        h->stream);
    return cuda_status();
}

// C = alpha op(A) op(B) + beta C by Algorithm 1 (arguments already checked).
// op(A) = A^T means the stored A is k x m: its "rows of op(A)" are the columns
// of the stored matrix, so the column kernels produce e and the K-major planes;
// likewise op(B) = B^T (stored n x k) goes through the row kernel.
// e_given / f_given (both or neither): caller-supplied line-1 exponents (lines 2-10 only).
// tri = 1 / 2 (SYRK, B is A with the other transpose, m == n): op(B) = op(A)^T
// shares op(A)'s exponents and residue planes, only the output tiles that meet
// the lower / upper triangle run, and only that triangle of C is read or written.
int dgemm_core(oz2_handle_t h, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
               int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int N,
               const int32_t* e_given = nullptr, const int32_t* f_given = nullptr, int tri = 0, int kskip = 0) {
    NvtxRange nvtx_("dgemm_core");
    if (m == 0 || n == 0) return OZ2_OK;
    const bool given = e_given && f_given;
    int rc, kstar = 0;
    if (!given && k > 0 && alpha != 0.0 && (rc = kstar_for(h, N, k, &kstar))) return rc;
    DevGuard g(h->device);
    if (k == 0 || alpha == 0.0) {                     // no product: C = beta C (0 if beta == 0)
        if (beta == 1.0) return OZ2_OK;
        oz2::launch_scale_c(C, m, n, ldc, beta, h->stream, tri);
        return cuda_status();
    }
    const std::vector<uint32_t> tiles = tri ? oz2::tri_tile_list(m, n, tri, gemm_sms(h)) : std::vector<uint32_t>();
    Layout L = layout_for(m, n, k, N, gemm_sms(h), ta == OZ2_OP_T ? std::max(m, n) : n, !tri, tiles.size());
    if (tri) L.off_Bres = L.off_Ares;                 // one set of planes (accu: B-hat = A-hat, same bytes)
    uint8_t* ws;
    if ((rc = get_workspace(h, L.total, &ws))) return rc;
    int8_t* Ares = (int8_t*)(ws + L.off_Ares);
    int8_t* Bres = tri ? Ares : (int8_t*)(ws + L.off_Bres);
    int32_t* e = given ? const_cast<int32_t*>(e_given) : (int32_t*)(ws + L.off_e);
    int32_t* f = given ? const_cast<int32_t*>(f_given) : (int32_t*)(ws + L.off_f);
    if (tri && !tiles.empty() &&
        cudaMemcpyAsync(ws + L.off_tiles, tiles.data(), sizeof(uint32_t) * tiles.size(), cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess)
        return OZ2_ERR_CUDA;
    uint8_t* scratch = ws + L.off_scratch;
    CUtensorMap tA, tB;
    if ((rc = make_plane_map(&tA, Ares, m, k, L.ldr, N, 128))) return rc;
    if ((rc = make_plane_map(&tB, Bres, n, k, L.ldr, N, 256 / oz2::gemm_cta_group()))) return rc;
    // Part 1 + 2-a (Alg. 1 lines 1-5) for op(A) and op(B).  With the accu rule
    // the exponents come first from both operands (accu_line1, timed in stage
    // ROWS), and the conversions below only form the residues.
    const bool accu = h->mode == OZ2_MODE_ACCU && !given;
    const bool skip_line1 = accu || given;              // e, f known before the residue passes
    const int what = skip_line1 ? 2 : 3;
    const int xb = given ? 64 : xbits_rule(h, N, kstar);
    auto convert_A = [&](cudaStream_t st) {
        if (ta == OZ2_OP_N) {
            oz2::launch_rows(A, m, k, lda, N, what, h->mode, kstar, e, Ares, L.ldr, st, 0, xb);
        } else {
            if (!skip_line1) oz2::launch_cols_exponents(A, k, m, lda, N, h->mode, kstar, e, ws + L.off_stats, st);
            oz2::launch_cols_residues(A, k, m, lda, e, N, Ares, L.ldr, st, 0, xb);
        }
    };
    auto convert_B_stats = [&](cudaStream_t st) {
        if (tri) return;                              // SYRK: op(B) = op(A)^T shares e and the planes
        if (tb == OZ2_OP_N && !skip_line1)
            oz2::launch_cols_exponents(B, k, n, ldb, N, h->mode, kstar, f, ws + L.off_stats, st);
    };
    auto convert_B_res = [&](cudaStream_t st) {
        if (tri) return;
        if (tb == OZ2_OP_N) oz2::launch_cols_residues(B, k, n, ldb, f, N, Bres, L.ldr, st, 0, xb);
        else oz2::launch_rows(B, n, k, ldb, N, what, h->mode, kstar, f, Bres, L.ldr, st, 0, xb);
    };
    mark(h);
    if (accu && (rc = accu_line1(h, ta, tb, m, n, k, A, lda, B, ldb, N, ws, L, e, f))) return rc;
    // A and B are independent passes; OZ2_CONV_OVERLAP=1 runs B's on a second
    // stream concurrently with A's (stage ROWS then times both, the column stages
    // read 0).  Default off: measured no gain, both passes are issue-bound.  (Not
    // with op(A) = A^T, whose column statistics share B's scratch.)
    const bool overlap = env_flag("OZ2_CONV_OVERLAP", 0) && ta == OZ2_OP_N && !skip_line1 && !tri;
    if (overlap) {
        if ((rc = ensure_aux(h))) return rc;
        cudaEventRecord(h->ev_fork, h->stream);
        cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0);
        convert_B_stats(h->s_aux);
        convert_B_res(h->s_aux);
        cudaEventRecord(h->ev_join, h->s_aux);
        convert_A(h->stream);
        cudaStreamWaitEvent(h->stream, h->ev_join, 0);
        mark(h);
        mark(h);
        mark(h);
    } else {
        convert_A(h->stream);
        mark(h);
        convert_B_stats(h->stream);
        mark(h);
        convert_B_res(h->stream);
        mark(h);
    }
    if (tri) {
        // SYRK: the triangle's tiles only, f = e (the columns of op(A)^T are the rows of op(A))
        if (oz2::launch_modmul_fused(&tA, &tB, m, n, k, N, scratch, e, e, C, ldc, (uint32_t*)(ws + L.off_sync),
                                     gemm_sms(h), h->stream, alpha, beta, tri, (const uint32_t*)(ws + L.off_tiles),
                                     (int)tiles.size()))
            return OZ2_ERR_CUDA;
        mark(h);
        mark(h);
        return cuda_status();
    }
    if (oz2::gemm_unit_parallel(m, n, gemm_sms(h)) && alpha == 1.0 && beta == 0.0 && !kskip) {
        // small problem (fewer output tiles than CTA pairs): the (tile, modulus)
        // units spread over all SMs (line 6-7 into uint8 planes), then lines 8-10
        // in a separate elementwise kernel
        uint8_t* R = ws + L.off_R;
        if (oz2::launch_modmul_residues(&tA, &tB, m, n, k, N, scratch, R, m, (uint32_t*)(ws + L.off_sync),
                                        gemm_sms(h), h->stream))
            return OZ2_ERR_CUDA;
        mark(h);
        oz2::launch_crt_sum(R, 1, (int64_t)N * m * n, m, n, e, f, N, C, ldc, h->stream);
        mark(h);
        return cuda_status();
    }
    // Part 2-b (line 6) with Parts 2-c, 3, 4 (lines 7-10) fused into the epilogue
    if (oz2::launch_modmul_fused(&tA, &tB, m, n, k, N, scratch, e, f, C, ldc, (uint32_t*)(ws + L.off_sync),
                                 gemm_sms(h), h->stream, alpha, beta, 0, nullptr, 0, kskip))
        return OZ2_ERR_CUDA;
    mark(h);
    mark(h);                                          // (no separate CRT stage)
    return cuda_status();
}

// 2-D host pipeline (FAST / EQ17, large m and n).  Row blocks of A and column
// panels of B go over the H2D stream interleaved so that the fractions of A and
// of B on the device stay level (B slightly ahead), each converted once when it
// lands into plane-major residues ([N][m][ldr], [N][n][ldr]).  A block that
// lands is multiplied at once with ALL panels already present, and a panel that
// lands with ALL blocks already present: one GEMM launch per arrival (the
// arrived blocks / panels are a contiguous row / column range of the planes),
// so every (block, panel) pair runs exactly once, in launches of many tiles.
// The last blocks of A shrink (512, 256, 256 rows) so the GEMM and the C
// copy-back after the final arrival are short.  Each product's C block leaves
// on the D2H stream as soon as it is written.  Bit-identical to one call: e_i
// depends on row i only, f_j on column j only.
int dgemm_host_2d(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc, int N, int kstar) {
    const int64_t pa = round_up(std::max<int64_t>(256, env_flag("OZ2_HOST_BLOCK", 1024)), 256);
    const int64_t pb = round_up(std::max<int64_t>(512, env_flag("OZ2_HOST_PANEL", 1024)), 512);
    std::vector<int64_t> r0s, nrs, c0s, ncs;
    {
        // A: blocks of pa rows, the last pa rows as pa/2, pa/4, pa/4 (multiples of 256)
        const int64_t tail = m > 2 * pa ? pa : 0;
        int64_t r = 0;
        for (; r + pa <= m - tail; r += pa) { r0s.push_back(r); nrs.push_back(pa); }
        if (r < m - tail) { r0s.push_back(r); nrs.push_back(m - tail - r); r = m - tail; }
        if (tail) {
            const int64_t t1 = round_up(tail / 2, 256), t2 = std::max<int64_t>(256, round_up(tail / 4, 256));
            for (int64_t sz : {t1, t2}) {
                if (r < m) { const int64_t rows = std::min(sz, m - r); r0s.push_back(r); nrs.push_back(rows); r += rows; }
            }
            if (r < m) { r0s.push_back(r); nrs.push_back(m - r); }
        }
        for (int64_t c = 0; c < n; c += pb) { c0s.push_back(c); ncs.push_back(std::min(pb, n - c)); }
    }
    const int64_t np = (int64_t)c0s.size(), nr = (int64_t)r0s.size();
    Layout L = layout_for(m, n, k, N, gemm_sms(h), pb);
    const size_t bytesA = sizeof(double) * (size_t)m * (size_t)k;
    const size_t bytesB = sizeof(double) * (size_t)k * (size_t)n;
    const size_t offA = (size_t)round_up((int64_t)L.total, 256);
    const size_t offB = (size_t)round_up((int64_t)(offA + bytesA), 256);
    const size_t offC = (size_t)round_up((int64_t)(offB + bytesB), 256);
    uint8_t* ws;
    int rc;
    if ((rc = get_workspace(h, offC + sizeof(double) * (size_t)m * (size_t)n, &ws))) return rc;
    double* dA = (double*)(ws + offA);
    double* dB = (double*)(ws + offB);
    double* dC = (double*)(ws + offC);
    if (!h->s_h2d && cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking) != cudaSuccess) return OZ2_ERR_CUDA;
    if (!h->s_d2h && cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking) != cudaSuccess) return OZ2_ERR_CUDA;
    const size_t nev = (size_t)(1 + 2 * (np + nr));
    while (h->pipe_ev.size() < nev) {
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return OZ2_ERR_CUDA;
        h->pipe_ev.push_back(ev);
    }
    cudaEvent_t evStart = h->pipe_ev[0];
    cudaEvent_t* evIn = &h->pipe_ev[1];                          // per piece: landed on the device
    cudaEvent_t* evOut = &h->pipe_ev[1 + np + nr];               // per piece: its product written
    if (cudaEventRecord(evStart, h->stream) != cudaSuccess) return OZ2_ERR_CUDA;
    cudaStreamWaitEvent(h->s_h2d, evStart, 0);
    cudaStreamWaitEvent(h->s_d2h, evStart, 0);
    // transfer order: keep the landed fraction of B at or just above that of A
    std::vector<std::pair<int, int64_t>> order;                  // (0 = panel of B, 1 = block of A, index)
    {
        int64_t ia = 0, ib = 0, rows_sent = 0, cols_sent = 0;
        while (ia < nr || ib < np) {
            const bool sendB = ib < np && (ia >= nr || (double)cols_sent / n <= (double)rows_sent / m + 1e-12);
            if (sendB) { order.push_back({0, ib}); cols_sent += ncs[ib]; ib++; }
            else { order.push_back({1, ia}); rows_sent += nrs[ia]; ia++; }
        }
    }
    for (size_t q = 0; q < order.size(); q++) {
        const auto& o = order[q];
        cudaError_t ce;
        if (o.first == 0) {
            const int64_t c0 = c0s[o.second], nc = ncs[o.second];
            ce = cudaMemcpy2DAsync(dB + c0, sizeof(double) * n, B + c0, sizeof(double) * ldb, sizeof(double) * nc, k,
                                   cudaMemcpyHostToDevice, h->s_h2d);
        } else {
            const int64_t r0 = r0s[o.second], rows = nrs[o.second];
            ce = cudaMemcpy2DAsync(dA + r0 * k, sizeof(double) * k, A + r0 * lda, sizeof(double) * lda,
                                   sizeof(double) * k, rows, cudaMemcpyHostToDevice, h->s_h2d);
        }
        if (ce == cudaSuccess) ce = cudaEventRecord(evIn[q], h->s_h2d);
        if (ce != cudaSuccess) return OZ2_ERR_CUDA;
    }
    int8_t* Ares = (int8_t*)(ws + L.off_Ares);                 // plane-major [N][m][ldr]
    int8_t* Bres = (int8_t*)(ws + L.off_Bres);                 // plane-major [N][n][ldr]
    int32_t* e = (int32_t*)(ws + L.off_e);
    int32_t* f = (int32_t*)(ws + L.off_f);
    const int64_t psA = m * L.ldr, psB = n * L.ldr;
    mark(h);
    mark(h);
    mark(h);
    mark(h);                                                   // conversions are timed inside the GEMM stage
    // rows [r0, r0 + rows) x columns [c0, c0 + nc): one fused GEMM launch, then its C block goes back
    auto product = [&](int64_t r0, int64_t rows, int64_t c0, int64_t nc, cudaEvent_t ev) -> int {
        CUtensorMap tA, tB;
        int rr;
        if ((rr = make_plane_map(&tA, Ares + r0 * L.ldr, rows, k, L.ldr, N, 128, psA))) return rr;
        if ((rr = make_plane_map(&tB, Bres + c0 * L.ldr, nc, k, L.ldr, N, 256 / oz2::gemm_cta_group(), psB))) return rr;
        if (oz2::launch_modmul_fused(&tA, &tB, rows, nc, k, N, ws + L.off_scratch, e + r0, f + c0, dC + r0 * n + c0, n,
                                     (uint32_t*)(ws + L.off_sync), gemm_sms(h), h->stream))
            return OZ2_ERR_CUDA;
        cudaEventRecord(ev, h->stream);
        cudaStreamWaitEvent(h->s_d2h, ev, 0);
        if (cudaMemcpy2DAsync(C + r0 * ldc + c0, sizeof(double) * ldc, dC + r0 * n + c0, sizeof(double) * n,
                              sizeof(double) * nc, rows, cudaMemcpyDeviceToHost, h->s_d2h) != cudaSuccess)
            return OZ2_ERR_CUDA;
        return OZ2_OK;
    };
    int64_t rows_in = 0, cols_in = 0;                          // landed prefixes of A's rows / B's columns
    for (size_t q = 0; q < order.size(); q++) {
        const int64_t x = order[q].second;
        cudaStreamWaitEvent(h->stream, evIn[q], 0);
        if (order[q].first == 0) {
            const int64_t c0 = c0s[x], nc = ncs[x];
            oz2::launch_cols_exponents(dB + c0, k, nc, n, N, h->mode, kstar, f + c0, ws + L.off_stats, h->stream);
            oz2::launch_cols_residues(dB + c0, k, nc, n, f + c0, N, Bres + c0 * L.ldr, L.ldr, h->stream, psB,
                                      xbits_rule(h, N, kstar));
            cols_in = c0 + nc;
            if (rows_in > 0 && (rc = product(0, rows_in, c0, nc, evOut[q]))) return rc;
        } else {
            const int64_t r0 = r0s[x], rows = nrs[x];
            oz2::launch_rows(dA + r0 * k, rows, k, k, N, 3, h->mode, kstar, e + r0, Ares + r0 * L.ldr, L.ldr,
                             h->stream, psA, xbits_rule(h, N, kstar));
            rows_in = r0 + rows;
            if (cols_in > 0 && (rc = product(r0, rows, 0, cols_in, evOut[q]))) return rc;
        }
    }
    mark(h);
    mark(h);
    if ((rc = cuda_status())) return rc;
    return cudaStreamSynchronize(h->s_d2h) == cudaSuccess && cudaStreamSynchronize(h->stream) == cudaSuccess
               ? OZ2_OK : OZ2_ERR_CUDA;
}

}  // namespace

extern "C" {

int oz2_dgemm_ex(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double* C, int64_t ldc, int N) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_op_args(OZ2_OP_N, OZ2_OP_N, m, n, k, A, lda, B, ldb, C, ldc, N);
    if (rc) return rc;
    return dgemm_core(h, OZ2_OP_N, OZ2_OP_N, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc, N);
}

int oz2_dgemm_op(oz2_handle_t h, int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc, int N) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_op_args(transA, transB, m, n, k, A, lda, B, ldb, C, ldc, N);
    if (rc) return rc;
    return dgemm_core(h, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, N);
}

int oz2_dtrmm(oz2_handle_t h, int side, int uplo, int transA, int diag, int64_t m, int64_t n, double alpha,
              const double* A, int64_t lda, double* B, int64_t ldb, int N) {
    NvtxRange nvtx_("oz2_dtrmm");
    if (!h) return OZ2_ERR_INVALID_ARG;
    if ((side != OZ2_LEFT && side != OZ2_RIGHT) || (uplo != OZ2_LOWER && uplo != OZ2_UPPER) ||
        (transA != OZ2_OP_N && transA != OZ2_OP_T) || (diag != OZ2_NON_UNIT && diag != OZ2_UNIT))
        return OZ2_ERR_INVALID_ARG;
    const int64_t na = side == OZ2_LEFT ? m : n;       // A is na x na
    int rc = check_common(m, n, na, N);
    if (rc) return rc;
    if (lda < (na > 0 ? na : 1) || ldb < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    if (m == 0 || n == 0) return OZ2_OK;
    if (!A || !B) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    // T = tri(A) (zeros outside the triangle, ones on a unit diagonal), then the
    // product with B written over B: the GEMM reads only the residue planes,
    // which are complete before its first store, so C may alias B (beta = 0)
    const size_t tb = sizeof(double) * (size_t)na * (size_t)na;
    if (h->tbuf_bytes < tb) {
        if (h->tbuf) { cudaStreamSynchronize(h->stream); cudaFree(h->tbuf); h->tbuf = nullptr; h->tbuf_bytes = 0; }
        if (cudaMalloc(&h->tbuf, tb) != cudaSuccess) return OZ2_ERR_CUDA;
        h->tbuf_bytes = tb;
    }
    double* T = (double*)h->tbuf;
    oz2::launch_tri_copy(A, na, lda, uplo, diag == OZ2_UNIT, T, h->stream);
    // op(A) lower iff (lower, N) or (upper, T); its zero K blocks are skipped per output tile
    const bool low = (uplo == OZ2_LOWER) == (transA == OZ2_OP_N);
    if (side == OZ2_LEFT)
        return dgemm_core(h, transA, OZ2_OP_N, m, n, m, alpha, T, m, B, ldb, 0.0, B, ldb, N, nullptr, nullptr, 0,
                          low ? 1 : 2);
    return dgemm_core(h, OZ2_OP_N, transA, m, n, n, alpha, B, ldb, T, n, 0.0, B, ldb, N, nullptr, nullptr, 0,
                      low ? 3 : 4);
}

int oz2_dsyrk(oz2_handle_t h, int uplo, int trans, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, double beta, double* C, int64_t ldc, int N) {
    NvtxRange nvtx_("oz2_dsyrk");
    if (!h) return OZ2_ERR_INVALID_ARG;
    if (uplo != OZ2_LOWER && uplo != OZ2_UPPER) return OZ2_ERR_INVALID_ARG;
    if (trans != OZ2_OP_N && trans != OZ2_OP_T) return OZ2_ERR_INVALID_ARG;
    // C := alpha op(A) op(A)^T + beta C: op(B) = op(A)^T is A itself with the other transpose
    const int tb = trans == OZ2_OP_N ? OZ2_OP_T : OZ2_OP_N;
    int rc = check_op_args(trans, tb, n, n, k, A, lda, A, lda, C, ldc, N);
    if (rc) return rc;
    return dgemm_core(h, trans, tb, n, n, k, alpha, A, lda, A, lda, beta, C, ldc, N, nullptr, nullptr, uplo);
}

// Prepared operands (oz2_prepare_a / oz2_prepare_b): exponents and residue
// planes of one operand, in memory owned by the object (one cudaMalloc each)
struct oz2_prepared {
    int device, side, N, mode;           // side: OZ2_LEFT (A, rows x k) or OZ2_RIGHT (B, k x rows)
    int64_t rows, k, ldr;
    void* mem;
    int32_t* exps;                       // e[rows] (A) or f[rows] (B)
    int8_t* planes;                      // [N][rows][ldr], K-major
};

namespace {
int prepare_common(oz2_handle_t h, int side, int64_t rows, int64_t k, const double* X, int64_t ld, int N,
                   oz2_prep_t* out) {
    NvtxRange nvtx_("prepare_common");
    if (!h || !out) return OZ2_ERR_INVALID_ARG;
    *out = nullptr;
    int rc = check_common(rows, rows, k, N);
    if (rc) return rc;
    if (h->mode == OZ2_MODE_ACCU) return OZ2_ERR_INVALID_ARG;        // accu couples A and B
    const int64_t need_ld = side == OZ2_LEFT ? (k > 0 ? k : 1) : (rows > 0 ? rows : 1);
    if (ld < need_ld || (k > 0 && rows > 0 && !X)) return OZ2_ERR_INVALID_ARG;
    int kstar = 0;
    if (k > 0 && (rc = kstar_for(h, N, k, &kstar))) return rc;
    DevGuard g(h->device);
    oz2_prepared* p = new (std::nothrow) oz2_prepared();
    if (!p) return OZ2_ERR_INVALID_ARG;
    p->device = h->device; p->side = side; p->N = N; p->mode = h->mode;
    p->rows = rows; p->k = k; p->ldr = round_up(k > 0 ? k : 1, 16);
    const size_t off_planes = (size_t)round_up((int64_t)sizeof(int32_t) * (rows > 0 ? rows : 1), 256);
    const size_t off_stats = (size_t)round_up((int64_t)(off_planes + (size_t)N * (size_t)rows * (size_t)p->ldr), 256);
    const size_t total = off_stats + (side == OZ2_RIGHT ? oz2::cols_stats_bytes(k, rows) : 0);
    if (cudaMalloc(&p->mem, total) != cudaSuccess) { delete p; return OZ2_ERR_CUDA; }
    uint8_t* base = (uint8_t*)p->mem;
    p->exps = (int32_t*)base;
    p->planes = (int8_t*)(base + off_planes);
    if (k > 0 && rows > 0) {
        if (side == OZ2_LEFT) {
            oz2::launch_rows(X, rows, k, ld, N, 3, h->mode, kstar, p->exps, p->planes, p->ldr, h->stream, 0,
                             xbits_rule(h, N, kstar));
        } else {
            oz2::launch_cols_exponents(X, k, rows, ld, N, h->mode, kstar, p->exps, base + off_stats, h->stream);
            oz2::launch_cols_residues(X, k, rows, ld, p->exps, N, p->planes, p->ldr, h->stream, 0,
                                      xbits_rule(h, N, kstar));
        }
    }
    if ((rc = cuda_status())) { cudaFree(p->mem); delete p; return rc; }
    *out = p;
    return OZ2_OK;
}

// lines 6-10 on converted operands: A' planes (ldr_a) x B' planes (ldr_b)
int prepared_product(oz2_handle_t h, int64_t m, int64_t n, int64_t k, int N, const int8_t* Ares, int64_t ldr_a,
                     const int32_t* e, const int8_t* Bres, int64_t ldr_b, const int32_t* f, double* C, int64_t ldc,
                     uint8_t* ws, const Layout& L) {
    int rc;
    CUtensorMap tA, tB;
    if ((rc = make_plane_map(&tA, Ares, m, k, ldr_a, N, 128))) return rc;
    if ((rc = make_plane_map(&tB, Bres, n, k, ldr_b, N, 256 / oz2::gemm_cta_group()))) return rc;
    if (oz2::launch_modmul_fused(&tA, &tB, m, n, k, N, ws + L.off_scratch, e, f, C, ldc,
                                 (uint32_t*)(ws + L.off_sync), gemm_sms(h), h->stream))
        return OZ2_ERR_CUDA;
    return cuda_status();
}
}  // namespace

int oz2_fp64mod_tables(int s, int64_t q, int64_t* moduli, uint32_t* M_words, int32_t* L, int32_t* T) {
    if (s < 2 || s > oz2::F64_MAX_S) return OZ2_ERR_NUM_MODULI;
    if (q < 1 || q > OZ2_MAX_K) return OZ2_ERR_INVALID_ARG;
    return oz2::f64_tables(s, q, moduli, M_words, L, T) ? OZ2_ERR_INVALID_ARG : OZ2_OK;
}

size_t oz2_fp64mod_workspace_bytes(int64_t m, int64_t n, int64_t k, int s) {
    if (m < 0 || n < 0 || k < 1 || s < 2 || s > oz2::F64_MAX_S) return 0;
    return oz2::f64_workspace_bytes(m, n, k, s);
}

int oz2_dgemm_fp64mod(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                      const double* B, int64_t ldb, int s, int v, double* C, int64_t ldc, int64_t strideC) {
    return oz2_dgemm_fp64mod_dw(h, m, n, k, A, nullptr, lda, B, nullptr, ldb, s, v, C, ldc, strideC);
}

int oz2_dgemm_fp64mod_dw(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, const double* A2,
                         int64_t lda, const double* B, const double* B2, int64_t ldb, int s, int v, double* C,
                         int64_t ldc, int64_t strideC) {
    NvtxRange nvtx_("oz2_dgemm_fp64mod_dw");
    if (!h) return OZ2_ERR_INVALID_ARG;
    if (s < 2 || s > oz2::F64_MAX_S) return OZ2_ERR_NUM_MODULI;
    if (m < 0 || n < 0 || k < 0 || v < 1 || v > 4) return OZ2_ERR_INVALID_ARG;
    if (k >= OZ2_MAX_K) return OZ2_ERR_K_TOO_LARGE;
    if (m > INT32_MAX || n > INT32_MAX || m * k > INT32_MAX || k * n > INT32_MAX || m * n > INT32_MAX)
        return OZ2_ERR_INVALID_ARG;                   // cuBLAS int dimensions / strides
    if (lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1) || ldc < (n > 0 ? n : 1) ||
        (v > 1 && strideC < m * ldc) || (m > 0 && n > 0 && (!C || (k > 0 && (!A || !B)))))
        return OZ2_ERR_INVALID_ARG;
    if (m == 0 || n == 0) return OZ2_OK;
    DevGuard g(h->device);
    if (k == 0) {
        for (int w = 0; w < v; w++) oz2::launch_scale_c(C + w * strideC, m, n, ldc, 0.0, h->stream);
        return cuda_status();
    }
    uint8_t* ws;
    int rc;
    if ((rc = get_workspace(h, oz2::f64_workspace_bytes(m, n, k, s), &ws))) return rc;
    const int r = oz2::launch_fp64mod(h->device, A, A2, m, k, lda, B, B2, n, ldb, s, v, C, ldc, strideC, ws,
                                      h->stream);
    if (r == -1) return OZ2_ERR_INVALID_ARG;
    if (r) return OZ2_ERR_CUDA;
    return cuda_status();
}

int oz2_reprepare(oz2_handle_t h, oz2_prep_t p, const double* X, int64_t ld) {
    NvtxRange nvtx_("oz2_reprepare");
    if (!h || !p || p->device != h->device || h->mode != p->mode) return OZ2_ERR_INVALID_ARG;
    const int64_t need_ld = p->side == OZ2_LEFT ? (p->k > 0 ? p->k : 1) : (p->rows > 0 ? p->rows : 1);
    if (ld < need_ld || (p->k > 0 && p->rows > 0 && !X)) return OZ2_ERR_INVALID_ARG;
    int kstar = 0, rc;
    if (p->k > 0 && (rc = kstar_for(h, p->N, p->k, &kstar))) return rc;
    DevGuard g(h->device);
    if (p->k > 0 && p->rows > 0) {
        uint8_t* base = (uint8_t*)p->mem;
        if (p->side == OZ2_LEFT) {
            oz2::launch_rows(X, p->rows, p->k, ld, p->N, 3, h->mode, kstar, p->exps, p->planes, p->ldr, h->stream, 0,
                             xbits_rule(h, p->N, kstar));
        } else {
            const size_t off_stats = (size_t)round_up(
                (int64_t)((size_t)((uint8_t*)p->planes - base) + (size_t)p->N * (size_t)p->rows * (size_t)p->ldr), 256);
            oz2::launch_cols_exponents(X, p->k, p->rows, ld, p->N, h->mode, kstar, p->exps, base + off_stats, h->stream);
            oz2::launch_cols_residues(X, p->k, p->rows, ld, p->exps, p->N, p->planes, p->ldr, h->stream, 0,
                                      xbits_rule(h, p->N, kstar));
        }
    }
    return cuda_status();
}

int oz2_prepare_a(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda, int N, oz2_prep_t* out) {
    return prepare_common(h, OZ2_LEFT, m, k, A, lda, N, out);
}

int oz2_prepare_b(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb, int N, oz2_prep_t* out) {
    return prepare_common(h, OZ2_RIGHT, n, k, B, ldb, N, out);
}

int oz2_release(oz2_prep_t p) {
    if (!p) return OZ2_ERR_INVALID_ARG;
    DevGuard g(p->device);
    const cudaError_t e = cudaFree(p->mem);
    delete p;
    return e == cudaSuccess ? OZ2_OK : OZ2_ERR_CUDA;
}

int oz2_dgemm_prepared(oz2_handle_t h, oz2_prep_t pb, int64_t m, const double* A, int64_t lda, double* C,
                       int64_t ldc) {
    NvtxRange nvtx_("oz2_dgemm_prepared");
    if (!h || !pb || pb->side != OZ2_RIGHT || pb->device != h->device || h->mode != pb->mode)
        return OZ2_ERR_INVALID_ARG;
    const int64_t k = pb->k, n = pb->rows;
    const int N = pb->N;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (lda < (k > 0 ? k : 1) || ldc < (n > 0 ? n : 1) || (m > 0 && n > 0 && (!C || (k > 0 && !A))))
        return OZ2_ERR_INVALID_ARG;
    if (m == 0 || n == 0) return OZ2_OK;
    DevGuard g(h->device);
    if (k == 0) {
        oz2::launch_scale_c(C, m, n, ldc, 0.0, h->stream);
        return cuda_status();
    }
    int kstar = 0;
    if ((rc = kstar_for(h, N, k, &kstar))) return rc;
    Layout L = layout_for(m, n, k, N, gemm_sms(h), 0, false);
    uint8_t* ws;
    if ((rc = get_workspace(h, L.total, &ws))) return rc;
    int8_t* Ares = (int8_t*)(ws + L.off_Ares);
    int32_t* e = (int32_t*)(ws + L.off_e);
    mark(h);
    oz2::launch_rows(A, m, k, lda, N, 3, h->mode, kstar, e, Ares, L.ldr, h->stream, 0, xbits_rule(h, N, kstar));
    mark(h);
    mark(h);
    mark(h);
    if ((rc = prepared_product(h, m, n, k, N, Ares, L.ldr, e, pb->planes, pb->ldr, pb->exps, C, ldc, ws, L)))
        return rc;
    mark(h);
    mark(h);
    return OZ2_OK;
}

int oz2_dgemm_prep2(oz2_handle_t h, oz2_prep_t pa, oz2_prep_t pb, double* C, int64_t ldc) {
    NvtxRange nvtx_("oz2_dgemm_prep2");
    if (!h || !pa || !pb || pa->side != OZ2_LEFT || pb->side != OZ2_RIGHT || pa->device != h->device ||
        pb->device != h->device || pa->N != pb->N || pa->k != pb->k || pa->mode != pb->mode)
        return OZ2_ERR_INVALID_ARG;
    const int64_t m = pa->rows, n = pb->rows, k = pa->k;
    const int N = pa->N;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (ldc < (n > 0 ? n : 1) || (m > 0 && n > 0 && !C)) return OZ2_ERR_INVALID_ARG;
    if (m == 0 || n == 0) return OZ2_OK;
    DevGuard g(h->device);
    if (k == 0) {
        oz2::launch_scale_c(C, m, n, ldc, 0.0, h->stream);
        return cuda_status();
    }
    Layout L = layout_for(m, n, 0, N, gemm_sms(h), 0, false);     // scratch + sync only (no planes)
    uint8_t* ws;
    if ((rc = get_workspace(h, L.total, &ws))) return rc;
    return prepared_product(h, m, n, k, N, pa->planes, pa->ldr, pa->exps, pb->planes, pb->ldr, pb->exps, C, ldc, ws, L);
}

// ---------------------------------------------------------------------------
// K-split pieces (2-D multi-GPU, kslice.cu)
// ---------------------------------------------------------------------------
int oz2_kslice_stats_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                          const int32_t* E_global, int32_t* E_out, uint64_t* S_out) {
    if (!h || h->mode == OZ2_MODE_ACCU || m < 0 || k < 0 || k >= OZ2_MAX_K || lda < (k > 0 ? k : 1)) return OZ2_ERR_INVALID_ARG;
    if (m > 0 && ((k > 0 && !A) || (!E_global && !E_out) || (E_global && !S_out))) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    oz2::launch_kslice_rows(A, m, k, lda, h->mode, E_global, E_out, (unsigned long long*)S_out, h->stream);
    return cuda_status();
}

int oz2_kslice_stats_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                          const int32_t* E_global, int32_t* E_out, uint64_t* S_out) {
    if (!h || h->mode == OZ2_MODE_ACCU || n < 0 || k < 0 || k >= OZ2_MAX_K || ldb < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    if (n > 0 && ((k > 0 && !B) || (!E_global && !E_out) || (E_global && !S_out))) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    uint8_t* ws;
    int rc;
    if ((rc = get_workspace(h, oz2::cols_stats_bytes(k, n), &ws))) return rc;
    oz2::launch_kslice_cols(B, k, n, ldb, h->mode, E_global, E_out, (unsigned long long*)S_out, ws, h->stream);
    return cuda_status();
}

int oz2_exponents_from_stats(oz2_handle_t h, int64_t count, const int32_t* E, const uint64_t* S, int64_t k_total,
                             int N, int32_t* e) {
    if (!h || h->mode == OZ2_MODE_ACCU || count < 0 || (count > 0 && (!E || !S || !e))) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(1, 1, k_total, N);
    if (rc) return rc;
    int kstar = 0;
    if ((rc = kstar_for(h, N, k_total, &kstar))) return rc;
    DevGuard g(h->device);
    oz2::launch_exponents_from_stats(E, (const unsigned long long*)S, count, N, h->mode, kstar, e, h->stream);
    return cuda_status();
}

int oz2_modmul_residues(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const int8_t* Ares, const int8_t* Bres,
                        int64_t ld_res, int N, uint8_t* R, int64_t rows_per_block) {
    NvtxRange nvtx_("oz2_modmul_residues");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (ld_res < k || ld_res % 16 || rows_per_block < 0 || (m > 0 && n > 0 && !R)) return OZ2_ERR_INVALID_ARG;
    if (rows_per_block == 0) rows_per_block = m;
    if (m == 0 || n == 0) return OZ2_OK;
    DevGuard g(h->device);
    if (k == 0) {
        const int64_t nblk = (m + rows_per_block - 1) / rows_per_block;
        return cudaMemsetAsync(R, 0, (size_t)nblk * N * rows_per_block * n, h->stream) == cudaSuccess ? OZ2_OK : OZ2_ERR_CUDA;
    }
    CUtensorMap tA, tB;
    if ((rc = make_plane_map(&tA, Ares, m, k, ld_res, N, 128))) return rc;
    if ((rc = make_plane_map(&tB, Bres, n, k, ld_res, N, 256 / oz2::gemm_cta_group()))) return rc;
    uint8_t* ws;
    const size_t scr = oz2::fused_scratch_bytes(m, n, N, gemm_sms(h));
    if ((rc = get_workspace(h, scr + 512, &ws))) return rc;
    if (oz2::launch_modmul_residues(&tA, &tB, m, n, k, N, ws, R, rows_per_block, (uint32_t*)(ws + scr + 256),
                                    gemm_sms(h), h->stream))
        return OZ2_ERR_CUDA;
    return cuda_status();
}

int oz2_crt_sum(oz2_handle_t h, int parts, int64_t m, int64_t n, const uint8_t* R, int64_t part_stride,
                const int32_t* e, const int32_t* f, int N, double* C, int64_t ldc, const int32_t* beta) {
    NvtxRange nvtx_("oz2_crt_sum");
    if (!h || parts < 1 || parts > (1 << 20)) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, 0, N);
    if (rc) return rc;
    if (ldc < (n > 0 ? n : 1) || (m > 0 && n > 0 && (!R || !e || !f || !C))) return OZ2_ERR_INVALID_ARG;
    DevGuard g(h->device);
    if (beta && (rc = ensure_cert(h))) return rc;
    oz2::launch_crt_sum(R, parts, part_stride, m, n, e, f, N, C, ldc, h->stream);
    if (beta) oz2::launch_refuse(beta, N, C, m, n, ldc, h->cert, h->stream);
    return cuda_status();
}

int oz2_dgemm_scaled(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                     const double* B, int64_t ldb, const int32_t* e, const int32_t* f, double* C, int64_t ldc,
                     int N) {
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_op_args(OZ2_OP_N, OZ2_OP_N, m, n, k, A, lda, B, ldb, C, ldc, N);
    if (rc) return rc;
    if (m > 0 && n > 0 && k > 0 && (!e || !f)) return OZ2_ERR_INVALID_ARG;
    if (!h->certify || m == 0 || n == 0 || k == 0)
        return dgemm_core(h, OZ2_OP_N, OZ2_OP_N, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc, N, e, f);
    // condition (13) certificate (certify.cu), then the product, then the refusal check
    DevGuard g(h->device);
    if ((rc = ensure_cert(h))) return rc;
    if ((rc = certify_into(h, m, n, k, A, lda, B, ldb, e, f, N, h->cert + 1))) return rc;
    if ((rc = dgemm_core(h, OZ2_OP_N, OZ2_OP_N, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc, N, e, f))) return rc;
    DevGuard g2(h->device);
    oz2::launch_refuse(h->cert + 1, N, C, m, n, ldc, h->cert, h->stream);
    return cuda_status();
}

int oz2_dgemm_strided_batched(oz2_handle_t h, int transA, int transB, int64_t m, int64_t n, int64_t k,
                              double alpha, const double* A, int64_t lda, int64_t strideA, const double* B,
                              int64_t ldb, int64_t strideB, double beta, double* C, int64_t ldc,
                              int64_t strideC, int64_t batch, int N) {
    NvtxRange nvtx_("oz2_dgemm_strided_batched");
    if (!h || batch < 0 || strideA < 0 || strideB < 0 || strideC < 0) return OZ2_ERR_INVALID_ARG;
    int rc = check_op_args(transA, transB, m, n, k, A, lda, B, ldb, C, ldc, N);
    if (rc) return rc;
    for (int64_t b = 0; b < batch; b++) {            // one workspace, reused in stream order
        rc = dgemm_core(h, transA, transB, m, n, k, alpha, A ? A + b * strideA : A, lda,
                        B ? B + b * strideB : B, ldb, beta, C + b * strideC, ldc, N);
        if (rc) return rc;
    }
    return OZ2_OK;
}

int oz2_dgemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
              double* C, int64_t ldc, int N) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return OZ2_ERR_NO_DEVICE;
    if (dev < 0 || dev >= 64) return OZ2_ERR_NO_DEVICE;
    if (!g_default[dev]) {
        oz2_handle_t hh;
        int rc = oz2_create(&hh, dev);
        if (rc) return rc;
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_default[dev]) g_default[dev] = hh; else oz2_destroy(hh);
    }
    return oz2_dgemm_ex(g_default[dev], m, n, k, A, lda, B, ldb, C, ldc, N);
}

int oz2_dgemm_host(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc, int N) {
    NvtxRange nvtx_("oz2_dgemm_host");
    if (!h) return OZ2_ERR_INVALID_ARG;
    int rc = check_common(m, n, k, N);
    if (rc) return rc;
    if (lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1) || ldc < (n > 0 ? n : 1)) return OZ2_ERR_INVALID_ARG;
    if (m == 0 || n == 0) return OZ2_OK;
    if (!C || (k > 0 && (!A || !B))) return OZ2_ERR_INVALID_ARG;
    int kstar = 0;
    if (k > 0 && (rc = kstar_for(h, N, k, &kstar))) return rc;
    DevGuard g(h->device);
    if (k == 0) {
        for (int64_t i = 0; i < m; i++) memset(C + i * ldc, 0, sizeof(double) * (size_t)n);
        return OZ2_OK;
    }
    if (h->mode == OZ2_MODE_ACCU) {
        // f depends on every row of A under the accu rule: no row-block pipeline
        Layout L = layout_for(m, n, k, N, gemm_sms(h), std::max(m, n));
        const size_t offA = (size_t)round_up((int64_t)L.total, 256);
        const size_t offB = (size_t)round_up((int64_t)(offA + sizeof(double) * (size_t)m * k), 256);
        const size_t offC = (size_t)round_up((int64_t)(offB + sizeof(double) * (size_t)k * n), 256);
        uint8_t* ws;
        if ((rc = get_workspace(h, offC + sizeof(double) * (size_t)m * n, &ws))) return rc;
        double* dA = (double*)(ws + offA);
        double* dB = (double*)(ws + offB);
        double* dC = (double*)(ws + offC);
        if (cudaMemcpy2DAsync(dA, sizeof(double) * k, A, sizeof(double) * lda, sizeof(double) * k, m,
                              cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
            cudaMemcpy2DAsync(dB, sizeof(double) * n, B, sizeof(double) * ldb, sizeof(double) * n, k,
                              cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
            return OZ2_ERR_CUDA;
        void* save_ptr = h->ws_user;
        size_t save_bytes = h->ws_user_bytes;
        h->ws_user = ws;
        h->ws_user_bytes = L.total;
        rc = dgemm_core(h, OZ2_OP_N, OZ2_OP_N, m, n, k, 1.0, dA, k, dB, n, 0.0, dC, n, N);
        h->ws_user = save_ptr;
        h->ws_user_bytes = save_bytes;
        if (rc) return rc;
        if (cudaMemcpy2DAsync(C, sizeof(double) * ldc, dC, sizeof(double) * n, sizeof(double) * n, m,
                              cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return OZ2_ERR_CUDA;
        return cudaStreamSynchronize(h->stream) == cudaSuccess ? OZ2_OK : OZ2_ERR_CUDA;
    }
    if (m >= 8192 && n >= 8192 && env_flag("OZ2_HOST_2D", 1)) return dgemm_host_2d(h, m, n, k, A, lda, B, ldb, C, ldc, N, kstar);
    // Pipeline over R row blocks of A and C (rows a multiple of 256): B goes
    // first on the H2D stream and is converted once; row block i is converted and
    // multiplied as soon as its copy lands, and its C block leaves on the D2H
    // stream while block i + 1 computes.  Results are bit-identical to one call
    // (e_i depends on row i only).
    // Block schedule: a small first block (the GEMMs start as soon as B and 1024
    // rows have landed), 4096-row middle blocks, then a shrinking tail (2048,
    // 1024, 512, 256, 256) so the last block's GEMM and copy-back are short.
    // Small m: equal blocks of >= 4096 rows.
    std::vector<int64_t> blk_r0, blk_rows;
    {
        std::vector<int64_t> sizes;
        if (m >= 12288) {
            const int64_t tail[5] = {2048, 1024, 512, 256, 256};
            int64_t mid = m - 1024 - 4096;
            sizes.push_back(1024);
            while (mid > 0) { const int64_t b = std::min<int64_t>(4096, mid); sizes.push_back(b); mid -= b; }
            for (int64_t t : tail) sizes.push_back(t);
        } else {
            const int64_t R = std::max<int64_t>(1, std::min<int64_t>(8, m / 4096));
            const int64_t eq = round_up((m + R - 1) / R, 256);
            for (int64_t r = 0; r < m; r += eq) sizes.push_back(std::min(eq, m - r));
        }
        int64_t r0 = 0;
        for (int64_t sz : sizes) { blk_r0.push_back(r0); blk_rows.push_back(sz); r0 += sz; }
    }
    const int64_t nblk = (int64_t)blk_r0.size();
    const int64_t mb = *std::max_element(blk_rows.begin(), blk_rows.end());
    Layout L = layout_for(mb, n, k, N, gemm_sms(h));          // A planes and e for one row block
    const size_t bytesA = sizeof(double) * (size_t)m * (size_t)k;
    const size_t bytesB = sizeof(double) * (size_t)k * (size_t)n;
    const size_t bytesC = sizeof(double) * (size_t)m * (size_t)n;
    const size_t offA = (size_t)round_up((int64_t)L.total, 256);
    const size_t offB = (size_t)round_up((int64_t)(offA + bytesA), 256);
    const size_t offC = (size_t)round_up((int64_t)(offB + bytesB), 256);
    uint8_t* ws;
    if ((rc = get_workspace(h, offC + bytesC, &ws))) return rc;
    double* dA = (double*)(ws + offA);
    double* dB = (double*)(ws + offB);
    double* dC = (double*)(ws + offC);
    if (!h->s_h2d && cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking) != cudaSuccess) return OZ2_ERR_CUDA;
    if (!h->s_d2h && cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking) != cudaSuccess) return OZ2_ERR_CUDA;
    const size_t nev = (size_t)(2 * nblk + 2);
    while (h->pipe_ev.size() < nev) {
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return OZ2_ERR_CUDA;
        h->pipe_ev.push_back(ev);
    }
    cudaEvent_t evB = h->pipe_ev[0], evStart = h->pipe_ev[1];
    cudaEvent_t* evA = &h->pipe_ev[2];
    cudaEvent_t* evC = &h->pipe_ev[2 + nblk];
    // the copy streams start after work already queued on the handle's stream
    if (cudaEventRecord(evStart, h->stream) != cudaSuccess) return OZ2_ERR_CUDA;
    cudaStreamWaitEvent(h->s_h2d, evStart, 0);
    cudaStreamWaitEvent(h->s_d2h, evStart, 0);
    if (cudaMemcpy2DAsync(dB, sizeof(double) * n, B, sizeof(double) * ldb, sizeof(double) * n, k,
                          cudaMemcpyHostToDevice, h->s_h2d) != cudaSuccess) return OZ2_ERR_CUDA;
    cudaEventRecord(evB, h->s_h2d);
    for (int64_t b = 0; b < nblk; b++) {
        const int64_t r0 = blk_r0[b], rows = blk_rows[b];
        if (cudaMemcpy2DAsync(dA + r0 * k, sizeof(double) * k, A + r0 * lda, sizeof(double) * lda,
                              sizeof(double) * k, rows, cudaMemcpyHostToDevice, h->s_h2d) != cudaSuccess)
            return OZ2_ERR_CUDA;
        cudaEventRecord(evA[b], h->s_h2d);
    }
    int8_t* Ares = (int8_t*)(ws + L.off_Ares);
    int8_t* Bres = (int8_t*)(ws + L.off_Bres);
    int32_t* e = (int32_t*)(ws + L.off_e);
    int32_t* f = (int32_t*)(ws + L.off_f);
    cudaStreamWaitEvent(h->stream, evB, 0);
    mark(h);
    mark(h);                                                  // rows of A are timed inside the GEMM stage here
    oz2::launch_cols_exponents(dB, k, n, n, N, h->mode, kstar, f, ws + L.off_stats, h->stream);
    mark(h);
    oz2::launch_cols_residues(dB, k, n, n, f, N, Bres, L.ldr, h->stream, 0, xbits_rule(h, N, kstar));
    mark(h);
    CUtensorMap tB;
    if ((rc = make_plane_map(&tB, Bres, n, k, L.ldr, N, 256 / oz2::gemm_cta_group()))) return rc;
    for (int64_t b = 0; b < nblk; b++) {
        const int64_t r0 = blk_r0[b], rows = blk_rows[b];
        cudaStreamWaitEvent(h->stream, evA[b], 0);
        oz2::launch_rows(dA + r0 * k, rows, k, k, N, 3, h->mode, kstar, e, Ares, L.ldr, h->stream, 0,
                         xbits_rule(h, N, kstar));
        CUtensorMap tA;
        if ((rc = make_plane_map(&tA, Ares, rows, k, L.ldr, N, 128))) return rc;
        if (oz2::launch_modmul_fused(&tA, &tB, rows, n, k, N, ws + L.off_scratch, e, f, dC + r0 * n, n,
                                     (uint32_t*)(ws + L.off_sync), gemm_sms(h), h->stream))
            return OZ2_ERR_CUDA;
        cudaEventRecord(evC[b], h->stream);
        cudaStreamWaitEvent(h->s_d2h, evC[b], 0);
        if (cudaMemcpy2DAsync(C + r0 * ldc, sizeof(double) * ldc, dC + r0 * n, sizeof(double) * n,
                              sizeof(double) * n, rows, cudaMemcpyDeviceToHost, h->s_d2h) != cudaSuccess)
            return OZ2_ERR_CUDA;
    }
    mark(h);
    mark(h);
    if ((rc = cuda_status())) return rc;
    return cudaStreamSynchronize(h->s_d2h) == cudaSuccess && cudaStreamSynchronize(h->stream) == cudaSuccess
               ? OZ2_OK : OZ2_ERR_CUDA;
}

}  // extern "C"
