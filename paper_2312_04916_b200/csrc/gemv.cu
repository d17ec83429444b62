// Backbone GEMVs with fused epilogues.
//
// EE_BF16_TILED (perf mode, weights packed by ee_pack_tiled, K % 512 == 0):
//   the TMA-bulk-fed persistent kernel of gemv_tma.cuh, launched with
//   programmatic dependent launch (weights stream before the dependency on
//   the previous kernel resolves).
// EE_BF16 (row-major weights, any K % 8 == 0): LDG + mma.sync kernel.
// EE_F32 (parity mode): SIMT FFMA kernel.
// All are row-stable: each output's reduction order depends only on (n, k).
#include <stdlib.h>

#include <algorithm>

#include "gemv_core.cuh"
#include "gemv_tma.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kUnroll = 4;
constexpr int kF32RW = 8, kF32RX = 4;

// ---- element-wise epilogue functors --------------------------------------
struct EpiStore {
    float* out;
    int64_t ldo;
    __device__ void operator()(int n, int r, float v) const { out[(int64_t)r * ldo + n] = v; }
};

struct EpiResidual {  // x + dot_rows(a, W)  (eepipe/inference.py:227, 229)
    float* x;
    int64_t ldx;
    __device__ void operator()(int n, int r, float v) const {
        float* p = x + (int64_t)r * ldx + n;
        *p = *p + v;
    }
};

template <typename T>
struct EpiGelu {  // gelu_fwd(dot_rows(h2, w1))  (eepipe/inference.py:229)
    T* out;
    int64_t ldo;
    __device__ void operator()(int n, int r, float v) const {
        out[(int64_t)r * ldo + n] = from_f32<T>(gelu_erf(v));
    }
};

template <typename T>
struct EpiQKV {  // q, k, v = dot_rows(h1, wq|wk|wv); KVCache.fill (inference.py:219-226)
    float* q;
    T* kc;
    T* vc;
    const int32_t* pos;
    int h;
    __device__ void operator()(int n, int r, float v) const {
        if (n < h) {
            q[(int64_t)r * h + n] = v;
        } else if (n < 2 * h) {
            kc[(int64_t)pos[r] * h + (n - h)] = from_f32<T>(v);
        } else {
            vc[(int64_t)pos[r] * h + (n - 2 * h)] = from_f32<T>(v);
        }
    }
};

// Adapter: sum the 4 consumer-warp partial tiles in fixed order, apply Fn.
template <class Fn>
struct TileApply {
    Fn fn;
    __device__ void tile(const float* red, int n0, int r0, int N, int m, int cols,
                         const float* inv) {
        using namespace tma_gemv;
        for (int i = threadIdx.x; i < kRows * cols; i += kConsumers * 32) {
            const int row = i & 15, col = i >> 4;
            const int o = row * kMaxCols + col;
            float v = ((red[o] + red[kRows * kMaxCols + o]) + red[2 * kRows * kMaxCols + o]) +
                      red[3 * kRows * kMaxCols + o];
            if (inv) v *= inv[col];
            const int n = n0 + row, r = r0 + col;
            if (n < N && r < m) fn(n, r, v);
        }
    }
    __device__ void finish() {}
};

// Residual epilogue that also refreshes the row statistics consumed by the
// next folded-norm GEMV: x += v, xb = bf16(x), ssq[r][n0/16] = sum of the 16
// squares in ascending order (same arithmetic as k_row_stats).
struct TileResidualStats {
    float* x;
    int64_t ldx;
    bf16* xb;
    float* ssq;
    __device__ void tile(const float* red, int n0, int r0, int N, int m, int cols,
                         const float* /*inv*/) {
        using namespace tma_gemv;
        __shared__ float vt[kRows][kMaxCols + 1];
        for (int i = threadIdx.x; i < kRows * cols; i += kConsumers * 32) {
            const int row = i & 15, col = i >> 4;
            const int o = row * kMaxCols + col;
            const float v = ((red[o] + red[kRows * kMaxCols + o]) + red[2 * kRows * kMaxCols + o]) +
                            red[3 * kRows * kMaxCols + o];
            const int n = n0 + row, r = r0 + col;
            float nv = 0.f;
            if (n < N && r < m) {
                float* p = x + (int64_t)r * ldx + n;
                nv = *p + v;
                *p = nv;
                xb[(int64_t)r * ldx + n] = __float2bfloat16_rn(nv);
            }
            vt[row][col] = nv;
        }
        consumers_sync();
        const int c = threadIdx.x;
        if (c < cols && r0 + c < m) {
            float s = 0.f;
#pragma unroll
            for (int row = 0; row < kRows; ++row) s = fmaf(vt[row][c], vt[row][c], s);
            ssq[(int64_t)(r0 + c) * (ldx >> 4) + (n0 >> 4)] = s;
        }
    }
    __device__ void finish() {}
};

// ---- TMA-fed kernel (tiled weights) ------------------------------------------
// weight-ring depth: 4 stages for 8-row groups, 3 for 16-row groups, so both
// run two CTAs per SM (~97 KB of shared memory each)
template <int NB>
constexpr int kGemvStages = NB == 1 ? 4 : 3;

// single-row passes (most decode passes): one activation row per stage and a
// 6-deep weight ring in the same ~109 KB (two CTAs per SM), so 6 of a tile's
// stages stream in before the dependency on the previous kernel resolves
constexpr int kGemvStages1 = 6;
// 2-4 rows: four activation rows per stage, a 5-deep ring (~107 KB)
constexpr int kGemvStages4 = 5;
template <int NB, int XR>
constexpr int gemv_stages() {
    return XR == 1 ? kGemvStages1 : XR == 4 ? kGemvStages4 : kGemvStages<NB>;
}

template <int NB, class Epi, int XR = 0>
__global__ void __launch_bounds__(tma_gemv::kThreads)
k_gemv_tma(const bf16* __restrict__ W, int N, int K, const bf16* __restrict__ X, int64_t ldx,
           int m, tma_gemv::RowNorm rn, Epi epi) {
    tma_gemv::gemv_body<NB, Epi, gemv_stages<NB, XR>(), XR>(W, N, K, X, ldx, m, rn, epi);
}

// ---- LDG kernels (row-major bf16, fp32 parity mode) ----------------------------
template <int NB, class Epi>
__global__ void __launch_bounds__(kThreads)
k_gemv_bf16(const bf16* __restrict__ W, int N, int64_t K, const bf16* __restrict__ X,
            int64_t ldx, int m, Epi epi) {
    __shared__ float red[kWarps][16][8 * NB];
    pdl_trigger_dev();
    pdl_wait_dev();
    const int warp = threadIdx.x >> 5;
    const int n0 = blockIdx.x * 16, r0 = blockIdx.y * 8 * NB;
    float acc[NB][4];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.f;
    warp_tile_bf16<NB, kUnroll>(W, K, n0, N, X, ldx, r0, m, warp, kWarps, acc);
    store_frag<NB>(red[warp], acc);
    __syncthreads();
    for (int i = threadIdx.x; i < 16 * 8 * NB; i += kThreads) {
        const int row = i & 15, col = i >> 4;
        float v = red[0][row][col];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += red[w][row][col];
        const int n = n0 + row, r = r0 + col;
        if (n < N && r < m) epi(n, r, v);
    }
}

template <class Epi>
__global__ void __launch_bounds__(kThreads)
k_gemv_f32(const float* __restrict__ W, int N, int64_t K, const float* __restrict__ X,
           int64_t ldx, int m, Epi epi) {
    __shared__ float red[kWarps][kF32RW][kF32RX];
    pdl_trigger_dev();
    pdl_wait_dev();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * kF32RW, r0 = blockIdx.y * kF32RX;
    float acc[kF32RW][kF32RX];
#pragma unroll
    for (int i = 0; i < kF32RW; ++i)
#pragma unroll
        for (int j = 0; j < kF32RX; ++j) acc[i][j] = 0.f;
    warp_tile_f32<kF32RW, kF32RX>(W, K, n0, N, X, ldx, r0, m, warp, kWarps, acc);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kF32RW; ++i)
#pragma unroll
            for (int j = 0; j < kF32RX; ++j) red[warp][i][j] = acc[i][j];
    }
    __syncthreads();
    if (threadIdx.x < kF32RW * kF32RX) {
        const int row = threadIdx.x % kF32RW, col = threadIdx.x / kF32RW;
        float v = red[0][row][col];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += red[w][row][col];
        const int n = n0 + row, r = r0 + col;
        if (n < N && r < m) epi(n, r, v);
    }
}

// ---- launchers ------------------------------------------------------------
template <int NB, class Epi, int XR = 0>
int run_tma_nb(const bf16* X, int64_t ldx, int64_t m, const void* W, int64_t N, int64_t K,
               tma_gemv::RowNorm rn, Epi epi, cudaStream_t s) {
    auto kern = k_gemv_tma<NB, Epi, XR>;
    const size_t smem = tma_gemv::smem_bytes(NB, gemv_stages<NB, XR>(), XR);
    static bool configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 15]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured[dev & 15] = true;
    }
    const int64_t tiles = (N + tma_gemv::kRows - 1) / tma_gemv::kRows;
    const int64_t rows_per_item = XR ? XR : 8 * NB;
    const int64_t groups = (m + rows_per_item - 1) / rows_per_item;
    const int64_t items = tiles * groups;
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(4, (226 * 1024) / (smem + 1024)));
    const int64_t slots = (int64_t)ee_sm_count() * per_sm;
    int64_t g = std::min<int64_t>(items, slots);
    // a grid that divides the items evenly (e.g. 768 QKV tiles on 256 CTAs x
    // 3 instead of 296 CTAs x 2.6) when one exists within 5/6 of the slots:
    // no CTA runs a last item alone (C3 5-row pass -2.4%, 1 row unchanged;
    // only up to 4 items per CTA: the C5 W1, 1792 tiles on 256 x 7, measured
    // slower than 296 x 6.05; EE_GEMV_BALANCE=0 for A/B).  Reduction orders
    // do not depend on the grid.
    static const bool balance = !getenv("EE_GEMV_BALANCE") || atoi(getenv("EE_GEMV_BALANCE")) != 0;
    if (balance && items > slots && items <= 4 * slots) {  // few items per CTA: the tail matters
        for (int64_t c = slots; c >= slots * 5 / 6; --c)
            if (items % c == 0) {
                g = c;
                break;
            }
    }
    const unsigned grid = (unsigned)g;
    cudaError_t e = launch_ex(kern, dim3(grid), dim3(tma_gemv::kThreads), smem, s,
                              (const bf16*)W, (int)N, (int)K, X, ldx, (int)m, rn, epi);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "gemv_tma launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

static bool gemv_nb1_only() {  // EE_GEMV_NB1=1: 8-row groups only (A/B runs)
    static const bool v = getenv("EE_GEMV_NB1") && atoi(getenv("EE_GEMV_NB1")) != 0;
    return v;
}
static bool gemv_deep4() {  // EE_GEMV_DEEP4=0: 2-4-row passes on the 8-row ring (A/B runs)
    static const bool v = !getenv("EE_GEMV_DEEP4") || atoi(getenv("EE_GEMV_DEEP4")) != 0;
    return v;
}
static bool gemv_deep1() {  // EE_GEMV_DEEP1=0: single-row passes on the 8-row ring (A/B runs)
    static const bool v = !getenv("EE_GEMV_DEEP1") || atoi(getenv("EE_GEMV_DEEP1")) != 0;
    return v;
}

template <class Epi>
int run_tma_epi(const bf16* X, int64_t ldx, int64_t m, const void* W, int64_t N, int64_t K,
                tma_gemv::RowNorm rn, Epi epi, cudaStream_t s) {
    EE_REQUIRE(K % kTiledKS == 0, EE_ESHAPE, "tiled gemv needs K %% %d == 0 (K=%lld)", kTiledKS,
               (long long)K);
    // 16-row groups for m > 8 (each weight stage serves 16 rows; a 3-deep
    // ring keeps it at two CTAs per SM).  A row's result does not depend on
    // the group width: the reduction order is per (n, k).
    if (m == 1 && gemv_deep1()) return run_tma_nb<1, Epi, 1>(X, ldx, m, W, N, K, rn, epi, s);
    if (m <= 4 && gemv_deep4()) return run_tma_nb<1, Epi, 4>(X, ldx, m, W, N, K, rn, epi, s);
    if (m <= 8 || gemv_nb1_only()) return run_tma_nb<1>(X, ldx, m, W, N, K, rn, epi, s);
    return run_tma_nb<2>(X, ldx, m, W, N, K, rn, epi, s);
}

template <class Fn>
int run_tma(const bf16* X, int64_t ldx, int64_t m, const void* W, int64_t N, int64_t K, Fn fn,
            cudaStream_t s, tma_gemv::RowNorm rn = {nullptr, 0.f}) {
    return run_tma_epi(X, ldx, m, W, N, K, rn, TileApply<Fn>{fn}, s);
}

template <class Epi>
int run_bf16(const void* x, int64_t m, int64_t K, const void* W, int64_t N, Epi epi,
             cudaStream_t s) {
    EE_REQUIRE(K % 8 == 0, EE_ESHAPE, "bf16 gemv needs K %% 8 == 0 (K=%lld)", (long long)K);
    const unsigned gx = (unsigned)((N + 15) / 16);
    cudaError_t e;
    if (m <= 8)
        e = launch_ex(k_gemv_bf16<1, Epi>, dim3(gx, 1), dim3(kThreads), 0, s, (const bf16*)W,
                      (int)N, K, (const bf16*)x, K, (int)m, epi);
    else
        e = launch_ex(k_gemv_bf16<2, Epi>, dim3(gx, (unsigned)((m + 15) / 16)), dim3(kThreads), 0,
                      s, (const bf16*)W, (int)N, K, (const bf16*)x, K, (int)m, epi);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "gemv_bf16 launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

template <class Epi>
int run_f32(const void* x, int64_t m, int64_t K, const void* W, int64_t N, Epi epi,
            cudaStream_t s) {
    const dim3 grid((unsigned)((N + kF32RW - 1) / kF32RW), (unsigned)((m + kF32RX - 1) / kF32RX));
    cudaError_t e = launch_ex(k_gemv_f32<Epi>, grid, dim3(kThreads), 0, s, (const float*)W, (int)N,
                              K, (const float*)x, K, (int)m, epi);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "gemv_f32 launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

template <class Epi>
int run_any(int dtype, const void* x, int64_t m, int64_t K, const void* W, int64_t N, Epi epi,
            cudaStream_t s) {
    if (dtype == EE_BF16_TILED) return run_tma((const bf16*)x, K, m, W, N, K, epi, s);
    if (dtype == EE_BF16) return run_bf16(x, m, K, W, N, epi, s);
    return ee_fail(EE_ECONFIG, "gemv: unknown dtype %d", dtype);
}

}  // namespace

int launch_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype, int epi,
                void* out, int64_t ldo, cudaStream_t s) {
    if (m == 0 || N == 0) return EE_OK;
    EE_REQUIRE(m > 0 && K > 0 && N > 0 && N < (1ll << 31) && K < (1ll << 30), EE_ESHAPE,
               "gemv: bad shape m=%lld K=%lld N=%lld", (long long)m, (long long)K, (long long)N);
    EE_REQUIRE(m <= 65535 * 16, EE_ESHAPE, "gemv: too many rows");
    if (dtype == EE_F32) {
        switch (epi) {
            case EE_EPI_STORE: return run_f32(x, m, K, W, N, EpiStore{(float*)out, ldo}, s);
            case EE_EPI_RESIDUAL: return run_f32(x, m, K, W, N, EpiResidual{(float*)out, ldo}, s);
            case EE_EPI_GELU: return run_f32(x, m, K, W, N, EpiGelu<float>{(float*)out, ldo}, s);
        }
        return ee_fail(EE_ECONFIG, "gemv: unknown epilogue %d", epi);
    }
    switch (epi) {
        case EE_EPI_STORE: return run_any(dtype, x, m, K, W, N, EpiStore{(float*)out, ldo}, s);
        case EE_EPI_RESIDUAL: return run_any(dtype, x, m, K, W, N, EpiResidual{(float*)out, ldo}, s);
        case EE_EPI_GELU: return run_any(dtype, x, m, K, W, N, EpiGelu<bf16>{(bf16*)out, ldo}, s);
    }
    return ee_fail(EE_ECONFIG, "gemv: unknown epilogue %d", epi);
}

int launch_qkv(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype, float* q,
               void* kc, void* vc, const int32_t* pos, cudaStream_t s) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && h > 0, EE_ESHAPE, "qkv: bad shape");
    if (dtype == EE_F32)
        return run_f32(xn, m, h, Wqkv, 3 * h, EpiQKV<float>{q, (float*)kc, (float*)vc, pos, (int)h}, s);
    return run_any(dtype, xn, m, h, Wqkv, 3 * h, EpiQKV<bf16>{q, (bf16*)kc, (bf16*)vc, pos, (int)h}, s);
}

int launch_gemv_tiled(const bf16* x, int64_t m, int64_t K, const void* W, int64_t N, int epi,
                      void* out, int64_t ldo, GemvNorm nrm, cudaStream_t s) {
    if (m == 0 || N == 0) return EE_OK;
    const tma_gemv::RowNorm rn{nrm.ssq, nrm.eps};
    switch (epi) {
        case EE_EPI_STORE: return run_tma(x, K, m, W, N, K, EpiStore{(float*)out, ldo}, s, rn);
        case EE_EPI_GELU: return run_tma(x, K, m, W, N, K, EpiGelu<bf16>{(bf16*)out, ldo}, s, rn);
        case EE_EPI_RESIDUAL:
            if (nrm.xb_out && nrm.ssq_out) {
                EE_REQUIRE(ldo % 16 == 0 && ldo == N, EE_ESHAPE, "residual stats need ldo == N");
                return run_tma_epi(x, K, m, W, N, K, rn,
                                   TileResidualStats{(float*)out, ldo, nrm.xb_out, nrm.ssq_out}, s);
            }
            return run_tma(x, K, m, W, N, K, EpiResidual{(float*)out, ldo}, s, rn);
    }
    return ee_fail(EE_ECONFIG, "gemv_tiled: unknown epilogue %d", epi);
}

int launch_qkv_tiled(const bf16* x, int64_t m, int64_t h, const void* Wqkv, GemvNorm nrm,
                     float* q, void* kc, void* vc, const int32_t* pos, cudaStream_t s) {
    if (m == 0) return EE_OK;
    return run_tma(x, h, m, Wqkv, 3 * h, h, EpiQKV<bf16>{q, (bf16*)kc, (bf16*)vc, pos, (int)h}, s,
                   tma_gemv::RowNorm{nrm.ssq, nrm.eps});
}

EE_TRACE_READER(ee_trace_gemv)

extern "C" int ee_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype,
                       int epilogue, void* out, int64_t ldo, void* stream) {
    return launch_gemv(x, m, K, W, N, dtype, epilogue, out, ldo, as_stream(stream));
}

extern "C" int ee_qkv_kvwrite(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype,
                              float* q_out, void* kcache, void* vcache, const int32_t* pos,
                              void* stream) {
    return launch_qkv(xn, m, h, Wqkv, dtype, q_out, kcache, vcache, pos, as_stream(stream));
}
