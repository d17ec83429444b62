// Backbone GEMVs with fused epilogues (store / residual / GELU / QKV+KV-write).
//
// Grid: x over 16-row weight tiles (bf16) or 8-row tiles (fp32), y over
// activation-row groups.  A CTA = 8 warps splitting K in interleaved 32-wide
// blocks; the 8 partial tiles are summed in warp order (fixed), so results
// are deterministic and independent of m.
#include "gemv_core.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kUnroll = 4;
constexpr int kF32RW = 8, kF32RX = 4;

// ---- epilogues -----------------------------------------------------------
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

// ---- kernels -------------------------------------------------------------
template <int NB, class Epi>
__global__ void __launch_bounds__(kThreads)
k_gemv_bf16(const bf16* __restrict__ W, int N, int64_t K, const bf16* __restrict__ X,
            int64_t ldx, int m, Epi epi) {
    __shared__ float red[kWarps][16][8 * NB];
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

template <class Epi>
int run_bf16(const void* x, int64_t m, int64_t K, const void* W, int64_t N, Epi epi,
             cudaStream_t s) {
    EE_REQUIRE(K % 8 == 0, EE_ESHAPE, "bf16 gemv needs K %% 8 == 0 (K=%lld)", (long long)K);
    const unsigned gx = (unsigned)((N + 15) / 16);
    if (m <= 8) {
        k_gemv_bf16<1, Epi><<<dim3(gx, 1), kThreads, 0, s>>>((const bf16*)W, (int)N, K,
                                                             (const bf16*)x, K, (int)m, epi);
    } else {
        const unsigned gy = (unsigned)((m + 15) / 16);
        k_gemv_bf16<2, Epi><<<dim3(gx, gy), kThreads, 0, s>>>((const bf16*)W, (int)N, K,
                                                              (const bf16*)x, K, (int)m, epi);
    }
    return ee_check_launch("gemv_bf16");
}

template <class Epi>
int run_f32(const void* x, int64_t m, int64_t K, const void* W, int64_t N, Epi epi,
            cudaStream_t s) {
    const dim3 grid((unsigned)((N + kF32RW - 1) / kF32RW), (unsigned)((m + kF32RX - 1) / kF32RX));
    k_gemv_f32<Epi><<<grid, kThreads, 0, s>>>((const float*)W, (int)N, K, (const float*)x, K,
                                              (int)m, epi);
    return ee_check_launch("gemv_f32");
}

}  // namespace

int launch_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype, int epi,
                void* out, int64_t ldo, cudaStream_t s) {
    if (m == 0 || N == 0) return EE_OK;
    EE_REQUIRE(m > 0 && K > 0 && N > 0 && N < (1ll << 31), EE_ESHAPE,
               "gemv: bad shape m=%lld K=%lld N=%lld", (long long)m, (long long)K, (long long)N);
    EE_REQUIRE(m <= 65535 * 16, EE_ESHAPE, "gemv: too many rows");
    if (dtype == EE_BF16) {
        switch (epi) {
            case EE_EPI_STORE: return run_bf16(x, m, K, W, N, EpiStore{(float*)out, ldo}, s);
            case EE_EPI_RESIDUAL: return run_bf16(x, m, K, W, N, EpiResidual{(float*)out, ldo}, s);
            case EE_EPI_GELU: return run_bf16(x, m, K, W, N, EpiGelu<bf16>{(bf16*)out, ldo}, s);
        }
    } else if (dtype == EE_F32) {
        switch (epi) {
            case EE_EPI_STORE: return run_f32(x, m, K, W, N, EpiStore{(float*)out, ldo}, s);
            case EE_EPI_RESIDUAL: return run_f32(x, m, K, W, N, EpiResidual{(float*)out, ldo}, s);
            case EE_EPI_GELU: return run_f32(x, m, K, W, N, EpiGelu<float>{(float*)out, ldo}, s);
        }
    } else {
        return ee_fail(EE_ECONFIG, "gemv: unknown dtype %d", dtype);
    }
    return ee_fail(EE_ECONFIG, "gemv: unknown epilogue %d", epi);
}

int launch_qkv(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype, float* q,
               void* kc, void* vc, const int32_t* pos, cudaStream_t s) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && h > 0, EE_ESHAPE, "qkv: bad shape");
    if (dtype == EE_BF16)
        return run_bf16(xn, m, h, Wqkv, 3 * h, EpiQKV<bf16>{q, (bf16*)kc, (bf16*)vc, pos, (int)h}, s);
    if (dtype == EE_F32)
        return run_f32(xn, m, h, Wqkv, 3 * h, EpiQKV<float>{q, (float*)kc, (float*)vc, pos, (int)h}, s);
    return ee_fail(EE_ECONFIG, "qkv: unknown dtype %d", dtype);
}

extern "C" int ee_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype,
                       int epilogue, void* out, int64_t ldo, void* stream) {
    return launch_gemv(x, m, K, W, N, dtype, epilogue, out, ldo, as_stream(stream));
}

extern "C" int ee_qkv_kvwrite(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype,
                              float* q_out, void* kcache, void* vcache, const int32_t* pos,
                              void* stream) {
    return launch_qkv(xn, m, h, Wqkv, dtype, q_out, kcache, vcache, pos, as_stream(stream));
}
