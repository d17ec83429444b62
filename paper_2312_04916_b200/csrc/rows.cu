// Row kernels: token+position embedding and RMSNorm(+gather, +cast).
//
// Both are HBM/L2-trivial (m <= a few rows at decode); they exist so that the
// residual stream stays float32 while GEMV inputs are produced once, already
// normalised and in the weight dtype.
#include "ee_common.cuh"

namespace {

constexpr int kRowThreads = 256;

// Fixed-order block sum: per-thread serial partials, then a fixed tree.
__device__ __forceinline__ float block_sum_fixed(float v, float* sh) {
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int s = kRowThreads / 2; s > 0; s >>= 1) {
        if (tid < s) sh[tid] += sh[tid + s];
        __syncthreads();
    }
    float r = sh[0];
    __syncthreads();
    return r;
}

template <typename T>
__global__ void __launch_bounds__(kRowThreads)
k_embed(const int32_t* __restrict__ tok, const int32_t* __restrict__ pos,
        const T* __restrict__ tok_emb, const T* __restrict__ pos_emb, int h,
        float* __restrict__ out) {
    pdl_trigger_dev();
    pdl_wait_dev();
    const int r = blockIdx.x;
    const T* te = tok_emb + (int64_t)tok[r] * h;
    const T* pe = pos_emb + (int64_t)pos[r] * h;
    float* o = out + (int64_t)r * h;
    for (int k = threadIdx.x; k < h; k += kRowThreads) o[k] = to_f32(te[k]) + to_f32(pe[k]);
}

// y = x * (mean(x^2) + eps)^(-1/2) * w   (eepipe/_pykernels.py:36-41)
template <typename TO>
__global__ void __launch_bounds__(kRowThreads)
k_rmsnorm_rows(const float* __restrict__ x, int64_t ldx, const int32_t* __restrict__ rows,
               int h, const float* __restrict__ w, float eps, TO* __restrict__ out) {
    __shared__ float sh[kRowThreads];
    pdl_trigger_dev();
    pdl_wait_dev();
    const int i = blockIdx.x;
    const int src = rows ? rows[i] : i;
    const float* xr = x + (int64_t)src * ldx;
    TO* o = out + (int64_t)i * h;
    if (w == nullptr) {
        for (int k = threadIdx.x; k < h; k += kRowThreads) o[k] = from_f32<TO>(xr[k]);
        return;
    }
    float ss = 0.f;
    for (int k = threadIdx.x; k < h; k += kRowThreads) ss = fmaf(xr[k], xr[k], ss);
    const float tot = block_sum_fixed(ss, sh);
    const float inv = 1.0f / sqrtf(tot / (float)h + eps);
    for (int k = threadIdx.x; k < h; k += kRowThreads) o[k] = from_f32<TO>(xr[k] * inv * w[k]);
}

}  // namespace

int launch_rmsnorm_rows(const float* x, int64_t ldx, const int32_t* rows, int64_t m, int64_t h,
                        const float* w, float eps, void* out, int dtype, cudaStream_t s) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && h > 0 && ldx >= h, EE_ESHAPE, "rmsnorm_rows: bad shape m=%lld h=%lld",
               (long long)m, (long long)h);
    cudaError_t e;
    dtype = act_dtype(dtype);
    if (dtype == EE_BF16)
        e = launch_ex(k_rmsnorm_rows<bf16>, dim3((unsigned)m), dim3(kRowThreads), 0, s, x, ldx, rows,
                      (int)h, w, eps, (bf16*)out);
    else if (dtype == EE_F32)
        e = launch_ex(k_rmsnorm_rows<float>, dim3((unsigned)m), dim3(kRowThreads), 0, s, x, ldx,
                      rows, (int)h, w, eps, (float*)out);
    else
        return ee_fail(EE_ECONFIG, "rmsnorm_rows: unknown dtype %d", dtype);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "rmsnorm_rows launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

extern "C" int ee_rmsnorm_rows(const float* x, int64_t ldx, const int32_t* rows, int64_t m,
                               int64_t h, const float* w, float eps, void* out, int dtype,
                               void* stream) {
    return launch_rmsnorm_rows(x, ldx, rows, m, h, w, eps, out, dtype, as_stream(stream));
}

extern "C" int ee_embed(const int32_t* tok, const int32_t* pos, int64_t m, const void* tok_emb,
                        const void* pos_emb, int64_t h, int dtype, float* out, void* stream) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && h > 0, EE_ESHAPE, "embed: bad shape");
    cudaStream_t s = as_stream(stream);
    cudaError_t e;
    dtype = act_dtype(dtype);
    if (dtype == EE_BF16)
        e = launch_ex(k_embed<bf16>, dim3((unsigned)m), dim3(kRowThreads), 0, s, tok, pos,
                      (const bf16*)tok_emb, (const bf16*)pos_emb, (int)h, out);
    else if (dtype == EE_F32)
        e = launch_ex(k_embed<float>, dim3((unsigned)m), dim3(kRowThreads), 0, s, tok, pos,
                      (const float*)tok_emb, (const float*)pos_emb, (int)h, out);
    else
        return ee_fail(EE_ECONFIG, "embed: unknown dtype %d", dtype);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "embed launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

// ---- row statistics for the folded-RMSNorm GEMVs ---------------------------
// xb = bf16(x) and ssq[r][t] = sum_{i<16} x[r][16t+i]^2 (ascending fmaf) —
// exactly what the residual GEMV epilogue produces for rows it updates, so a
// row's statistics do not depend on which kernel last wrote it.
namespace {
__global__ void __launch_bounds__(256)
k_row_stats(const float* __restrict__ x, int64_t ldx, int m, int h, bf16* __restrict__ xb,
            float* __restrict__ ssq) {
    pdl_trigger_dev();
    pdl_wait_dev();
    const int nt = h >> 4;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)m * nt) return;
    const int r = (int)(i / nt), t = (int)(i % nt);
    const float* xr = x + (int64_t)r * ldx + t * 16;
    bf16* br = xb + (int64_t)r * h + t * 16;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const float v = xr[k];
        s = fmaf(v, v, s);
        br[k] = __float2bfloat16_rn(v);
    }
    ssq[(int64_t)r * nt + t] = s;
}
}  // namespace

int launch_row_stats(const float* x, int64_t ldx, int64_t m, int64_t h, void* xb, float* ssq,
                     cudaStream_t s) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && h > 0 && h % 16 == 0, EE_ESHAPE, "row_stats: h must be a multiple of 16");
    const int64_t n = m * (h / 16);
    cudaError_t e = launch_ex(k_row_stats, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, x,
                              ldx, (int)m, (int)h, (bf16*)xb, ssq);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "row_stats launch: %s", cudaGetErrorString(e));
    return EE_OK;
}

extern "C" int ee_row_stats(const float* x, int64_t ldx, int64_t m, int64_t h, void* xb,
                            float* ssq, void* stream) {
    return launch_row_stats(x, ldx, m, h, xb, ssq, as_stream(stream));
}

// embedding + (tiled mode) row statistics of the new rows in one call
extern "C" int ee_embed_stats(const int32_t* tok, const int32_t* pos, int64_t m, const void* tok_emb,
                              const void* pos_emb, int64_t h, int dtype, float* out, void* xb,
                              float* ssq, void* stream) {
    int rc = ee_embed(tok, pos, m, tok_emb, pos_emb, h, dtype, out, stream);
    if (rc || m == 0 || xb == nullptr || ssq == nullptr) return rc;
    return launch_row_stats(out, h, m, h, xb, ssq, as_stream(stream));
}

// asynchronous host -> device copy (pinned source) on `stream`
extern "C" int ee_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    if (bytes == 0) return EE_OK;
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream));
    EE_REQUIRE(e == cudaSuccess, EE_ECUDA, "copy_h2d: %s", cudaGetErrorString(e));
    return EE_OK;
}
