// Fused multi-tensor optimizer step (SGD / Adam) over every parameter of a
// model in ONE launch, restating `SGD.step` / `Adam.step`
// (eepipe/training.py:24-53) in float32 on the device:
//
//   g = grad * scale                         (scale = 1 / num_microbatches)
//   SGD :  p -= lr * g
//   Adam:  m += (1 - b1) (g - m);  v += (1 - b2) (g*g - v)
//          p -= step_size * m / (sqrt(v) + eps),
//          step_size = lr * sqrt(1 - b2^t) / (1 - b1^t)   (computed by the host
//          in double, the reference's bias-correction form)
//
// The per-tensor table (ee_opt_tensor_t) lives in device memory; tensors are
// laid end to end in one virtual index space [0, total) (`start` = prefix
// offset) that the grid strides over in 2048-element chunks, so hundreds of
// small tensors cost one launch.  HBM-bound: per element it reads g, p, m, v
// and writes p, m, v (+ the optional low-precision copy of p).
#include "ee_common.cuh"

namespace {

constexpr int kOptThreads = 256;
constexpr int kChunk = 2048;  // elements per CTA iteration (8 per thread)

template <typename G>
__device__ __forceinline__ float grad_at(const void* g, int64_t i) {
    return to_f32<G>(reinterpret_cast<const G*>(g)[i]);
}

template <typename G, bool ADAM>
__global__ void __launch_bounds__(kOptThreads)
k_opt_step(const ee_opt_tensor_t* __restrict__ table, int n_tensors, int64_t total, float lr,
           float b1, float b2, float eps, float scale, float step_size) {
    __shared__ int s_first;
    for (int64_t c0 = (int64_t)blockIdx.x * kChunk; c0 < total; c0 += (int64_t)gridDim.x * kChunk) {
        // first tensor overlapping the chunk (binary search on start offsets)
        if (threadIdx.x == 0) {
            int lo = 0, hi = n_tensors - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (table[mid].start <= c0) lo = mid; else hi = mid - 1;
            }
            s_first = lo;
        }
        __syncthreads();
        const int64_t c1 = min(c0 + kChunk, total);
        for (int ti = s_first; ti < n_tensors; ++ti) {
            const ee_opt_tensor_t t = table[ti];
            if (t.start >= c1) break;
            const int64_t a = max(c0, t.start), b = min(c1, t.start + t.n);
            for (int64_t e = a + threadIdx.x; e < b; e += kOptThreads) {
                const int64_t i = e - t.start;
                const float g = grad_at<G>(t.grad, i) * scale;
                float p = t.param[i];
                if (ADAM) {
                    float m = t.m[i], v = t.v[i];
                    m += (1.f - b1) * (g - m);
                    v += (1.f - b2) * (g * g - v);
                    p -= step_size * m / (sqrtf(v) + eps);
                    t.m[i] = m;
                    t.v[i] = v;
                } else {
                    p -= lr * g;
                }
                t.param[i] = p;
                if (t.param_lp) reinterpret_cast<bf16*>(t.param_lp)[i] = __float2bfloat16_rn(p);
            }
        }
        __syncthreads();
    }
}

}  // namespace

extern "C" int ee_optimizer_step(const ee_opt_tensor_t* table, int32_t n_tensors, int64_t total,
                                 int kind, int grad_dtype, float lr, float beta1, float beta2,
                                 float eps, float grad_scale, float step_size, void* stream) {
    EE_REQUIRE(n_tensors >= 0 && total >= 0, EE_ESHAPE, "optimizer: negative sizes");
    EE_REQUIRE(kind == EE_OPT_SGD || kind == EE_OPT_ADAM, EE_ECONFIG, "optimizer: unknown kind %d",
               kind);
    EE_REQUIRE(grad_dtype == EE_F32 || grad_dtype == EE_BF16, EE_ECONFIG,
               "optimizer: gradients must be float32 or bf16");
    if (n_tensors == 0 || total == 0) return EE_OK;
    EE_REQUIRE(table != nullptr, EE_ESHAPE, "optimizer: null tensor table");
    cudaStream_t s = as_stream(stream);
    const int64_t chunks = (total + kChunk - 1) / kChunk;
    const int64_t cap = (int64_t)ee_sm_count() * 8;
    const int grid = (int)(chunks < cap ? chunks : cap);
    const bool adam = kind == EE_OPT_ADAM;
    if (grad_dtype == EE_F32) {
        if (adam)
            k_opt_step<float, true><<<grid, kOptThreads, 0, s>>>(table, n_tensors, total, lr, beta1,
                                                                beta2, eps, grad_scale, step_size);
        else
            k_opt_step<float, false><<<grid, kOptThreads, 0, s>>>(table, n_tensors, total, lr, beta1,
                                                                 beta2, eps, grad_scale, step_size);
    } else {
        if (adam)
            k_opt_step<bf16, true><<<grid, kOptThreads, 0, s>>>(table, n_tensors, total, lr, beta1,
                                                               beta2, eps, grad_scale, step_size);
        else
            k_opt_step<bf16, false><<<grid, kOptThreads, 0, s>>>(table, n_tensors, total, lr, beta1,
                                                                beta2, eps, grad_scale, step_size);
    }
    return ee_check_launch("optimizer_step");
}
