// Fused multi-tensor optimizer step (SGD / Adam) over every parameter of a
// model in ONE launch, restating `SGD.step` / `Adam.step`
// (eepipe/training.py:24-53) in float32 on the device:
//
//   g = grad * scale                         (scale = 1 / num_microbatches)
//   SGD :  p -= lr * g
//   ACCUM: p += g   (float32 gradient accumulation across microbatches; p is
//          the accumulator, no moments)
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
constexpr int kChunk = 4096;  // elements per CTA iteration (16 per thread)

template <typename G>
__device__ __forceinline__ float grad_at(const void* g, int64_t i) {
    return to_f32<G>(reinterpret_cast<const G*>(g)[i]);
}

template <typename G>
__device__ __forceinline__ void grad4(const void* g, int64_t i, float* o) {
    if constexpr (sizeof(G) == 4) {
        const float4 v = reinterpret_cast<const float4*>(g)[i >> 2];
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const uint2 u = reinterpret_cast<const uint2*>(g)[i >> 2];
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
}

template <int KIND>
__device__ __forceinline__ void update1(float g, float& p, float& m, float& v, float lr, float b1,
                                        float b2, float eps, float step_size) {
    if (KIND == EE_OPT_ACCUM) {
        p += g;  // float32 gradient accumulator += grad * scale
    } else if (KIND == EE_OPT_ADAM) {
        m += (1.f - b1) * (g - m);
        v += (1.f - b2) * (g * g - v);
        p -= step_size * m / (sqrtf(v) + eps);
    } else {
        p -= lr * g;
    }
}

// One tensor's slice [a, b) (offsets within the tensor).  Vector path (4
// elements per thread step, 16-byte float32 / 8-byte bf16 accesses) when the
// tensor's arrays are aligned; scalar otherwise.
template <typename G, int KIND>
__device__ __forceinline__ void update_range(const ee_opt_tensor_t& t, int64_t a, int64_t b,
                                             float lr, float b1, float b2, float eps, float scale,
                                             float step_size) {
    const bool vec = ((t.n & 3) == 0) && ((a & 3) == 0) && ((b & 3) == 0) &&
                     (((uintptr_t)t.param | (uintptr_t)t.m | (uintptr_t)t.v) & 15) == 0 &&
                     (((uintptr_t)t.grad) & (sizeof(G) == 4 ? 15 : 7)) == 0 &&
                     (((uintptr_t)t.param_lp) & 7) == 0;
    if (vec) {
        for (int64_t i = a + 4 * threadIdx.x; i < b; i += 4 * kOptThreads) {
            float g[4];
            grad4<G>(t.grad, i, g);
            float4 p = reinterpret_cast<float4*>(t.param)[i >> 2];
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f), v = m;
            if (KIND == EE_OPT_ADAM) {
                m = reinterpret_cast<float4*>(t.m)[i >> 2];
                v = reinterpret_cast<float4*>(t.v)[i >> 2];
            }
            update1<KIND>(g[0] * scale, p.x, m.x, v.x, lr, b1, b2, eps, step_size);
            update1<KIND>(g[1] * scale, p.y, m.y, v.y, lr, b1, b2, eps, step_size);
            update1<KIND>(g[2] * scale, p.z, m.z, v.z, lr, b1, b2, eps, step_size);
            update1<KIND>(g[3] * scale, p.w, m.w, v.w, lr, b1, b2, eps, step_size);
            reinterpret_cast<float4*>(t.param)[i >> 2] = p;
            if (KIND == EE_OPT_ADAM) {
                reinterpret_cast<float4*>(t.m)[i >> 2] = m;
                reinterpret_cast<float4*>(t.v)[i >> 2] = v;
            }
            if (KIND != EE_OPT_ACCUM && t.param_lp) {
                uint2 u;
                *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(p.x, p.y);
                *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(p.z, p.w);
                reinterpret_cast<uint2*>(t.param_lp)[i >> 2] = u;
            }
        }
    } else {
        for (int64_t i = a + threadIdx.x; i < b; i += kOptThreads) {
            const float g = grad_at<G>(t.grad, i) * scale;
            float p = t.param[i];
            float m = 0.f, v = 0.f;
            if (KIND == EE_OPT_ADAM) {
                m = t.m[i];
                v = t.v[i];
            }
            update1<KIND>(g, p, m, v, lr, b1, b2, eps, step_size);
            t.param[i] = p;
            if (KIND == EE_OPT_ADAM) {
                t.m[i] = m;
                t.v[i] = v;
            }
            if (KIND != EE_OPT_ACCUM && t.param_lp)
                reinterpret_cast<bf16*>(t.param_lp)[i] = __float2bfloat16_rn(p);
        }
    }
}

template <typename G, int KIND>
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
            const int64_t a = max(c0, t.start) - t.start, b = min(c1, t.start + t.n) - t.start;
            if (a < b) update_range<G, KIND>(t, a, b, lr, b1, b2, eps, scale, step_size);
        }
        __syncthreads();
    }
}

}  // namespace

extern "C" int ee_optimizer_step(const ee_opt_tensor_t* table, int32_t n_tensors, int64_t total,
                                 int kind, int grad_dtype, float lr, float beta1, float beta2,
                                 float eps, float grad_scale, float step_size, void* stream) {
    EE_REQUIRE(n_tensors >= 0 && total >= 0, EE_ESHAPE, "optimizer: negative sizes");
    EE_REQUIRE(kind == EE_OPT_SGD || kind == EE_OPT_ADAM || kind == EE_OPT_ACCUM, EE_ECONFIG,
               "optimizer: unknown kind %d", kind);
    EE_REQUIRE(grad_dtype == EE_F32 || grad_dtype == EE_BF16, EE_ECONFIG,
               "optimizer: gradients must be float32 or bf16");
    if (n_tensors == 0 || total == 0) return EE_OK;
    EE_REQUIRE(table != nullptr, EE_ESHAPE, "optimizer: null tensor table");
    cudaStream_t s = as_stream(stream);
    const int64_t chunks = (total + kChunk - 1) / kChunk;
    const int64_t cap = (int64_t)ee_sm_count() * 8;
    const int grid = (int)(chunks < cap ? chunks : cap);
#define EE_OPT_LAUNCH(G, K)                                                                  \
    k_opt_step<G, K><<<grid, kOptThreads, 0, s>>>(table, n_tensors, total, lr, beta1, beta2, eps, \
                                                  grad_scale, step_size)
    if (grad_dtype == EE_F32) {
        if (kind == EE_OPT_ADAM) EE_OPT_LAUNCH(float, EE_OPT_ADAM);
        else if (kind == EE_OPT_SGD) EE_OPT_LAUNCH(float, EE_OPT_SGD);
        else EE_OPT_LAUNCH(float, EE_OPT_ACCUM);
    } else {
        if (kind == EE_OPT_ADAM) EE_OPT_LAUNCH(bf16, EE_OPT_ADAM);
        else if (kind == EE_OPT_SGD) EE_OPT_LAUNCH(bf16, EE_OPT_SGD);
        else EE_OPT_LAUNCH(bf16, EE_OPT_ACCUM);
    }
#undef EE_OPT_LAUNCH
    return ee_check_launch("optimizer_step");
}
