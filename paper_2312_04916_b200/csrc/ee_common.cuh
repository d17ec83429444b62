// Shared device/host helpers for libee.so (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ee.h"

typedef __nv_bfloat16 bf16;

// ---- error plumbing (abi.cu) -------------------------------------------
int ee_fail(int code, const char* fmt, ...);
int ee_check_launch(const char* what);

#define EE_REQUIRE(cond, code, ...)          \
    do {                                     \
        if (!(cond)) return ee_fail(code, __VA_ARGS__); \
    } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- scalar conversions ---------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f32<bf16>(float v) { return __float2bfloat16_rn(v); }

// exact-erf GELU in float32 (eepipe/_pykernels.py:27-28)
__device__ __forceinline__ float gelu_erf(float x) {
    return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}

// ---- memory helpers -------------------------------------------------------
// Streaming 16-byte load: weights are read exactly once per pass, so keep
// them out of L1 and hint a 256-byte L2 prefetch.
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Cached 16-byte load (activations re-read by every CTA).
__device__ __forceinline__ uint4 ld_cached16(const void* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}

// ---- tensor-core fragment MMA (bf16 x bf16 -> f32, m16n8k16) -------------
__device__ __forceinline__ void mma_16816(float c[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---- host-side launch helpers (defined in the .cu files) -----------------
int launch_rmsnorm_rows(const float* x, int64_t ldx, const int32_t* rows, int64_t m, int64_t h,
                        const float* w, float eps, void* out, int dtype, cudaStream_t s);
int launch_gemv(const void* x, int64_t m, int64_t K, const void* W, int64_t N, int dtype,
                int epi, void* out, int64_t ldo, cudaStream_t s);
int launch_qkv(const void* xn, int64_t m, int64_t h, const void* Wqkv, int dtype, float* q,
               void* kc, void* vc, const int32_t* pos, cudaStream_t s);
int launch_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                     const void* kc, const void* vc, int64_t nh, int64_t dh, int dtype, void* out,
                     void* ws, size_t ws_bytes, cudaStream_t s);
size_t attention_ws_bytes(int64_t m, int64_t nh, int64_t dh, int64_t s_max);
size_t exit_head_ws_bytes(int64_t m, int64_t h, int64_t V);

// ---- programmatic dependent launch ----------------------------------------
// Every kernel of the decode chain is launched with programmatic stream
// serialization: it may start while its predecessor drains, does its
// independent prologue (weight streaming, barrier init), then waits with
// griddepcontrol.wait before touching the predecessor's outputs.
__device__ __forceinline__ void pdl_wait_dev() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_dev() { asm volatile("griddepcontrol.launch_dependents;"); }

bool ee_pdl_enabled();  // EE_PDL=0 disables (debug)

// ---- timeline probes (profiling builds only: -DEE_TRACE) -------------------
// Per translation unit: slot i holds the min (EE_TMIN) or max (EE_TMAX) of
// %globaltimer over the CTAs that reach the probe (thread 0 of each CTA);
// EE_TRACE_READER(name) defines extern "C" name(uint64_t* out, int reset).
#ifdef EE_TRACE
static __device__ unsigned long long g_trace[16];
__device__ __forceinline__ unsigned long long ee_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define EE_TMIN(i) do { if (threadIdx.x == 0) atomicMin(&g_trace[i], ee_gtime()); } while (0)
#define EE_TMAX(i) do { if (threadIdx.x == 0) atomicMax(&g_trace[i], ee_gtime()); } while (0)
#define EE_TRACE_READER(name)                                                              \
    extern "C" int name(unsigned long long* out, int reset) {                             \
        cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));                                \
        if (reset) {                                                                        \
            unsigned long long init[16];                                                    \
            for (int i = 0; i < 16; ++i) init[i] = (i & 1) ? 0ull : ~0ull;                  \
            cudaMemcpyToSymbol(g_trace, init, sizeof(init));                                \
        }                                                                                   \
        return 0;                                                                           \
    }
#else
#define EE_TMIN(i) do { } while (0)
#define EE_TMAX(i) do { } while (0)
#define EE_TRACE_READER(name)
#endif
extern thread_local int g_pdl_off;  // debug (EE_PDL_SKIP): nonzero disables PDL on this thread's next launches

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ee_pdl_enabled() && !g_pdl_off ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

int ee_sm_count();  // cached per process


// ---- tiled bf16 weight layout (pack.cu) -------------------------------------
constexpr int kTiledKS = 512;  // k elements per tile stage
// activation / KV dtype for a weight dtype (tiled bf16 weights -> bf16)
static inline int act_dtype(int dt) { return dt == EE_F32 ? EE_F32 : (dt == EE_BF16_TILED ? EE_BF16 : dt); }
int launch_row_stats(const float* x, int64_t ldx, int64_t m, int64_t h, void* xb, float* ssq,
                     cudaStream_t s);
// tiled-mode GEMV with folded RMSNorm (ssq != nullptr) and, for residual
// epilogues, refreshed row statistics (xb_out/ssq_out != nullptr)
struct GemvNorm {
    const float* ssq;  // input-row sum-of-squares partials (K/16 per row) or nullptr
    float eps;
    bf16* xb_out;      // residual epilogue: bf16 copy of the updated rows
    float* ssq_out;    // residual epilogue: their sum-of-squares partials
};
int launch_gemv_tiled(const bf16* x, int64_t m, int64_t K, const void* W, int64_t N, int epi,
                      void* out, int64_t ldo, GemvNorm nrm, cudaStream_t s);
// multi-row (prefill) tcgen05 GEMM over tiled weights (prefill_gemm.cu);
// epi: 0 = q/K/V write (folded norm), 1 = GELU (folded norm), 2 = residual +
// row statistics
int launch_prefill_tiled(const bf16* x, int64_t m, int64_t K, const void* W, int64_t N, int epi,
                         const float* ssq_in, float eps, float* q, void* kc, void* vc,
                         const int32_t* pos, int64_t h, void* out, float* xres, bf16* xb,
                         float* ssq_out, void* ws, size_t ws_bytes, cudaStream_t s);
constexpr int kPrefillMinRows = 17;  // passes with more rows use the GEMM
int decode_layer_launches(const ee_decoder_t* D, int64_t m);
int launch_qkv_tiled(const bf16* x, int64_t m, int64_t h, const void* Wqkv, GemvNorm nrm,
                     float* q, void* kc, void* vc, const int32_t* pos, cudaStream_t s);
