// Training MLP block GEMMs with the GELU fused into the epilogue, on the
// CTA-pair tcgen05 GEMM of tc_gemm.cuh (TMA SW128 operands, TMEM
// accumulators, 8 epilogue warps):
//
//   up:        pre = X W1,  act = GELU_erf(pre)            (both stored bf16)
//   down-bwd:  dpre = (dY W2^T) * GELU_erf'(pre)          (bf16)
//
// restating the `gelu_fwd` / `gelu_bwd` of the block (eepipe/_pykernels.py:
// 27-33, eepipe/model.py:214-216) around the two matmuls that feed / consume
// them, so the (T, 4h) activation and its gradient are written once by the
// GEMM instead of by a GEMM plus an element-wise pass (and read again).  The
// element-wise arithmetic follows the unfused bf16 path: the GEMM result is
// rounded to bf16 first (that is the tensor the element-wise op would read),
// GELU / its derivative are evaluated in float32 on it.
//
// Layouts: X (T, h), dY (T, h), pre / act / dpre (T, N) row-major bf16;
// W1 is (h, N) row-major (read MN-major), W2 is (N, h) row-major (K-major).
#include <cuda.h>

#include "tc_gemm.cuh"

namespace {

constexpr int kBN = 256;

__device__ __forceinline__ float gelu_grad(float x) {
    const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752440f));
    const float pdf = 0.39894228040143267794f * expf(-0.5f * x * x);
    return cdf + x * pdf;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&t);
}

struct EpiGeluUp {
    static constexpr bool kTwoPass = false;
    static constexpr bool kSplitK = false;
    static constexpr bool kStreamK = true;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = false;  // two outputs: per-thread row stores
    bf16* pre;
    bf16* act;
    int ld;
    __device__ void begin_tile(int, int, int, bool) {}
    __device__ void end_tile(int, int, int, bool) {}
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        float p[16], a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            p[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
            a[j] = gelu_erf(p[j]);
        }
        bf16* po = pre + (int64_t)row * ld + col;
        bf16* ao = act + (int64_t)row * ld + col;
        if (nvalid == 16) {
            uint4 u[2], w[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                u[q] = make_uint4(pack2(p[8 * q], p[8 * q + 1]), pack2(p[8 * q + 2], p[8 * q + 3]),
                                  pack2(p[8 * q + 4], p[8 * q + 5]), pack2(p[8 * q + 6], p[8 * q + 7]));
                w[q] = make_uint4(pack2(a[8 * q], a[8 * q + 1]), pack2(a[8 * q + 2], a[8 * q + 3]),
                                  pack2(a[8 * q + 4], a[8 * q + 5]), pack2(a[8 * q + 6], a[8 * q + 7]));
            }
            reinterpret_cast<uint4*>(po)[0] = u[0];
            reinterpret_cast<uint4*>(po)[1] = u[1];
            reinterpret_cast<uint4*>(ao)[0] = w[0];
            reinterpret_cast<uint4*>(ao)[1] = w[1];
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) {
                    po[j] = __float2bfloat16_rn(p[j]);
                    ao[j] = __float2bfloat16_rn(a[j]);
                }
        }
    }
};

struct EpiGeluBwd {
    static constexpr bool kTwoPass = false;
    static constexpr bool kSplitK = false;
    static constexpr bool kStreamK = true;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = true;   // TMA-stored output boxes (tc_gemm.cuh)
    static constexpr bool kReduceAdd = false;
    using OutT = bf16;
    const bf16* pre;
    bf16* dpre;
    int ld;
    int out_map(CUtensorMap* m, int M, int N) const { return tc::make_tmap_out(m, dpre, 2, M, N, ld); }
    __device__ void stage(int row, int col, const float* v, int nvalid, bf16* o) {
        const bf16* pi = pre + (int64_t)row * ld + col;
        float x[16];
        if (nvalid == 16) {
            const uint4 u0 = reinterpret_cast<const uint4*>(pi)[0];
            const uint4 u1 = reinterpret_cast<const uint4*>(pi)[1];
            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                x[2 * q] = f.x;
                x[2 * q + 1] = f.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = j < nvalid ? __bfloat162float(pi[j]) : 0.f;
        }
        uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            o32[q] = pack2(__bfloat162float(__float2bfloat16_rn(v[2 * q])) * gelu_grad(x[2 * q]),
                           __bfloat162float(__float2bfloat16_rn(v[2 * q + 1])) * gelu_grad(x[2 * q + 1]));
    }
    __device__ void begin_tile(int, int, int, bool) {}
    __device__ void end_tile(int, int, int, bool) {}
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        const bf16* pi = pre + (int64_t)row * ld + col;
        bf16* go = dpre + (int64_t)row * ld + col;
        float x[16];
        if (nvalid == 16) {
            const uint4 u0 = reinterpret_cast<const uint4*>(pi)[0];
            const uint4 u1 = reinterpret_cast<const uint4*>(pi)[1];
            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                x[2 * q] = f.x;
                x[2 * q + 1] = f.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = j < nvalid ? __bfloat162float(pi[j]) : 0.f;
        }
        float g[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) g[j] = __bfloat162float(__float2bfloat16_rn(v[j])) * gelu_grad(x[j]);
        if (nvalid == 16) {
            uint4 u[2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
                u[q] = make_uint4(pack2(g[8 * q], g[8 * q + 1]), pack2(g[8 * q + 2], g[8 * q + 3]),
                                  pack2(g[8 * q + 4], g[8 * q + 5]), pack2(g[8 * q + 6], g[8 * q + 7]));
            reinterpret_cast<uint4*>(go)[0] = u[0];
            reinterpret_cast<uint4*>(go)[1] = u[1];
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) go[j] = __float2bfloat16_rn(g[j]);
        }
    }
};

}  // namespace

extern "C" int ee_mlp_up_gelu(const void* X, const void* W1, int64_t T, int64_t h, int64_t N,
                              void* pre, void* act, void* stream) {
    EE_REQUIRE(T > 0 && h > 0 && N > 0 && h % 8 == 0 && N % 8 == 0, EE_ESHAPE,
               "mlp_up_gelu: h and N must be positive multiples of 8 (T=%lld h=%lld N=%lld)",
               (long long)T, (long long)h, (long long)N);
    EE_REQUIRE(T < (1ll << 31) && N < (1ll << 31) && h < (1ll << 31), EE_ESHAPE,
               "mlp_up_gelu: too large");
    return tc::launch_tc_gemm2<kBN, false, true, false>(
        X, W1, (int)T, (int)N, (int)h, EpiGeluUp{(bf16*)pre, (bf16*)act, (int)N},
        as_stream(stream));
}

extern "C" int ee_mlp_gelu_bwd(const void* dY, const void* W2, int64_t T, int64_t h, int64_t N,
                               const void* pre, void* dpre, void* stream) {
    EE_REQUIRE(T > 0 && h > 0 && N > 0 && h % 8 == 0 && N % 8 == 0, EE_ESHAPE,
               "mlp_gelu_bwd: h and N must be positive multiples of 8 (T=%lld h=%lld N=%lld)",
               (long long)T, (long long)h, (long long)N);
    EE_REQUIRE(T < (1ll << 31) && N < (1ll << 31) && h < (1ll << 31), EE_ESHAPE,
               "mlp_gelu_bwd: too large");
    return tc::launch_tc_gemm2<kBN, false, false, false>(
        dY, W2, (int)T, (int)N, (int)h, EpiGeluBwd{(const bf16*)pre, (bf16*)dpre, (int)N},
        as_stream(stream));
}
