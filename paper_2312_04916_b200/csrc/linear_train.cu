// Training backbone linears on the CTA-pair tcgen05 GEMM of tc_gemm.cuh
// (TMA SW128 operands, TMEM accumulators, 8 epilogue warps), replacing the
// library (cuBLAS) forward and input-gradient matmuls of `run_layer`
// (eepipe/model.py:207-216; matmul fwd / bwd eepipe/autodiff.py:158-179):
//
//   forward:  Y  = X W  [+ R]        X (T, K) bf16, W (K, N) bf16 (read MN-major)
//   dgrad:    dX = dY W^T [+ R]      dY (T, N) bf16, W (K, N) (read K-major)
//
// Outputs bf16 row-major; the optional residual R (bf16, same shape as the
// output) is added to the float32 accumulator before the single rounding
// (the `addmm(beta = 1)` the unfused path used: one rounding, no separate
// add pass over the (T, N) rows).  The weight gradient of the same linears
// is ee_wgrad_accum (exit_head_train.cu): float32 accumulation in place.
#include <cuda.h>

#include "tc_gemm.cuh"

namespace {

constexpr int kBN = 256;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&t);
}

struct EpiBf16 {
    static constexpr bool kTwoPass = false;
    static constexpr bool kSplitK = false;
    static constexpr bool kStreamK = true;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = true;   // TMA-stored output boxes (tc_gemm.cuh)
    static constexpr bool kReduceAdd = false;
    using OutT = bf16;
    bf16* out;
    const bf16* res;  // nullable
    int ld;
    int out_map(CUtensorMap* m, int M, int N) const { return tc::make_tmap_out(m, out, 2, M, N, ld); }
    // 16 outputs of a chunk: accumulator + residual, one rounding
    __device__ void stage(int row, int col, const float* v0, int nvalid, bf16* o) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = v0[j];
        if (res && nvalid > 0) {
            const int64_t off = (int64_t)row * ld + col;
            if (nvalid == 16) {
                const uint4 r0 = reinterpret_cast<const uint4*>(res + off)[0];
                const uint4 r1 = reinterpret_cast<const uint4*>(res + off)[1];
                const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                    v[2 * q] += f.x;
                    v[2 * q + 1] += f.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j < nvalid) v[j] += __bfloat162float(res[off + j]);
            }
        }
        uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
#pragma unroll
        for (int q = 0; q < 8; ++q) o32[q] = pack2(v[2 * q], v[2 * q + 1]);
    }
    // the half-row's residual (BN/2 bf16 = 256 B, two lines) is pulled into
    // L1 before the accumulator chunks stream out of TMEM, so the per-chunk
    // residual loads hit L1 instead of waiting on HBM one chunk at a time
    __device__ void begin_tile(int row, int col0, int, bool valid) {
        if (res && valid) {
            const bf16* p = res + (int64_t)row * ld + col0;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 64));
        }
    }
    __device__ void end_tile(int, int, int, bool) {}
    __device__ void chunk(int row, int col, const float* v0, int nvalid) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = v0[j];
        const int64_t off = (int64_t)row * ld + col;
        if (nvalid == 16) {
            if (res) {
                const uint4 r0 = reinterpret_cast<const uint4*>(res + off)[0];
                const uint4 r1 = reinterpret_cast<const uint4*>(res + off)[1];
                const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                    v[2 * q] += f.x;
                    v[2 * q + 1] += f.y;
                }
            }
            uint4 u[2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
                u[q] = make_uint4(pack2(v[8 * q], v[8 * q + 1]), pack2(v[8 * q + 2], v[8 * q + 3]),
                                  pack2(v[8 * q + 4], v[8 * q + 5]), pack2(v[8 * q + 6], v[8 * q + 7]));
            reinterpret_cast<uint4*>(out + off)[0] = u[0];
            reinterpret_cast<uint4*>(out + off)[1] = u[1];
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) {
                    const float r = res ? __bfloat162float(res[off + j]) : 0.f;
                    out[off + j] = __float2bfloat16_rn(v[j] + r);
                }
        }
    }
};

int check(const char* what, int64_t T, int64_t K, int64_t N) {
    EE_REQUIRE(T > 0 && K > 0 && N > 0 && K % 8 == 0 && N % 8 == 0, EE_ESHAPE,
               "%s: K and N must be positive multiples of 8 (T=%lld K=%lld N=%lld)", what,
               (long long)T, (long long)K, (long long)N);
    EE_REQUIRE(T < (1ll << 31) && K < (1ll << 31) && N < (1ll << 31), EE_ESHAPE, "%s: too large",
               what);
    return EE_OK;
}

}  // namespace

extern "C" int ee_linear_fwd(const void* X, const void* W, int64_t T, int64_t K, int64_t N,
                             const void* R, void* Y, void* stream) {
    int rc;
    if ((rc = check("linear_fwd", T, K, N))) return rc;
    return tc::launch_tc_gemm2<kBN, false, true, false>(
        X, W, (int)T, (int)N, (int)K, EpiBf16{(bf16*)Y, (const bf16*)R, (int)N}, as_stream(stream));
}

extern "C" int ee_linear_dgrad(const void* dY, const void* W, int64_t T, int64_t K, int64_t N,
                               const void* R, void* dX, void* stream) {
    int rc;
    if ((rc = check("linear_dgrad", T, K, N))) return rc;
    return tc::launch_tc_gemm2<kBN, false, false, false>(
        dY, W, (int)T, (int)K, (int)N, EpiBf16{(bf16*)dX, (const bf16*)R, (int)K},
        as_stream(stream));
}

// q / k / v of one block as ONE GEMM each way: the three (K, N) weight
// matrices are adjacent in the flat parameter buffer (W_j = W + j K N), so
// they are read as one stacked operand (tc_gemm.cuh, bsub):
//   fwd:    Y (T, parts N) = X [W_0 | ... | W_{p-1}]
//   dgrad:  dX (T, K) = dY (T, parts N) [W_0 | ... | W_{p-1}]^T [+ R]
// One wide GEMM instead of three 2048-wide ones: fewer partial waves and
// epilogue tails (eepipe/model.py:207-216 computes h1 @ wq, h1 @ wk, h1 @ wv).
extern "C" int ee_linear_fwd_stacked(const void* X, const void* W, int64_t T, int64_t K, int64_t N,
                                     int64_t parts, void* Y, void* stream) {
    int rc;
    if ((rc = check("linear_fwd_stacked", T, K, N * parts))) return rc;
    EE_REQUIRE(parts >= 1 && N % 128 == 0 && K % 64 == 0, EE_ESHAPE,
               "linear_fwd_stacked: N %% 128 and K %% 64 must be 0 (K=%lld N=%lld)", (long long)K,
               (long long)N);
    return tc::launch_tc_gemm2<kBN, false, true, false>(
        X, W, (int)T, (int)(N * parts), (int)K, EpiBf16{(bf16*)Y, nullptr, (int)(N * parts)},
        as_stream(stream), 1, (int)N);
}

extern "C" int ee_linear_dgrad_stacked(const void* dY, const void* W, int64_t T, int64_t K,
                                       int64_t N, int64_t parts, const void* R, void* dX,
                                       void* stream) {
    int rc;
    if ((rc = check("linear_dgrad_stacked", T, K, N * parts))) return rc;
    EE_REQUIRE(parts >= 1 && N % 128 == 0, EE_ESHAPE,
               "linear_dgrad_stacked: N %% 128 must be 0 (N=%lld)", (long long)N);
    return tc::launch_tc_gemm2<kBN, false, false, false>(
        dY, W, (int)T, (int)K, (int)(N * parts), EpiBf16{(bf16*)dX, (const bf16*)R, (int)K},
        as_stream(stream), 1, (int)N);
}

#ifdef EE_TRACE
extern "C" int ee_trace_gemm(unsigned long long* tl, int* units) {
    cudaMemcpyFromSymbol(tl, tc::g_gemm_tl, sizeof(tc::g_gemm_tl));
    return (int)cudaMemcpyFromSymbol(units, tc::g_gemm_unit, sizeof(tc::g_gemm_unit));
}
#endif
