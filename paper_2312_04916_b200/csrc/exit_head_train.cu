// Fused training exit head: weighted cross-entropy of one exit and its
// gradients on tcgen05 tensor cores, without the (n, V) LOGITS ever being
// written to HBM.
//
// Restates `run_head` (x @ out^T, eepipe/model.py:219-230) + `cross_entropy`
// (eepipe/autodiff.py:301-323, _pykernels.py:64-85) + the matmul backward
// (eepipe/autodiff.py:170-177):
//   S = X W^T,  lse_i = log sum_v exp S_iv,  loss = w/n sum_i (lse_i - S_i,t_i)
//   G = w/n (softmax(S) - onehot(t)),  dX = G W,  dW += G^T X
// as four tcgen05 GEMMs (tc_gemm.cuh) whose epilogues do the softmax work:
//   K1  S = X W^T          epilogue: per (row, 256-col tile) online max /
//                          sum-exp + the target logit (logits stay in TMEM)
//   M   merge partials in fixed order -> lse, loss (deterministic)
//   K2  S = X W^T (again)  epilogue: G = w/n (exp(S - lse) - [v == t]) in
//                          bf16, stored row-major (G) and transposed (G^T)
//   K3  dX  = G  . (W^T)^T  (A = G   [n x V], B = W^T [h x V], K = V)
//   K4  dW += G^T . (X^T)^T (A = G^T [V x n], B = X^T [h x n], K = n)
// Only the logit GRADIENT G (bf16) reaches HBM, and only because the two
// backward GEMMs contract it along different axes; the logits themselves,
// the softmax probabilities and the reference's cached (n, V) float64 probs
// (_ckernels.pyx:130-151) never exist in memory.  Executed FLOPs are
// 8 n h V (S is recomputed once); the roofline is quoted on the algorithmic
// 6 n h V.
#include <cuda.h>

#include "tc_gemm.cuh"

namespace {

constexpr int kBN = 256;

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct TrainWs {
    bf16 *xt, *wt, *g, *gt;
    float *pmax, *psum, *tgt, *lse, *rowloss;
};

TrainWs carve(void* ws, int64_t n, int64_t h, int64_t V, bool need_wt) {
    TrainWs w;
    char* p = (char*)ws;
    const int64_t ntn = (V + kBN - 1) / kBN;
    w.xt = (bf16*)p; p += al((size_t)h * n * 2);
    w.wt = need_wt ? (bf16*)p : nullptr; p += need_wt ? al((size_t)h * V * 2) : 0;
    w.pmax = (float*)p; p += al((size_t)n * ntn * 4);
    w.psum = (float*)p; p += al((size_t)n * ntn * 4);
    w.tgt = (float*)p; p += al((size_t)n * 4);
    w.lse = (float*)p; p += al((size_t)n * 4);
    w.rowloss = (float*)p; p += al((size_t)n * 4);
    w.g = (bf16*)p; p += al((size_t)n * V * 2);
    w.gt = (bf16*)p; p += al((size_t)n * V * 2);
    return w;
}

size_t carve_bytes(int64_t n, int64_t h, int64_t V, bool need_wt) {
    const int64_t ntn = (V + kBN - 1) / kBN;
    return al((size_t)h * n * 2) + (need_wt ? al((size_t)h * V * 2) : 0) +
           2 * al((size_t)n * ntn * 4) + 3 * al((size_t)n * 4) + 2 * al((size_t)n * V * 2);
}

// ---- epilogues ----------------------------------------------------------------
struct EpiLse {  // K1: per (row, tile) online max / sum-exp, target logit
    const int64_t* targets;
    float *pmax, *psum, *tgt;
    int ntn;
    float m, s;
    int64_t t;
    __device__ void begin_tile(int row, int, int, bool valid) {
        m = -INFINITY;
        s = 0.f;
        t = valid ? targets[row] : -1;
    }
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        float cm = -INFINITY;
        for (int j = 0; j < nvalid; ++j) cm = fmaxf(cm, v[j]);
        const float nm = fmaxf(m, cm);
        float acc = s * expf(m - nm);
        for (int j = 0; j < nvalid; ++j) acc += expf(v[j] - nm);
        s = acc;
        m = nm;
        if (t >= col && t < col + nvalid) tgt[row] = v[t - col];
    }
    __device__ void end_tile(int row, int, int nb, bool valid) {
        if (valid) {
            pmax[(int64_t)row * ntn + nb] = m;
            psum[(int64_t)row * ntn + nb] = s;
        }
    }
};

struct EpiGrad {  // K2: G = scale * (exp(S - lse) - onehot), bf16, G and G^T
    const int64_t* targets;
    const float* lse;
    float scale;
    bf16 *g, *gt;
    int M, N;
    float l;
    int64_t t;
    __device__ void begin_tile(int row, int, int, bool valid) {
        if (valid) {
            l = lse[row];
            t = targets[row];
        }
    }
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        float gv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            gv[j] = scale * expf(v[j] - l) - ((int64_t)(col + j) == t ? scale : 0.f);
        bf16* gr = g + (int64_t)row * N + col;
        if (nvalid == 16) {
            uint32_t w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                __nv_bfloat162 b = __floats2bfloat162_rn(gv[2 * j], gv[2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&b);
            }
            reinterpret_cast<uint4*>(gr)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(gr)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
            for (int j = 0; j < nvalid; ++j) gr[j] = __float2bfloat16_rn(gv[j]);
        }
        for (int j = 0; j < nvalid; ++j) gt[(int64_t)(col + j) * M + row] = __float2bfloat16_rn(gv[j]);
    }
    __device__ void end_tile(int, int, int, bool) {}
};

template <bool ACCUM>
struct EpiF32 {  // K3 store / K4 accumulate
    float* out;
    int ldo;
    __device__ void begin_tile(int, int, int, bool) {}
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        float* o = out + (int64_t)row * ldo + col;
        if (nvalid == 16) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
                float4 c = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                if (ACCUM) {
                    const float4 p = *reinterpret_cast<const float4*>(o + j);
                    c.x += p.x;
                    c.y += p.y;
                    c.z += p.z;
                    c.w += p.w;
                }
                *reinterpret_cast<float4*>(o + j) = c;
            }
        } else {
            for (int j = 0; j < nvalid; ++j) o[j] = ACCUM ? o[j] + v[j] : v[j];
        }
    }
    __device__ void end_tile(int, int, int, bool) {}
};

// ---- small kernels ---------------------------------------------------------
__global__ void k_transpose_bf16(const bf16* __restrict__ in, int64_t rows, int64_t cols,
                                 bf16* __restrict__ out) {
    __shared__ bf16 tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

// per-row merge of the tile partials in ascending tile order
__global__ void k_lse_merge(const float* __restrict__ pmax, const float* __restrict__ psum,
                            const float* __restrict__ tgt, int n, int ntn, float* __restrict__ lse,
                            float* __restrict__ rowloss) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* pm = pmax + (int64_t)i * ntn;
    const float* ps = psum + (int64_t)i * ntn;
    float M = -INFINITY;
    for (int b = 0; b < ntn; ++b) M = fmaxf(M, pm[b]);
    float S = 0.f;
    for (int b = 0; b < ntn; ++b) S += ps[b] * expf(pm[b] - M);
    const float l = M + logf(S);
    lse[i] = l;
    rowloss[i] = l - tgt[i];
}

// fixed-shape tree sum of the per-row losses -> weight/n * sum (one CTA)
__global__ void k_loss_sum(const float* __restrict__ rowloss, int n, float scale,
                           float* __restrict__ loss) {
    __shared__ float sh[1024];
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += 1024) s += rowloss[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = sh[0] * scale;
}

int transpose(const bf16* in, int64_t rows, int64_t cols, bf16* out, cudaStream_t s) {
    const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    k_transpose_bf16<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, out);
    return ee_check_launch("transpose");
}

}  // namespace

namespace tc {
int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EE_REQUIRE(((uintptr_t)base & 15) == 0 && cols % 8 == 0, EE_ESHAPE,
               "tensor map: base must be 16-B aligned and cols %% 8 == 0");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    // resolved through the runtime so libee.so does not link libcuda (the
    // build container has no driver; the GPU box does)
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return ee_fail(EE_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        encode = (EncodeFn)fn;
    }
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EE_REQUIRE(r == CUDA_SUCCESS, EE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return EE_OK;
}
}  // namespace tc

size_t exit_head_train_ws_bytes(int64_t n, int64_t h, int64_t V) {
    return carve_bytes(n, h, V, true);
}

extern "C" int ee_exit_head_train(const void* x, int64_t n, int64_t h, const void* W, const void* Wt,
                                  int64_t V, const int64_t* targets, float weight, float* loss,
                                  float* dx, float* dw_acc, void* ws, size_t ws_bytes,
                                  void* stream) {
    EE_REQUIRE(n > 0 && h > 0 && V > 0 && n % 8 == 0 && h % 8 == 0 && V % 8 == 0, EE_ESHAPE,
               "exit_head_train: n, h, V must be positive multiples of 8 (n=%lld h=%lld V=%lld)",
               (long long)n, (long long)h, (long long)V);
    EE_REQUIRE(n < (1ll << 31) / 1 && V < (1ll << 31), EE_ESHAPE, "exit_head_train: too large");
    EE_REQUIRE(ws && ws_bytes >= carve_bytes(n, h, V, Wt == nullptr), EE_ESHAPE,
               "exit_head_train: workspace too small (%zu < %zu)", ws_bytes,
               carve_bytes(n, h, V, Wt == nullptr));
    cudaStream_t s = as_stream(stream);
    TrainWs w = carve(ws, n, h, V, Wt == nullptr);
    const int ntn = (int)((V + kBN - 1) / kBN);
    const float scale = weight / (float)n;
    int rc;
    // operands for the backward GEMMs (K-major everywhere)
    if ((rc = transpose((const bf16*)x, n, h, w.xt, s))) return rc;
    const bf16* wt = (const bf16*)Wt;
    if (!wt) {
        if ((rc = transpose((const bf16*)W, V, h, w.wt, s))) return rc;
        wt = w.wt;
    }
    // K1: online log-sum-exp partials + target logits
    if ((rc = tc::launch_tc_gemm<kBN>(x, W, (int)n, (int)V, (int)h,
                                      EpiLse{targets, w.pmax, w.psum, w.tgt, ntn, 0.f, 0.f, 0}, s)))
        return rc;
    k_lse_merge<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w.pmax, w.psum, w.tgt, (int)n, ntn,
                                                            w.lse, w.rowloss);
    if ((rc = ee_check_launch("lse_merge"))) return rc;
    k_loss_sum<<<1, 1024, 0, s>>>(w.rowloss, (int)n, scale, loss);
    if ((rc = ee_check_launch("loss_sum"))) return rc;
    // K2: logit gradient (bf16), both layouts
    if ((rc = tc::launch_tc_gemm<kBN>(
             x, W, (int)n, (int)V, (int)h,
             EpiGrad{targets, w.lse, scale, w.g, w.gt, (int)n, (int)V, 0.f, 0}, s)))
        return rc;
    // K3: dX = G . W
    if ((rc = tc::launch_tc_gemm<kBN>(w.g, wt, (int)n, (int)h, (int)V, EpiF32<false>{dx, (int)h}, s)))
        return rc;
    // K4: dW += G^T . X
    return tc::launch_tc_gemm<kBN>(w.gt, w.xt, (int)V, (int)h, (int)n, EpiF32<true>{dw_acc, (int)h},
                                   s);
}
