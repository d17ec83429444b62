// Fused inference exit head:
//   [gather rows] -> [RMSNorm] -> logits over the vocabulary -> split-V
//   (max, sum-exp, argmax) per 16-row vocabulary tile -> fixed-order merge ->
//   (token, confidence, fire).  Logits never touch HBM (optional debug dump).
//
// Restates `head_logits` + `exit_decision` (eepipe/inference.py:118-133,
// 175-185):  m = max(l); p = exp(l - m) / sum; token = argmax (lowest index
// wins); conf = p[token] = 1 / sum exp(l - m); fire = thr < 1 && conf > thr.
//
// bf16: the TMA-bulk-fed GEMV body (gemv_tma.cuh) with the RMSNorm fused in
// its prologue and a softmax-partial epilogue; tiles are statically
// round-robined over a persistent grid whose size does not depend on the
// row count; each CTA folds its tiles' partials in tile order into one
// running partial per row, and the last CTA to finish merges the CTA
// partials in CTA order with a fixed-shape tree (deterministic, row-stable).  fp32 (parity mode): RMSNorm launch + SIMT dot products with
// the same partial/merge scheme.
#include <algorithm>

#include "gemv_core.cuh"
#include "gemv_tma.cuh"

namespace {

constexpr int kMaxCols = 16;

struct HeadWs {
    int* done_ctr;
    int* flag;
    int* unit_ctr;
    float* pm;
    float* ps;
    int* pi;
    float* xn;  // fp32 path: normalised rows (kMaxCols x h)
};

__host__ __device__ inline HeadWs head_ws(void* base, int64_t units) {
    HeadWs w;
    char* b = (char*)base;
    w.done_ctr = (int*)b;
    w.flag = (int*)(b + 4);
    w.unit_ctr = (int*)(b + 8);
    w.pm = (float*)(b + 256);
    w.ps = w.pm + units * kMaxCols;
    w.pi = (int*)(w.ps + units * kMaxCols);
    w.xn = (float*)(w.pi + units * kMaxCols);
    return w;
}

__device__ __forceinline__ void combine(float& m1, float& s1, int& i1, float m2, float s2, int i2) {
    if (s2 == 0.f) return;  // empty partial
    if (s1 == 0.f) {
        m1 = m2;
        s1 = s2;
        i1 = i2;
        return;
    }
    const float M = fmaxf(m1, m2);
    const float s = s1 * expf(m1 - M) + s2 * expf(m2 - M);
    const int i = (m1 > m2) ? i1 : ((m2 > m1) ? i2 : min(i1, i2));
    m1 = M;
    s1 = s;
    i1 = i;
}

// Fixed-order merge of all unit partials, one WARP per column (columns
// round-robin over the NT/32 warps): lane l folds units l, l+32, ... in
// ascending order, then a xor butterfly with a commutative combine (every
// lane ends with identical bits).  No block-wide barriers inside the merge.
template <int NT>
__device__ void merge_and_decide(const HeadWs& w, int64_t units, int m, float thr, int32_t* token,
                                 float* conf, uint8_t* fire, int32_t* nonfinite, int tid,
                                 void (*sync)()) {
    const int lane = tid & 31, wid = tid >> 5;
    for (int c = wid; c < m; c += NT / 32) {
        float M = -INFINITY, S = 0.f;
        int I = 0x7fffffff;
        // 16 partials per lane in flight per batch, folded in ascending unit order
        for (int64_t u0 = lane; u0 < units; u0 += 32 * 16) {
            float pm[16], ps[16];
            int pi[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int64_t u = u0 + 32 * k;
                if (u < units) {
                    pm[k] = __ldcg(w.pm + u * kMaxCols + c);
                    ps[k] = __ldcg(w.ps + u * kMaxCols + c);
                    pi[k] = __ldcg(w.pi + u * kMaxCols + c);
                }
            }
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (u0 + 32 * k < units) combine(M, S, I, pm[k], ps[k], pi[k]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, M, o);
            const float s2 = __shfl_xor_sync(0xffffffffu, S, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, I, o);
            combine(M, S, I, m2, s2, i2);
        }
        if (lane == 0) {
            const float cf = 1.0f / S;
            token[c] = I;
            conf[c] = cf;
            fire[c] = (thr < 1.0f && cf > thr) ? 1 : 0;
        }
    }
    // the outputs may live in host-mapped memory that the host polls through
    // *nonfinite (written last): make them visible system-wide first
    __threadfence_system();
    sync();
    if (tid == 0) {
        *nonfinite = __ldcg(w.flag);
        *w.flag = 0;
        *w.done_ctr = 0;
        *w.unit_ctr = 0;
    }
}

__device__ void sync_consumers() { tma_gemv::consumers_sync(); }
__device__ void sync_block() { __syncthreads(); }

// ---- bf16: epilogue for the TMA body ---------------------------------------
struct HeadEpi {
    HeadWs w;
    int V, m;
    float thr;
    int32_t *token, *nonfinite;
    float* conf;
    uint8_t* fire;
    float* dbg;
    bool bad;
    // running partials of this CTA, combined over its tiles in increasing
    // tile order: thread 16 j holds columns j and j + 8 (rounds k = 0, 1)
    float rm[2] = {-INFINITY, -INFINITY}, rs[2] = {0.f, 0.f};
    int ri[2] = {0x7fffffff, 0x7fffffff};

    __device__ void tile(const float* red, int n0, int r0, int N, int mm, int cols,
                         const float* /*inv*/) {
        using namespace tma_gemv;
        const int tid = threadIdx.x;
        const int nr = min(kRows, V - n0);
        auto val = [&](int i, int c) {
            const int o = i * kMaxCols + c;
            return ((red[o] + red[kRows * kMaxCols + o]) + red[2 * kRows * kMaxCols + o]) +
                   red[3 * kRows * kMaxCols + o];
        };
        // 16 threads per column (one vocabulary row each), fixed xor
        // butterflies for the tile max / argmax and the sum of exponentials
        for (int c0 = 0; c0 < m; c0 += kConsumers * 32 / kRows) {
            const int c = c0 + (tid >> 4);
            const int i = tid & 15;
            const bool act = c < m;
            const float v = (act && i < nr) ? val(i, c) : -INFINITY;
            if (act && i < nr) bad |= !isfinite(v);
            float mx = v;
            int idx = (act && i < nr) ? n0 + i : 0x7fffffff;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                if (m2 > mx || (m2 == mx && i2 < idx)) {
                    mx = m2;
                    idx = i2;
                }
            }
            float e = (act && i < nr) ? expf(v - mx) : 0.f;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            // lane i == 0 of each column group folds the tile into the CTA's
            // running partial of that column (tiles in increasing order)
            if (act && i == 0) {
                const int k = c0 / (kConsumers * 32 / kRows);
                combine(rm[k], rs[k], ri[k], mx, e, idx);
            }
        }
        if (dbg) {
            for (int i = tid; i < kRows * m; i += kConsumers * 32) {
                const int row = i & 15, c = i >> 4;
                if (row < nr) dbg[(int64_t)c * V + n0 + row] = val(row, c);
            }
        }
    }

    __device__ void finish() {
        using namespace tma_gemv;
        __shared__ int s_last;
        // one partial per CTA (unit = CTA index); the last CTA merges the
        // CTA partials in CTA order: a fixed two-level order (tiles of a CTA
        // ascending, then CTAs ascending) for a fixed grid size
        if ((threadIdx.x & 15) == 0) {
            const int64_t u = blockIdx.x;
            constexpr int per_round = kConsumers * 32 / kRows;  // 8 columns
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int c = k * per_round + (threadIdx.x >> 4);
                if (c < m) {
                    w.pm[u * kMaxCols + c] = rm[k];
                    w.ps[u * kMaxCols + c] = rs[k];
                    w.pi[u * kMaxCols + c] = ri[k];
                }
            }
        }
        if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(w.flag, 1);
        __threadfence();
        consumers_sync();
        if (threadIdx.x == 0) s_last = (atomicAdd(w.done_ctr, 1) == (int)gridDim.x - 1);
        consumers_sync();
        if (!s_last) return;
        __threadfence();
        merge_and_decide<kConsumers * 32>(w, gridDim.x, m, thr, token, conf, fire, nonfinite,
                                          threadIdx.x, sync_consumers);
    }
};

// weight-ring depth per row configuration: two CTAs per SM either way
// (4 x 24 KB stages for 8-row groups, 3 x 32 KB for 16-row groups), so the
// fixed grid of 2 x SMs runs in one wave
template <int NB>
constexpr int kHeadStages = NB == 1 ? 4 : 3;

template <int NB>
__global__ void __launch_bounds__(tma_gemv::kThreads)
k_exit_head_tma(const bf16* __restrict__ W, int V, int K, const bf16* __restrict__ X, int m,
                HeadEpi epi) {
    tma_gemv::gemv_body<NB, HeadEpi, kHeadStages<NB>>(W, V, K, X, K, m,
                                                      tma_gemv::RowNorm{nullptr, 0.f}, epi);
}

// ---- fp32 parity path --------------------------------------------------------
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ int grab_unit(int* ctr) {
    int u = 0;
    if ((threadIdx.x & 31) == 0) u = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, u, 0);
}

template <typename TW>
__global__ void __launch_bounds__(kThreads)
k_exit_head_simt(const float* __restrict__ X, int m, int64_t K, const TW* __restrict__ W, int V,
                float thr, int32_t* token, float* conf, uint8_t* fire, int32_t* nonfinite,
                float* logits_dbg, void* ws) {
    constexpr int RW = 8, RX = 4;
    __shared__ float tiles[kWarps][RW][kMaxCols];
    __shared__ int s_last;
    pdl_trigger_dev();
    pdl_wait_dev();
    const int64_t units = (V + RW - 1) / RW;
    const HeadWs w = head_ws(ws, units);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float (*tile)[kMaxCols] = tiles[warp];
    bool bad = false;
    for (int u = grab_unit(w.unit_ctr); u < units; u = grab_unit(w.unit_ctr)) {
        const int n0 = u * RW;
        for (int r0 = 0; r0 < m; r0 += RX) {
            float acc[RW][RX];
#pragma unroll
            for (int i = 0; i < RW; ++i)
#pragma unroll
                for (int j = 0; j < RX; ++j) acc[i][j] = 0.f;
            warp_tile_f32<RW, RX>(W, K, n0, V, X, K, r0, m, 0, 1, acc);
            if (lane == 0) {
#pragma unroll
                for (int i = 0; i < RW; ++i)
#pragma unroll
                    for (int j = 0; j < RX; ++j)
                        if (r0 + j < kMaxCols) tile[i][r0 + j] = acc[i][j];
            }
        }
        __syncwarp();
        if (lane < m) {
            const int nr = min(RW, V - n0);
            float mx = -INFINITY;
            int idx = n0;
            for (int i = 0; i < nr; ++i) {
                const float v = tile[i][lane];
                bad |= !isfinite(v);
                if (v > mx) {
                    mx = v;
                    idx = n0 + i;
                }
            }
            float sum = 0.f;
            for (int i = 0; i < nr; ++i) sum += expf(tile[i][lane] - mx);
            w.pm[(int64_t)u * kMaxCols + lane] = mx;
            w.ps[(int64_t)u * kMaxCols + lane] = sum;
            w.pi[(int64_t)u * kMaxCols + lane] = idx;
        }
        if (logits_dbg) {
            for (int i = lane; i < RW * m; i += 32) {
                const int row = i % RW, c = i / RW;
                if (n0 + row < V) logits_dbg[(int64_t)c * V + n0 + row] = tile[row][c];
            }
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(w.flag, 1);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(w.done_ctr, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    merge_and_decide<kThreads>(w, units, m, thr, token, conf, fire, nonfinite, threadIdx.x,
                               sync_block);
}

}  // namespace

// Workspace: 256 B of counters + (max, sum, idx) per (unit, column) for the
// smaller fp32 unit (8 rows) + kMaxCols normalised fp32 rows.  Zero once at
// allocation; every call leaves the counters zeroed.
size_t exit_head_ws_bytes(int64_t /*m*/, int64_t h, int64_t V) {
    const int64_t units = (V + 7) / 8;
    return 256 + (size_t)units * kMaxCols * 12 + (size_t)kMaxCols * h * 4;
}

extern "C" int ee_exit_head_infer(const float* x, int64_t ldx, const int32_t* rows, int64_t m,
                                  int64_t h, const float* norm_w, float eps, const void* W,
                                  int64_t V, int dtype, float threshold, int32_t* token,
                                  float* conf, uint8_t* fire, int32_t* nonfinite,
                                  float* logits_dbg, void* ws, size_t ws_bytes, void* stream) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && m <= kMaxCols, EE_ESHAPE, "exit_head: 1 <= m <= %d rows per call (m=%lld)",
               kMaxCols, (long long)m);
    EE_REQUIRE(h > 0 && V > 0 && V < (1ll << 30), EE_ESHAPE, "exit_head: bad shape");
    EE_REQUIRE(threshold > 0.f && threshold <= 1.f, EE_ECONFIG, "threshold must lie in (0, 1]");
    EE_REQUIRE(ws != nullptr && ws_bytes >= exit_head_ws_bytes(m, h, V), EE_ESHAPE,
               "exit_head: workspace too small");
    cudaStream_t s = as_stream(stream);
    const int sms = ee_sm_count();
    if (dtype == EE_BF16_TILED) {
        EE_REQUIRE(h % kTiledKS == 0, EE_ESHAPE, "exit_head tiled needs h %% %d == 0", kTiledKS);
        const int64_t units = (V + 15) / 16;
        HeadWs w = head_ws(ws, (V + 7) / 8);
        HeadEpi epi{w, (int)V, (int)m, threshold, token, nonfinite, conf, fire, logits_dbg, false};
        // gather + RMSNorm (or plain cast) of the evaluated rows -> bf16 (m, h)
        int rc = launch_rmsnorm_rows(x, ldx, rows, m, h, norm_w, eps, w.xn, EE_BF16, s);
        if (rc) return rc;
        const bf16* xn = (const bf16*)w.xn;
        const int nb = m <= 8 ? 1 : 2;
        const size_t smem = tma_gemv::smem_bytes(nb, nb == 1 ? kHeadStages<1> : kHeadStages<2>);
        // the grid (and with it the two-level merge order) does not depend
        // on m: 2 CTAs per SM
        const unsigned grid = (unsigned)std::min<int64_t>(units, (int64_t)sms * 2);
        static int conf_smem[2][16] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        cudaError_t e;
        if (nb == 1) {
            if ((int)smem > conf_smem[0][dev & 15]) {
                cudaFuncSetAttribute(k_exit_head_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
                conf_smem[0][dev & 15] = (int)smem;
            }
            e = launch_ex(k_exit_head_tma<1>, dim3(grid), dim3(tma_gemv::kThreads), smem, s,
                          (const bf16*)W, (int)V, (int)h, xn, (int)m, epi);
        } else {
            if ((int)smem > conf_smem[1][dev & 15]) {
                cudaFuncSetAttribute(k_exit_head_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
                conf_smem[1][dev & 15] = (int)smem;
            }
            e = launch_ex(k_exit_head_tma<2>, dim3(grid), dim3(tma_gemv::kThreads), smem, s,
                          (const bf16*)W, (int)V, (int)h, xn, (int)m, epi);
        }
        if (e != cudaSuccess) return ee_fail(EE_ECUDA, "exit_head launch: %s", cudaGetErrorString(e));
        return EE_OK;
    }
    if (dtype == EE_F32 || dtype == EE_BF16) {
        // SIMT path: parity mode (fp32) and small row-major bf16 heads
        HeadWs w = head_ws(ws, (V + 7) / 8);
        int rc = launch_rmsnorm_rows(x, ldx, rows, m, h, norm_w, eps, w.xn, EE_F32, s);
        if (rc) return rc;
        const int64_t units = (V + 7) / 8;
        const unsigned grid = (unsigned)std::min<int64_t>((units + kWarps - 1) / kWarps, (int64_t)sms * 4);
        cudaError_t e;
        if (dtype == EE_F32)
            e = launch_ex(k_exit_head_simt<float>, dim3(grid), dim3(kThreads), 0, s,
                          (const float*)w.xn, (int)m, h, (const float*)W, (int)V, threshold, token,
                          conf, fire, nonfinite, logits_dbg, ws);
        else
            e = launch_ex(k_exit_head_simt<bf16>, dim3(grid), dim3(kThreads), 0, s,
                          (const float*)w.xn, (int)m, h, (const bf16*)W, (int)V, threshold, token,
                          conf, fire, nonfinite, logits_dbg, ws);
        if (e != cudaSuccess) return ee_fail(EE_ECUDA, "exit_head launch: %s", cudaGetErrorString(e));
        return EE_OK;
    }
    return ee_fail(EE_ECONFIG, "exit_head: unknown dtype %d", dtype);
}
