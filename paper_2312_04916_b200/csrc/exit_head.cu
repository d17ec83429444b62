// Fused inference exit head: [norm already applied] -> logits over the
// vocabulary -> split-V online (max, sum-exp, argmax) -> fixed-order merge ->
// (token, confidence, fire).  Logits never touch HBM (optional debug dump).
//
// Restates `head_logits` + `exit_decision` (eepipe/inference.py:118-133,
// 175-185):  m = max(l); p = exp(l - m) / sum; token = argmax (lowest index
// wins); conf = p[token] = 1 / sum exp(l - m); fire = thr < 1 && conf > thr.
//
// Work unit = 16 vocabulary rows x full h (bf16 tensor-core GEMV core) or
// 8 rows (fp32 SIMT).  Units are handed out dynamically to warps of a
// persistent grid (load balance across 148 SMs with no tail); each unit's
// partial depends only on the unit, so the result is deterministic and
// row-stable.  The last CTA to finish merges the partials in unit order with
// a fixed-shape tree.
#include <algorithm>

#include "gemv_core.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxCols = 16;
constexpr int kUnroll = 4;

struct HeadWs {
    int* unit_ctr;
    int* done_ctr;
    int* flag;
    float* pm;
    float* ps;
    int* pi;
};

__host__ __device__ inline HeadWs head_ws(void* base, int64_t units) {
    HeadWs w;
    char* b = (char*)base;
    w.unit_ctr = (int*)b;
    w.done_ctr = (int*)(b + 4);
    w.flag = (int*)(b + 8);
    w.pm = (float*)(b + 256);
    w.ps = w.pm + units * kMaxCols;
    w.pi = (int*)(w.ps + units * kMaxCols);
    return w;
}

// Serial (max, argmax, sum-exp) of one column over a unit's rows, ascending n.
template <int R>
__device__ __forceinline__ void unit_partial(const float (*tile)[kMaxCols], int c, int n0, int V,
                                             float& mx, float& sum, int& idx, bool& bad) {
    mx = -INFINITY;
    idx = n0;
    const int nr = min(R, V - n0);
    for (int i = 0; i < nr; ++i) {
        const float v = tile[i][c];
        bad |= !isfinite(v);
        if (v > mx) {
            mx = v;
            idx = n0 + i;
        }
    }
    sum = 0.f;
    for (int i = 0; i < nr; ++i) sum += expf(tile[i][c] - mx);
}

__device__ __forceinline__ void combine(float& m1, float& s1, int& i1, float m2, float s2, int i2) {
    if (s2 == 0.f) return;  // empty partial (no units for this thread)
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

// Last CTA: fixed-order merge of all unit partials for each column.
__device__ void merge_and_decide(const HeadWs& w, int64_t units, int m, float thr, int32_t* token,
                                 float* conf, uint8_t* fire, int32_t* nonfinite) {
    __shared__ float sm_m[kThreads], sm_s[kThreads];
    __shared__ int sm_i[kThreads];
    const int tid = threadIdx.x;
    for (int c = 0; c < m; ++c) {
        float M = -INFINITY, S = 0.f;
        int I = 0x7fffffff;
        for (int64_t u = tid; u < units; u += kThreads)
            combine(M, S, I, __ldcg(w.pm + u * kMaxCols + c), __ldcg(w.ps + u * kMaxCols + c),
                    __ldcg(w.pi + u * kMaxCols + c));
        sm_m[tid] = M;
        sm_s[tid] = S;
        sm_i[tid] = I;
        __syncthreads();
        for (int s = kThreads / 2; s > 0; s >>= 1) {
            if (tid < s) {
                float a = sm_m[tid], b = sm_s[tid];
                int i = sm_i[tid];
                combine(a, b, i, sm_m[tid + s], sm_s[tid + s], sm_i[tid + s]);
                sm_m[tid] = a;
                sm_s[tid] = b;
                sm_i[tid] = i;
            }
            __syncthreads();
        }
        if (tid == 0) {
            const float cf = 1.0f / sm_s[0];
            token[c] = sm_i[0];
            conf[c] = cf;
            fire[c] = (thr < 1.0f && cf > thr) ? 1 : 0;
        }
        __syncthreads();
    }
    if (tid == 0) {
        *nonfinite = __ldcg(w.flag);
        *w.flag = 0;
        *w.unit_ctr = 0;
        *w.done_ctr = 0;
    }
}

__device__ __forceinline__ int grab_unit(int* ctr) {
    int u = 0;
    if ((threadIdx.x & 31) == 0) u = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, u, 0);
}

__device__ __forceinline__ bool finish_cta(const HeadWs& w) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(w.done_ctr, 1) == (int)gridDim.x - 1);
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

template <int NB>
__global__ void __launch_bounds__(kThreads)
k_exit_head_bf16(const bf16* __restrict__ X, int m, int64_t K, const bf16* __restrict__ W, int V,
                 float thr, int32_t* token, float* conf, uint8_t* fire, int32_t* nonfinite,
                 float* logits_dbg, void* ws) {
    __shared__ float tiles[kWarps][16][kMaxCols];
    const int64_t units = (V + 15) / 16;
    const HeadWs w = head_ws(ws, units);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float (*tile)[kMaxCols] = tiles[warp];
    bool bad = false;
    for (int u = grab_unit(w.unit_ctr); u < units; u = grab_unit(w.unit_ctr)) {
        float acc[NB][4];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.f;
        const int n0 = u * 16;
        warp_tile_bf16<NB, kUnroll>(W, K, n0, V, X, K, 0, m, 0, 1, acc);
        {
            const int g = lane >> 2, t = lane & 3;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                tile[g][nb * 8 + 2 * t] = acc[nb][0];
                tile[g][nb * 8 + 2 * t + 1] = acc[nb][1];
                tile[g + 8][nb * 8 + 2 * t] = acc[nb][2];
                tile[g + 8][nb * 8 + 2 * t + 1] = acc[nb][3];
            }
        }
        __syncwarp();
        if (lane < m) {
            float mx, sum;
            int idx;
            unit_partial<16>(tile, lane, n0, V, mx, sum, idx, bad);
            w.pm[(int64_t)u * kMaxCols + lane] = mx;
            w.ps[(int64_t)u * kMaxCols + lane] = sum;
            w.pi[(int64_t)u * kMaxCols + lane] = idx;
        }
        if (logits_dbg) {
            for (int i = lane; i < 16 * m; i += 32) {
                const int row = i & 15, c = i >> 4;
                if (n0 + row < V) logits_dbg[(int64_t)c * V + n0 + row] = tile[row][c];
            }
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(w.flag, 1);
    if (finish_cta(w)) merge_and_decide(w, units, m, thr, token, conf, fire, nonfinite);
}

__global__ void __launch_bounds__(kThreads)
k_exit_head_f32(const float* __restrict__ X, int m, int64_t K, const float* __restrict__ W, int V,
                float thr, int32_t* token, float* conf, uint8_t* fire, int32_t* nonfinite,
                float* logits_dbg, void* ws) {
    constexpr int RW = 8, RX = 4;
    __shared__ float tiles[kWarps][RW][kMaxCols];
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
            float mx, sum;
            int idx;
            unit_partial<RW>(tile, lane, n0, V, mx, sum, idx, bad);
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
    if (finish_cta(w)) merge_and_decide(w, units, m, thr, token, conf, fire, nonfinite);
}

}  // namespace

// Workspace: 256 B of counters + (max, sum, idx) per (unit, column).  Sized
// for the fp32 unit (8 rows), which is the larger count.  Zero once at
// allocation; every call leaves the counters zeroed.
size_t exit_head_ws_bytes(int64_t /*m*/, int64_t V) {
    const int64_t units = (V + 7) / 8;
    return 256 + (size_t)units * kMaxCols * 12;
}

extern "C" int ee_exit_head_infer(const void* xn, int64_t m, int64_t h, const void* W, int64_t V,
                                  int dtype, float threshold, int32_t* token, float* conf,
                                  uint8_t* fire, int32_t* nonfinite, float* logits_dbg, void* ws,
                                  size_t ws_bytes, void* stream) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && m <= kMaxCols, EE_ESHAPE, "exit_head: 1 <= m <= %d rows per call (m=%lld)",
               kMaxCols, (long long)m);
    EE_REQUIRE(h > 0 && V > 0 && V < (1ll << 30), EE_ESHAPE, "exit_head: bad shape");
    EE_REQUIRE(threshold > 0.f && threshold <= 1.f, EE_ECONFIG, "threshold must lie in (0, 1]");
    EE_REQUIRE(ws != nullptr && ws_bytes >= exit_head_ws_bytes(m, V), EE_ESHAPE,
               "exit_head: workspace too small");
    cudaStream_t s = as_stream(stream);
    int sms = ee_device_sms();
    if (sms <= 0) sms = 148;
    if (dtype == EE_BF16) {
        EE_REQUIRE(h % 8 == 0, EE_ESHAPE, "exit_head bf16 needs h %% 8 == 0");
        const int64_t units = (V + 15) / 16;
        const unsigned grid = (unsigned)std::min<int64_t>((units + kWarps - 1) / kWarps, (int64_t)sms * 4);
        if (m <= 8)
            k_exit_head_bf16<1><<<grid, kThreads, 0, s>>>((const bf16*)xn, (int)m, h, (const bf16*)W,
                                                          (int)V, threshold, token, conf, fire,
                                                          nonfinite, logits_dbg, ws);
        else
            k_exit_head_bf16<2><<<grid, kThreads, 0, s>>>((const bf16*)xn, (int)m, h, (const bf16*)W,
                                                          (int)V, threshold, token, conf, fire,
                                                          nonfinite, logits_dbg, ws);
    } else if (dtype == EE_F32) {
        const int64_t units = (V + 7) / 8;
        const unsigned grid = (unsigned)std::min<int64_t>((units + kWarps - 1) / kWarps, (int64_t)sms * 4);
        k_exit_head_f32<<<grid, kThreads, 0, s>>>((const float*)xn, (int)m, h, (const float*)W,
                                                  (int)V, threshold, token, conf, fire, nonfinite,
                                                  logits_dbg, ws);
    } else {
        return ee_fail(EE_ECONFIG, "exit_head: unknown dtype %d", dtype);
    }
    return ee_check_launch("exit_head_infer");
}
