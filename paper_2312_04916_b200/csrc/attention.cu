// Multi-row causal decode attention over the KV cache of one layer.
//
// Row r (position p) attends over cache positions 0..p; heads split the
// hidden axis as reshape(nh, dh) (eepipe/inference.py:207, 225), scale
// 1/sqrt(dh) (eepipe/inference.py:203).
//
// Decode attention is latency-bound (a few MB of K/V per layer spread over
// heads), so the kernel is organised to minimise DEPENDENT memory round
// trips and to overlap with its neighbours under programmatic dependent
// launch:
//   * one CTA (128 threads) per (head, row, 32-position block); the block
//     partition is keyed by POSITION ONLY (block b = [32b, 32b+32) ∩ [0,p]),
//     so the result does not depend on how many rows share the launch
//     (row-stable);
//   * every thread issues all of its K and V loads at once (a quarter of one
//     K row and of one V row each: 4 + 4 16-byte loads);
//   * blocks that lie entirely below the smallest position written by this
//     pass are read BEFORE griddepcontrol.wait — those K/V entries were
//     written by earlier passes, so the loads overlap the QKV GEMV that is
//     still running;
//   * the block partial (max, sum-exp, acc[dh]) goes to a workspace; the
//     last CTA of a (row, head) merges the partials in ascending block order
//     (fixed order, deterministic).
#include "ee_common.cuh"

namespace {

constexpr int kBlk = 32;
constexpr int kThreads = 128;
constexpr int kMaxDh = 128;  // per-thread quarter rows: dh <= 128
constexpr int kRowsPerLaunch = 64;
constexpr int kMaxBlocks = 64;  // s_max <= 2048

template <typename T> struct Q;  // 16-byte vector of T
template <> struct Q<bf16> {
    static constexpr int N = 8;
    __device__ static void cvt(const uint4& u, float* v) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    }
};
template <> struct Q<float> {
    static constexpr int N = 4;
    __device__ static void cvt(const uint4& u, float* v) {
        v[0] = __uint_as_float(u.x);
        v[1] = __uint_as_float(u.y);
        v[2] = __uint_as_float(u.z);
        v[3] = __uint_as_float(u.w);
    }
};

// Per (thread) share of a 32 x dh block: row j = tid / 4, quarter qd = tid % 4
// covering dims [qd*dq, (qd+1)*dq), dq = dh / 4, in 16-byte vectors.
template <typename T>
struct BlockLoad {
    static constexpr int VN = Q<T>::N;
    static constexpr int kMaxVec = kMaxDh / 4 / VN;  // vectors per quarter row
    uint4 k[kMaxVec], v[kMaxVec];
    __device__ void issue(const T* kc, const T* vc, int64_t row_off, int nvec, bool valid) {
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) {
            if (valid && i < nvec) {
                k[i] = *reinterpret_cast<const uint4*>(kc + row_off + i * VN);
                v[i] = *reinterpret_cast<const uint4*>(vc + row_off + i * VN);
            }
        }
    }
};

template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads)
k_attn_decode(const float* __restrict__ q, const int32_t* __restrict__ pos, int m,
              const T* __restrict__ kc, const T* __restrict__ vc, int nh, int dh, float scale,
              T* __restrict__ out, float* __restrict__ part, int* __restrict__ ctr) {
    __shared__ float s_q[kMaxDh];
    __shared__ float s_p[kBlk];
    __shared__ __align__(16) float s_v[kBlk][kMaxDh + 4];
    __shared__ float s_stat[2];
    __shared__ int s_last;
    constexpr int VN = Q<T>::N;

    pdl_trigger_dev();
    const int hh = blockIdx.x, r = blockIdx.y, b = blockIdx.z;
    const int h = nh * dh;
    const int p = pos[r];  // host-written control data: safe before the wait
    const int nblk = p / kBlk + 1;
    if (b >= nblk) {
        pdl_wait_dev();
        return;
    }
    int pmin = p;
    for (int i = 0; i < m; ++i) pmin = min(pmin, pos[i]);
    const int tid = threadIdx.x;
    const int j = tid >> 2, qd = tid & 3;
    const int dq = dh >> 2;
    const int nvec = dq / VN;
    const int j0 = b * kBlk;
    const int nj = min(kBlk, p + 1 - j0);
    const bool valid = j < nj;
    const int64_t row_off = (int64_t)(j0 + j) * h + hh * dh + qd * dq;

    BlockLoad<T> ld;
    const bool old = (j0 + kBlk) <= pmin;  // every position of the block predates this pass
    if (VEC && old) ld.issue(kc, vc, row_off, nvec, valid);
    pdl_wait_dev();
    if (VEC && !old) ld.issue(kc, vc, row_off, nvec, valid);

    for (int d = tid; d < dh; d += kThreads) s_q[d] = q[(int64_t)r * h + hh * dh + d];
    __syncthreads();

    // score of position j0 + j: 4 threads x (dh/4) dims, fixed-order combine
    float sc = 0.f;
    if (VEC) {
#pragma unroll
        for (int i = 0; i < BlockLoad<T>::kMaxVec; ++i) {
            if (i < nvec) {
                float kv[VN];
                Q<T>::cvt(ld.k[i], kv);
#pragma unroll
                for (int e = 0; e < VN; ++e) sc = fmaf(s_q[qd * dq + i * VN + e], kv[e], sc);
            }
        }
    } else if (valid) {
        for (int e = 0; e < dq; ++e) sc = fmaf(s_q[qd * dq + e], to_f32(kc[row_off + e]), sc);
    }
    sc += __shfl_xor_sync(0xffffffffu, sc, 1);
    sc += __shfl_xor_sync(0xffffffffu, sc, 2);
    // V rows to shared memory for the position-ordered reduction
    if (VEC) {
#pragma unroll
        for (int i = 0; i < BlockLoad<T>::kMaxVec; ++i) {
            if (i < nvec) {
                float vv[VN];
                Q<T>::cvt(ld.v[i], vv);
#pragma unroll
                for (int e = 0; e < VN; ++e) s_v[j][qd * dq + i * VN + e] = valid ? vv[e] : 0.f;
            }
        }
    } else {
        for (int e = 0; e < dq; ++e) s_v[j][qd * dq + e] = valid ? to_f32(vc[row_off + e]) : 0.f;
    }
    if (qd == 0) s_p[j] = valid ? sc * scale : -INFINITY;
    __syncthreads();
    if (tid < 32) {
        float s = s_p[tid];
        float mx = s;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e = tid < nj ? expf(s - mx) : 0.f;
        float l = e;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        s_p[tid] = e;
        if (tid == 0) {
            s_stat[0] = mx;
            s_stat[1] = l;
        }
    }
    __syncthreads();
    const int64_t slot = ((int64_t)r * nh + hh) * kMaxBlocks + b;
    const int stride = dh + 2;
    for (int d = tid; d < dh; d += kThreads) {
        float a = 0.f;
        for (int jj = 0; jj < nj; ++jj) a = fmaf(s_p[jj], s_v[jj][d], a);
        if (nblk == 1)
            out[(int64_t)r * h + hh * dh + d] = from_f32<T>(a / s_stat[1]);
        else
            part[slot * stride + 2 + d] = a;
    }
    if (nblk == 1) return;
    if (tid == 0) {
        part[slot * stride] = s_stat[0];
        part[slot * stride + 1] = s_stat[1];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ctr[r * nh + hh], 1) == nblk - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // fixed-order merge over blocks 0..nblk-1
    const float* base = part + ((int64_t)r * nh + hh) * kMaxBlocks * stride;
    float M = -INFINITY;
    for (int bb = 0; bb < nblk; ++bb) M = fmaxf(M, __ldcg(base + bb * stride));
    float L = 0.f;
    for (int bb = 0; bb < nblk; ++bb) L += __ldcg(base + bb * stride + 1) * expf(__ldcg(base + bb * stride) - M);
    for (int d = tid; d < dh; d += kThreads) {
        float o = 0.f;
        for (int bb = 0; bb < nblk; ++bb)
            o += __ldcg(base + bb * stride + 2 + d) * expf(__ldcg(base + bb * stride) - M);
        out[(int64_t)r * h + hh * dh + d] = from_f32<T>(o / L);
    }
    if (tid == 0) ctr[r * nh + hh] = 0;  // leave the workspace re-usable
}

size_t counters_bytes(int64_t nh) { return (((size_t)kRowsPerLaunch * nh * 4) + 255) & ~(size_t)255; }

}  // namespace

// Workspace: [counters: 64*nh int32][partials: 64*nh*64*(dh+2) float32].
// Zero once at allocation; every call leaves the counters zeroed.
size_t attention_ws_bytes(int64_t /*m*/, int64_t nh, int64_t dh, int64_t /*s_max*/) {
    return counters_bytes(nh) + (size_t)kRowsPerLaunch * nh * kMaxBlocks * (dh + 2) * sizeof(float);
}

int launch_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                     const void* kc, const void* vc, int64_t nh, int64_t dh, int dtype, void* out,
                     void* ws, size_t ws_bytes, cudaStream_t s) {
    if (m == 0) return EE_OK;
    dtype = act_dtype(dtype);
    const int vn = dtype == EE_BF16 ? 8 : 4;
    EE_REQUIRE(m > 0 && nh > 0 && dh > 0 && max_pos >= 0, EE_ESHAPE, "attention: bad shape");
    EE_REQUIRE(dh <= kMaxDh && dh % 4 == 0, EE_ESHAPE,
               "attention: head_dim must be <= %d and a multiple of 4, got %lld", kMaxDh,
               (long long)dh);
    const bool vec = dh % (4 * vn) == 0;
    EE_REQUIRE(max_pos < kMaxBlocks * kBlk, EE_ESHAPE, "attention: position %d beyond %d",
               max_pos, kMaxBlocks * kBlk);
    EE_REQUIRE(ws != nullptr && ws_bytes >= attention_ws_bytes(m, nh, dh, 0), EE_ESHAPE,
               "attention: workspace too small");
    int* ctr = (int*)ws;
    float* part = (float*)((char*)ws + counters_bytes(nh));
    const float scale = 1.0f / sqrtf((float)dh);
    const int64_t h = nh * dh;
    const int nblk = max_pos / kBlk + 1;
    for (int64_t r0 = 0; r0 < m; r0 += kRowsPerLaunch) {
        const int64_t mr = m - r0 < kRowsPerLaunch ? m - r0 : kRowsPerLaunch;
        const dim3 grid((unsigned)nh, (unsigned)mr, (unsigned)nblk);
        cudaError_t e;
        if (dtype == EE_BF16)
            e = launch_ex(vec ? k_attn_decode<bf16, true> : k_attn_decode<bf16, false>, grid,
                          dim3(kThreads), 0, s, q + r0 * h, pos + r0, (int)mr, (const bf16*)kc,
                          (const bf16*)vc, (int)nh, (int)dh, scale, (bf16*)out + r0 * h, part, ctr);
        else if (dtype == EE_F32)
            e = launch_ex(vec ? k_attn_decode<float, true> : k_attn_decode<float, false>, grid,
                          dim3(kThreads), 0, s, q + r0 * h, pos + r0, (int)mr, (const float*)kc,
                          (const float*)vc, (int)nh, (int)dh, scale, (float*)out + r0 * h, part,
                          ctr);
        else
            return ee_fail(EE_ECONFIG, "attention: unknown dtype %d", dtype);
        if (e != cudaSuccess) return ee_fail(EE_ECUDA, "attention launch: %s", cudaGetErrorString(e));
    }
    return EE_OK;
}

extern "C" int ee_decode_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                                   const void* kcache, const void* vcache, int64_t nh, int64_t dh,
                                   int dtype, void* out, void* ws, size_t ws_bytes, void* stream) {
    return launch_attention(q, m, pos, max_pos, kcache, vcache, nh, dh, dtype, out, ws, ws_bytes,
                            as_stream(stream));
}
