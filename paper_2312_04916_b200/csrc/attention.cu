// Multi-row causal decode attention over the KV cache of one layer.
//
// Row r (position p) attends over cache positions 0..p; heads split the
// hidden axis as reshape(nh, dh) (eepipe/inference.py:207, 225), scale
// 1/sqrt(dh).  Work is split into KV chunks of kChunk positions keyed by
// POSITION ONLY (chunk c covers [64c, 64c+64) ∩ [0, p]), one CTA per
// (head, row, chunk), 4 warps:
//   scores: warp w takes positions j ≡ w (mod 4); each lane owns 4
//           consecutive head dims (one 8-B bf16 / 16-B fp32 load per
//           position), fixed xor-butterfly per score;
//   P·V:    warp w accumulates the same positions, lane owns 4 dims;
//           the 4 warp partials are summed in warp order.
// Each CTA writes (max, sum-exp, acc[dh]); the last CTA of a (row, head)
// merges the chunks in ascending order.  Nothing depends on how many rows
// share the launch, so the result is row-stable.
#include "ee_common.cuh"

namespace {

constexpr int kChunk = 64;
constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerLaunch = 64;
constexpr int kMaxDh = 256;

__device__ __forceinline__ void load4(const float* p, float v[4]) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x;
    v[1] = u.y;
    v[2] = u.z;
    v[3] = u.w;
}
__device__ __forceinline__ void load4(const bf16* p, float v[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    v[0] = fa.x;
    v[1] = fa.y;
    v[2] = fb.x;
    v[3] = fb.y;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_attn_decode(const float* __restrict__ q, const int32_t* __restrict__ pos,
              const T* __restrict__ kc, const T* __restrict__ vc, int nh, int dh, float scale,
              T* __restrict__ out, float* __restrict__ part, int* __restrict__ ctr,
              int chunks_cap) {
    __shared__ __align__(16) float qs[kMaxDh];
    __shared__ float sc[kChunk];
    __shared__ __align__(16) float red[kWarps][kMaxDh];
    __shared__ float s_m, s_l;
    __shared__ int s_last;

    pdl_trigger_dev();
    pdl_wait_dev();
    const int hh = blockIdx.x, r = blockIdx.y, c = blockIdx.z;
    const int h = nh * dh;
    const int p = pos[r];
    const int nchunks = p / kChunk + 1;
    if (c >= nchunks) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int d = tid; d < dh; d += kThreads) qs[d] = q[(int64_t)r * h + hh * dh + d];
    __syncthreads();

    const int j0 = c * kChunk;
    const int nj = min(kChunk, p + 1 - j0);
    const T* kbase = kc + (int64_t)j0 * h + hh * dh;
    const T* vbase = vc + (int64_t)j0 * h + hh * dh;

    // scores: warp w owns positions w, w+4, ... (16 per warp for a full chunk);
    // all K loads of a group of 8 positions are issued before any reduction
    // so the warp has 8 independent requests in flight.
    for (int j8 = warp; j8 < nj; j8 += 8 * kWarps) {
        float s[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = 0.f;
        for (int d = lane * 4; d < dh; d += 128) {
            float kv[8][4];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int jj = j8 + u * kWarps;
                if (jj < nj) load4(kbase + (int64_t)jj * h + d, kv[u]);
                else kv[u][0] = kv[u][1] = kv[u][2] = kv[u][3] = 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s[u] = fmaf(qs[d], kv[u][0], s[u]);
                s[u] = fmaf(qs[d + 1], kv[u][1], s[u]);
                s[u] = fmaf(qs[d + 2], kv[u][2], s[u]);
                s[u] = fmaf(qs[d + 3], kv[u][3], s[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float v = warp_sum(s[u]);
            const int jj = j8 + u * kWarps;
            if (lane == 0 && jj < nj) sc[jj] = v * scale;
        }
    }
    __syncthreads();
    if (warp == 0) {
        float mx = -INFINITY;
        for (int jj = lane; jj < nj; jj += 32) mx = fmaxf(mx, sc[jj]);
        mx = warp_max(mx);
        float l = 0.f;
        for (int jj = lane; jj < nj; jj += 32) {
            const float e = expf(sc[jj] - mx);
            sc[jj] = e;
            l += e;
        }
        l = warp_sum(l);
        if (lane == 0) {
            s_m = mx;
            s_l = l;
        }
    }
    __syncthreads();

    // P·V: warp w over positions j ≡ w (mod 4), lane owns dims [4*lane + 128*i, +4)
    for (int d = lane * 4; d < dh; d += 128) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        for (int j8 = warp; j8 < nj; j8 += 8 * kWarps) {
            float vv[8][4];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int jj = j8 + u * kWarps;
                if (jj < nj) load4(vbase + (int64_t)jj * h + d, vv[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int jj = j8 + u * kWarps;
                if (jj < nj) {
                    const float pj = sc[jj];
                    a0 = fmaf(pj, vv[u][0], a0);
                    a1 = fmaf(pj, vv[u][1], a1);
                    a2 = fmaf(pj, vv[u][2], a2);
                    a3 = fmaf(pj, vv[u][3], a3);
                }
            }
        }
        red[warp][d] = a0;
        red[warp][d + 1] = a1;
        red[warp][d + 2] = a2;
        red[warp][d + 3] = a3;
    }
    __syncthreads();

    const int64_t slot = ((int64_t)r * nh + hh) * chunks_cap;
    const int stride = dh + 2;
    for (int d = tid; d < dh; d += kThreads) {
        const float a = ((red[0][d] + red[1][d]) + red[2][d]) + red[3][d];
        if (nchunks == 1)
            out[(int64_t)r * h + hh * dh + d] = from_f32<T>(a / s_l);
        else
            part[(slot + c) * stride + 2 + d] = a;
    }
    if (nchunks == 1) return;
    if (tid == 0) {
        part[(slot + c) * stride] = s_m;
        part[(slot + c) * stride + 1] = s_l;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ctr[r * nh + hh], 1) == nchunks - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // Fixed-order merge over chunks 0..nchunks-1.
    float M = -INFINITY;
    for (int cc = 0; cc < nchunks; ++cc) M = fmaxf(M, __ldcg(part + (slot + cc) * stride));
    float L = 0.f;
    for (int cc = 0; cc < nchunks; ++cc)
        L += __ldcg(part + (slot + cc) * stride + 1) * expf(__ldcg(part + (slot + cc) * stride) - M);
    for (int d = tid; d < dh; d += kThreads) {
        float o = 0.f;
        for (int cc = 0; cc < nchunks; ++cc)
            o += __ldcg(part + (slot + cc) * stride + 2 + d) *
                 expf(__ldcg(part + (slot + cc) * stride) - M);
        out[(int64_t)r * h + hh * dh + d] = from_f32<T>(o / L);
    }
    if (tid == 0) ctr[r * nh + hh] = 0;  // leave the workspace re-usable
}

size_t counters_bytes(int64_t nh) { return (((size_t)kRowsPerLaunch * nh * 4) + 255) & ~(size_t)255; }

}  // namespace

// Workspace: [counters: 64*nh int32][partials: 64*nh*chunks*(dh+2) float32].
// Must be zero-filled once at allocation; every call leaves it zeroed.
size_t attention_ws_bytes(int64_t /*m*/, int64_t nh, int64_t dh, int64_t s_max) {
    const int64_t chunks = (s_max + kChunk - 1) / kChunk;
    return counters_bytes(nh) + (size_t)kRowsPerLaunch * nh * chunks * (dh + 2) * sizeof(float);
}

int launch_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                     const void* kc, const void* vc, int64_t nh, int64_t dh, int dtype, void* out,
                     void* ws, size_t ws_bytes, cudaStream_t s) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(m > 0 && nh > 0 && dh > 0 && max_pos >= 0, EE_ESHAPE, "attention: bad shape");
    EE_REQUIRE(dh % 4 == 0 && dh <= kMaxDh, EE_ESHAPE,
               "attention: head_dim must be a multiple of 4 and <= %d (got %lld)", kMaxDh,
               (long long)dh);
    const int chunks = max_pos / kChunk + 1;
    const size_t cbytes = counters_bytes(nh);
    EE_REQUIRE(ws != nullptr && ws_bytes >= cbytes, EE_ESHAPE, "attention: workspace too small");
    const int64_t chunks_cap =
        (int64_t)((ws_bytes - cbytes) / ((size_t)kRowsPerLaunch * nh * (dh + 2) * sizeof(float)));
    EE_REQUIRE(chunks_cap >= chunks, EE_ESHAPE,
               "attention: workspace holds %lld chunks, need %d (max_pos %d)",
               (long long)chunks_cap, chunks, max_pos);
    dtype = act_dtype(dtype);
    int* ctr = (int*)ws;
    float* part = (float*)((char*)ws + cbytes);
    const float scale = 1.0f / sqrtf((float)dh);
    const int64_t h = nh * dh;
    for (int64_t r0 = 0; r0 < m; r0 += kRowsPerLaunch) {
        const int64_t mr = m - r0 < kRowsPerLaunch ? m - r0 : kRowsPerLaunch;
        const dim3 grid((unsigned)nh, (unsigned)mr, (unsigned)chunks);
        cudaError_t e;
        if (dtype == EE_BF16)
            e = launch_ex(k_attn_decode<bf16>, grid, dim3(kThreads), 0, s, q + r0 * h, pos + r0,
                          (const bf16*)kc, (const bf16*)vc, (int)nh, (int)dh, scale,
                          (bf16*)out + r0 * h, part, ctr, (int)chunks_cap);
        else if (dtype == EE_F32)
            e = launch_ex(k_attn_decode<float>, grid, dim3(kThreads), 0, s, q + r0 * h, pos + r0,
                          (const float*)kc, (const float*)vc, (int)nh, (int)dh, scale,
                          (float*)out + r0 * h, part, ctr, (int)chunks_cap);
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
