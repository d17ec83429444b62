// Multi-row causal decode attention over the KV cache of one layer.
//
// Row r (position p) attends over cache positions 0..p; heads split the
// hidden axis as reshape(nh, dh) (eepipe/inference.py:207, 225), scale
// 1/sqrt(dh).  Work is split into KV chunks of kChunk positions keyed by
// POSITION ONLY (chunk c covers [64c, 64c+64) ∩ [0, p]), one CTA per
// (head, row, chunk).  Each CTA writes (max, sum-exp, acc[dh]); the last CTA
// of a (row, head) to finish merges the chunks in ascending order.  Nothing
// depends on how many rows share the launch, so the result is row-stable.
//
// Bytes: K and V rows of the prefix are read once per (row, head); for the
// rows of one recompute pass the shared prefix is L2-resident after the first
// row touches it.
#include "ee_common.cuh"

namespace {

constexpr int kChunk = 64;
constexpr int kThreads = 128;
constexpr int kRowsPerLaunch = 64;

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
    extern __shared__ float sm[];
    float* qs = sm;           // [dh]
    float* sc = sm + dh;      // [kChunk]
    __shared__ float s_m, s_l;
    __shared__ int s_last;

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
    for (int jj = warp; jj < nj; jj += kThreads / 32) {
        const T* kr = kc + (int64_t)(j0 + jj) * h + hh * dh;
        float s = 0.f;
        for (int d = lane; d < dh; d += 32) s = fmaf(qs[d], to_f32(kr[d]), s);
        s = warp_sum(s);
        if (lane == 0) sc[jj] = s * scale;
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

    const int64_t slot = ((int64_t)r * nh + hh) * chunks_cap;
    const int stride = dh + 2;
    for (int d = tid; d < dh; d += kThreads) {
        const T* vcol = vc + (int64_t)j0 * h + hh * dh + d;
        float a = 0.f;
        for (int jj = 0; jj < nj; ++jj) a = fmaf(sc[jj], to_f32(vcol[(int64_t)jj * h]), a);
        if (nchunks == 1) {
            out[(int64_t)r * h + hh * dh + d] = from_f32<T>(a / s_l);
        } else {
            part[(slot + c) * stride + 2 + d] = a;
        }
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
    const int chunks = max_pos / kChunk + 1;
    const size_t cbytes = counters_bytes(nh);
    EE_REQUIRE(ws != nullptr && ws_bytes >= cbytes, EE_ESHAPE, "attention: workspace too small");
    const int64_t chunks_cap =
        (int64_t)((ws_bytes - cbytes) / ((size_t)kRowsPerLaunch * nh * (dh + 2) * sizeof(float)));
    EE_REQUIRE(chunks_cap >= chunks, EE_ESHAPE,
               "attention: workspace holds %lld chunks, need %d (max_pos %d)",
               (long long)chunks_cap, chunks, max_pos);
    int* ctr = (int*)ws;
    float* part = (float*)((char*)ws + cbytes);
    const float scale = 1.0f / sqrtf((float)dh);
    const size_t shm = (size_t)(dh + kChunk) * sizeof(float);
    const int64_t h = nh * dh;
    for (int64_t r0 = 0; r0 < m; r0 += kRowsPerLaunch) {
        const int64_t mr = m - r0 < kRowsPerLaunch ? m - r0 : kRowsPerLaunch;
        const dim3 grid((unsigned)nh, (unsigned)mr, (unsigned)chunks);
        if (dtype == EE_BF16)
            k_attn_decode<bf16><<<grid, kThreads, shm, s>>>(
                q + r0 * h, pos + r0, (const bf16*)kc, (const bf16*)vc, (int)nh, (int)dh, scale,
                (bf16*)out + r0 * h, part, ctr, (int)chunks_cap);
        else if (dtype == EE_F32)
            k_attn_decode<float><<<grid, kThreads, shm, s>>>(
                q + r0 * h, pos + r0, (const float*)kc, (const float*)vc, (int)nh, (int)dh, scale,
                (float*)out + r0 * h, part, ctr, (int)chunks_cap);
        else
            return ee_fail(EE_ECONFIG, "attention: unknown dtype %d", dtype);
        int rc = ee_check_launch("decode_attention");
        if (rc) return rc;
    }
    return EE_OK;
}

extern "C" int ee_decode_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                                   const void* kcache, const void* vcache, int64_t nh, int64_t dh,
                                   int dtype, void* out, void* ws, size_t ws_bytes, void* stream) {
    return launch_attention(q, m, pos, max_pos, kcache, vcache, nh, dh, dtype, out, ws, ws_bytes,
                            as_stream(stream));
}
