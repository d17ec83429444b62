// Multi-row causal decode attention over the KV cache of one layer.
//
// Row r (position p) attends over cache positions 0..p; heads split the
// hidden axis as reshape(nh, dh) (eepipe/inference.py:207, 225), scale
// 1/sqrt(dh) (eepipe/inference.py:203).
//
// Decode attention is latency-bound (a few MB of K/V per layer spread over
// heads): what matters is the number of DEPENDENT steps between the QKV GEMV
// finishing and the Wo GEMV starting.  Organisation:
//   * one CTA (8 warps) per (head, row, 256-position chunk); warp w owns the
//     32-position block 8 c + w, lane j its position: q.K in registers,
//     warp max / sum-exp by shuffles, P.V with each lane owning dh/32 output
//     dimensions (coalesced V rows);
//   * blocks and chunks are keyed by POSITION ONLY, and every merge runs in a
//     fixed order (warps of a chunk in block order through shared memory,
//     chunks in chunk order), so a row's result does not depend on how many
//     rows share the launch (row-stable) and is deterministic;
//   * rows up to position 255 need no cross-CTA step at all; longer rows
//     publish one partial per chunk and the last CTA of the (row, head)
//     merges them;
//   * K/V rows that predate this pass (positions below every row of the
//     launch) are prefetched into L2 BEFORE griddepcontrol.wait, overlapping
//     the QKV GEMV that is still writing the new rows.
#include "ee_common.cuh"

namespace {

constexpr int kBlk = 32;                      // positions per warp block
constexpr int kWarpsA = 8;                    // blocks per chunk
constexpr int kChunk = kBlk * kWarpsA;        // 256 positions per CTA
constexpr int kThreadsA = kWarpsA * 32;
constexpr int kMaxDh = 128;
constexpr int kRowsPerLaunch = 64;
constexpr int kMaxChunks = 8;                 // s_max <= 2048

template <typename T> __device__ __forceinline__ void load4(const T* p, float* v);
template <> __device__ __forceinline__ void load4<bf16>(const bf16* p, float* v) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
template <> __device__ __forceinline__ void load4<float>(const float* p, float* v) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <typename T, bool DH128>
__global__ void __launch_bounds__(kThreadsA)
k_attn_decode(const float* __restrict__ q, const int32_t* __restrict__ pos, int m,
              const T* __restrict__ kc, const T* __restrict__ vc, int nh, int dh, float scale,
              T* __restrict__ out, float* __restrict__ part, int* __restrict__ ctr) {
    __shared__ float s_q[kMaxDh];
    __shared__ float s_m[kWarpsA], s_l[kWarpsA];
    __shared__ float s_acc[kWarpsA][kMaxDh];
    __shared__ int s_last;

    pdl_trigger_dev();
    const int hh = blockIdx.x, r = blockIdx.y, ch = blockIdx.z;
    const int h = nh * dh;
    const int p = pos[r];  // host-written control data: safe before the wait
    const int nch = p / kChunk + 1;
    if (ch >= nch) {
        pdl_wait_dev();
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = ch * kChunk + warp * kBlk;          // this warp's block
    const int jj = j0 + lane;                          // this lane's position
    const bool valid = jj <= p;
    const bool wvalid = j0 <= p;
    const T* krow = kc + (int64_t)jj * h + hh * dh;
    const T* vrow = vc + (int64_t)jj * h + hh * dh;
    {
        int pmin = p;
        for (int i = 0; i < m; ++i) pmin = min(pmin, pos[i]);
        if (valid && jj < pmin) {  // written by an earlier pass: fetch while QKV runs
            const int bytes = dh * (int)sizeof(T);
            for (int o = 0; o < bytes; o += 128) {
                prefetch_l2((const char*)krow + o);
                prefetch_l2((const char*)vrow + o);
            }
        }
    }
    pdl_wait_dev();
    for (int d = threadIdx.x; d < dh; d += kThreadsA) s_q[d] = q[(int64_t)r * h + hh * dh + d];
    __syncthreads();

    float mx = -INFINITY, l = 0.f;
    float acc[kMaxDh / 32][4];
    if (wvalid) {
        // score of this lane's position: fixed-order dot product.  DH = 128
        // (the configs' head dim) issues the whole K row and this lane's V
        // columns of the block before using any of them: one memory round
        // trip per warp
        float sc = 0.f;
        const int nj = min(kBlk, p + 1 - j0);
        const T* vb = vc + (int64_t)j0 * h + hh * dh;
#pragma unroll
        for (int g = 0; g < kMaxDh / 128; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
        if constexpr (DH128) {
            // bf16 only: the raw K row (16 x 16 B) and this lane's 4 V columns
            // of the block's 32 positions (32 x 8 B) stay packed in registers
            uint4 kraw[16];
            uint2 vraw[kBlk];
            if (valid) {
#pragma unroll
                for (int i = 0; i < 16; ++i) kraw[i] = reinterpret_cast<const uint4*>(krow)[i];
            }
#pragma unroll
            for (int j = 0; j < kBlk; ++j)
                if (j < nj) vraw[j] = *reinterpret_cast<const uint2*>(vb + (int64_t)j * h + 4 * lane);
            if (valid) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint32_t w4[4] = {kraw[i].x, kraw[i].y, kraw[i].z, kraw[i].w};
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const float2 f =
                            __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e2]));
                        sc = fmaf(s_q[8 * i + 2 * e2], f.x, sc);
                        sc = fmaf(s_q[8 * i + 2 * e2 + 1], f.y, sc);
                    }
                }
            }
            const float sv = valid ? sc * scale : -INFINITY;
            mx = sv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float e = valid ? expf(sv - mx) : 0.f;
            l = e;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
            for (int j = 0; j < kBlk; ++j) {
                const float pj = __shfl_sync(0xffffffffu, e, j);
                if (j < nj) {
                    const float2 a =
                        __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vraw[j].x));
                    const float2 b =
                        __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vraw[j].y));
                    acc[0][0] = fmaf(pj, a.x, acc[0][0]);
                    acc[0][1] = fmaf(pj, a.y, acc[0][1]);
                    acc[0][2] = fmaf(pj, b.x, acc[0][2]);
                    acc[0][3] = fmaf(pj, b.y, acc[0][3]);
                }
            }
        } else {
            if (valid) {
                for (int d = 0; d < dh; d += 4) {
                    float kv[4];
                    load4<T>(krow + d, kv);
                    sc = fmaf(s_q[d], kv[0], sc);
                    sc = fmaf(s_q[d + 1], kv[1], sc);
                    sc = fmaf(s_q[d + 2], kv[2], sc);
                    sc = fmaf(s_q[d + 3], kv[3], sc);
                }
            }
            const float sv = valid ? sc * scale : -INFINITY;
            mx = sv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float e = valid ? expf(sv - mx) : 0.f;
            l = e;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
            // P.V: lane owns output dims [4 lane, 4 lane + 4)
            for (int j = 0; j < nj; ++j) {
                const float pj = __shfl_sync(0xffffffffu, e, j);
                if (4 * lane < dh) {
                    float v4[4];
                    load4<T>(vb + (int64_t)j * h + 4 * lane, v4);
                    acc[0][0] = fmaf(pj, v4[0], acc[0][0]);
                    acc[0][1] = fmaf(pj, v4[1], acc[0][1]);
                    acc[0][2] = fmaf(pj, v4[2], acc[0][2]);
                    acc[0][3] = fmaf(pj, v4[3], acc[0][3]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < kMaxDh / 128; ++g) {
            const int d0 = 4 * (lane + 32 * g);
            if (d0 < dh) {
                s_acc[warp][d0] = acc[g][0];
                s_acc[warp][d0 + 1] = acc[g][1];
                s_acc[warp][d0 + 2] = acc[g][2];
                s_acc[warp][d0 + 3] = acc[g][3];
            }
        }
    }
    if (lane == 0) {
        s_m[warp] = mx;
        s_l[warp] = l;
    }
    __syncthreads();
    // merge the chunk's blocks in block order
    const int nb = min(kWarpsA, (p - ch * kChunk) / kBlk + 1);
    float M = -INFINITY;
    for (int w = 0; w < nb; ++w) M = fmaxf(M, s_m[w]);
    float L = 0.f;
    for (int w = 0; w < nb; ++w) L += s_l[w] * expf(s_m[w] - M);
    const int64_t slot = ((int64_t)r * nh + hh) * kMaxChunks + ch;
    const int stride = dh + 2;
    for (int d = threadIdx.x; d < dh; d += kThreadsA) {
        float o = 0.f;
        for (int w = 0; w < nb; ++w) o += s_acc[w][d] * expf(s_m[w] - M);
        if (nch == 1) out[(int64_t)r * h + hh * dh + d] = from_f32<T>(o / L);
        else part[slot * stride + 2 + d] = o;
    }
    if (nch == 1) return;
    if (threadIdx.x == 0) {
        part[slot * stride] = M;
        part[slot * stride + 1] = L;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&ctr[r * nh + hh], 1) == nch - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // fixed-order merge over chunks 0..nch-1
    const float* base = part + ((int64_t)r * nh + hh) * kMaxChunks * stride;
    float MM = -INFINITY;
    for (int c = 0; c < nch; ++c) MM = fmaxf(MM, __ldcg(base + c * stride));
    float LL = 0.f;
    for (int c = 0; c < nch; ++c) LL += __ldcg(base + c * stride + 1) * expf(__ldcg(base + c * stride) - MM);
    for (int d = threadIdx.x; d < dh; d += kThreadsA) {
        float o = 0.f;
        for (int c = 0; c < nch; ++c)
            o += __ldcg(base + c * stride + 2 + d) * expf(__ldcg(base + c * stride) - MM);
        out[(int64_t)r * h + hh * dh + d] = from_f32<T>(o / LL);
    }
    if (threadIdx.x == 0) ctr[r * nh + hh] = 0;  // leave the workspace re-usable
}

size_t counters_bytes(int64_t nh) { return (((size_t)kRowsPerLaunch * nh * 4) + 255) & ~(size_t)255; }

}  // namespace

// Workspace: [counters: 64*nh int32][partials: 64*nh*kMaxChunks*(dh+2) float32].
// Zero once at allocation; every call leaves the counters zeroed.
size_t attention_ws_bytes(int64_t /*m*/, int64_t nh, int64_t dh, int64_t /*s_max*/) {
    return counters_bytes(nh) + (size_t)kRowsPerLaunch * nh * kMaxChunks * (dh + 2) * sizeof(float);
}

int launch_attention(const float* q, int64_t m, const int32_t* pos, int32_t max_pos,
                     const void* kc, const void* vc, int64_t nh, int64_t dh, int dtype, void* out,
                     void* ws, size_t ws_bytes, cudaStream_t s) {
    if (m == 0) return EE_OK;
    dtype = act_dtype(dtype);
    EE_REQUIRE(m > 0 && nh > 0 && dh > 0 && max_pos >= 0, EE_ESHAPE, "attention: bad shape");
    EE_REQUIRE(dh <= kMaxDh && dh % 4 == 0, EE_ESHAPE,
               "attention: head_dim must be <= %d and a multiple of 4, got %lld", kMaxDh,
               (long long)dh);
    EE_REQUIRE(max_pos < kMaxChunks * kChunk, EE_ESHAPE, "attention: position %d beyond %d",
               max_pos, kMaxChunks * kChunk);
    EE_REQUIRE(ws != nullptr && ws_bytes >= attention_ws_bytes(m, nh, dh, 0), EE_ESHAPE,
               "attention: workspace too small");
    int* ctr = (int*)ws;
    float* part = (float*)((char*)ws + counters_bytes(nh));
    const float scale = 1.0f / sqrtf((float)dh);
    const int64_t h = nh * dh;
    const int nch = max_pos / kChunk + 1;
    for (int64_t r0 = 0; r0 < m; r0 += kRowsPerLaunch) {
        const int64_t mr = m - r0 < kRowsPerLaunch ? m - r0 : kRowsPerLaunch;
        const dim3 grid((unsigned)nh, (unsigned)mr, (unsigned)nch);
        cudaError_t e;
        if (dtype == EE_BF16)
            e = launch_ex(dh == 128 ? k_attn_decode<bf16, true> : k_attn_decode<bf16, false>, grid, dim3(kThreadsA), 0, s, q + r0 * h, pos + r0,
                          (int)mr, (const bf16*)kc, (const bf16*)vc, (int)nh, (int)dh, scale,
                          (bf16*)out + r0 * h, part, ctr);
        else if (dtype == EE_F32)
            e = launch_ex(k_attn_decode<float, false>, grid, dim3(kThreadsA), 0, s, q + r0 * h, pos + r0,
                          (int)mr, (const float*)kc, (const float*)vc, (int)nh, (int)dh, scale,
                          (float*)out + r0 * h, part, ctr);
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
