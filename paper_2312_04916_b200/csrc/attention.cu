// Multi-row causal decode attention over the KV cache of one layer.
//
// Row r (position p) attends over cache positions 0..p; heads split the
// hidden axis as reshape(nh, dh) (eepipe/inference.py:207, 225), scale
// 1/sqrt(dh) (eepipe/inference.py:203).
//
// Decode attention is latency-bound (a few MB of K/V per layer spread over
// heads): what matters is the number of DEPENDENT steps between the QKV GEMV
// finishing and the Wo GEMV starting.  Organisation:
//   * one CTA (8 warps) per (head, row, 256-position chunk) -- for bf16 with
//     head_dim 128 per (head, group of <= 16 rows, chunk), the rows sharing
//     each K/V load (k_attn_rows128: K tile cp.async'd into shared memory
//     with an XOR swizzle, V columns in registers); warp w owns the block
//     8 c + w, lane j its position: q.K in registers, warp max / sum-exp by
//     shuffles, P.V with each lane owning dh/32 output dimensions (coalesced
//     V rows);
//   * blocks and chunks are keyed by POSITION ONLY, and every merge runs in a
//     fixed order (warps of a chunk in block order through shared memory,
//     chunks in chunk order), so a row's result does not depend on how many
//     rows share the launch (row-stable) and is deterministic;
//   * rows up to position 255 need no cross-CTA step at all; longer rows
//     publish one partial per chunk and the last CTA of the (row, head)
//     merges them;
//   * nothing but the host-written positions is touched before
//     griddepcontrol.wait.  (An L2 prefetch of the K/V rows that predate the
//     pass, issued before the wait to overlap the QKV GEMV, made multi-chunk
//     rows (positions >= 256) nondeterministic run to run on B200: removed.)
#include "attn_core.cuh"

namespace {

using attn::kBlk;
using attn::kChunk;
using attn::kMaxChunks;
using attn::kMaxDh;
using attn::kRowsPerLaunch;
using attn::kWarpsA;
constexpr int kThreadsA = kWarpsA * 32;

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

template <typename T>
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
    pdl_wait_dev();
    for (int d = threadIdx.x; d < dh; d += kThreadsA) s_q[d] = q[(int64_t)r * h + hh * dh + d];
    __syncthreads();

    float mx = -INFINITY, l = 0.f;
    float acc[kMaxDh / 32][4];
    if (wvalid) {
        // score of this lane's position: fixed-order dot product
        float sc = 0.f;
        const int nj = min(kBlk, p + 1 - j0);
        const T* vb = vc + (int64_t)j0 * h + hh * dh;
#pragma unroll
        for (int g = 0; g < kMaxDh / 128; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
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
    for (int w = 0; w < nb; ++w) L = fmaf(s_l[w], expf(s_m[w] - M), L);
    const int64_t slot = ((int64_t)r * nh + hh) * kMaxChunks + ch;
    const int stride = dh + 2;
    for (int d = threadIdx.x; d < dh; d += kThreadsA) {
        float o = 0.f;
        for (int w = 0; w < nb; ++w) o = fmaf(s_acc[w][d], expf(s_m[w] - M), o);
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
    for (int d = threadIdx.x; d < dh; d += kThreadsA)
        out[(int64_t)r * h + hh * dh + d] = from_f32<T>(attn::chunk_merge(base, stride, nch, d));
    if (threadIdx.x == 0) ctr[r * nh + hh] = 0;  // leave the workspace re-usable
}

// bf16, head_dim 128 (the configs' head dim): one CTA per (head, group of up
// to 16 rows, 256-position chunk); the group size is chosen per launch so the
// grid just fills the GPU.  Rows of a pass share the layer's K/V
// prefix, so each warp loads its 32-position block ONCE (block_issue128_k, up
// to the group's last position: K into a swizzled shared-memory tile, V into
// registers) and scores every row of the group from it (block_eval128_k);
// per-row results go through shared memory
// and are merged exactly as in k_attn_decode, so a row's output does not
// depend on which rows share its group.
constexpr int kRowsCta = 16;
constexpr int kRowsKernelMinChunks = 1;  // K staged in smem: faster at every context (m = 1 too)

// dynamic shared memory: K tiles [kWarpsA][kBlk][dh] bf16 (swizzled), q [rows][dh] and
// per-row block results [rows][kWarpsA][dh] float32
__host__ __device__ constexpr size_t rows128_smem(int rows) {
    return (size_t)kWarpsA * kBlk * kMaxDh * 2 + (size_t)rows * (kMaxDh + kWarpsA * kMaxDh) * sizeof(float);
}

__global__ void __launch_bounds__(kThreadsA)
k_attn_rows128(const float* __restrict__ q, const int32_t* __restrict__ pos, int m,
               const bf16* __restrict__ kc, const bf16* __restrict__ vc, int nh, float scale,
               bf16* __restrict__ out, float* __restrict__ part, int* __restrict__ ctr, int g) {
    extern __shared__ __align__(16) float smem_rows[];
    __shared__ float s_m[kRowsCta][kWarpsA], s_l[kRowsCta][kWarpsA];
    __shared__ int s_last[kRowsCta];
    constexpr int dh = kMaxDh;
    pdl_trigger_dev();
    const int hh = blockIdx.x, ch = blockIdx.z;
    const int r0 = blockIdx.y * g;  // this CTA's rows: [r0, r0 + mr), g <= kRowsCta
    const int mr = min(g, m - r0);
    const int h = nh * dh;
    bf16* s_k = reinterpret_cast<bf16*>(smem_rows);                        // [kWarpsA][kBlk][dh]
    float* s_q = smem_rows + kWarpsA * kBlk * dh / 2;                      // [mr][dh]
    float* s_acc = s_q + mr * dh;                                          // [mr][kWarpsA][dh]
    // host-written control data: safe before the wait
    int pmax = -1;
    for (int i = 0; i < mr; ++i) pmax = max(pmax, pos[r0 + i]);
    if (pmax < ch * kChunk) {
        pdl_wait_dev();
        return;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int j0 = ch * kChunk + warp * kBlk;
    pdl_wait_dev();
    // the block's K / V loads go out first, the q rows are staged meanwhile
    attn::BlockRegsV R;
    bf16* sk = s_k + warp * kBlk * dh;  // this warp's K tile
    if (j0 <= pmax) attn::block_issue128_k(R, sk, kc, vc, h, hh * dh, j0, pmax);
    for (int t = tid; t < mr * (dh / 4); t += kThreadsA) {
        const int i = t / (dh / 4), c = t % (dh / 4);
        reinterpret_cast<float4*>(s_q + i * dh)[c] =
            reinterpret_cast<const float4*>(q + (int64_t)(r0 + i) * h + hh * dh)[c];
    }
    __syncthreads();
    if (j0 <= pmax) {
        attn::block_wait128_k();
        for (int i = 0; i < mr; ++i) {
            const int p = pos[r0 + i];
            if (j0 > p) continue;  // warp-uniform
            float mx, l, acc[4];
            attn::block_eval128_k(R, sk, s_q + i * dh, j0, p, scale, mx, l, acc);
            reinterpret_cast<float4*>(s_acc + (i * kWarpsA + warp) * dh)[lane] =
                make_float4(acc[0], acc[1], acc[2], acc[3]);
            if (lane == 0) {
                s_m[i][warp] = mx;
                s_l[i][warp] = l;
            }
        }
    }
    __syncthreads();
    // per (row, dim): the chunk's blocks in block order (k_attn_decode's
    // expressions)
    const int stride = dh + 2;
    for (int t = tid; t < mr * dh; t += kThreadsA) {
        const int i = t / dh, d = t % dh;
        const int p = pos[r0 + i];
        if (p < ch * kChunk) continue;
        const int nb = min(kWarpsA, (p - ch * kChunk) / kBlk + 1);
        float M = -INFINITY;
        for (int w = 0; w < nb; ++w) M = fmaxf(M, s_m[i][w]);
        float L = 0.f;
        for (int w = 0; w < nb; ++w) L = fmaf(s_l[i][w], expf(s_m[i][w] - M), L);
        float o = 0.f;
        for (int w = 0; w < nb; ++w) o = fmaf(s_acc[(i * kWarpsA + w) * dh + d], expf(s_m[i][w] - M), o);
        const int r = r0 + i;
        if (p / kChunk == 0) {
            out[(int64_t)r * h + hh * dh + d] = __float2bfloat16_rn(o / L);
        } else {
            const int64_t slot = ((int64_t)r * nh + hh) * kMaxChunks + ch;
            part[slot * stride + 2 + d] = o;
            if (d == 0) {
                part[slot * stride] = M;
                part[slot * stride + 1] = L;
            }
        }
    }
    if (pmax < kChunk) return;  // every row of the group fits one chunk
    __threadfence();
    __syncthreads();
    if (tid < mr) {
        const int p = pos[r0 + tid];
        s_last[tid] = p >= ch * kChunk && p >= kChunk &&
                      atomicAdd(&ctr[(r0 + tid) * nh + hh], 1) == p / kChunk;
    }
    __syncthreads();
    bool any = false;
    for (int i = 0; i < mr; ++i) any |= s_last[i] != 0;
    if (!any) return;
    __threadfence();
    // rows this CTA completed: fixed-order merge over chunks 0..nch-1
    for (int t = tid; t < mr * dh; t += kThreadsA) {
        const int i = t / dh, d = t % dh;
        if (!s_last[i]) continue;
        const int r = r0 + i;
        const int nch = pos[r] / kChunk + 1;
        const float* base = part + ((int64_t)r * nh + hh) * kMaxChunks * stride;
        out[(int64_t)r * h + hh * dh + d] = __float2bfloat16_rn(attn::chunk_merge(base, stride, nch, d));
    }
    if (tid < mr && s_last[tid]) ctr[(r0 + tid) * nh + hh] = 0;  // re-usable workspace
}

}  // namespace

// Workspace layout: attn_core.cuh (counters, then partial slots).
size_t attention_ws_bytes(int64_t /*m*/, int64_t nh, int64_t dh, int64_t /*s_max*/) {
    return attn::counters_bytes(nh) + attn::partial_slots(nh) * (dh + 2) * sizeof(float);
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
    float* part = (float*)((char*)ws + attn::counters_bytes(nh));
    const float scale = 1.0f / sqrtf((float)dh);
    const int64_t h = nh * dh;
    const int nch = max_pos / kChunk + 1;
    for (int64_t r0 = 0; r0 < m; r0 += kRowsPerLaunch) {
        const int64_t mr = m - r0 < kRowsPerLaunch ? m - r0 : kRowsPerLaunch;
        const dim3 grid((unsigned)nh, (unsigned)mr, (unsigned)nch);
        cudaError_t e;
        // bf16, head_dim 128: the rows kernel (K/V block loads shared by the
        // group's rows, K staged swizzled in shared memory, V in registers);
        // other shapes / fp32: one CTA per row (same arithmetic)
        if (dtype == EE_BF16 && dh == kMaxDh && nch >= kRowsKernelMinChunks) {
            // rows per CTA: just enough to fill the GPU with one CTA per SM
            // (more rows per CTA share more K/V loads but evaluate serially)
            const int64_t want = (mr * nh * nch + ee_sm_count() - 1) / ee_sm_count();
            const int g = (int)(want < 1 ? 1 : (want > kRowsCta ? kRowsCta : want));
            const int groups = (int)((mr + g - 1) / g);
            const size_t smem = rows128_smem((int)(mr < g ? mr : g));
            static bool configured[16] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!configured[dev & 15]) {
                cudaFuncSetAttribute(k_attn_rows128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)rows128_smem(kRowsCta));
                configured[dev & 15] = true;
            }
            e = launch_ex(k_attn_rows128, dim3((unsigned)nh, (unsigned)groups, (unsigned)nch),
                          dim3(kThreadsA), smem, s, q + r0 * h, pos + r0, (int)mr,
                          (const bf16*)kc, (const bf16*)vc, (int)nh, scale, (bf16*)out + r0 * h,
                          part, ctr, g);
        } else if (dtype == EE_BF16)
            e = launch_ex(k_attn_decode<bf16>, grid, dim3(kThreadsA), 0, s, q + r0 * h, pos + r0,
                          (int)mr, (const bf16*)kc, (const bf16*)vc, (int)nh, (int)dh, scale,
                          (bf16*)out + r0 * h, part, ctr);
        else if (dtype == EE_F32)
            e = launch_ex(k_attn_decode<float>, grid, dim3(kThreadsA), 0, s, q + r0 * h, pos + r0,
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
