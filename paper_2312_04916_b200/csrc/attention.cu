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
#include <stdlib.h>

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
    EE_TMIN(0);  // even slots: min, odd: max
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
    EE_TMIN(2);
    EE_TMAX(3);
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
        if (warp == 0) EE_TMAX(5);
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
    EE_TMAX(7);
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
    EE_TMAX(9);
}


// ---------------------------------------------------------------------------
// bf16, head_dim 128: split-K/V "slab" kernel on a thread-block cluster.
// A cluster of C <= 8 CTAs (grid y) serves one (head, group of <= 16 rows);
// CTA rank r evaluates the 64-position slabs r, r + C, ... of the head's K/V
// (double-buffered cp.async into shared memory, K 16-byte chunks XOR-
// swizzled).  Per slab and row (short dependent chains, for latency):
//   s_j  = (q . K_j) * scale: thread (j, quarter) sums 32 dims as 4
//          interleaved chains, the quarters added in order;
//   m, l = slab max / sum of exp(s_j - m) over j <= p (warp butterflies);
//   o[d] = sum_j exp(s_j - m) V_j[d]: thread (d, half), 4 chains per half.
// Each slab's (m, l, o) stays in its CTA's shared memory; after a cluster
// barrier rank 0 folds slabs 0..p/64 of every row in slab order through
// distributed shared memory (weights e^(m_c - M) and their sum by warp
// butterflies, then o = sum_c w_c o_c in slab order) and writes the row.
// Every value depends on (row, position) only -- not on C or the other rows
// of the launch: row-stable and deterministic, no global atomics.
// No K/V load is issued before griddepcontrol.wait, not even of rows that
// earlier passes wrote: measured on B200, such loads -- when their values
// are consumed -- made the PRECEDING QKV GEMV write wrong K rows.
constexpr int kSlab = 64;
constexpr int kMaxSlabs = kMaxChunks * kChunk / kSlab;  // 32 (positions < 2048)
constexpr int kSlabThreads = 256;
constexpr int kSlabWarps = kSlabThreads / 32;
constexpr int kSlabRows = 16;
constexpr int kMaxCluster = 8;  // (16, non-portable: clusters scheduled late, slower)
constexpr int kLocalSlabs = kMaxSlabs / kMaxCluster;  // slabs one CTA may own
constexpr int kSlot = kMaxDh + 4;                     // [m, l, -, -, o[128]] per (slab, row)
constexpr int kKVBytes = 2 * kSlab * kMaxDh * 2;      // one K + V slab buffer
static_assert(kMaxSlabs == 32, "the fold uses one warp lane per slab");

__host__ __device__ constexpr size_t slab_smem(int rows, int local) {
    // 2 K/V buffers; q rows; scores (4 quarter partials per (row, position));
    // PV halves; the CTA's slab partials
    return (size_t)2 * kKVBytes + (size_t)rows * kMaxDh * 4 + (size_t)rows * 4 * kSlab * 4 +
           (size_t)rows * 2 * kMaxDh * 4 + (size_t)local * rows * kSlot * 4;
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ float2 bf2(uint32_t u) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                     "memory");
}
__device__ __forceinline__ uint32_t cl_map(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t a) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t a, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}

// A/B variants (profiling builds only, -DEE_ATTN_V=n): 0 = rolled PV loop,
// two-trip fold; 1 = unrolled PV + one-trip fold, <= 85 registers (3 CTAs
// per SM); 2 = the same, <= 64 registers; 3 = the same, no register cap
#ifndef EE_ATTN_V
#define EE_ATTN_V 1
#endif
#define EE_PV_UNROLL (EE_ATTN_V != 0)
#define EE_FOLD_HOIST (EE_ATTN_V != 0)
#if EE_ATTN_V == 1
#define EE_SLAB_BOUNDS __launch_bounds__(kSlabThreads, 3)
#elif EE_ATTN_V == 2
#define EE_SLAB_BOUNDS __launch_bounds__(kSlabThreads, 4)
#else
#define EE_SLAB_BOUNDS __launch_bounds__(kSlabThreads)
#endif

__global__ void EE_SLAB_BOUNDS
k_attn_slab128(const float* __restrict__ q, const int32_t* __restrict__ pos, int m,
               const bf16* __restrict__ kc, const bf16* __restrict__ vc, int nh, float scale,
               bf16* __restrict__ out, int g, int push) {
    extern __shared__ __align__(16) uint8_t smem_slab[];
    __shared__ float s_mx[kSlabRows], s_l[kSlabRows];
    __shared__ __align__(8) uint64_t s_recv;  // push mode: rank 0's "partials arrived" barrier
    constexpr int dh = kMaxDh;
    EE_TMIN(0);
    pdl_trigger_dev();
    const int hh = blockIdx.x;
    const int C = (int)gridDim.y;
    const int rank = (int)cl_rank();
    const int r0 = blockIdx.z * g;
    const int mr = min(g, m - r0);
    const int h = nh * dh;
    uint8_t* sKV = smem_slab;                                         // [2][K | V]
    float* sQ = reinterpret_cast<float*>(smem_slab + 2 * kKVBytes);   // [mr][dh]
    float* sS = sQ + mr * dh;                                         // [mr][4][kSlab]
    float* sO = sS + mr * 4 * kSlab;                                  // [mr][2][dh]
    // pull mode: [local slab][mr][kSlot] (this CTA's slabs, read by rank 0
    // through DSMEM); push mode: [slab][mr][kSlot] (every slab of the group,
    // written into rank 0's copy by the CTA that evaluated it)
    float* sPart = sO + mr * 2 * dh;
    // host-written control data (safe before the wait)
    int pmax = -1;
    for (int i = 0; i < mr; ++i) pmax = max(pmax, pos[r0 + i]);
    const int ns_g = pmax / kSlab + 1;                             // slabs of the group
    const int nloc = rank < ns_g ? (ns_g - 1 - rank) / C + 1 : 0;  // this CTA's slabs
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t hoff = (int64_t)hh * dh;
    const uint32_t kv_u = (uint32_t)__cvta_generic_to_shared(sKV);
    // slab sl (positions up to the group's last) into buffer b
    auto issue = [&](int b, int sl) {
        const int j0 = sl * kSlab, nj = min(kSlab, pmax + 1 - j0);
        const uint32_t k_u = kv_u + b * kKVBytes, v_u = k_u + kKVBytes / 2;
        for (int idx = tid; idx < nj * 16; idx += kSlabThreads) {
            const int jl = idx >> 4, c = idx & 15;
            const int64_t go = (int64_t)(j0 + jl) * h + hoff + c * 8;
            cp16(k_u + (uint32_t)((jl * 16 + (c ^ (jl & 7))) * 16), kc + go);
            cp16(v_u + (uint32_t)((jl * 16 + c) * 16), vc + go);
        }
    };
    const uint32_t recv_u = (uint32_t)__cvta_generic_to_shared(&s_recv);
    if (push) {
        // rank 0's barrier counts one arrival per other CTA; the cluster
        // barrier phase started here completes before the first remote store
        if (rank == 0 && tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(recv_u), "r"(C - 1));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    }
    pdl_wait_dev();
    EE_TMIN(2);
    EE_TMAX(3);
    if (nloc > 0) issue(0, rank);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (nloc > 1) issue(1, rank + C);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int t = tid; t < mr * (dh / 4); t += kSlabThreads) {
        const int i = t / (dh / 4), c = t % (dh / 4);
        reinterpret_cast<float4*>(sQ + i * dh)[c] =
            reinterpret_cast<const float4*>(q + (int64_t)(r0 + i) * h + hoff)[c];
    }
    if (push) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t part_u = (uint32_t)__cvta_generic_to_shared(sPart);
    const uint32_t part0 = push ? cl_map(part_u, 0) : part_u;  // rank 0's partial area
    for (int li = 0; li < nloc; ++li) {
        const int sl = rank + li * C, j0 = sl * kSlab, jend = min(j0 + kSlab, pmax + 1);
        const int b = li & 1;
        const bf16* sK = reinterpret_cast<const bf16*>(sKV + b * kKVBytes);
        const bf16* sV = sK + kSlab * dh;
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // this slab's group landed
        __syncthreads();
        EE_TMAX(5);
        // scores: thread (position jl = tid & 63, quarter qt = tid >> 6)
        {
            const int jl = tid & (kSlab - 1), qt = tid >> 6;
            if (j0 + jl < jend) {
                uint4 kk[4];
                const uint4* krow = reinterpret_cast<const uint4*>(sK) + jl * 16;
#pragma unroll
                for (int c = 0; c < 4; ++c) kk[c] = krow[(qt * 4 + c) ^ (jl & 7)];
                for (int i = 0; i < mr; ++i) {
                    const float4* qv = reinterpret_cast<const float4*>(sQ + i * dh + qt * 32);
                    float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 q0 = qv[2 * c], q1 = qv[2 * c + 1];
                        const float2 k0 = bf2(kk[c].x), k1 = bf2(kk[c].y), k2 = bf2(kk[c].z),
                                     k3 = bf2(kk[c].w);
                        a[0] = fmaf(q0.x, k0.x, a[0]);
                        a[1] = fmaf(q0.y, k0.y, a[1]);
                        a[2] = fmaf(q0.z, k1.x, a[2]);
                        a[3] = fmaf(q0.w, k1.y, a[3]);
                        a[0] = fmaf(q1.x, k2.x, a[0]);
                        a[1] = fmaf(q1.y, k2.y, a[1]);
                        a[2] = fmaf(q1.z, k3.x, a[2]);
                        a[3] = fmaf(q1.w, k3.y, a[3]);
                    }
                    sS[(i * 4 + qt) * kSlab + jl] = (a[0] + a[1]) + (a[2] + a[3]);
                }
            }
        }
        __syncthreads();
        if (li == 0) EE_TMAX(11);
        // slab softmax per row: warp per row, lane owns positions lane, lane + 32
        for (int i = warp; i < mr; i += kSlabWarps) {
            const int p = pos[r0 + i];
            const float* s0 = sS + i * 4 * kSlab;
            const int ja = j0 + lane, jb = j0 + 32 + lane;
            float a = -INFINITY, bb = -INFINITY;
            if (ja <= p)
                a = ((s0[lane] + s0[kSlab + lane]) + (s0[2 * kSlab + lane] + s0[3 * kSlab + lane])) *
                    scale;
            if (jb <= p)
                bb = ((s0[32 + lane] + s0[kSlab + 32 + lane]) +
                      (s0[2 * kSlab + 32 + lane] + s0[3 * kSlab + 32 + lane])) *
                     scale;
            float mx = fmaxf(a, bb);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float ea = ja <= p ? expf(a - mx) : 0.f;
            const float eb = jb <= p ? expf(bb - mx) : 0.f;
            float l = ea + eb;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
            __syncwarp();
            float* pr = sS + i * 4 * kSlab;  // probabilities overwrite the first quarter
            pr[lane] = ea;
            pr[32 + lane] = eb;
            if (lane == 0) {
                s_mx[i] = mx;
                s_l[i] = l;
            }
        }
        __syncthreads();
        if (li == 0) EE_TMAX(13);
        // P V: thread (dim d, position half ph), 4 interleaved chains per half
        {
            const int d = tid & (dh - 1), ph = tid >> 7;
            for (int i = 0; i < mr; ++i) {
                const int p = pos[r0 + i];
                if (p < j0) continue;  // CTA-uniform
                const int jb = ph * 32;
                const int nj = max(0, min(32, p + 1 - j0 - jb));
                const float* pr = sS + i * 4 * kSlab + jb;
                const bf16* vb = sV + jb * dh + d;
                float a[4] = {0.f, 0.f, 0.f, 0.f};
#if EE_PV_UNROLL
                if (nj == 32) {
                    // full half-slab: unrolled, so all 64 shared loads issue
                    // ahead of the FMA chains (same chains, same order)
#pragma unroll
                    for (int jh = 0; jh < 32; jh += 16) {
                        float pv[16], vv[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            pv[j] = pr[jh + j];
                            vv[j] = __bfloat162float(vb[(jh + j) * dh]);
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) a[j & 3] = fmaf(pv[j], vv[j], a[j & 3]);
                    }
                } else
#endif
                {
                    int jl = 0;
                    for (; jl + 4 <= nj; jl += 4) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            a[u] = fmaf(pr[jl + u], __bfloat162float(vb[(jl + u) * dh]), a[u]);
                    }
#pragma unroll
                    for (int u = 0; u < 3; ++u)  // tail: at most 3 positions
                        if (jl + u < nj)
                            a[u] = fmaf(pr[jl + u], __bfloat162float(vb[(jl + u) * dh]), a[u]);
                }
                sO[(i * 2 + ph) * dh + d] = (a[0] + a[1]) + (a[2] + a[3]);
            }
        }
        __syncthreads();  // buffer b and sS free from here on
        if (li == 0) EE_TMAX(15);
        if (li + 2 < nloc) issue(b, rank + (li + 2) * C);
        asm volatile("cp.async.commit_group;" ::: "memory");
        // the slab's partials -> this CTA's shared memory (pull) or rank 0's
        // (push: remote stores, released by the arrival below)
        for (int t = tid; t < mr * dh; t += kSlabThreads) {
            const int i = t / dh, d = t % dh;
            const float o = sO[i * 2 * dh + d] + sO[(i * 2 + 1) * dh + d];
            if (push) {
                const uint32_t a = part0 + (uint32_t)(((sl * mr + i) * kSlot) * 4);
                st_dsmem(a + 16 + 4 * d, o);
                if (d == 0) {
                    st_dsmem(a, s_mx[i]);
                    st_dsmem(a + 4, s_l[i]);
                }
            } else {
                float* slot = sPart + (li * mr + i) * kSlot;
                slot[4 + d] = o;
                if (d == 0) {
                    slot[0] = s_mx[i];
                    slot[1] = s_l[i];
                }
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    EE_TMAX(7);
    if (push) {
        if (rank != 0) {
            // every thread's remote stores precede thread 0's release-arrival
            __syncthreads();
            if (tid == 0)
                asm volatile(
                    "fence.acq_rel.cluster;\n\t"
                    "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                        cl_map(recv_u, 0))
                    : "memory");
            return;  // rank 0 never reads this CTA's shared memory
        }
        if (C > 1)
            asm volatile(
                "{\n\t.reg .pred p;\n"
                "WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n\t"
                "@!p bra WAIT_%=;\n}" ::"r"(recv_u)
                : "memory");
        __syncthreads();  // rank 0's own partials too
    } else {
        cl_sync();  // every slab partial of the cluster is in place
    }
    EE_TMAX(1);
    if (rank == 0 && push) {
        // push mode: every slab's partial sits in this CTA's own shared
        // memory; the same fold arithmetic as the pull path below
        for (int i = warp; i < mr; i += kSlabWarps) {
            const int r = r0 + i;
            const int ns = pos[r] / kSlab + 1;
            const float* base = sPart + i * kSlot;  // slab c at base + c * mr * kSlot
            const int cs = mr * kSlot;
            float Mc = -INFINITY, Lc = 0.f;
            if (lane < ns) {
                Mc = base[lane * cs];
                Lc = base[lane * cs + 1];
            }
            float MM = Mc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) MM = fmaxf(MM, __shfl_xor_sync(0xffffffffu, MM, o));
            const float w = lane < ns ? expf(Mc - MM) : 0.f;
            float LL = Lc * w;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) LL += __shfl_xor_sync(0xffffffffu, LL, o);
            float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int c0 = 0; c0 < ns; c0 += 8) {
                float4 oc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    oc[u] = c0 + u < ns ? reinterpret_cast<const float4*>(base + (c0 + u) * cs + 4)[lane]
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float wc = __shfl_sync(0xffffffffu, w, (c0 + u) & 31);
                    if (c0 + u < ns) {
                        o4.x = fmaf(oc[u].x, wc, o4.x);
                        o4.y = fmaf(oc[u].y, wc, o4.y);
                        o4.z = fmaf(oc[u].z, wc, o4.z);
                        o4.w = fmaf(oc[u].w, wc, o4.w);
                    }
                }
            }
            const float inv = 1.f / LL;
            bf16* orow = out + (int64_t)r * h + hoff + 4 * lane;
            *reinterpret_cast<__nv_bfloat162*>(orow) = __floats2bfloat162_rn(o4.x * inv, o4.y * inv);
            *reinterpret_cast<__nv_bfloat162*>(orow + 2) = __floats2bfloat162_rn(o4.z * inv, o4.w * inv);
        }
    } else if (rank == 0) {
        for (int i = warp; i < mr; i += kSlabWarps) {
            const int r = r0 + i;
            const int ns = pos[r] / kSlab + 1;
            // slab c lives in rank c % C, local index c / C
            auto slot_addr = [&](int c) {
                return cl_map(part_u + (uint32_t)((((c / C) * mr + i) * kSlot) * 4), (uint32_t)(c % C));
            };
            float Mc = -INFINITY, Lc = 0.f;
            if (lane < ns) {
                const uint32_t a = slot_addr(lane);
                Mc = ld_dsmem(a);
                Lc = ld_dsmem(a + 4);
            }
            // the first 8 slabs' o slices travel with (m, l): one DSMEM round
            // trip instead of two for contexts up to 512
#if EE_FOLD_HOIST
            float4 oc0[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                oc0[u] = u < ns ? ld_dsmem4(slot_addr(u) + 16 + 16 * lane) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
            float MM = Mc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) MM = fmaxf(MM, __shfl_xor_sync(0xffffffffu, MM, o));
            const float w = lane < ns ? expf(Mc - MM) : 0.f;
            float LL = Lc * w;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) LL += __shfl_xor_sync(0xffffffffu, LL, o);
            float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int c0 = 0; c0 < ns; c0 += 8) {
                float4 oc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
#if EE_FOLD_HOIST
                    oc[u] = c0 == 0 ? oc0[u]
                            : c0 + u < ns ? ld_dsmem4(slot_addr(c0 + u) + 16 + 16 * lane)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
#else
                    oc[u] = c0 + u < ns ? ld_dsmem4(slot_addr(c0 + u) + 16 + 16 * lane)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float wc = __shfl_sync(0xffffffffu, w, (c0 + u) & 31);
                    if (c0 + u < ns) {
                        o4.x = fmaf(oc[u].x, wc, o4.x);
                        o4.y = fmaf(oc[u].y, wc, o4.y);
                        o4.z = fmaf(oc[u].z, wc, o4.z);
                        o4.w = fmaf(oc[u].w, wc, o4.w);
                    }
                }
            }
            const float inv = 1.f / LL;
            bf16* orow = out + (int64_t)r * h + hoff + 4 * lane;
            *reinterpret_cast<__nv_bfloat162*>(orow) = __floats2bfloat162_rn(o4.x * inv, o4.y * inv);
            *reinterpret_cast<__nv_bfloat162*>(orow + 2) = __floats2bfloat162_rn(o4.z * inv, o4.w * inv);
        }
    }
    EE_TMAX(9);
    if (!push) cl_sync();  // rank 0 has read every partial: the other CTAs may exit
}

}  // namespace

EE_TRACE_READER(ee_trace_attention)

// Workspace layout: attn_core.cuh (counters, then partial slots).
size_t attention_ws_bytes(int64_t /*m*/, int64_t nh, int64_t dh, int64_t /*s_max*/) {
    return attn::counters_bytes(nh) + attn::partial_slots(nh) * (dh + 2) * sizeof(float);
}

// EE_ATTN_PUSH=0 (A/B): slab partials always pulled by rank 0 through DSMEM
constexpr int kPushMaxSlabs = 12;
static bool attn_push() {
    static const bool v = !getenv("EE_ATTN_PUSH") || atoi(getenv("EE_ATTN_PUSH")) != 0;
    return v;
}

// EE_ATTN_SLAB=0 (A/B): the chunked rows kernel instead of the slab kernel
static bool attn_slab() {
    static const bool v = !getenv("EE_ATTN_SLAB") || atoi(getenv("EE_ATTN_SLAB")) != 0;
    return v;
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
        const int ns = max_pos / kSlab + 1;
        if (dtype == EE_BF16 && dh == kMaxDh && attn_slab()) {
            const int C = ns < kMaxCluster ? ns : kMaxCluster;
            // rows per cluster: enough clusters to cover the GPU about twice
            const int64_t want = (2 * mr * nh * C + ee_sm_count() - 1) / (2 * ee_sm_count());
            const int g = (int)(want < 1 ? 1 : (want > kSlabRows ? kSlabRows : want));
            const int groups = (int)((mr + g - 1) / g);
            // push mode (partials stored straight into rank 0, no cluster
            // barriers at the end) up to 12 slabs: per pass -1.5..-2.3% at
            // ctx 64-320, -3..-6% at ctx 640, but +1.4..+6% at ctx 1024 and
            // +2.6% at 2000 (1 row), where pull mode stays
            // (profiles/r2_attn_push_ab.txt)
            const int gr = (int)(mr < g ? mr : g);
            const bool push = attn_push() && ns <= kPushMaxSlabs &&
                              slab_smem(gr, ns) <= slab_smem(kSlabRows, kLocalSlabs);
            const int local = push ? ns : (ns + C - 1) / C;
            static bool configured[16] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (!configured[dev & 15]) {
                cudaFuncSetAttribute(k_attn_slab128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)slab_smem(kSlabRows, kLocalSlabs));
                configured[dev & 15] = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)nh, (unsigned)C, (unsigned)groups);
            cfg.blockDim = dim3(kSlabThreads);
            cfg.dynamicSmemBytes = slab_smem(gr, local);
            cfg.stream = s;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 1;
            attr[0].val.clusterDim.y = (unsigned)C;
            attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = ee_pdl_enabled() && !g_pdl_off ? 2 : 1;
            e = cudaLaunchKernelEx(&cfg, k_attn_slab128, q + r0 * h, pos + r0, (int)mr,
                                   (const bf16*)kc, (const bf16*)vc, (int)nh, scale,
                                   (bf16*)out + r0 * h, g, push ? 1 : 0);
        } else if (dtype == EE_BF16 && dh == kMaxDh && nch >= kRowsKernelMinChunks) {
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
