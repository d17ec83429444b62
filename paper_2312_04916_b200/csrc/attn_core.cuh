// Decode-attention arithmetic (attention.cu).  Every (row, head) is
// evaluated with the same operations in the same order whatever else shares
// the launch (row-stable):
//
//   block  b (32 positions 32b .. 32b+31, lane j = position 32b + j):
//          s_j = (q . K_j) * scale (fixed-order dot),  m_b = max_j s_j,
//          l_b = sum_j exp(s_j - m_b),  a_b[d] = sum_j exp(s_j - m_b) V_j[d]
//   chunk  c (blocks 8c .. 8c+7):  M_c = max m_b,  L_c = sum l_b e^(m_b-M_c),
//          o_c[d] = sum a_b[d] e^(m_b - M_c)          (blocks in order)
//   row    one chunk: out = o_0 / L_0; otherwise the same merge over chunks
//          in chunk order: out = (sum o_c e^(M_c-MM)) / (sum L_c e^(M_c-MM))
//
// Heads split the hidden axis as reshape(nh, dh) (eepipe/inference.py:207,
// 225), scale 1/sqrt(dh) (eepipe/inference.py:203).
#pragma once

#include "ee_common.cuh"

namespace attn {

constexpr int kBlk = 32;                 // positions per block (one warp)
constexpr int kWarpsA = 8;               // blocks per chunk
constexpr int kChunk = kBlk * kWarpsA;   // 256 positions
constexpr int kMaxDh = 128;
constexpr int kRowsPerLaunch = 64;
constexpr int kMaxChunks = 8;            // positions < 2048
constexpr int kMaxBlocks = kMaxChunks * kWarpsA;

// Workspace: [ctr: kRowsPerLaunch*nh int32] (rounded to 256 B) then
// [partials: kRowsPerLaunch*nh*kMaxChunks slots of (dh+2) floats].  Zeroed
// once at allocation; every call leaves the counters zeroed.
__host__ __device__ inline size_t counters_bytes(int64_t nh) {
    return (((size_t)kRowsPerLaunch * nh * 4) + 255) & ~(size_t)255;
}
__host__ __device__ inline size_t partial_slots(int64_t nh) {
    return (size_t)kRowsPerLaunch * nh * kMaxChunks;
}

// One 32-position block of one head, bf16 K/V, dh = 128, in two steps so
// several rows can score it (k_attn_rows128), with the K tile staged in
// shared memory and the V columns in registers: block_issue128_k copies the
// block's K rows
// (32 x 256 B, coalesced) with cp.async into the warp's tile sk, 16-byte
// chunk c of row j at chunk c ^ (j & 7) (conflict-free row reads), and
// block_eval128_k evaluates one row (position p <= plim, q in shared
// memory), reading this lane's K row back in two 8-chunk halves.  Same
// arithmetic, same order as k_attn_decode's generic path.
struct BlockRegsV {
    uint2 v[kBlk];
};

// issue: the K tile copy (cp.async, committed) and the V register loads;
// block_wait128_k completes the K copy for the whole warp
__device__ __forceinline__ void block_issue128_k(BlockRegsV& R, bf16* sk, const bf16* __restrict__ kc,
                                                 const bf16* __restrict__ vc, int64_t h, int hoff,
                                                 int j0, int plim) {
    const int lane = threadIdx.x & 31;
    const int nj = min(kBlk, plim + 1 - j0);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sk);
#pragma unroll
    for (int t = 0; t < kBlk * 16 / 32; ++t) {
        const int idx = lane + 32 * t;
        const int j = idx >> 4, c = idx & 15;
        if (j < nj)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             sbase + (uint32_t)((j * 16 + (c ^ (j & 7))) * 16)),
                         "l"(kc + (int64_t)(j0 + j) * h + hoff + c * 8)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const bf16* vb = vc + (int64_t)j0 * h + hoff + 4 * lane;
#pragma unroll
    for (int j = 0; j < kBlk; ++j)
        if (j < nj) R.v[j] = *reinterpret_cast<const uint2*>(vb + (int64_t)j * h);
}

__device__ __forceinline__ void block_wait128_k() {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
}

__device__ __forceinline__ void block_eval128_k(const BlockRegsV& R, const bf16* sk, const float* sq,
                                                int j0, int p, float scale, float& mx, float& l,
                                                float acc[4]) {
    const int lane = threadIdx.x & 31;
    const bool valid = j0 + lane <= p;
    const int nj = min(kBlk, p + 1 - j0);
    float sc = 0.f;
    if (valid) {
        const uint4* krow = reinterpret_cast<const uint4*>(sk) + lane * 16;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint4 kk[8];
#pragma unroll
            for (int q8 = 0; q8 < 8; ++q8) kk[q8] = krow[(half * 8 + q8) ^ (lane & 7)];
#pragma unroll
            for (int q8 = 0; q8 < 8; ++q8) {
                const int i = half * 8 + q8;
                const uint32_t w4[4] = {kk[q8].x, kk[q8].y, kk[q8].z, kk[q8].w};
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e2]));
                    sc = fmaf(sq[8 * i + 2 * e2], f.x, sc);
                    sc = fmaf(sq[8 * i + 2 * e2 + 1], f.y, sc);
                }
            }
        }
    }
    const float sval = valid ? sc * scale : -INFINITY;
    mx = sval;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float e = valid ? expf(sval - mx) : 0.f;
    l = e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
#pragma unroll
    for (int j = 0; j < kBlk; ++j) {
        const float pj = __shfl_sync(0xffffffffu, e, j);
        if (j < nj) {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&R.v[j].x));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&R.v[j].y));
            acc[0] = fmaf(pj, a.x, acc[0]);
            acc[1] = fmaf(pj, a.y, acc[1]);
            acc[2] = fmaf(pj, b.x, acc[2]);
            acc[3] = fmaf(pj, b.y, acc[3]);
        }
    }
}

// Cross-chunk merge of one (row, head, dim): chunk partials (M_c, L_c, o_c)
// at base + c*stride (+0, +1, +2+d), c < nch, all loaded up front (one L2
// round trip), then folded in chunk order:
//   out = (sum_c o_c e^(M_c-MM)) / (sum_c L_c e^(M_c-MM)),  MM = max_c M_c
__device__ __forceinline__ float chunk_merge(const float* base, int stride, int nch, int d) {
    float Mc[kMaxChunks], Lc[kMaxChunks], oc[kMaxChunks];
#pragma unroll
    for (int c = 0; c < kMaxChunks; ++c) {
        if (c < nch) {
            Mc[c] = __ldcg(base + c * stride);
            Lc[c] = __ldcg(base + c * stride + 1);
            oc[c] = __ldcg(base + c * stride + 2 + d);
        }
    }
    float MM = -INFINITY;
#pragma unroll
    for (int c = 0; c < kMaxChunks; ++c)
        if (c < nch) MM = fmaxf(MM, Mc[c]);
    float LL = 0.f, o = 0.f;
#pragma unroll
    for (int c = 0; c < kMaxChunks; ++c)
        if (c < nch) LL = fmaf(Lc[c], expf(Mc[c] - MM), LL);
#pragma unroll
    for (int c = 0; c < kMaxChunks; ++c)
        if (c < nch) o = fmaf(oc[c], expf(Mc[c] - MM), o);
    return o / LL;
}

}  // namespace attn
