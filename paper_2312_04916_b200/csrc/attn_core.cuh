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
// several rows can score it (k_attn_rows128): block_load128 issues the raw K
// row of this lane's position (16 x 16 B, registers) and copies the block's V
// rows (32 x 256 B) into the warp's shared-memory tile sv with cp.async, for
// every position <= plim -- one memory round trip per block -- and
// block_eval128 evaluates one row (position p <= plim, q in shared memory).
struct BlockRegs {
    uint4 k[16];
};

__device__ __forceinline__ void block_load128(BlockRegs& R, bf16* sv, const bf16* __restrict__ kc,
                                              const bf16* __restrict__ vc, int64_t h, int hoff,
                                              int j0, int plim) {
    const int lane = threadIdx.x & 31;
    const int jj = j0 + lane;
    const int nj = min(kBlk, plim + 1 - j0);
    const bf16* vb = vc + (int64_t)j0 * h + hoff + 4 * lane;
    const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(sv + 4 * lane);
    for (int j = 0; j < nj; ++j)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sdst + j * kMaxDh * 2),
                     "l"(vb + (int64_t)j * h)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (jj <= plim) {
        const uint4* krow = reinterpret_cast<const uint4*>(kc + (int64_t)jj * h + hoff);
#pragma unroll
        for (int i = 0; i < 16; ++i) R.k[i] = krow[i];
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
}

__device__ __forceinline__ void block_eval128(const BlockRegs& R, const bf16* sv, const float* sq,
                                              int j0, int p, float scale, float& mx, float& l,
                                              float acc[4]) {
    const int lane = threadIdx.x & 31;
    const bool valid = j0 + lane <= p;
    const int nj = min(kBlk, p + 1 - j0);
    float sc = 0.f;
    if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint32_t w4[4] = {R.k[i].x, R.k[i].y, R.k[i].z, R.k[i].w};
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e2]));
                sc = fmaf(sq[8 * i + 2 * e2], f.x, sc);
                sc = fmaf(sq[8 * i + 2 * e2 + 1], f.y, sc);
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
            const uint2 vv = *reinterpret_cast<const uint2*>(sv + j * kMaxDh + 4 * lane);
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv.x));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv.y));
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
