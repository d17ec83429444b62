// Row-stable GEMV cores shared by the backbone GEMVs and the exit head.
//
// Decode is HBM-bound (arithmetic intensity ~= rows FLOP/B with rows <= 5),
// so the design goal is: stream every weight byte exactly once with many
// 16-byte requests in flight, and make the per-element reduction order a
// function of (n, k) only — never of how many rows share the launch (the
// reference's `dot_rows` contract, eepipe/_pykernels.py:14-17).
//
// bf16 path: one warp owns a 16 (weight rows) x 8*NB (activation rows) tile
// and walks k in blocks of 32.  Each lane loads 16 contiguous bytes of two
// weight rows (rows g and g+8, k = 32*kb + 8*t .. +7) and 16 bytes of its
// activation row, and feeds them to two m16n8k16 tensor-core MMAs.  The k
// index of the MMA fragments is a fixed permutation of the true k (the same
// permutation on both operands), so no shuffles are needed to build
// fragments.  Each output column (activation row) is computed independently
// by the MMA, so the result is row-stable by construction.
//
// fp32 path (parity mode): SIMT FFMA, lane-serial over k = 32*j + lane, then
// a fixed xor-butterfly, then a fixed-order cross-warp sum.
#pragma once

#include "ee_common.cuh"

// Accumulate acc[NB][4] (mma C fragments) for W rows n0..n0+15 and X rows
// r0..r0+8*NB-1 over k-blocks kb0, kb0+kbstep, ... (blocks of 32).
// Out-of-range rows are clamped (their outputs are discarded by the caller;
// columns and rows never mix inside an MMA).  K % 8 == 0 is required.
template <int NB, int U>
__device__ __forceinline__ void warp_tile_bf16(const bf16* __restrict__ W, int64_t K, int n0,
                                               int N, const bf16* __restrict__ X, int64_t ldx,
                                               int r0, int m, int kb0, int kbstep,
                                               float (&acc)[NB][4]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const bf16* wa = W + (int64_t)min(n0 + g, N - 1) * K + t * 8;
    const bf16* wb = W + (int64_t)min(n0 + g + 8, N - 1) * K + t * 8;
    const bf16* xp[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) xp[nb] = X + (int64_t)min(r0 + nb * 8 + g, m - 1) * ldx + t * 8;

    const int nfull = (int)(K >> 5);
    int kb = kb0;
    for (; kb + (U - 1) * kbstep < nfull; kb += U * kbstep) {
        uint4 a[U], b[U], x[U][NB];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t off = (int64_t)(kb + u * kbstep) * 32;
            a[u] = ld_stream16(wa + off);
            b[u] = ld_stream16(wb + off);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) x[u][nb] = ld_cached16(xp[nb] + off);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                mma_16816(acc[nb], a[u].x, b[u].x, a[u].y, b[u].y, x[u][nb].x, x[u][nb].y);
                mma_16816(acc[nb], a[u].z, b[u].z, a[u].w, b[u].w, x[u][nb].z, x[u][nb].w);
            }
        }
    }
    for (; kb < nfull; kb += kbstep) {
        const int64_t off = (int64_t)kb * 32;
        const uint4 a = ld_stream16(wa + off), b = ld_stream16(wb + off);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const uint4 x = ld_cached16(xp[nb] + off);
            mma_16816(acc[nb], a.x, b.x, a.y, b.y, x.x, x.y);
            mma_16816(acc[nb], a.z, b.z, a.w, b.w, x.z, x.w);
        }
    }
    // Partial last block (K % 32 != 0): owned by the warp whose sequence
    // lands exactly on it; lanes past K contribute exact zeros.
    if ((K & 31) && kb == nfull) {
        const int64_t off = (int64_t)nfull * 32;
        const bool ok = off + t * 8 < K;
        const uint4 z = make_uint4(0, 0, 0, 0);
        const uint4 a = ok ? ld_stream16(wa + off) : z, b = ok ? ld_stream16(wb + off) : z;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const uint4 x = ok ? ld_cached16(xp[nb] + off) : z;
            mma_16816(acc[nb], a.x, b.x, a.y, b.y, x.x, x.y);
            mma_16816(acc[nb], a.z, b.z, a.w, b.w, x.z, x.w);
        }
    }
}

// Scatter a warp's C fragments to a [16][8*NB] float tile (row = W row).
template <int NB>
__device__ __forceinline__ void store_frag(float (*tile)[8 * NB], const float (&acc)[NB][4]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        tile[g][nb * 8 + 2 * t] = acc[nb][0];
        tile[g][nb * 8 + 2 * t + 1] = acc[nb][1];
        tile[g + 8][nb * 8 + 2 * t] = acc[nb][2];
        tile[g + 8][nb * 8 + 2 * t + 1] = acc[nb][3];
    }
}

// fp32 SIMT tile: RW weight rows x RX activation rows, lanes over
// k = 32*(w0 + j*wstep) + lane.  Result reduced over the warp with a fixed
// xor butterfly (every lane ends with the full warp sum).
template <int RW, int RX, typename TW = float>
__device__ __forceinline__ void warp_tile_f32(const TW* __restrict__ W, int64_t K, int n0,
                                              int N, const float* __restrict__ X, int64_t ldx,
                                              int r0, int m, int w0, int wstep,
                                              float (&acc)[RW][RX]) {
    const int lane = threadIdx.x & 31;
    const TW* wr[RW];
    const float* xr[RX];
#pragma unroll
    for (int i = 0; i < RW; ++i) wr[i] = W + (int64_t)min(n0 + i, N - 1) * K;
#pragma unroll
    for (int j = 0; j < RX; ++j) xr[j] = X + (int64_t)min(r0 + j, m - 1) * ldx;
    for (int64_t k = (int64_t)w0 * 32 + lane; k < K; k += (int64_t)wstep * 32) {
        float xv[RX];
#pragma unroll
        for (int j = 0; j < RX; ++j) xv[j] = __ldg(xr[j] + k);
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const float wv = to_f32<TW>(wr[i][k]);
#pragma unroll
            for (int j = 0; j < RX; ++j) acc[i][j] = fmaf(wv, xv[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < RW; ++i)
#pragma unroll
        for (int j = 0; j < RX; ++j)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[i][j] += __shfl_xor_sync(0xffffffffu, acc[i][j], o);
}
