// HBM weight layout for the TMA-fed GEMV: "tiled" bf16.
//
// A (N, K) row-major bf16 matrix (K-major rows, the reference matrix
// transposed) is re-laid out as
//     [N/16 tiles][K/512 k-stages][16 rows][512 k]      (zero rows pad N)
// so that the 16 x 512 block a CTA consumes per pipeline stage is one
// contiguous 16 KB run — ONE bulk async copy per stage (small copies are
// TMA-issue-bound on B200: 1 KB pieces stream at ~2.4-4.3 TB/s, 16 KB pieces
// at ~5.8 TB/s, tools/bw_probe.cu).  Inside a row, the 16-byte chunk c is
// stored at chunk position c ^ (row & 7): the consumers' 16-B LDS of rows
// g and g+8 then hit 8 distinct bank groups (4 wavefronts per warp access,
// the minimum) without padding.  An optional per-column scale folds an
// RMSNorm weight into the matrix (decode.cu).
#include "ee_common.cuh"

namespace {

__global__ void k_pack_tiled(const uint4* __restrict__ src, int64_t N, int64_t K,
                             const float* __restrict__ col_scale, uint4* __restrict__ dst,
                             int64_t total_chunks) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total_chunks) return;
    // dst chunk index -> (tile, ks, r, p)
    const int64_t kst = K / kTiledKS;
    const int p = (int)(i & 63);
    const int r = (int)((i >> 6) & 15);
    const int64_t blk = i >> 10;  // tile * kst + ks
    const int64_t ks = blk % kst, tile = blk / kst;
    const int64_t n = tile * 16 + r;
    const int c = p ^ (r & 7);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n < N) {
        v = src[(n * K + ks * kTiledKS) / 8 + c];
        if (col_scale) {
            const float* cs = col_scale + ks * kTiledKS + c * 8;
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                __nv_bfloat162 o = __floats2bfloat162_rn(f.x * cs[2 * e], f.y * cs[2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t*>(&o);
            }
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    dst[i] = v;
}

}  // namespace

extern "C" size_t ee_tiled_weight_bytes(int64_t N, int64_t K) {
    if (N <= 0 || K <= 0 || K % kTiledKS) return 0;
    return (size_t)((N + 15) / 16) * 16 * K * 2;
}

extern "C" int ee_pack_tiled(const void* W, int64_t N, int64_t K, const float* col_scale,
                             void* out, void* stream) {
    EE_REQUIRE(ee_tiled_weight_bytes(N, K) > 0, EE_ESHAPE,
               "pack_tiled: K must be a positive multiple of %d (K=%lld)", kTiledKS, (long long)K);
    const int64_t chunks = (int64_t)ee_tiled_weight_bytes(N, K) / 16;
    const int threads = 256;
    k_pack_tiled<<<(unsigned)((chunks + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
        (const uint4*)W, N, K, col_scale, (uint4*)out, chunks);
    return ee_check_launch("pack_tiled");
}
