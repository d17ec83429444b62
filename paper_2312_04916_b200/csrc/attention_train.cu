// Causal multi-head attention for the training backbone on tcgen05 tensor
// cores (flash-attention style: the (S x S) scores never reach HBM),
// restating `causal_attention` forward / backward (eepipe/autodiff.py:
// 265-298) and the boundary kernels `attention_fwd` / `attention_bwd`
// (eepipe/_pykernels.py:52-62, eepipe/_ckernels.pyx:170-236):
//   P = softmax(Q K^T / sqrt(dh) + causal mask),  O = P V
//   dV = P^T dO,  dP = dO V^T,  dS = P (dP - rowsum(dO o O)),
//   dQ = dS K / sqrt(dh),  dK = dS^T Q / sqrt(dh)
//
// Layout: Q, K, V, O, dO, dQ, dK, dV are (B*S, ld) bf16 row-major with head
// hh in columns [hh*128, hh*128 + 128) -- the projections' own output layout
// (no (B, H, S, dh) transposes); lse / D are float32 [B][H][S].  head_dim
// 128, S a multiple of 128.  One CTA per (128-row tile, head, batch):
//   warp 0 lane 0   TMA producer (2-D tensor maps, 128-byte swizzle)
//   warp 1 lane 0   tcgen05.mma issuer (UMMA 128 x 128 x 16, fp32 in TMEM)
//   warps 2..5      one thread per tile row (= TMEM lane): softmax / dS in
//                   registers, P / dS written to shared memory in the UMMA
//                   K-major SW128 layout; the same bytes serve as the
//                   MN-major (transposed) operand of dV / dK.
// Deterministic: every sum has a fixed order (no atomics): dK/dV accumulate
// over q tiles in one CTA, dQ over key tiles in another (k_attn_bwd_q).
#include <cuda.h>

#include "tc_gemm.cuh"

namespace {

using namespace tc;

constexpr int kT = 128;                 // rows per tile (queries or keys)
constexpr int kDh = 128;                // head dim
constexpr int kBox = kT * 128;          // one 64-column box of 128 rows: 16 KB
constexpr int kTile = 2 * kBox;         // 128 x 128 bf16: 32 KB
constexpr int kAttnThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// K-major operand (rows x 128, two 64-column boxes): k-th 16-wide slice of box kb
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int kb, int k) {
    return sw128_desc(tile + kb * kBox + k * 32, 1, 64);
}
// the SAME bytes read MN-major (MN = the 128 columns, K = the 128 rows):
// k-th 16-row slice, MN chunks (the two boxes) 16 KB apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int kk) {
    return sw128_desc(tile + kk * 2048, kBox / 16, 64);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&t);
}
// 16 values (columns c0..c0+15 of tile row r) -> bf16 into a K-major SW128 tile
__device__ __forceinline__ void store_row16(uint8_t* tile, int r, int c0, const float* v) {
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
        const int c = c0 + 8 * h8;
        const int kb = c >> 6, chunk = (c & 63) >> 3;
        uint4 u = make_uint4(pack2(v[8 * h8], v[8 * h8 + 1]), pack2(v[8 * h8 + 2], v[8 * h8 + 3]),
                             pack2(v[8 * h8 + 4], v[8 * h8 + 5]), pack2(v[8 * h8 + 6], v[8 * h8 + 7]));
        *reinterpret_cast<uint4*>(tile + kb * kBox + r * 128 + ((chunk ^ (r & 7)) << 4)) = u;
    }
}

__device__ __forceinline__ void alloc_tmem512(uint32_t* slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void free_tmem512(uint32_t tmem) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

constexpr uint32_t kIdescKK = idesc_bf16(128, 128, false, false);  // A, B K-major
constexpr uint32_t kIdescKM = idesc_bf16(128, 128, false, true);   // A K-major, B MN-major
constexpr uint32_t kIdescMM = idesc_bf16(128, 128, true, true);    // A, B MN-major

// load one 128 x 128 tile (two 64-column boxes) of head column col, rows row0
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* m, int col, int row0,
                                          uint64_t* bar) {
    tma_load_2d(dst, m, col, row0, bar);
    tma_load_2d(dst + kBox, m, col + 64, row0, bar);
}

// ============================================================================
// forward: CTA = (q tile, head, batch); key tiles 0..qt, double-buffered S
// ============================================================================
struct FwdBars {
    uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], s_free[2], p_full, o_done;
    uint32_t tmem;
};
constexpr size_t kFwdSmem = 1024 + 6 * (size_t)kTile + sizeof(FwdBars) + 64;

__global__ void __launch_bounds__(kAttnThreads, 1)
k_attn_fwd(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
           const __grid_constant__ CUtensorMap tv, int S, int H, bf16* __restrict__ out, int ldo,
           float* __restrict__ lse, float scale) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sQ = sm;
    uint8_t* sK = sm + kTile;          // [2]
    uint8_t* sV = sm + 3 * kTile;      // [2]
    uint8_t* sP = sm + 5 * kTile;
    FwdBars* bar = reinterpret_cast<FwdBars*>(sm + 6 * kTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    const int qt = nqt - 1 - (int)blockIdx.x;  // longest rows first
    const int hh = blockIdx.y, b = blockIdx.z;
    const int row0 = b * S + qt * kT;
    const int col = hh * kDh;
    const int nkt = qt + 1;
    if (threadIdx.x == 0) {
        mb_init(&bar->q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mb_init(&bar->kv_full[i], 1);
            mb_init(&bar->kv_empty[i], 1);
            mb_init(&bar->s_full[i], 1);
            mb_init(&bar->s_free[i], 128);
        }
        mb_init(&bar->p_full, 128);
        mb_init(&bar->o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) alloc_tmem512(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    if (warp == 0) {
        if (lane == 0) {
            mb_expect_tx(&bar->q_full, kTile);
            load_tile(sQ, &tq, col, row0, &bar->q_full);
            for (int kt = 0; kt < nkt; ++kt) {
                const int s = kt & 1;
                if (kt >= 2) mb_wait(&bar->kv_empty[s], ((kt >> 1) - 1) & 1);
                mb_expect_tx(&bar->kv_full[s], 2 * kTile);
                load_tile(sK + s * kTile, &tk, col, b * S + kt * kT, &bar->kv_full[s]);
                load_tile(sV + s * kTile, &tv, col, b * S + kt * kT, &bar->kv_full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mb_wait(&bar->q_full, 0);
            tc_fence_after();
            const uint32_t q = su32(sQ);
            auto issue_s = [&](int kt) {
                const int s = kt & 1;
                mb_wait(&bar->kv_full[s], (kt >> 1) & 1);
                if (kt >= 2) mb_wait(&bar->s_free[s], ((kt >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t kk = su32(sK + s * kTile);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc_mma(tmem + s * kT, desc_k(q, kb, k), desc_k(kk, kb, k), kIdescKK,
                               (kb | k) != 0);
                tc_commit(&bar->s_full[s]);
            };
            issue_s(0);
            const uint32_t p = su32(sP);
            for (int kt = 0; kt < nkt; ++kt) {
                if (kt + 1 < nkt) issue_s(kt + 1);
                mb_wait(&bar->p_full, kt & 1);
                tc_fence_after();
                const uint32_t v = su32(sV + (kt & 1) * kTile);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc_mma(tmem + 2 * kT, desc_k(p, kb, k), desc_mn(v, kb * 4 + k), kIdescKM,
                               (kt | kb | k) != 0);
                tc_commit(&bar->o_done);
                tc_commit(&bar->kv_empty[kt & 1]);
            }
        }
    } else {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // tile row = TMEM lane
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const float sl2 = scale * kLog2e;
        float m = -INFINITY, l = 0.f;
        float v[kT];
        for (int kt = 0; kt < nkt; ++kt) {
            const int s = kt & 1;
            mb_wait(&bar->s_full[s], (kt >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < kT; c += 16) tmem_ld16_nowait(tmem + lane_off + s * kT + c, v + c);
            tmem_wait_ld();
            tc_fence_before();
            mb_arrive(&bar->s_free[s]);
            const bool diag = kt == qt;
            float mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < kT; ++j) {
                const float x = (diag && j > r) ? -INFINITY : v[j] * sl2;
                v[j] = x;
                mx = fmaxf(mx, x);
            }
            const float mn = fmaxf(m, mx);
            const float alpha = exp2f(m - mn);
            float sum = 0.f;
#pragma unroll
            for (int j = 0; j < kT; ++j) {
                const float e = exp2f(v[j] - mn);
                v[j] = e;
                sum += e;
            }
            l = l * alpha + sum;
            m = mn;
            if (kt > 0) {
                mb_wait(&bar->o_done, (kt - 1) & 1);  // PV(kt-1) done: O stable, P free
                tc_fence_after();
                if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                    for (int c = 0; c < kDh; c += 16) {
                        float o[16];
                        tmem_ld16(tmem + lane_off + 2 * kT + c, o);
#pragma unroll
                        for (int j = 0; j < 16; ++j) o[j] *= alpha;
                        tmem_st16(tmem + lane_off + 2 * kT + c, o);
                    }
                    tmem_wait_st();
                }
            }
#pragma unroll
            for (int c = 0; c < kT; c += 16) store_row16(sP, r, c, v + c);
            fence_async_smem();
            tc_fence_before();
            mb_arrive(&bar->p_full);
        }
        mb_wait(&bar->o_done, (nkt - 1) & 1);
        tc_fence_after();
        const float inv = 1.f / l;
        bf16* orow = out + (int64_t)(row0 + r) * ldo + col;
#pragma unroll 1
        for (int c = 0; c < kDh; c += 16) {
            float o[16];
            tmem_ld16(tmem + lane_off + 2 * kT + c, o);
            uint4 u0 = make_uint4(pack2(o[0] * inv, o[1] * inv), pack2(o[2] * inv, o[3] * inv),
                                  pack2(o[4] * inv, o[5] * inv), pack2(o[6] * inv, o[7] * inv));
            uint4 u1 = make_uint4(pack2(o[8] * inv, o[9] * inv), pack2(o[10] * inv, o[11] * inv),
                                  pack2(o[12] * inv, o[13] * inv), pack2(o[14] * inv, o[15] * inv));
            reinterpret_cast<uint4*>(orow + c)[0] = u0;
            reinterpret_cast<uint4*>(orow + c)[1] = u1;
        }
        lse[((int64_t)b * H + hh) * S + qt * kT + r] = (m + log2f(l)) * kLn2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
    }
}

// D[b][h][s] = sum_d dO * O (float32), one warp per (row, head)
__global__ void k_attn_dot(const bf16* __restrict__ dout, int ldd, const bf16* __restrict__ o,
                           int ldo, int S, int H, int rows, float* __restrict__ D) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows * H) return;
    const int row = w / H, hh = w % H;
    const uint2 a = *reinterpret_cast<const uint2*>(dout + (int64_t)row * ldd + hh * kDh + 4 * lane);
    const uint2 c = *reinterpret_cast<const uint2*>(o + (int64_t)row * ldo + hh * kDh + 4 * lane);
    const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.x));
    const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.y));
    const float2 c0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.x));
    const float2 c1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.y));
    float s = a0.x * c0.x + a0.y * c0.y + a1.x * c1.x + a1.y * c1.y;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
        const int b = row / S, si = row % S;
        D[((int64_t)b * H + hh) * S + si] = s;
    }
}

// P (and dS) of one 16-column chunk of tile row r from S and dP in TMEM
struct RowGrad {
    float lse2;  // lse * log2(e)
    float d;     // rowsum(dO o O)
    float sl2;   // scale * log2(e)
    float scale;
};
__device__ __forceinline__ void p_ds_chunk(const RowGrad& g, const float* sv, const float* dpv,
                                           bool diag, int r, int c0, float* p, float* ds) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const bool masked = diag && (c0 + j) > r;
        const float pj = masked ? 0.f : exp2f(sv[j] * g.sl2 - g.lse2);
        p[j] = pj;
        ds[j] = pj * (dpv[j] - g.d) * g.scale;
    }
}

// ============================================================================
// backward dK, dV: CTA = (key tile, head, batch); q tiles kt..nqt-1
//   TMEM: S [0,128) dP [128,256) dV [256,384) dK [384,512)
// ============================================================================
struct BwdBars {
    uint64_t kv_full, qd_full, qd_empty, s_full, st_free, p_full;
    uint32_t tmem;
};
constexpr size_t kBwdKvSmem = 1024 + 6 * (size_t)kTile + sizeof(BwdBars) + 64;

__global__ void __launch_bounds__(kAttnThreads, 1)
k_attn_bwd_kv(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
              const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
              int S, int H, const float* __restrict__ lse, const float* __restrict__ D,
              bf16* __restrict__ dk, int lddk, bf16* __restrict__ dv, int lddv, float scale) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sK = sm;
    uint8_t* sV = sm + kTile;
    uint8_t* sQ = sm + 2 * kTile;
    uint8_t* sDO = sm + 3 * kTile;
    uint8_t* sP = sm + 4 * kTile;
    uint8_t* sDS = sm + 5 * kTile;
    BwdBars* bar = reinterpret_cast<BwdBars*>(sm + 6 * kTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    const int kt = (int)blockIdx.x;  // key tile
    const int hh = blockIdx.y, b = blockIdx.z;
    const int col = hh * kDh;
    const int n = nqt - kt;  // q tiles kt .. nqt-1
    if (threadIdx.x == 0) {
        mb_init(&bar->kv_full, 1);
        mb_init(&bar->qd_full, 1);
        mb_init(&bar->qd_empty, 1);
        mb_init(&bar->s_full, 1);
        mb_init(&bar->st_free, 128);
        mb_init(&bar->p_full, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) alloc_tmem512(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    if (warp == 0) {
        if (lane == 0) {
            mb_expect_tx(&bar->kv_full, 2 * kTile);
            load_tile(sK, &tk, col, b * S + kt * kT, &bar->kv_full);
            load_tile(sV, &tv, col, b * S + kt * kT, &bar->kv_full);
            for (int i = 0; i < n; ++i) {
                if (i > 0) mb_wait(&bar->qd_empty, (i - 1) & 1);
                const int q0 = b * S + (kt + i) * kT;
                mb_expect_tx(&bar->qd_full, 2 * kTile);
                load_tile(sQ, &tq, col, q0, &bar->qd_full);
                load_tile(sDO, &tdo, col, q0, &bar->qd_full);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mb_wait(&bar->kv_full, 0);
            const uint32_t k = su32(sK), v = su32(sV), q = su32(sQ), dO = su32(sDO);
            const uint32_t p = su32(sP), ds = su32(sDS);
            for (int i = 0; i < n; ++i) {
                mb_wait(&bar->qd_full, i & 1);
                if (i > 0) mb_wait(&bar->st_free, (i - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        tc_mma(tmem, desc_k(q, kb, kk), desc_k(k, kb, kk), kIdescKK, (kb | kk) != 0);
                        tc_mma(tmem + kT, desc_k(dO, kb, kk), desc_k(v, kb, kk), kIdescKK,
                               (kb | kk) != 0);
                    }
                tc_commit(&bar->s_full);
                mb_wait(&bar->p_full, i & 1);
                tc_fence_after();
                // dV += P^T dO, dK += dS^T Q  (M = keys, K = q rows, N = dh)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    tc_mma(tmem + 2 * kT, desc_mn(p, kk), desc_mn(dO, kk), kIdescMM, (i | kk) != 0);
                    tc_mma(tmem + 3 * kT, desc_mn(ds, kk), desc_mn(q, kk), kIdescMM, (i | kk) != 0);
                }
                tc_commit(&bar->qd_empty);
            }
        }
    } else {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        RowGrad g;
        g.sl2 = scale * kLog2e;
        g.scale = scale;
        for (int i = 0; i < n; ++i) {
            const int qt = kt + i;
            const int64_t si = ((int64_t)b * H + hh) * S + qt * kT + r;
            g.lse2 = lse[si] * kLog2e;
            g.d = D[si];
            mb_wait(&bar->s_full, i & 1);
            tc_fence_after();
            const bool diag = i == 0;  // q tile == key tile
#pragma unroll 1
            for (int c = 0; c < kT; c += 16) {
                float sv[16], dpv[16], p[16], ds[16];
                tmem_ld16_nowait(tmem + lane_off + c, sv);
                tmem_ld16_nowait(tmem + lane_off + kT + c, dpv);
                tmem_wait_ld();
                p_ds_chunk(g, sv, dpv, diag, r, c, p, ds);
                store_row16(sP, r, c, p);
                store_row16(sDS, r, c, ds);
            }
            tc_fence_before();
            mb_arrive(&bar->st_free);
            fence_async_smem();
            tc_fence_before();
            mb_arrive(&bar->p_full);
        }
        // the final dV / dK: wait for the last accumulation (qd_empty of i = n-1)
        mb_wait(&bar->qd_empty, (n - 1) & 1);
        tc_fence_after();
        const int64_t row = (int64_t)b * S + kt * kT + r;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {
            bf16* dst = which == 0 ? dv + row * lddv + col : dk + row * lddk + col;
#pragma unroll 1
            for (int c = 0; c < kDh; c += 16) {
                float o[16];
                tmem_ld16(tmem + lane_off + (2 + which) * kT + c, o);
                uint4 u0 = make_uint4(pack2(o[0], o[1]), pack2(o[2], o[3]), pack2(o[4], o[5]),
                                      pack2(o[6], o[7]));
                uint4 u1 = make_uint4(pack2(o[8], o[9]), pack2(o[10], o[11]), pack2(o[12], o[13]),
                                      pack2(o[14], o[15]));
                reinterpret_cast<uint4*>(dst + c)[0] = u0;
                reinterpret_cast<uint4*>(dst + c)[1] = u1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
    }
}

// ============================================================================
// backward dQ: CTA = (q tile, head, batch); key tiles 0..qt, K/V double-buffered
//   TMEM: S [0,128) dP [128,256) dQ [256,384)
// ============================================================================
struct BwdQBars {
    uint64_t qd_full, kv_full[2], kv_empty[2], s_full, st_free, ds_full, ds_free;
    uint32_t tmem;
};
constexpr size_t kBwdQSmem = 1024 + 7 * (size_t)kTile + sizeof(BwdQBars) + 64;

__global__ void __launch_bounds__(kAttnThreads, 1)
k_attn_bwd_q(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
             const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
             int S, int H, const float* __restrict__ lse, const float* __restrict__ D,
             bf16* __restrict__ dq, int lddq, float scale) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sQ = sm;
    uint8_t* sDO = sm + kTile;
    uint8_t* sK = sm + 2 * kTile;  // [2]
    uint8_t* sV = sm + 4 * kTile;  // [2]
    uint8_t* sDS = sm + 6 * kTile;
    BwdQBars* bar = reinterpret_cast<BwdQBars*>(sm + 7 * kTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    const int qt = nqt - 1 - (int)blockIdx.x;
    const int hh = blockIdx.y, b = blockIdx.z;
    const int col = hh * kDh;
    const int nkt = qt + 1;
    if (threadIdx.x == 0) {
        mb_init(&bar->qd_full, 1);
        for (int i = 0; i < 2; ++i) {
            mb_init(&bar->kv_full[i], 1);
            mb_init(&bar->kv_empty[i], 1);
        }
        mb_init(&bar->s_full, 1);
        mb_init(&bar->st_free, 128);
        mb_init(&bar->ds_full, 128);
        mb_init(&bar->ds_free, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) alloc_tmem512(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    if (warp == 0) {
        if (lane == 0) {
            const int q0 = b * S + qt * kT;
            mb_expect_tx(&bar->qd_full, 2 * kTile);
            load_tile(sQ, &tq, col, q0, &bar->qd_full);
            load_tile(sDO, &tdo, col, q0, &bar->qd_full);
            for (int kt = 0; kt < nkt; ++kt) {
                const int s = kt & 1;
                if (kt >= 2) mb_wait(&bar->kv_empty[s], ((kt >> 1) - 1) & 1);
                mb_expect_tx(&bar->kv_full[s], 2 * kTile);
                load_tile(sK + s * kTile, &tk, col, b * S + kt * kT, &bar->kv_full[s]);
                load_tile(sV + s * kTile, &tv, col, b * S + kt * kT, &bar->kv_full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mb_wait(&bar->qd_full, 0);
            const uint32_t q = su32(sQ), dO = su32(sDO), ds = su32(sDS);
            for (int kt = 0; kt < nkt; ++kt) {
                const int s = kt & 1;
                mb_wait(&bar->kv_full[s], (kt >> 1) & 1);
                if (kt > 0) mb_wait(&bar->st_free, (kt - 1) & 1);
                tc_fence_after();
                const uint32_t k = su32(sK + s * kTile), v = su32(sV + s * kTile);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        tc_mma(tmem, desc_k(q, kb, kk), desc_k(k, kb, kk), kIdescKK, (kb | kk) != 0);
                        tc_mma(tmem + kT, desc_k(dO, kb, kk), desc_k(v, kb, kk), kIdescKK,
                               (kb | kk) != 0);
                    }
                tc_commit(&bar->s_full);
                mb_wait(&bar->ds_full, kt & 1);
                tc_fence_after();
                // dQ += dS K   (A = dS K-major over keys, B = K tile MN-major)
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc_mma(tmem + 2 * kT, desc_k(ds, kb, kk), desc_mn(k, kb * 4 + kk), kIdescKM,
                               (kt | kb | kk) != 0);
                tc_commit(&bar->ds_free);
                tc_commit(&bar->kv_empty[s]);
            }
        }
    } else {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int64_t si = ((int64_t)b * H + hh) * S + qt * kT + r;
        RowGrad g;
        g.sl2 = scale * kLog2e;
        g.scale = scale;
        g.lse2 = lse[si] * kLog2e;
        g.d = D[si];
        for (int kt = 0; kt < nkt; ++kt) {
            mb_wait(&bar->s_full, kt & 1);
            if (kt > 0) mb_wait(&bar->ds_free, (kt - 1) & 1);  // dQ MMA of kt-1 read dS
            tc_fence_after();
            const bool diag = kt == qt;
#pragma unroll 1
            for (int c = 0; c < kT; c += 16) {
                float sv[16], dpv[16], p[16], d[16];
                tmem_ld16_nowait(tmem + lane_off + c, sv);
                tmem_ld16_nowait(tmem + lane_off + kT + c, dpv);
                tmem_wait_ld();
                p_ds_chunk(g, sv, dpv, diag, r, c, p, d);
                store_row16(sDS, r, c, d);
            }
            tc_fence_before();
            mb_arrive(&bar->st_free);
            fence_async_smem();
            tc_fence_before();
            mb_arrive(&bar->ds_full);
        }
        mb_wait(&bar->ds_free, (nkt - 1) & 1);
        tc_fence_after();
        bf16* dst = dq + ((int64_t)b * S + qt * kT + r) * lddq + col;
#pragma unroll 1
        for (int c = 0; c < kDh; c += 16) {
            float o[16];
            tmem_ld16(tmem + lane_off + 2 * kT + c, o);
            uint4 u0 = make_uint4(pack2(o[0], o[1]), pack2(o[2], o[3]), pack2(o[4], o[5]),
                                  pack2(o[6], o[7]));
            uint4 u1 = make_uint4(pack2(o[8], o[9]), pack2(o[10], o[11]), pack2(o[12], o[13]),
                                  pack2(o[14], o[15]));
            reinterpret_cast<uint4*>(dst + c)[0] = u0;
            reinterpret_cast<uint4*>(dst + c)[1] = u1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
    }
}

int check_attn(int64_t B, int64_t S, int64_t H, int64_t ld, const void* p) {
    EE_REQUIRE(B > 0 && H > 0 && S > 0 && S % kT == 0, EE_ESHAPE,
               "attention_train: S must be a positive multiple of %d (B=%lld S=%lld H=%lld)", kT,
               (long long)B, (long long)S, (long long)H);
    EE_REQUIRE(ld >= H * kDh && ld % 8 == 0 && p != nullptr && ((uintptr_t)p & 15) == 0, EE_ESHAPE,
               "attention_train: head_dim 128, row stride >= H*128 (multiple of 8), 16-B aligned");
    EE_REQUIRE(B * S < (1ll << 31), EE_ESHAPE, "attention_train: too many rows");
    return EE_OK;
}

template <class K>
void set_smem(K kern, size_t bytes) {
    static bool done[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!done[dev & 15]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        done[dev & 15] = true;
    }
}

}  // namespace

extern "C" int ee_attn_train_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk,
                                 const void* v, int64_t ldv, int64_t B, int64_t S, int64_t H,
                                 void* out, int64_t ldo, float* lse, void* stream) {
    int rc;
    if ((rc = check_attn(B, S, H, ldq, q)) || (rc = check_attn(B, S, H, ldk, k)) ||
        (rc = check_attn(B, S, H, ldv, v)) || (rc = check_attn(B, S, H, ldo, out)))
        return rc;
    EE_REQUIRE(lse != nullptr, EE_ESHAPE, "attention_train: null lse");
    CUtensorMap tq, tk, tv;
    const int64_t rows = B * S, cols = H * kDh;
    if ((rc = make_tmap_bf16_ld(&tq, q, rows, cols, ldq, kT)) ||
        (rc = make_tmap_bf16_ld(&tk, k, rows, cols, ldk, kT)) ||
        (rc = make_tmap_bf16_ld(&tv, v, rows, cols, ldv, kT)))
        return rc;
    set_smem(k_attn_fwd, kFwdSmem);
    const dim3 grid((unsigned)(S / kT), (unsigned)H, (unsigned)B);
    k_attn_fwd<<<grid, kAttnThreads, kFwdSmem, as_stream(stream)>>>(
        tq, tk, tv, (int)S, (int)H, (bf16*)out, (int)ldo, lse, 1.0f / sqrtf((float)kDh));
    return ee_check_launch("attn_train_fwd");
}

extern "C" int ee_attn_train_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk,
                                 const void* v, int64_t ldv, const void* o, int64_t ldo,
                                 const void* dout, int64_t ldd, const float* lse, int64_t B,
                                 int64_t S, int64_t H, void* dq, int64_t lddq, void* dk,
                                 int64_t lddk, void* dv, int64_t lddv, float* dsum, void* stream) {
    int rc;
    if ((rc = check_attn(B, S, H, ldq, q)) || (rc = check_attn(B, S, H, ldk, k)) ||
        (rc = check_attn(B, S, H, ldv, v)) || (rc = check_attn(B, S, H, ldo, o)) ||
        (rc = check_attn(B, S, H, ldd, dout)) || (rc = check_attn(B, S, H, lddq, dq)) ||
        (rc = check_attn(B, S, H, lddk, dk)) || (rc = check_attn(B, S, H, lddv, dv)))
        return rc;
    EE_REQUIRE(lse != nullptr && dsum != nullptr, EE_ESHAPE, "attention_train: null lse / D");
    cudaStream_t s = as_stream(stream);
    const int64_t rows = B * S, cols = H * kDh;
    {
        const int64_t warps = rows * H;
        k_attn_dot<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(
            (const bf16*)dout, (int)ldd, (const bf16*)o, (int)ldo, (int)S, (int)H, (int)rows, dsum);
        if ((rc = ee_check_launch("attn_train_dot"))) return rc;
    }
    CUtensorMap tq, tk, tv, tdo;
    if ((rc = make_tmap_bf16_ld(&tq, q, rows, cols, ldq, kT)) ||
        (rc = make_tmap_bf16_ld(&tk, k, rows, cols, ldk, kT)) ||
        (rc = make_tmap_bf16_ld(&tv, v, rows, cols, ldv, kT)) ||
        (rc = make_tmap_bf16_ld(&tdo, dout, rows, cols, ldd, kT)))
        return rc;
    const float scale = 1.0f / sqrtf((float)kDh);
    const dim3 grid((unsigned)(S / kT), (unsigned)H, (unsigned)B);
    set_smem(k_attn_bwd_kv, kBwdKvSmem);
    k_attn_bwd_kv<<<grid, kAttnThreads, kBwdKvSmem, s>>>(tq, tk, tv, tdo, (int)S, (int)H, lse, dsum,
                                                          (bf16*)dk, (int)lddk, (bf16*)dv,
                                                          (int)lddv, scale);
    if ((rc = ee_check_launch("attn_train_bwd_kv"))) return rc;
    set_smem(k_attn_bwd_q, kBwdQSmem);
    k_attn_bwd_q<<<grid, kAttnThreads, kBwdQSmem, s>>>(tq, tk, tv, tdo, (int)S, (int)H, lse, dsum,
                                                        (bf16*)dq, (int)lddq, scale);
    return ee_check_launch("attn_train_bwd_q");
}
