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
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
        : "memory");
}
// D (TMEM) (+)= A (TMEM: row = lane, K-major bf16 pairs per column) . B (smem)
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
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

// store one 128 x 64 SW128 box of shared memory to (col, row0) of the map's
// matrix (bulk group; the issuing thread waits for the smem reads before exit)
__device__ __forceinline__ void tma_store_box(const CUtensorMap* m, const uint8_t* src, int col,
                                              int row0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
        "r"(su32(src)), "r"(col), "r"(row0)
        : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// epilogue of an fp32 TMEM accumulator (lanes = tile rows) through shared
// memory: this thread's row r, columns [c_lo, c_hi) -> bf16 SW128 boxes at
// `tile`; then the `nthreads` threads that share named barrier `bar_id` sync
// and the first of them stores boxes [box_lo, box_lo + nbox) with TMA.
__device__ __forceinline__ void tmem_epilogue_tma(uint32_t tacc, uint8_t* tile, int r, int c_lo,
                                                  int c_hi, int bar_id, int nthreads, bool issuer,
                                                  const CUtensorMap* m, int col, int row0,
                                                  int box_lo, int nbox) {
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += 16) {
        float o[16];
        tmem_ld16(tacc + c, o);
        store_row16(tile, r, c, o);
    }
    fence_async_smem();
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    if (issuer) {
        for (int x = box_lo; x < box_lo + nbox; ++x)
            tma_store_box(m, tile + x * kBox, col + 64 * x, row0);
        tma_store_commit_wait_read();
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
// forward: CTA = (pair of q tiles A = qt, B = qt - 1, head, batch), key tiles
// 0..qt streamed once for both (K and V through a 3-slot ring).  Two softmax
// warpgroups (A: warps 2-5, B: warps 6-9; warp w owns TMEM lanes of quarter
// w % 4) so that one tile's exponentials overlap the other tile's MMAs:
//   MMA issue order per key tile j:  S_A(j+1), PV_A(j), S_B(j+1), PV_B(j)
//   TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512)
// P goes through shared memory (K-major SW128), so S_t(j+1) can be computed
// while the softmax of tile j still works on its registers.  Lazy
// rescaling: a row keeps its exponent offset m until its running max
// exceeds m by more than 8 (log2 units; P <= 256), so O is rewritten in TMEM
// only when the max jumps.  (Measured alternatives, B200, C2 shape: P in
// TMEM read by a TS-MMA 84 us -- S_t(j+1) then has to wait for PV_t(j);
// event-driven MMA issue 76 us; this order 73 us.)
// ============================================================================
#ifdef EE_TRACE
// per-event timestamps of CTA 0 (events: 0 S issued, 1 PV issued, 2 S seen by
// the softmax, 3 P published) x tile x key tile
__device__ unsigned long long g_fwd_tl[4][2][32];
#define FWD_TL(e, t, j)                                                  \
    do {                                                                 \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 32) \
            g_fwd_tl[e][t][j] = ee_gtime();                              \
    } while (0)
// start / end of every CTA (kernel 0 fwd, 1 bwd_kv, 2 bwd_q; first 2048 CTAs)
__device__ unsigned long long g_cta_tl[3][2048][4];
#define CTA_TL(k, e)                                                                  \
    do {                                                                              \
        const unsigned id = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
        if ((threadIdx.x == ((e) == 0 ? 0u : 32u) || (e) >= 2) && id < 2048) g_cta_tl[k][id][e] = ee_gtime(); \
    } while (0)
#else
#define FWD_TL(e, t, j) do { } while (0)
#define CTA_TL(k, e) do { } while (0)
#endif
constexpr int kFwdThreads = 320;
constexpr int kRing = 3;                 // K / V ring slots (one 32 KB tile each)
constexpr float kRescaleLog2 = 8.f;

struct FwdBars {
    uint64_t q_full, full[kRing], empty[kRing];
    uint64_t s_full[2], s_free[2], p_full[2], o_done[2];
    uint32_t tmem;
};
// Q_A, Q_B, ring, P_A, P_B
constexpr size_t kFwdSmem = 1024 + (4 + kRing) * (size_t)kTile + sizeof(FwdBars) + 64;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(kFwdThreads, 1)
k_attn_fwd(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
           const __grid_constant__ CUtensorMap tv, int S, int H, bf16* __restrict__ out, int ldo,
           float* __restrict__ lse, float scale) {
    extern __shared__ uint8_t smem_raw[];
    CTA_TL(0, 0);
    uint8_t* sm = tc::align1024(smem_raw);
    uint8_t* sQ = sm;                        // [2] (A, B)
    uint8_t* sRing = sm + 2 * kTile;         // [kRing]
    uint8_t* sP = sm + (2 + kRing) * kTile;  // [2]
    FwdBars* bar = reinterpret_cast<FwdBars*>(sm + (4 + kRing) * kTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    // grid (heads, pairs, batch): the pair index is the SLOW dimension, so the
    // longest pairs of every head are dispatched first (longest-processing-
    // time order across the whole grid)
    const int qa = nqt - 1 - 2 * (int)blockIdx.y;
    const int qb = qa - 1;                          // -1: no second tile
    const int hh = blockIdx.x, b = blockIdx.z;
    const int col = hh * kDh;
    const int na = qa + 1, nb = qb + 1;             // key tiles of A / B
    if (threadIdx.x == 0) {
        mb_init(&bar->q_full, 1);
        for (int i = 0; i < kRing; ++i) {
            mb_init(&bar->full[i], 1);
            mb_init(&bar->empty[i], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mb_init(&bar->s_full[t], 1);
            mb_init(&bar->s_free[t], 128);
            mb_init(&bar->p_full[t], 128);
            mb_init(&bar->o_done[t], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) alloc_tmem512(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            mb_expect_tx(&bar->q_full, (nb > 0 ? 2 : 1) * kTile);
            load_tile(sQ, &tq, col, b * S + qa * kT, &bar->q_full);
            if (nb > 0) load_tile(sQ + kTile, &tq, col, b * S + qb * kT, &bar->q_full);
            for (int L = 0; L < 2 * na; ++L) {  // K(0) V(0) K(1) V(1) ...
                const int s = L % kRing, u = L / kRing;
                if (u > 0) mb_wait(&bar->empty[s], (u - 1) & 1);
                mb_expect_tx(&bar->full[s], kTile);
                load_tile(sRing + s * kTile, (L & 1) ? &tv : &tk, col, b * S + (L >> 1) * kT,
                          &bar->full[s]);
            }
        }
    } else if (warp == 1) {
        {
            const bool leader = elect_one();
            // ---------------- MMA issuer ----------------
            mb_wait(&bar->q_full, 0);
            tc_fence_after();
            auto slot = [&](int L) { return L % kRing; };
            auto wait_full = [&](int L) {
                mb_wait(&bar->full[slot(L)], (L / kRing) & 1);
                tc_fence_after();
            };
            auto issue_s = [&](int t, int j) {  // S_t = Q_t K(j)^T
                const uint32_t q = su32(sQ + t * kTile), kk = su32(sRing + slot(2 * j) * kTile);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (leader) tc_mma(tmem + t * kT, desc_k(q, kb, k), desc_k(kk, kb, k), kIdescKK,
                               (kb | k) != 0);
                if (leader) tc_commit(&bar->s_full[t]);
                FWD_TL(0, t, j);
            };
            auto issue_pv = [&](int t, int j) {  // O_t += P_t V(j)
                const uint32_t p = su32(sP + t * kTile), v = su32(sRing + slot(2 * j + 1) * kTile);
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (leader) tc_mma(tmem + (2 + t) * kT, desc_k(p, kb, k), desc_mn(v, kb * 4 + k), kIdescKM,
                               (j | kb | k) != 0);
                if (leader) tc_commit(&bar->o_done[t]);
                FWD_TL(1, t, j);
            };
            wait_full(0);
            issue_s(0, 0);
            if (nb > 0) issue_s(1, 0);
            if (leader) tc_commit(&bar->empty[slot(0)]);
            for (int j = 0; j < na; ++j) {
                const bool nxt = j + 1 < na, bnow = j < nb, bnxt = j + 1 < nb;
                if (nxt) {
                    wait_full(2 * j + 2);
                    mb_wait(&bar->s_free[0], j & 1);  // softmax A has read S_A(j)
                    tc_fence_after();
                    issue_s(0, j + 1);
                }
                wait_full(2 * j + 1);
                mb_wait(&bar->p_full[0], j & 1);
                tc_fence_after();
                issue_pv(0, j);
                if (bnxt) {
                    mb_wait(&bar->s_free[1], j & 1);
                    tc_fence_after();
                    issue_s(1, j + 1);
                }
                if (nxt) if (leader) tc_commit(&bar->empty[slot(2 * j + 2)]);  // K(j+1) read by both S
                if (bnow) {
                    mb_wait(&bar->p_full[1], j & 1);
                    tc_fence_after();
                    issue_pv(1, j);
                }
                if (leader) tc_commit(&bar->empty[slot(2 * j + 1)]);  // V(j) read by both PV
            }
        }
    } else {
        // ---------------- softmax warpgroups ----------------
        const int t = (warp - 2) >> 2;   // 0: tile A, 1: tile B
        const int qt = t == 0 ? qa : qb;
        const int n = t == 0 ? na : nb;
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // tile row = TMEM lane
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const uint32_t tS = tmem + lane_off + t * kT, tO = tmem + lane_off + (2 + t) * kT;
        uint8_t* myP = sP + t * kTile;
        const float sl2 = scale * kLog2e;
        float m = -INFINITY, l = 0.f;
        float v[kT];
        for (int j = 0; j < n; ++j) {
            mb_wait(&bar->s_full[t], j & 1);
            tc_fence_after();
            if (threadIdx.x == 64 + 128 * t) FWD_TL(2, t, j);
#pragma unroll
            for (int c = 0; c < kT; c += 16) tmem_ld16_nowait(tS + c, v + c);
            tmem_wait_ld();
            tc_fence_before();
            mb_arrive(&bar->s_free[t]);
            const bool diag = j == qt;
            float mx = -INFINITY;
            if (diag) {
#pragma unroll
                for (int c = 0; c < kT; ++c) {
                    if (c > r) v[c] = -INFINITY;
                    mx = fmaxf(mx, v[c]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < kT; ++c) mx = fmaxf(mx, v[c]);
            }
            const float mrow = mx * sl2;
            // lazy rescale: move the offset only when the max outgrows it
            const bool move = j == 0 || mrow > m + kRescaleLog2;
            const float mnew = move ? mrow : m;
            const float alpha = j == 0 ? 0.f : ex2(m - mnew);
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < kT; ++c) {
                v[c] = ex2(fmaf(v[c], sl2, -mnew));
                s4[c & 3] += v[c];
            }
            l = fmaf(l, alpha, (s4[0] + s4[1]) + (s4[2] + s4[3]));
            m = mnew;
            if (j > 0) {
                mb_wait(&bar->o_done[t], (j - 1) & 1);  // PV(j-1) done: O stable, P free
                tc_fence_after();
                if (__any_sync(0xffffffffu, move)) {
#pragma unroll 1
                    for (int c = 0; c < kDh; c += 16) {
                        float o[16];
                        tmem_ld16(tO + c, o);
#pragma unroll
                        for (int q = 0; q < 16; ++q) o[q] *= alpha;
                        tmem_st16(tO + c, o);
                    }
                    tmem_wait_st();
                }
            }
#pragma unroll
            for (int c = 0; c < kT; c += 16) store_row16(myP, r, c, v + c);
            fence_async_smem();
            tc_fence_before();
            if (threadIdx.x == 64 + 128 * t) FWD_TL(3, t, j);
            mb_arrive(&bar->p_full[t]);
        }
        if (n > 0) {
            mb_wait(&bar->o_done[t], (n - 1) & 1);
            tc_fence_after();
            const float inv = 1.f / l;
            bf16* orow = out + (int64_t)(b * S + qt * kT + r) * ldo + col;
#pragma unroll 1
            for (int c = 0; c < kDh; c += 16) {
                float o[16];
                tmem_ld16(tO + c, o);
                uint4 u0 = make_uint4(pack2(o[0] * inv, o[1] * inv), pack2(o[2] * inv, o[3] * inv),
                                      pack2(o[4] * inv, o[5] * inv), pack2(o[6] * inv, o[7] * inv));
                uint4 u1 = make_uint4(pack2(o[8] * inv, o[9] * inv), pack2(o[10] * inv, o[11] * inv),
                                      pack2(o[12] * inv, o[13] * inv), pack2(o[14] * inv, o[15] * inv));
                reinterpret_cast<uint4*>(orow + c)[0] = u0;
                reinterpret_cast<uint4*>(orow + c)[1] = u1;
            }
            lse[((int64_t)b * H + hh) * S + qt * kT + r] = (m + log2f(l)) * kLn2;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
        CTA_TL(0, 1);
    }
}

// D[b][h][s] = sum_d dO * O (float32), one warp per (row, head)
// 16 lanes per (row, head): 8 dims each (16-byte loads), xor-butterfly over
// the 16 lanes; a warp covers kDotPairs (row, head) pairs, two at a time
constexpr int kDotPairs = 8;
__global__ void k_attn_dot(const bf16* __restrict__ dout, int ldd, const bf16* __restrict__ o,
                           int ldo, int S, int H, int rows, float* __restrict__ D) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int half = lane >> 4, l16 = lane & 15;
#pragma unroll
    for (int it = 0; it < kDotPairs / 2; ++it) {
        const int pidx = warp * kDotPairs + it * 2 + half;  // (row, head) pair
        const bool ok = pidx < rows * H;
        float sacc = 0.f;
        int row = 0, hh = 0;
        if (ok) {
            row = pidx / H;
            hh = pidx % H;
            const uint4 a = *reinterpret_cast<const uint4*>(dout + (int64_t)row * ldd + hh * kDh + 8 * l16);
            const uint4 c = *reinterpret_cast<const uint4*>(o + (int64_t)row * ldo + hh * kDh + 8 * l16);
            const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 af = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[q]));
                const float2 cf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cw[q]));
                sacc = fmaf(af.x, cf.x, sacc);
                sacc = fmaf(af.y, cf.y, sacc);
            }
        }
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
        if (ok && l16 == 0) {
            const int b = row / S, si = row % S;
            D[((int64_t)b * H + hh) * S + si] = sacc;
        }
    }
}

// ============================================================================
// backward dK, dV: CTA = (key tile, head, batch); q tiles kt..nqt-1, in the
// TRANSPOSED formulation (rows = keys = TMEM lanes), each q tile as two
// 64-row halves h handled by two warpgroups (h = 0: warps 2-5, h = 1: warps
// 6-9) so one half's exponentials overlap the other half's MMAs:
//   S_h^T = K Q_h^T,  dP_h^T = V dO_h^T                    (M = keys, N = 64)
//   P_h^T = exp2(S_h^T c - lse_q),  dS_h^T = P_h^T (dP_h^T - D_q) / sqrt(dh)
//   dV += P_h^T dO_h,  dK += dS_h^T Q_h    (A = P^T / dS^T straight from TMEM)
// P and dS never touch shared memory; (Q_i, dO_i) plus the q tile's lse / D
// stream through a 2-stage ring.  TMEM: S_0^T [0,64) dP_0^T [64,128)
// S_1^T [128,192) dP_1^T [192,256) dV [256,384) dK [384,512); P^T / dS^T
// overwrite the first 32 columns of S^T / dP^T, so S_h^T(i+1) is issued once
// the dV / dK MMAs of half h of tile i completed.
// ============================================================================
#ifndef EE_ATTN_SPLIT_KV
#define EE_ATTN_SPLIT_KV 1
#endif
#ifndef EE_ATTN_SPLIT_Q
#define EE_ATTN_SPLIT_Q 2
#endif
constexpr int kBwdStages = 2;
constexpr int kHalf = kT / 2;
// softmax warps per TMEM lane quarter and half (each takes kHalf / split of
// the half's columns); 2 for dQ, 1 for dK / dV (18 warps cap a thread at 96
// registers, which the dK / dV kernel exceeds)
constexpr int kSplitKv = EE_ATTN_SPLIT_KV, kSplitQ = EE_ATTN_SPLIT_Q;
constexpr int kBwdKvThreads = 64 + 256 * kSplitKv, kBwdQThreads = 64 + 256 * kSplitQ;
struct BwdBars {
    uint64_t kv_full, full[kBwdStages], empty[kBwdStages], s_full[2], p_full[2], mma_done[2];
    uint32_t tmem;
};
constexpr int kBwdStage = 2 * kTile + 2 * kT * 4;  // Q, dO tiles + lse, D of the q tile
constexpr size_t kBwdKvSmem = 1024 + 2 * (size_t)kTile + kBwdStages * (size_t)kBwdStage +
                              sizeof(BwdBars) + 64;
constexpr uint32_t kIdescKK64 = idesc_bf16(128, 64, false, false);  // N = 64 q rows

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kBwdKvThreads, 1)
k_attn_bwd_kv(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
              const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
              const __grid_constant__ CUtensorMap tdk, const __grid_constant__ CUtensorMap tdv,
              int S, int H, const float* __restrict__ lse, const float* __restrict__ D,
              float scale) {
    constexpr int kSplit = kSplitKv, kCols = kHalf / kSplit;
    extern __shared__ uint8_t smem_raw[];
    CTA_TL(1, 0);
    uint8_t* sm = tc::align1024(smem_raw);
    uint8_t* sK = sm;
    uint8_t* sV = sm + kTile;
    uint8_t* sStage = sm + 2 * kTile;  // [kBwdStages] x (Q, dO, lse, D)
    BwdBars* bar = reinterpret_cast<BwdBars*>(sm + 2 * kTile + kBwdStages * kBwdStage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    const int kt = (int)blockIdx.y;  // key tile; slow grid dimension: longest first
    const int hh = blockIdx.x, b = blockIdx.z;
    const int col = hh * kDh;
    const int n = nqt - kt;  // q tiles kt .. nqt-1
    const float* lse_bh = lse + ((int64_t)b * H + hh) * S;
    const float* d_bh = D + ((int64_t)b * H + hh) * S;
    if (threadIdx.x == 0) {
        mb_init(&bar->kv_full, 1);
        for (int i = 0; i < kBwdStages; ++i) {
            mb_init(&bar->full[i], 1);
            mb_init(&bar->empty[i], 1);
        }
        for (int h = 0; h < 2; ++h) {
            mb_init(&bar->s_full[h], 1);
            mb_init(&bar->p_full[h], 128 * kSplit);
            mb_init(&bar->mma_done[h], 1);
        }
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
                const int st = i % kBwdStages, u = i / kBwdStages;
                if (u > 0) mb_wait(&bar->empty[st], (u - 1) & 1);
                uint8_t* g = sStage + st * kBwdStage;
                const int qt = kt + i, q0 = b * S + qt * kT;
                mb_expect_tx(&bar->full[st], kBwdStage);
                load_tile(g, &tq, col, q0, &bar->full[st]);
                load_tile(g + kTile, &tdo, col, q0, &bar->full[st]);
                bulk_g2s(g + 2 * kTile, lse_bh + qt * kT, kT * 4, &bar->full[st]);
                bulk_g2s(g + 2 * kTile + kT * 4, d_bh + qt * kT, kT * 4, &bar->full[st]);
            }
        }
    } else if (warp == 1) {
        {
            const bool leader = elect_one();
            mb_wait(&bar->kv_full, 0);
            tc_fence_after();
            const uint32_t k = su32(sK), v = su32(sV);
            // S_h^T, dP_h^T of tile i: K-major B = rows [64h, 64h+64) of Q / dO
            auto issue_s = [&](int i, int h) {
                const int st = i % kBwdStages;
                const uint32_t q = su32(sStage + st * kBwdStage) + h * kHalf * 128, dO = q + kTile;
                const uint32_t ts = tmem + h * kT;
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (leader) tc_mma(ts, desc_k(k, kb, kk), desc_k(q, kb, kk), kIdescKK64, (kb | kk) != 0);
                        if (leader) tc_mma(ts + kHalf, desc_k(v, kb, kk), desc_k(dO, kb, kk), kIdescKK64,
                               (kb | kk) != 0);
                    }
                if (leader) tc_commit(&bar->s_full[h]);
                FWD_TL(0, h, i);
            };
            // dV += P_h^T dO_h, dK += dS_h^T Q_h  (K = the half's 64 q rows)
            auto issue_acc = [&](int i, int h) {
                const int st = i % kBwdStages;
                const uint32_t q = su32(sStage + st * kBwdStage), dO = q + kTile;
                const uint32_t ts = tmem + h * kT;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (leader) tc_mma_ts(tmem + 2 * kT, ts + kk * 8, desc_mn(dO, 4 * h + kk), kIdescKM,
                              (i | h | kk) != 0);
                    if (leader) tc_mma_ts(tmem + 3 * kT, ts + kHalf + kk * 8, desc_mn(q, 4 * h + kk), kIdescKM,
                              (i | h | kk) != 0);
                }
                if (leader) tc_commit(&bar->mma_done[h]);
                FWD_TL(1, h, i);
            };
            mb_wait(&bar->full[0], 0);
            tc_fence_after();
            issue_s(0, 0);
            issue_s(0, 1);
            if (lane == 0) CTA_TL(1, 2);
            for (int i = 0; i < n; ++i) {
                const bool nxt = i + 1 < n;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    mb_wait(&bar->p_full[h], i & 1);
                    tc_fence_after();
                    issue_acc(i, h);
                    if (h == 1) if (leader) tc_commit(&bar->empty[i % kBwdStages]);  // Q / dO of tile i read
                    if (nxt) {
                        mb_wait(&bar->full[(i + 1) % kBwdStages], ((i + 1) / kBwdStages) & 1);
                        mb_wait(&bar->mma_done[h], i & 1);  // P_h^T / dS_h^T(i) consumed
                        tc_fence_after();
                        issue_s(i + 1, h);
                    }
                }
            }
        }
    } else {
        // kSplit warps per TMEM lane quarter and half: sub-group `sub` owns the
        // half's q columns [sub * kCols, sub * kCols + kCols)
        const int sw = warp - 2;
        const int hf = sw / (4 * kSplit);  // this group's q half
        const int sub = (sw >> 2) % kSplit;
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // key row = TMEM lane
        const int lead = 64 + hf * 128 * kSplit;  // first thread of the half's group
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const uint32_t tS = tmem + lane_off + hf * kT + sub * kCols, tP = tS + kHalf;
        const float sl2 = scale * kLog2e;
        for (int i = 0; i < n; ++i) {
            const float* sLse = reinterpret_cast<const float*>(sStage + (i % kBwdStages) * kBwdStage +
                                                                 2 * kTile) + hf * kHalf + sub * kCols;
            const float* sD = sLse + kT;
            mb_wait(&bar->full[i % kBwdStages], (i / kBwdStages) & 1);  // lse / D landed
            mb_wait(&bar->s_full[hf], i & 1);
            tc_fence_after();
            if (threadIdx.x == lead) FWD_TL(2, hf, i);
            const bool diag = i == 0;  // q tile == key tile: q index < key r is masked
            const int c0 = hf * kHalf + sub * kCols;  // q index of this thread's first column
            float sv[kCols / 16][16], dpv[kCols / 16][16];
#pragma unroll
            for (int cc = 0; cc < kCols / 16; ++cc) {
                tmem_ld16_nowait(tS + cc * 16, sv[cc]);
                tmem_ld16_nowait(tP + cc * 16, dpv[cc]);
            }
            {   // this half's lse -> lse * log2(e) and D -> D / sqrt(dh), in place
                // (one multiply per column instead of one per element)
                const int tw = threadIdx.x - lead;
                if (tw < kHalf) {
                    float* l = const_cast<float*>(sLse) - sub * kCols + tw;
                    float* d = l + kT;
                    *l *= kLog2e;
                    *d *= scale;
                }
                tmem_wait_ld();
                // also orders every sub-group's S^T / dP^T reads before any
                // P^T / dS^T write (they pack over the other sub-group's columns)
                asm volatile("bar.sync %0, %1;" ::"r"(1 + hf), "r"(128 * kSplit) : "memory");
            }
#pragma unroll
            for (int cc = 0; cc < kCols / 16; ++cc) {
                const int c = cc * 16;
                uint32_t pk[8], dk8[8];
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const float4 l4 = *reinterpret_cast<const float4*>(sLse + c + j);
                    const float4 d4 = *reinterpret_cast<const float4*>(sD + c + j);
                    const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
                    float pe[4], de[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        pe[e] = ex2(fmaf(sv[cc][j + e], sl2, -lv[e]));
                        if (diag && c0 + c + j + e < r) pe[e] = 0.f;
                        de[e] = pe[e] * fmaf(dpv[cc][j + e], scale, -dv4[e]);
                    }
                    pk[j / 2] = pack2(pe[0], pe[1]);
                    pk[j / 2 + 1] = pack2(pe[2], pe[3]);
                    dk8[j / 2] = pack2(de[0], de[1]);
                    dk8[j / 2 + 1] = pack2(de[2], de[3]);
                }
                // P^T over the half's S^T columns [(sub*kCols + c)/2, +8), dS^T
                // likewise over dP^T's (all read before the barrier above)
                const uint32_t po = tmem + lane_off + hf * kT + (sub * kCols + c) / 2;
                tmem_st8u(po, pk);
                tmem_st8u(po + kHalf, dk8);
            }
            tmem_wait_st();
            tc_fence_before();
            if (threadIdx.x == lead) FWD_TL(3, hf, i);
            mb_arrive(&bar->p_full[hf]);
        }
        // the final dV (warpgroup 0) / dK (warpgroup 1)
        mb_wait(&bar->mma_done[0], (n - 1) & 1);
        mb_wait(&bar->mma_done[1], (n - 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 64) CTA_TL(1, 3);
        // dV (half 0) / dK (half 1) through the free stage-0 Q / dO buffers
        const int c_lo = sub * (kDh / kSplit), c_hi = c_lo + kDh / kSplit;
        tmem_epilogue_tma(tmem + lane_off + (2 + hf) * kT, sStage + hf * 2 * kBox, r, c_lo, c_hi,
                          3 + hf * kSplit + sub, 128, threadIdx.x == 64 + 32 * (sw & ~3),
                          hf == 0 ? &tdv : &tdk, col, b * S + kt * kT, c_lo / 64, (c_hi - c_lo) / 64);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
        CTA_TL(1, 1);
    }
}

// ============================================================================
// backward dQ: CTA = (q tile, head, batch); key tiles 0..qt through a 2-stage
// K / V ring, each as two 64-key halves h handled by two warpgroups (h = 0:
// warps 2-5, h = 1: warps 6-9) so one half's exponentials overlap the other
// half's MMAs.  S_h = Q K_h^T, dP_h = dO V_h^T (M = q rows = TMEM lanes,
// N = 64), dS_h = P_h (dP_h - D) / sqrt(dh) written as bf16 pairs over the
// first 32 columns of dP_h, dQ += dS_h K_h with A = dS_h straight from TMEM
// (K_h read MN-major).
//   TMEM: S_0 [0,64) dP_0 [64,128) S_1 [128,192) dP_1 [192,256) dQ [256,384)
// ============================================================================
struct BwdQBars {
    uint64_t qd_full, full[kBwdStages], empty[kBwdStages], s_full[2], ds_full[2], mma_done[2];
    uint32_t tmem;
};
constexpr size_t kBwdQSmem = 1024 + 2 * (size_t)kTile + 2 * kBwdStages * (size_t)kTile +
                             sizeof(BwdQBars) + 64;

__global__ void __launch_bounds__(kBwdQThreads, 1)
k_attn_bwd_q(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
             const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
             const __grid_constant__ CUtensorMap tdq, int S, int H,
             const float* __restrict__ lse, const float* __restrict__ D, float scale) {
    constexpr int kSplit = kSplitQ, kCols = kHalf / kSplit;
    extern __shared__ uint8_t smem_raw[];
    CTA_TL(2, 0);
    uint8_t* sm = tc::align1024(smem_raw);
    uint8_t* sQ = sm;
    uint8_t* sDO = sm + kTile;
    uint8_t* sKV = sm + 2 * kTile;  // [kBwdStages] x (K, V)
    BwdQBars* bar = reinterpret_cast<BwdQBars*>(sm + 2 * kTile + 2 * kBwdStages * kTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqt = S / kT;
    const int qt = nqt - 1 - (int)blockIdx.y;  // slow grid dimension: longest first
    const int hh = blockIdx.x, b = blockIdx.z;
    const int col = hh * kDh;
    const int nkt = qt + 1;
    if (threadIdx.x == 0) {
        mb_init(&bar->qd_full, 1);
        for (int i = 0; i < kBwdStages; ++i) {
            mb_init(&bar->full[i], 1);
            mb_init(&bar->empty[i], 1);
        }
        for (int h = 0; h < 2; ++h) {
            mb_init(&bar->s_full[h], 1);
            mb_init(&bar->ds_full[h], 128 * kSplit);
            mb_init(&bar->mma_done[h], 1);
        }
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
                const int st = kt % kBwdStages, u = kt / kBwdStages;
                if (u > 0) mb_wait(&bar->empty[st], (u - 1) & 1);
                uint8_t* g = sKV + st * 2 * kTile;
                mb_expect_tx(&bar->full[st], 2 * kTile);
                load_tile(g, &tk, col, b * S + kt * kT, &bar->full[st]);
                load_tile(g + kTile, &tv, col, b * S + kt * kT, &bar->full[st]);
            }
        }
    } else if (warp == 1) {
        {
            const bool leader = elect_one();
            mb_wait(&bar->qd_full, 0);
            const uint32_t q = su32(sQ), dO = su32(sDO);
            // S_h, dP_h of key tile kt: K-major B = rows [64h, 64h+64) of K / V
            auto issue_s = [&](int kt, int h) {
                const uint32_t k = su32(sKV + (kt % kBwdStages) * 2 * kTile) + h * kHalf * 128,
                               v = k + kTile;
                const uint32_t ts = tmem + h * kT;
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (leader) tc_mma(ts, desc_k(q, kb, kk), desc_k(k, kb, kk), kIdescKK64, (kb | kk) != 0);
                        if (leader) tc_mma(ts + kHalf, desc_k(dO, kb, kk), desc_k(v, kb, kk), kIdescKK64,
                               (kb | kk) != 0);
                    }
                if (leader) tc_commit(&bar->s_full[h]);
            };
            // dQ += dS_h K_h   (K = the half's 64 keys, K tile MN-major)
            auto issue_acc = [&](int kt, int h) {
                const uint32_t k = su32(sKV + (kt % kBwdStages) * 2 * kTile);
                const uint32_t ts = tmem + h * kT;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (leader) tc_mma_ts(tmem + 2 * kT, ts + kHalf + kk * 8, desc_mn(k, 4 * h + kk), kIdescKM,
                              (kt | h | kk) != 0);
                if (leader) tc_commit(&bar->mma_done[h]);
            };
            mb_wait(&bar->full[0], 0);
            tc_fence_after();
            issue_s(0, 0);
            issue_s(0, 1);
            for (int kt = 0; kt < nkt; ++kt) {
                const bool nxt = kt + 1 < nkt;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    mb_wait(&bar->ds_full[h], kt & 1);
                    tc_fence_after();
                    issue_acc(kt, h);
                    if (h == 1) if (leader) tc_commit(&bar->empty[kt % kBwdStages]);  // K / V of tile kt read
                    if (nxt) {
                        mb_wait(&bar->full[(kt + 1) % kBwdStages], ((kt + 1) / kBwdStages) & 1);
                        mb_wait(&bar->mma_done[h], kt & 1);  // dS_h(kt) consumed
                        tc_fence_after();
                        issue_s(kt + 1, h);
                    }
                }
            }
        }
    } else {
        const int sw = warp - 2;
        const int hf = sw / (4 * kSplit);  // this group's key half
        const int sub = (sw >> 2) % kSplit;
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const uint32_t tS = tmem + lane_off + hf * kT + sub * kCols, tP = tS + kHalf;
        const int64_t si = ((int64_t)b * H + hh) * S + qt * kT + r;
        const float sl2 = scale * kLog2e;
        const float lse2 = lse[si] * kLog2e, ds_off = D[si] * scale;
        const int c0 = hf * kHalf + sub * kCols;  // key index of this thread's first column
        for (int kt = 0; kt < nkt; ++kt) {
            mb_wait(&bar->s_full[hf], kt & 1);
            tc_fence_after();
            const bool diag = kt == qt;
            float sv[kCols / 16][16], dpv[kCols / 16][16];
#pragma unroll
            for (int cc = 0; cc < kCols / 16; ++cc) {
                tmem_ld16_nowait(tS + cc * 16, sv[cc]);
                tmem_ld16_nowait(tP + cc * 16, dpv[cc]);
            }
            tmem_wait_ld();
            if (kSplit > 1)  // every sub-group's reads before dS packs over them
                asm volatile("bar.sync %0, %1;" ::"r"(1 + hf), "r"(128 * kSplit) : "memory");
#pragma unroll
            for (int cc = 0; cc < kCols / 16; ++cc) {
                const int c = cc * 16;
                uint32_t dk8[8];
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    float p0 = ex2(fmaf(sv[cc][j], sl2, -lse2));
                    float p1 = ex2(fmaf(sv[cc][j + 1], sl2, -lse2));
                    if (diag && c0 + c + j > r) p0 = 0.f;
                    if (diag && c0 + c + j + 1 > r) p1 = 0.f;
                    dk8[j / 2] = pack2(p0 * fmaf(dpv[cc][j], scale, -ds_off),
                                       p1 * fmaf(dpv[cc][j + 1], scale, -ds_off));
                }
                // dS over the half's dP columns [(sub*kCols + c)/2, +8)
                tmem_st8u(tmem + lane_off + hf * kT + kHalf + (sub * kCols + c) / 2, dk8);
            }
            tmem_wait_st();
            tc_fence_before();
            mb_arrive(&bar->ds_full[hf]);
        }
        {   // dQ: the 2 * kSplit groups take kDh / (2 * kSplit) columns each, through
            // the free K / V stage 0; box x = hf is stored by its half group's first thread
            constexpr int kEpi = kDh / (2 * kSplit);
            const int g = hf * kSplit + sub;
            mb_wait(&bar->mma_done[0], (nkt - 1) & 1);
            mb_wait(&bar->mma_done[1], (nkt - 1) & 1);
            tc_fence_after();
            tmem_epilogue_tma(tmem + lane_off + 2 * kT, sKV, r, g * kEpi, (g + 1) * kEpi, 1 + hf,
                              128 * kSplit, threadIdx.x == 64 + 128 * kSplit * hf, &tdq, col,
                              b * S + qt * kT, hf, 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        free_tmem512(tmem);
        CTA_TL(2, 1);
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

#ifdef EE_TRACE
extern "C" int ee_trace_attn_fwd(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_fwd_tl, sizeof(g_fwd_tl));
}
extern "C" int ee_trace_attn_cta(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_cta_tl, sizeof(g_cta_tl));
}
#endif

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
    const dim3 grid((unsigned)H, (unsigned)((S / kT + 1) / 2), (unsigned)B);
    k_attn_fwd<<<grid, kFwdThreads, kFwdSmem, as_stream(stream)>>>(
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
        const int64_t dwarps = (warps + kDotPairs - 1) / kDotPairs;
        k_attn_dot<<<(unsigned)((dwarps + 7) / 8), 256, 0, s>>>(
            (const bf16*)dout, (int)ldd, (const bf16*)o, (int)ldo, (int)S, (int)H, (int)rows, dsum);
        if ((rc = ee_check_launch("attn_train_dot"))) return rc;
    }
    CUtensorMap tq, tk, tv, tdo, tdq, tdk, tdv;
    if ((rc = make_tmap_bf16_ld(&tq, q, rows, cols, ldq, kT)) ||
        (rc = make_tmap_bf16_ld(&tk, k, rows, cols, ldk, kT)) ||
        (rc = make_tmap_bf16_ld(&tv, v, rows, cols, ldv, kT)) ||
        (rc = make_tmap_bf16_ld(&tdo, dout, rows, cols, ldd, kT)) ||
        (rc = make_tmap_bf16_ld(&tdq, dq, rows, cols, lddq, kT)) ||
        (rc = make_tmap_bf16_ld(&tdk, dk, rows, cols, lddk, kT)) ||
        (rc = make_tmap_bf16_ld(&tdv, dv, rows, cols, lddv, kT)))
        return rc;
    const float scale = 1.0f / sqrtf((float)kDh);
    const dim3 grid((unsigned)H, (unsigned)(S / kT), (unsigned)B);
    set_smem(k_attn_bwd_kv, kBwdKvSmem);
    k_attn_bwd_kv<<<grid, kBwdKvThreads, kBwdKvSmem, s>>>(tq, tk, tv, tdo, tdk, tdv, (int)S, (int)H,
                                                          lse, dsum, scale);
    if ((rc = ee_check_launch("attn_train_bwd_kv"))) return rc;
    set_smem(k_attn_bwd_q, kBwdQSmem);
    k_attn_bwd_q<<<grid, kBwdQThreads, kBwdQSmem, s>>>(tq, tk, tv, tdo, tdq, (int)S, (int)H, lse,
                                                        dsum, scale);
    return ee_check_launch("attn_train_bwd_q");
}
