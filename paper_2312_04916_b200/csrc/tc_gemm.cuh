// Warp-specialised tcgen05 GEMM for sm_100a:   C[M, N] = A[M, K] · B[N, K]^T
// (both operands K-major bf16, fp32 accumulation in tensor memory), with
// pluggable epilogues.  Used by the fused training exit head
// (exit_head_train.cu).
//
//   warp 0 (one lane)  TMA producer: 128x64 A tile + BNx64 B tile per stage
//                      (cp.async.bulk.tensor.2d, SWIZZLE_128B), 4-stage ring
//                      of full/empty mbarriers.
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                      UMMA 128 x BN x 16, accumulator in TMEM; smem stages
//                      are released with tcgen05.commit -> empty[s].
//                      Two TMEM accumulators (2 x BN columns) so the
//                      epilogue of tile i overlaps the MMAs of tile i+1.
//   warps 2..9         epilogue: two warps per TMEM lane quarter, each owning
//                      half of the tile's columns; tcgen05.ld 32x32b.x16
//                      (row = TMEM lane), per-row epilogue functor, then
//                      release the TMEM buffer (tmem_empty mbarrier).
// Persistent grid (one CTA per SM), static tile schedule with M fastest so
// CTAs working at the same time share the B tile in L2.
#pragma once

#include <cuda.h>

#include "ee_common.cuh"

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + kEpiWarps * 32;
constexpr int kABytes = BM * BK * 2;

template <int BN>
struct Cfg {
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
    static constexpr size_t kSmem = (size_t)kStages * kStageBytes + 1024 /*align*/ + 256;
};

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// one elected lane of a converged warp.  The MMA-issuing warps run their
// loops warp-uniformly and only the elected lane issues tcgen05.mma /
// commit: the operand descriptors then live in uniform registers (no
// per-MMA R2UR conversion from a single divergent lane).
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(p));
    return p != 0;
}

// dynamic shared memory rounded up to 1024 B (SW128 atoms) by pointer
// arithmetic on the shared array itself, so the compiler keeps the shared
// address space (an integer round trip would turn every access generic)
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return p + ((1024u - (su32(p) & 1023u)) & 1023u);
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TCW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TCW_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue over one (row, half-tile) of the accumulator.  Two-pass
// epilogues get the whole half-row (BN/2 fp32) in registers with one
// tcgen05.wait (pre() over every chunk, then chunk() over every chunk);
// one-pass epilogues stream it 16 columns at a time.
template <int BN, class Epi>
__device__ __forceinline__ void epilogue_half_row(Epi& epi, uint32_t base, int row, int M, int N,
                                                  int col0) {
    if constexpr (Epi::kTwoPass) {
        float v[BN / 2];
#pragma unroll
        for (int c = 0; c < BN / 2; c += 16) tmem_ld16_nowait(base + c, v + c);
        tmem_wait_ld();
        if (row < M) {
            if (col0 + BN / 2 <= N) {  // interior tile: nvalid folds to 16
#pragma unroll
                for (int c = 0; c < BN / 2; c += 16) epi.pre(row, col0 + c, v + c, 16);
#pragma unroll
                for (int c = 0; c < BN / 2; c += 16) epi.chunk(row, col0 + c, v + c, 16);
            } else {
#pragma unroll
                for (int c = 0; c < BN / 2; c += 16) {
                    const int nvalid = min(16, N - (col0 + c));
                    if (nvalid > 0) epi.pre(row, col0 + c, v + c, nvalid);
                }
#pragma unroll
                for (int c = 0; c < BN / 2; c += 16) {
                    const int nvalid = min(16, N - (col0 + c));
                    if (nvalid > 0) epi.chunk(row, col0 + c, v + c, nvalid);
                }
            }
        }
    } else {
        const bool interior = col0 + BN / 2 <= N;
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 16) {
            float v[16];
            tmem_ld16(base + c, v);
            if (row < M) {
                if (interior) {
                    epi.chunk(row, col0 + c, v, 16);
                } else {
                    const int nvalid = min(16, N - (col0 + c));
                    if (nvalid > 0) epi.chunk(row, col0 + c, v, nvalid);
                }
            }
        }
    }
}

// Canonical UMMA shared-memory descriptors, 128-byte swizzle, version 1.
// K-major tile (rows x 64 k): rows of 128 B, 8-row atoms 1024 B apart (SBO),
//   LBO unused (1); the k-th UMMA_K=16 slice starts 32*k bytes in.
// MN-major tile (64 k rows x MN): 64-element MN chunks of 64 rows x 128 B
//   (8 KB, one TMA box each) -> LBO = 8 KB between MN chunks, SBO = 1 KB
//   between 8-row k groups; the k-th UMMA_K=16 slice starts 2 KB*k in.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t lbo16, uint32_t sbo16) {
    return (uint64_t)((smem_addr & 0x3FFFF) >> 4) | ((uint64_t)lbo16 << 16) |
           ((uint64_t)sbo16 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t tile_addr, int k) {
    return MN ? sw128_desc(tile_addr + k * 2048, 512, 64) : sw128_desc(tile_addr + k * 32, 1, 64);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, majors, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Kernel.  Epi::chunk(row, col0, v[16], nvalid) is called per 16-column chunk
// for every row of the tile (by the epilogue thread owning that row and
// column half, in ascending column order); Epi::begin_tile / end_tile
// bracket one (row, half-tile) with part = 2 * n_tile + half.  An epilogue
// with kTwoPass = true first sees every chunk of the (row, half-tile) through
// Epi::pre (same order), then through Epi::chunk (epilogue_half_row).
// A_MN / B_MN: operand stored MN-major (row-major (K, MN) in HBM) instead of
// K-major; N_FASTEST: tile order (pick so the larger operand is shared by
// the CTAs running at the same time).
template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M,
          int N, int K, Epi epi) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
    const int ntiles = tiles_m * tiles_n;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mb_init(&tfull[b], 1);
            mb_init(&tempty[b], kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tb) : "memory");
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
                const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
                for (int kb = 0; kb < nk; ++kb) {
                    mb_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * C::kStageBytes;
                    mb_expect_tx(&full[s], C::kStageBytes);
                    if (A_MN) {
                        for (int c = 0; c < BM / 64; ++c)
                            tma_load_2d(st + c * 8192, &ta, mb * BM + c * 64, kb * BK, &full[s]);
                    } else {
                        tma_load_2d(st, &ta, kb * BK, mb * BM, &full[s]);
                    }
                    if (B_MN) {
                        for (int c = 0; c < BN / 64; ++c)
                            tma_load_2d(st + kABytes + c * 8192, &tb, nb * BN + c * 64, kb * BK,
                                        &full[s]);
                    } else {
                        tma_load_2d(st + kABytes, &tb, kb * BK, nb * BN, &full[s]);
                    }
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        {
            // ---------------- MMA issuer (warp-uniform, one elected lane issues) ----------------
            const bool leader = elect_one();
            constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mb_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mb_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = su32(smem + s * C::kStageBytes);
                    const uint32_t b0 = a0 + kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        if (leader) tc_mma(d, op_desc<A_MN>(a0, k), op_desc<B_MN>(b0, k), idesc, (kb | k) != 0);
                    if (leader) tc_commit(&empty[s]);  // smem stage free once these MMAs completed
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (leader) tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else {
        // ---------------- epilogue (warps 2..9) ----------------
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int half = (warp - 2) >> 2;  // which half of the tile's columns
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
            const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
            mb_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = mb * BM + row_in_tile;
            const int col0 = nb * BN + half * (BN / 2);
            const int part = nb * 2 + half;  // partial index for per-tile reductions
            epi.begin_tile(row, col0, part, row < M);
            const uint32_t base =
                tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * (BN / 2);
            epilogue_half_row<BN>(epi, base, row, M, N, col0);
            epi.end_tile(row, col0, part, row < M);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(C::kTmemCols));
    }
}

// ---- CTA-pair (cta_group::2) variant -----------------------------------------
// A cluster of two CTAs on one TPC computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (UMMA 256 x BN x 16): CTA r stages rows
// [128 r, 128 r + 128) of A and columns [BN/2 r, BN/2 r + BN/2) of B, so each
// SM streams half of B through shared memory (the 1-CTA 128 x 256 tile is
// shared-memory-bandwidth bound at ~75% of the tensor pipe).  The leader
// (rank 0) issues every MMA; both CTAs' TMA loads complete on the leader's
// full[s] barrier; commits are multicast to both CTAs' empty / tmem_full
// barriers; both CTAs' epilogue warps release the accumulator on the
// leader's tmem_empty.  Each CTA's TMEM holds the accumulator rows of its
// own 128 A rows, so the epilogue is identical to the 1-CTA kernel.
constexpr int kStages2 = 6;

template <int BN>
struct Cfg2 {
    static constexpr int kBBytes = (BN / 2) * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr size_t kSmem = (size_t)kStages2 * kStageBytes + 1024 + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void mb_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at this smem offset in both CTAs of the pair once
// all previously issued MMAs have completed
__device__ __forceinline__ void tc_commit2(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], m;\n\t}" ::"r"(su32(bar))
        : "memory");
}

// split-K: item i -> (split s = i / ntiles, tile t = i % ntiles); split s
// covers k-blocks [nk s / S, nk (s+1) / S); an epilogue with kSplitK = true
// is told the split (set_split) and writes its own partial output
template <class Epi>
__device__ __forceinline__ void epi_set_split(Epi& epi, int s, int t) {
    if constexpr (Epi::kSplitK) epi.set_split(s, t);
}

template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_tc_gemm2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M,
           int N, int K, Epi epi, int splits) {
    using C = Cfg2<BN>;
    constexpr int BM2 = 2 * BM;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * C::kStageBytes);
    uint64_t* empty = full + kStages2;
    uint64_t* tfull = empty + kStages2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int tiles_m = (M + BM2 - 1) / BM2, tiles_n = (N + BN - 1) / BN;
    const int ntiles = tiles_m * tiles_n;
    const int nk = (K + BK - 1) / BK;
    const int nitems = ntiles * splits;
    auto kr = [&](int it, int& k0, int& k1) {
        const int sp = it / ntiles;
        k0 = (int)((int64_t)nk * sp / splits);
        k1 = (int)((int64_t)nk * (sp + 1) / splits);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mb_init(&tfull[b], 1);
            mb_init(&tempty[b], 2 * kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
    __syncthreads();     // (explicit CTA barrier too: the TMEM address is read from smem)
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs) ----------------
            asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tb) : "memory");
            int s = 0;
            uint32_t ph = 0;
            for (int it = cid; it < nitems; it += ncl) {
                const int t = it % ntiles;
                const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
                const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
                const int m0 = mb * BM2 + (int)rank * BM;
                const int n0 = nb * BN + (int)rank * (BN / 2);
                int k0, k1;
                kr(it, k0, k1);
                for (int kb = k0; kb < k1; ++kb) {
                    mb_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * C::kStageBytes;
                    const uint32_t bar = map_rank(&full[s], 0);
                    if (rank == 0) mb_expect_tx(&full[s], 2 * C::kStageBytes);
                    if (A_MN) {
                        for (int c = 0; c < BM / 64; ++c)
                            tma_load_2d_pair(st + c * 8192, &ta, m0 + c * 64, kb * BK, bar);
                    } else {
                        tma_load_2d_pair(st, &ta, kb * BK, m0, bar);
                    }
                    if (B_MN) {
                        for (int c = 0; c < BN / 128; ++c)
                            tma_load_2d_pair(st + kABytes + c * 8192, &tb, n0 + c * 64, kb * BK, bar);
                    } else {
                        tma_load_2d_pair(st + kABytes, &tb, kb * BK, n0, bar);
                    }
                    if (++s == kStages2) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer (leader CTA only; warp-uniform, one lane issues) ----------------
            const bool leader = elect_one();
            constexpr uint32_t idesc = idesc_bf16(BM2, BN, A_MN, B_MN);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            for (int it = cid; it < nitems; it += ncl) {
                int k0, k1;
                kr(it, k0, k1);
                mb_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = k0; kb < k1; ++kb) {
                    mb_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = su32(smem + s * C::kStageBytes);
                    const uint32_t b0 = a0 + kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        if (leader)
                            tc_mma2(d, op_desc<A_MN>(a0, k), op_desc<B_MN>(b0, k), idesc,
                                    (kb > k0 || k > 0) ? 1u : 0u);
                    if (leader) tc_commit2(&empty[s]);  // both CTAs' stage s free once these MMAs completed
                    if (++s == kStages2) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (leader) tc_commit2(&tfull[acc]);  // both CTAs' accumulators ready
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else {
        // ---------------- epilogue (warps 2..9 of both CTAs) ----------------
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row_in_tile = (int)rank * BM + quarter * 32 + lane;
        const uint32_t leader_tempty0 = map_rank(&tempty[0], 0);
        int acc = 0;
        uint32_t aph = 0;
        for (int it = cid; it < nitems; it += ncl) {
            const int t = it % ntiles;
            const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
            const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
            epi_set_split(epi, it / ntiles, t);
            mb_wait(&tfull[acc], aph);
            tc_fence_after();
            const int row = mb * BM2 + row_in_tile;
            const int col0 = nb * BN + half * (BN / 2);
            const int part = nb * 2 + half;
            epi.begin_tile(row, col0, part, row < M);
            const uint32_t base =
                tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * (BN / 2);
            epilogue_half_row<BN>(epi, base, row, M, N, col0);
            epi.end_tile(row, col0, part, row < M);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive_remote(leader_tempty0 + acc * 8);
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // all MMAs consumed, all remote arrivals landed
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(C::kTmemCols));
    }
}

// Host: 2-D bf16 tensor map of a row-major (rows x cols) matrix, box
// (64 cols x box_rows rows), 128-byte swizzle, zero fill out of bounds.
int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);
// the same over a matrix with row stride ld >= cols (elements)
int make_tmap_bf16_ld(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                      int box_rows);

// C[M, N] = A . B^T with A given as (M, K) row-major (A_MN = false) or as
// (K, M) row-major (A_MN = true); B likewise as (N, K) or (K, N).
template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
int launch_tc_gemm(const void* A, const void* B, int M, int N, int K, Epi epi, cudaStream_t s) {
    CUtensorMap ta, tb;
    int rc;
    if ((rc = A_MN ? make_tmap_bf16(&ta, A, K, M, BK) : make_tmap_bf16(&ta, A, M, K, BM))) return rc;
    if ((rc = B_MN ? make_tmap_bf16(&tb, B, K, N, BK) : make_tmap_bf16(&tb, B, N, K, BN))) return rc;
    auto kern = k_tc_gemm<BN, A_MN, B_MN, N_FASTEST, Epi>;
    static bool configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 15]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<BN>::kSmem);
        configured[dev & 15] = true;
    }
    const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    const int grid = tiles < ee_sm_count() ? tiles : ee_sm_count();
    kern<<<grid, kThreads, Cfg<BN>::kSmem, s>>>(ta, tb, M, N, K, epi);
    return ee_check_launch("tc_gemm");
}


// CTA-pair launch: M tiles of 256 rows, grid = 2 x min(tiles, SMs / 2).
template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
int launch_tc_gemm2(const void* A, const void* B, int M, int N, int K, Epi epi, cudaStream_t s,
                    int splits = 1) {
    CUtensorMap ta, tb;
    int rc;
    if ((rc = A_MN ? make_tmap_bf16(&ta, A, K, M, BK) : make_tmap_bf16(&ta, A, M, K, BM))) return rc;
    if ((rc = B_MN ? make_tmap_bf16(&tb, B, K, N, BK) : make_tmap_bf16(&tb, B, N, K, BN / 2)))
        return rc;
    auto kern = k_tc_gemm2<BN, A_MN, B_MN, N_FASTEST, Epi>;
    static bool configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 15]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg2<BN>::kSmem);
        configured[dev & 15] = true;
    }
    const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN) * splits;
    const int pairs = ee_sm_count() / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    kern<<<grid, kThreads, Cfg2<BN>::kSmem, s>>>(ta, tb, M, N, K, epi, splits);
    return ee_check_launch("tc_gemm2");
}

}  // namespace tc
