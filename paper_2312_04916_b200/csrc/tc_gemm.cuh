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
    // + per-epilogue-warp 4 KB staging boxes for TMA-stored epilogues
    static constexpr size_t kStageOff = (size_t)kStages2 * kStageBytes + 1024;  // from aligned base
    static constexpr size_t kSmemStaged = kStageOff + kEpiWarps * 4096 + 1024;
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

// TMA-stored epilogues (Epi::kStaged): each epilogue warp converts its 32
// rows x (128 B of output columns) into a 4 KB SW128 box in shared memory and
// one lane stores the box with cp.async.bulk.tensor (or reduce-adds it:
// Epi::kReduceAdd, float32 accumulation in L2 without a read in the SM) --
// coalesced and asynchronous, instead of 32 scattered row segments per
// store instruction.  Epi::stage(row, col, v[16], nvalid, o[16]) makes the
// 16 outputs of a chunk; the box is clipped to the matrix by the TMA unit.
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <bool kAdd>
__device__ __forceinline__ void tma_store_box2d(const CUtensorMap* m, const void* src, int c0, int r0) {
    if constexpr (kAdd)
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
            "r"(su32(src)), "r"(c0), "r"(r0)
            : "memory");
    else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
                     "r"(su32(src)), "r"(c0), "r"(r0)
                     : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <class Epi>
struct StagedOut {
    static constexpr bool value = false;
};

// Stream-K tail.  A persistent grid of ncl clusters over T tiles leaves
// 1 - (T mod ncl) / ncl of the last wave idle (the 256-tile backbone shapes
// on 74 clusters: 86.5% busy).  With the tail on, the LAST sk_tiles tiles
// (the partial wave plus one whole wave) have their k-blocks, flattened
// tile-major, cut into ncl equal ranges of w blocks, one per cluster; the
// first dp_items tiles run whole, round-robin, afterwards.  A cluster runs
// its range first, one piece per tile touched:
//   * the piece at the range's end, without the tile's last k-block, is a
//     "writer" and runs first: fp32 partial into the cluster's own slot,
//     then a release flag (= this launch's epoch);
//   * the piece at the range's start, with the tile's last k-block but not
//     its first, is the "owner" and runs last: it waits for the flags of
//     the lower clusters holding the tile's earlier k-blocks, adds their
//     partials (cluster order = k order) to its accumulator, then takes the
//     normal epilogue;
//   * pieces covering a whole tile take the normal epilogue.
// Owners only wait on LOWER clusters' first pieces: no deadlock (clusters
// are dispatched in index order) and no wait in practice.  The summation
// order is a function of the shape only, so results are deterministic.
// Used where it measured faster (tools/time_gemm.py, C2 shapes): a partial
// last wave (plain schedule < 92% busy), at least one whole wave, and >= 64
// k-blocks per tile -- e.g. the 256-tile dgrad / wgrad / W2 shapes (-3..-6%);
// not the 2048 x 2048 (64 tiles) weight gradient or K = 2048 forwards, which
// measured 2-10% slower with it.
struct SkArgs {
    int dp_items = 0;           // whole tiles first (all items when sk_tiles == 0)
    int sk_tiles = 0;           // tiles in the stream-K region (0: off)
    int w = 0;                  // k-blocks per cluster range
    float* ws = nullptr;        // [ncl][2 ranks][128 x BN] fp32 partial slots
    uint32_t* flags = nullptr;  // [ncl][2]
    uint32_t epoch = 0;
};
enum : int { kUnitWhole = 0, kUnitWriter = 1, kUnitOwner = 2 };
#ifdef EE_TRACE
// per cluster (<= 80) and unit (<= 12): MMA start / MMA issued / epilogue
// start / epilogue end (%globaltimer), and (tile, k0, k1, role) of the unit
static __device__ unsigned long long g_gemm_tl[80][12][4];
static __device__ int g_gemm_unit[80][12][4];
#define GEMM_TL(c, j, e) do { if ((c) < 80 && (j) < 12) g_gemm_tl[c][j][e] = ee_gtime(); } while (0)
#define GEMM_UNIT(c, j, u)                                                             \
    do {                                                                               \
        if ((c) < 80 && (j) < 12) {                                                    \
            g_gemm_unit[c][j][0] = (u).t; g_gemm_unit[c][j][1] = (u).k0;                \
            g_gemm_unit[c][j][2] = (u).k1; g_gemm_unit[c][j][3] = (u).role;             \
        }                                                                              \
    } while (0)
#else
#define GEMM_TL(c, j, e) do { } while (0)
#define GEMM_UNIT(c, j, u) do { } while (0)
#endif
struct Unit {
    int t, s, k0, k1, role;
};
// the unit sequence of one cluster; the producer, the MMA issuer and the
// epilogue warps each walk an identical copy.  Stream-K pieces come first, in
// the order [writer (range end), whole tiles, owner (range start)], then the
// whole tiles of the round-robin part: the owner waits for the lower
// cluster's FIRST piece, long finished by then.  (Owner second instead of
// last, so that its epilogue overlaps later mainloops, measured slower: the
// short owner piece then waits for the writer's epilogue.)
struct UnitIter {
    int cid, ncl, ntiles, nk, splits;
    const SkArgs* sk;
    int it;       // round-robin cursor
    int j, np;    // stream-K piece cursor / count
    int ta, tb;   // first / last tile of the range (stream-K tile numbering)
    int64_t a, b; // range [a, b) of flattened k-blocks
    __device__ UnitIter(int cid_, int ncl_, int ntiles_, int nk_, int splits_, const SkArgs* sk_)
        : cid(cid_), ncl(ncl_), ntiles(ntiles_), nk(nk_), splits(splits_), sk(sk_), it(cid_), j(0),
          np(0), ta(0), tb(0), a(0), b(0) {
        if (sk->sk_tiles > 0) {
            const int64_t total = (int64_t)sk->sk_tiles * nk;
            a = min((int64_t)cid * sk->w, total);
            b = min((int64_t)(cid + 1) * sk->w, total);
            if (b > a) {
                ta = (int)(a / nk);
                tb = (int)((b - 1) / nk);
                np = tb - ta + 1;
            }
        }
    }
    __device__ bool next(Unit& u) {
        if (j < np) {
            // piece order: tb, ta + 1, ..., tb - 1, ta
            const int t = j == 0 ? tb : (j == np - 1 ? ta : ta + j);
            ++j;
            const int64_t ts = (int64_t)t * nk;
            u.t = sk->dp_items + t;
            u.s = 0;
            u.k0 = (int)((a > ts ? a : ts) - ts);
            u.k1 = (int)((b < ts + nk ? b : ts + nk) - ts);
            u.role = u.k1 < nk ? kUnitWriter : (u.k0 > 0 ? kUnitOwner : kUnitWhole);
            return true;
        }
        const int dp_limit = sk->sk_tiles > 0 ? sk->dp_items : ntiles * splits;
        if (it < dp_limit) {
            u.t = it % ntiles;
            u.s = it / ntiles;
            u.k0 = (int)((int64_t)nk * u.s / splits);
            u.k1 = (int)((int64_t)nk * (u.s + 1) / splits);
            u.role = kUnitWhole;
            it += ncl;
            return true;
        }
        return false;
    }
};
// partial slot layout: [half][quarter][chunk][lane][16] fp32, so the writer's
// and the owner's accesses (same thread -> same row) are contiguous per warp
template <int BN>
__device__ __forceinline__ float* sk_slot(const SkArgs& sk, int cl, uint32_t rank, int half,
                                          int quarter, int lane) {
    // chunk ch, quarter-of-chunk q of this lane at + ch * 512 + q * 128
    return sk.ws + (size_t)(cl * 2 + (int)rank) * (128 * BN) +
           (size_t)((half * 4 + quarter) * (BN / 32)) * 512 + lane * 4;
}
// the 16 partial values of chunk ch (4 coalesced 512-byte warp loads)
template <int BN>
__device__ __forceinline__ void sk_load(const SkArgs& sk, int c, uint32_t rank, int half, int quarter,
                                        int lane, int ch, float4* f) {
    const float4* p =
        reinterpret_cast<const float4*>(sk_slot<BN>(sk, c, rank, half, quarter, lane) + (size_t)ch * 512);
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = __ldcg(p + q * 32);
}
// chunk ch (16 columns) of the half-row += every contributing partial, in
// cluster order
template <int BN>
__device__ __forceinline__ void sk_add(const SkArgs& sk, int c_first, int c_last, uint32_t rank,
                                       int half, int quarter, int lane, int ch, float* v) {
    for (int c = c_first; c <= c_last; ++c) {
        float4 f[4];
        sk_load<BN>(sk, c, rank, half, quarter, lane, ch, f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[4 * q] += f[q].x;
            v[4 * q + 1] += f[q].y;
            v[4 * q + 2] += f[q].z;
            v[4 * q + 3] += f[q].w;
        }
    }
}
__device__ __forceinline__ void sk_wait(const uint32_t* flag, uint32_t epoch) {
    uint32_t f;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
    } while (f != epoch);
}
// the owner's epilogue: epilogue_half_row with the lower clusters' partials
// added to the accumulator chunks first
template <int BN, class Epi>
__device__ __forceinline__ void epilogue_half_row_sk(Epi& epi, uint32_t base, int row, int M, int N,
                                                     int col0, const SkArgs& sk, int c_first,
                                                     int c_last, uint32_t rank, int half,
                                                     int quarter, int lane) {
    if constexpr (Epi::kTwoPass) {
        float v[BN / 2];
#pragma unroll
        for (int c = 0; c < BN / 2; c += 16) tmem_ld16_nowait(base + c, v + c);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 2; c += 16)
            sk_add<BN>(sk, c_first, c_last, rank, half, quarter, lane, c / 16, v + c);
        if (row < M) {
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
    } else {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 16) {
            float v[16];
            tmem_ld16(base + c, v);
            sk_add<BN>(sk, c_first, c_last, rank, half, quarter, lane, c / 16, v);
            if (row < M) {
                const int nvalid = min(16, N - (col0 + c));
                if (nvalid > 0) epi.chunk(row, col0 + c, v, nvalid);
            }
        }
    }
}

// one (row, half-tile) through the warp's staging box: chunks of 16 columns
// from TMEM (+ stream-K partials for an owner), Epi::stage, SW128 box writes,
// one TMA store per 128 B of output columns
template <int BN, class Epi>
__device__ __forceinline__ void epilogue_half_row_staged(Epi& epi, uint32_t base, int row, int M, int N,
                                                         int col0, int row0, uint8_t* stg,
                                                         const CUtensorMap* tout, int lane, bool owner,
                                                         const SkArgs& sk, int c_first, int c_last,
                                                         uint32_t rank, int half, int quarter,
                                                         int osub) {
    using O = typename Epi::OutT;
    constexpr int kBoxCols = 128 / (int)sizeof(O);  // 64 bf16 / 32 fp32 columns
    constexpr int kUnits = 16 * (int)sizeof(O) / 16;  // 16-byte units per chunk
    // owner: the partials of all chunks are loaded a whole box ahead of use
    // (one cluster's partial in registers per chunk of the box; others, rare,
    // are added with plain loads)
    constexpr int kCh = kBoxCols / 16;
    float4 pf[kCh][4];
    if (Epi::kStreamK && owner)
#pragma unroll
        for (int cc = 0; cc < kCh; ++cc) sk_load<BN>(sk, c_first, rank, half, quarter, lane, cc, pf[cc]);
#pragma unroll 1
    for (int g = 0; g < (BN / 2) / kBoxCols; ++g) {
        if (lane == 0) bulk_wait_read0();  // the previous box has left shared memory
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < kCh; ++cc) {
            const int c = g * kBoxCols + cc * 16;
            float v[16];
            tmem_ld16(base + c, v);
            if (Epi::kStreamK && owner) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    v[4 * q] += pf[cc][q].x;
                    v[4 * q + 1] += pf[cc][q].y;
                    v[4 * q + 2] += pf[cc][q].z;
                    v[4 * q + 3] += pf[cc][q].w;
                }
                if (g + 1 < (BN / 2) / kBoxCols)  // next box's chunk cc in flight
                    sk_load<BN>(sk, c_first, rank, half, quarter, lane, c / 16 + kCh, pf[cc]);
                if (c_last > c_first) sk_add<BN>(sk, c_first + 1, c_last, rank, half, quarter, lane, c / 16, v);
            }
            alignas(16) O o[16];
            const int nvalid = row < M ? min(16, N - (col0 + c)) : 0;
            epi.stage(row, col0 + c, v, nvalid, o);
#pragma unroll
            for (int k = 0; k < kUnits; ++k)
                *reinterpret_cast<uint4*>(stg + lane * 128 + (((cc * kUnits + k) ^ (lane & 7)) << 4)) =
                    reinterpret_cast<const uint4*>(o)[k];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && col0 + g * kBoxCols < N && row0 < M) {
            // stacked output (osub > 0): column block j below block j - 1
            const int c = col0 + g * kBoxCols;
            tma_store_box2d<Epi::kReduceAdd>(tout, stg, osub ? c % osub : c,
                                             osub ? (c / osub) * M + row0 : row0);
        }
    }
}

template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_tc_gemm2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M,
           int N, int K, Epi epi, int splits, const __grid_constant__ SkArgs sk,
           const __grid_constant__ CUtensorMap tout, int bsub, int osub) {
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
            UnitIter ui(cid, ncl, ntiles, nk, splits, &sk);
            Unit u;
            while (ui.next(u)) {
                const int t = u.t;
                const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
                const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
                const int m0 = mb * BM2 + (int)rank * BM;
                const int n0 = nb * BN + (int)rank * (BN / 2);
                for (int kb = u.k0; kb < u.k1; ++kb) {
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
                    // stacked B (bsub > 0, launch_tc_gemm2): logical column
                    // block j of width bsub lives below block j - 1 in memory
                    if (B_MN) {
                        const int bc = bsub ? n0 % bsub : n0;
                        const int br = bsub ? (n0 / bsub) * K + kb * BK : kb * BK;
                        for (int c = 0; c < BN / 128; ++c)
                            tma_load_2d_pair(st + kABytes + c * 8192, &tb, bc + c * 64, br, bar);
                    } else {
                        const int kk = kb * BK;
                        tma_load_2d_pair(st + kABytes, &tb, bsub ? kk % bsub : kk,
                                         bsub ? (kk / bsub) * N + n0 : n0, bar);
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
            UnitIter ui(cid, ncl, ntiles, nk, splits, &sk);
            Unit u;
            int jt = 0;
            while (ui.next(u)) {
                const int k0 = u.k0, k1 = u.k1;
                mb_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                if (lane == 0) {
                    GEMM_TL(cid, jt, 0);
                    GEMM_UNIT(cid, jt, u);
                }
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
                if (lane == 0) GEMM_TL(cid, jt, 1);
                ++jt;
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
        UnitIter ui(cid, ncl, ntiles, nk, splits, &sk);
        Unit u;
        int jt = 0;
        while (ui.next(u)) {
            const int t = u.t;
            const int mb = N_FASTEST ? t / tiles_n : t % tiles_m;
            const int nb = N_FASTEST ? t % tiles_n : t / tiles_m;
            epi_set_split(epi, u.s, t);
            mb_wait(&tfull[acc], aph);
            tc_fence_after();
            if (rank == 0 && warp == 2 && lane == 0) GEMM_TL(cid, jt, 2);
            const int row = mb * BM2 + row_in_tile;
            const int col0 = nb * BN + half * (BN / 2);
            const int part = nb * 2 + half;
            const uint32_t base =
                tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * (BN / 2);
            if (Epi::kStreamK && u.role == kUnitWriter) {
                // this piece's fp32 partial into the cluster's slot
                float* dst = sk_slot<BN>(sk, cid, rank, half, quarter, lane);
#pragma unroll 1
                for (int c = 0; c < BN / 2; c += 16) {
                    float v[16];
                    tmem_ld16(base + c, v);
                    float4* d4 = reinterpret_cast<float4*>(dst + (size_t)(c / 16) * 512);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        __stcg(d4 + q * 32, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                }
            } else {
                epi.begin_tile(row, col0, part, row < M);
                const bool owner = Epi::kStreamK && u.role == kUnitOwner;
                int c_first = 0;
                if (owner) {
                    // the lower clusters holding k-blocks [0, k0) of this tile
                    c_first = (int)((int64_t)(t - sk.dp_items) * nk / sk.w);
                    for (int c = c_first; c < cid; ++c) sk_wait(sk.flags + c * 2 + rank, sk.epoch);
                }
                if constexpr (Epi::kStaged) {
                    uint8_t* stg = smem + Cfg2<BN>::kStageOff + (size_t)(warp - 2) * 4096;
                    epilogue_half_row_staged<BN>(epi, base, row, M, N, col0,
                                                 mb * BM2 + (int)rank * BM + quarter * 32, stg, &tout,
                                                 lane, owner, sk, c_first, cid - 1, rank, half, quarter,
                                                 osub);
                } else if (owner) {
                    epilogue_half_row_sk<BN>(epi, base, row, M, N, col0, sk, c_first, cid - 1, rank,
                                             half, quarter, lane);
                } else {
                    epilogue_half_row<BN>(epi, base, row, M, N, col0);
                }
                epi.end_tile(row, col0, part, row < M);
            }
            tc_fence_before();
            __syncwarp();
            if (rank == 0 && warp == 2 && lane == 0) GEMM_TL(cid, jt, 3);
            ++jt;
            if (lane == 0) mb_arrive_remote(leader_tempty0 + acc * 8);
            if (Epi::kStreamK && u.role == kUnitWriter) {
                // every epilogue warp of this CTA has stored its rows: publish
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sk.flags + cid * 2 + rank),
                                 "r"(sk.epoch)
                                 : "memory");
                }
            }
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }
    if constexpr (Epi::kStaged)
        if (warp >= 2 && lane == 0) bulk_wait_all0();  // this warp's output boxes written
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
// output map of a TMA-stored epilogue: (rows x cols) row stride ld, element
// size 2 (bf16) or 4 (float32), box 128 B of columns x 32 rows, SW128
int make_tmap_out(CUtensorMap* map, const void* base, int elem_bytes, int64_t rows, int64_t cols,
                  int64_t ld);

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


// Stream-K workspace of one stream: partial slots + flags, grown on demand;
// the epoch makes flags from earlier launches stale without a memset.
// Launches on one stream are ordered, so one workspace per stream suffices;
// concurrent streams (the weight-gradient side stream) get their own.
struct SkWs {
    int dev = -1;
    cudaStream_t stream = nullptr;
    float* ws = nullptr;
    uint32_t* flags = nullptr;
    size_t ws_bytes = 0;
    int nflags = 0;
    uint32_t epoch = 0;
};
SkWs* sk_workspace(cudaStream_t s, size_t ws_bytes, int nflags);  // nullptr: none free
bool sk_enabled();  // EE_GEMM_STREAMK=0 turns the tail off (A/B)

// the stream-K plan for T tiles of nk k-blocks on ncl clusters (sk_tiles = 0:
// plain round-robin); see SkArgs
inline SkArgs sk_plan(int tiles, int nk, int ncl) {
    SkArgs a;
    if (ncl <= 0 || tiles % ncl == 0 || tiles < ncl || nk < 64 || !sk_enabled()) return a;
    const int full = tiles / ncl, rem = tiles % ncl;
    if ((double)tiles / ((double)(full + 1) * ncl) >= 0.92) return a;  // tail already small
    a.sk_tiles = rem + (full >= 1 ? ncl : 0);  // the partial wave plus one whole wave
    a.dp_items = tiles - a.sk_tiles;
    a.w = (int)(((int64_t)a.sk_tiles * nk + ncl - 1) / ncl);
    if (a.w < 8) a.sk_tiles = 0;  // short k: not worth the partials
    return a;
}

// CTA-pair launch: M tiles of 256 rows, grid = 2 x min(tiles, SMs / 2), or
// 2 x SMs / 2 with the stream-K tail (epilogues with kStreamK, splits == 1,
// not while the stream is being captured: the epoch is a launch argument).
//
// Stacked operands (several same-shape matrices adjacent in memory, e.g. the
// q / k / v projections in the flat parameter buffer), one GEMM for all:
//   bsub > 0: B is the logical concatenation along its N (B_MN) or K (K-major)
//     axis of blocks of width bsub, block j stored below block j - 1
//     (B_MN: (K, bsub) blocks; K-major: (N, bsub) blocks);
//   osub > 0: the output likewise, (M, osub) blocks (staged epilogues only).
// Tiles and TMA boxes never straddle a block: bsub / osub multiples of 128
// (and K % 64 == 0 for a stacked B_MN, M % 32 == 0 for a stacked output).
template <int BN, bool A_MN, bool B_MN, bool N_FASTEST, class Epi>
int launch_tc_gemm2(const void* A, const void* B, int M, int N, int K, Epi epi, cudaStream_t s,
                    int splits = 1, int bsub = 0, int osub = 0) {
    CUtensorMap ta, tb;
    int rc;
    EE_REQUIRE(bsub == 0 || (bsub % 128 == 0 && (B_MN ? N % bsub == 0 && K % BK == 0 : K % bsub == 0)),
               EE_ESHAPE, "tc_gemm2: bad stacked B (bsub %d, N %d, K %d)", bsub, N, K);
    EE_REQUIRE(osub == 0 || (Epi::kStaged && osub % 128 == 0 && N % osub == 0 && M % 32 == 0),
               EE_ESHAPE, "tc_gemm2: bad stacked output (osub %d, M %d, N %d)", osub, M, N);
    if ((rc = A_MN ? make_tmap_bf16(&ta, A, K, M, BK) : make_tmap_bf16(&ta, A, M, K, BM))) return rc;
    if (bsub)
        rc = B_MN ? make_tmap_bf16(&tb, B, (int64_t)(N / bsub) * K, bsub, BK)
                  : make_tmap_bf16(&tb, B, (int64_t)(K / bsub) * N, bsub, BN / 2);
    else
        rc = B_MN ? make_tmap_bf16(&tb, B, K, N, BK) : make_tmap_bf16(&tb, B, N, K, BN / 2);
    if (rc) return rc;
    auto kern = k_tc_gemm2<BN, A_MN, B_MN, N_FASTEST, Epi>;
    static bool configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    constexpr size_t kSmemL = Epi::kStaged ? Cfg2<BN>::kSmemStaged : Cfg2<BN>::kSmem;
    if (!configured[dev & 15]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemL);
        configured[dev & 15] = true;
    }
    CUtensorMap tout;
    memset(&tout, 0, sizeof(tout));
    if constexpr (Epi::kStaged) {
        if ((rc = osub ? epi.out_map(&tout, (N / osub) * M, osub) : epi.out_map(&tout, M, N)))
            return rc;
    }
    const int tiles1 = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
    const int tiles = tiles1 * splits;
    const int pairs = ee_sm_count() / 2;
    int ncl = tiles < pairs ? tiles : pairs;
    SkArgs sk;
    if constexpr (Epi::kStreamK) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (splits == 1 && cudaStreamIsCapturing(s, &cap) == cudaSuccess &&
            cap == cudaStreamCaptureStatusNone) {
            sk = sk_plan(tiles1, (K + BK - 1) / BK, pairs);
            if (sk.sk_tiles > 0) {
                SkWs* w = sk_workspace(s, (size_t)pairs * 2 * 128 * BN * sizeof(float), pairs * 2);
                if (w) {
                    sk.ws = w->ws;
                    sk.flags = w->flags;
                    sk.epoch = ++w->epoch;
                    ncl = pairs;
                } else {
                    sk = SkArgs{};
                }
            }
        }
    }
    kern<<<2 * ncl, kThreads, kSmemL, s>>>(ta, tb, M, N, K, epi, splits, sk, tout, bsub, osub);
    return ee_check_launch("tc_gemm2");
}

}  // namespace tc
