// TMA-bulk-fed, row-stable GEMV for bf16 weights in the tiled layout
// (pack.cu) on sm_100a.
//
//   v[r, n] = sum_k x[r, k] * W[n, k]     (x: bf16 rows, W: tiled bf16)
//
// Structure (persistent CTA, 5 warps, 2 CTAs per SM):
//   warp 4, one elected lane = producer.  Streams the CTA's weight tiles
//     through a ring of kStages shared-memory stages; a stage is one 16 x 512
//     bf16 block = ONE 16 KB bulk async copy
//     (`cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes`,
//     SASS UBLKCP) completing on the stage's `wfull` mbarrier.  Weights never
//     depend on the previous kernel, so the producer fills the whole ring
//     BEFORE `griddepcontrol.wait`: under programmatic dependent launch the
//     next GEMV's weights stream in while the previous kernel drains.  After
//     the wait it also copies the stage's chunk of the activation rows
//     (`xfull` mbarrier), so consumers never touch global memory.
//   warps 0..3 = consumers: wait wfull[s] and xfull[s], build m16n8k16
//     fragments with 16-B LDS (weights XOR-swizzled per row by the packer,
//     activations padded: both conflict-free), mma.sync into fp32, release
//     empty[s].  The 16 k-blocks of a stage are split round-robin over the 4
//     warps and the 4 partial tiles are summed in warp order, so the
//     reduction order of every output depends only on (n, k), never on the
//     number of rows m (row-stable, the `dot_rows` contract of
//     eepipe/_pykernels.py:14-17).
#pragma once

#include "ee_common.cuh"

namespace tma_gemv {

constexpr int kConsumers = 4;
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kRows = 16;
constexpr int kStages = 4;
constexpr int KS = kTiledKS;                  // 512 k per stage
constexpr int kWBytes = kRows * KS * 2;       // 16 KB weight block per stage
constexpr int kXPitch = KS * 2 + 16;          // padded activation row
constexpr int kMaxCols = 16;                  // activation rows per work item (NB = 2)

// a stage = the 16 KB weight block + the activation rows it serves (xrows
// reserved: 8 NB by default; a single-row pass reserves 1 and spends the
// room on a deeper weight ring)
__host__ __device__ constexpr int stage_bytes(int NB, int xrows = 0) {
    return kWBytes + (xrows ? xrows : 8 * NB) * kXPitch;
}
__host__ inline size_t smem_bytes(int NB, int stages = kStages, int xrows = 0) {
    return (size_t)stages * stage_bytes(NB, xrows) + 3 * stages * 8 +
           (size_t)kConsumers * kRows * kMaxCols * 4 + kMaxCols * 4 + 64;
}

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Weight stages carry an L2 evict-first hint: every weight byte is read once
// per pass, so its lines should go first and leave the L2 to the data that
// is re-read (the KV cache rows of earlier positions, the activation rows).
// EE_GEMV_EVICT_FIRST=0 (profiling A/B builds) drops the hint.
#ifndef EE_GEMV_EVICT_FIRST
#define EE_GEMV_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
#if EE_GEMV_EVICT_FIRST
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
        "[%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    (void)pol;
    bulk_g2s(dst, src, bytes, bar);
#endif
}
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
}
__device__ __forceinline__ uint4 lds16(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(addr));
    return r;
}

// Folded RMSNorm: when `ssq` is given, the activation rows are the RAW
// residual rows (bf16 copy) and the norm weight has been folded into W's
// columns at pack time; the consumers compute 1/rms per row from the
// per-16-column sum-of-squares partials ssq[row][0..K/16) (summed in a fixed
// order) and the epilogue scales each output by it:
//   sum_k W[n,k] (x[k] w[k] / rms) = (1/rms) sum_k (W[n,k] w[k]) x[k].
struct RowNorm {
    const float* ssq;  // (rows, K/16) or nullptr
    float eps;
};

// Work item i -> tile = i / groups, column group = i % groups; a CTA takes
// items blockIdx.x, +gridDim.x, ...  Epi provides tile(red, n0, r0, N, m,
// cols, inv) and finish(), both called by the 128 consumer threads (inv is
// the per-column 1/rms or nullptr).  K must be a multiple of 512, W in the
// tiled layout.
template <int NB, class Epi, int kStages = tma_gemv::kStages, int kXRows = 0>
__device__ __forceinline__ void gemv_body(const bf16* __restrict__ W, int N, int K,
                                          const bf16* __restrict__ X, int64_t ldx, int m,
                                          RowNorm rn, Epi& epi) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int cols = kXRows ? kXRows : 8 * NB;  // rows per work item
    constexpr int sbytes = stage_bytes(NB, kXRows);
    uint8_t* ring = smem;
    uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + kStages * sbytes);
    uint64_t* xfull = wfull + kStages;
    uint64_t* empty = xfull + kStages;
    float* red = reinterpret_cast<float*>(empty + kStages);  // [kConsumers][16][kMaxCols]
    float* inv = red + kConsumers * kRows * kMaxCols;        // [kMaxCols]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = (N + kRows - 1) / kRows;
    const int groups = (m + cols - 1) / cols;
    const int items = tiles * groups;
    const int nks = K / KS;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&xfull[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_trigger_dev();
    // trace slots (profiling builds): 4 per kernel kind, qkv / wo / w1 / w2
    const int tslot = 4 * (N == 3 * K ? 0 : N == K ? 1 : N == 4 * K ? 2 : 3);
    (void)tslot;
    EE_TMIN(tslot);

    if (warp == kConsumers) {
        // ---------------- producer (one lane) ----------------
        if (lane != 0) return;
        const int my_items =
            items > (int)blockIdx.x ? (items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const int total = my_items * nks;
        const uint64_t pol = policy_evict_first();
        auto issue_w = [&](int q) {
            const int it = (int)blockIdx.x + (q / nks) * (int)gridDim.x;
            const int ks = q % nks;
            const int slot = q % kStages;
            mbar_expect_tx(&wfull[slot], kWBytes);
            bulk_g2s_hint(ring + slot * sbytes, W + ((int64_t)(it / groups) * nks + ks) * (kRows * KS),
                          kWBytes, &wfull[slot], pol);
        };
        auto issue_x = [&](int q) {
            const int it = (int)blockIdx.x + (q / nks) * (int)gridDim.x;
            const int ks = q % nks;
            const int slot = q % kStages;
            const int r0 = (it % groups) * cols;
            const int mr = min(cols, m - r0);
            uint8_t* dst = ring + slot * sbytes + kWBytes;
            mbar_expect_tx(&xfull[slot], (uint32_t)(mr * KS * 2));
            for (int r = 0; r < mr; ++r)
                bulk_g2s(dst + r * kXPitch, X + (int64_t)(r0 + r) * ldx + (int64_t)ks * KS, KS * 2,
                         &xfull[slot]);
        };
        // 1) weights for the first ring's worth of stages, before the
        //    dependency on the previous kernel is resolved
        const int pre = min(total, kStages);
        for (int q = 0; q < pre; ++q) issue_w(q);
        // 2) activations are produced by the previous kernel
        pdl_wait_dev();
        for (int q = 0; q < pre; ++q) issue_x(q);
        // 3) steady state
        for (int q = pre; q < total; ++q) {
            mbar_wait(&empty[q % kStages], ((q / kStages) - 1) & 1);
            issue_w(q);
            issue_x(q);
        }
        return;
    }

    // ---------------- consumers ----------------
    pdl_wait_dev();  // epilogues read/write buffers shared with the predecessor
    EE_TMIN(tslot + 2);
    const int g = lane >> 2, t = lane & 3;
    const uint32_t ring_u32 = smem_u32(ring);
    int q = 0;
    int cur_grp = -1;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        // row groups fastest: the CTAs that process one weight tile for the
        // different row groups run concurrently, so the tile is fetched from
        // HBM once and served from L2 to the others (multi-row prefill)
        const int tile = it / groups;
        const int grp = it % groups;
        const int n0 = tile * kRows;
        const int r0 = grp * cols;
        const int mr = min(cols, m - r0);
        if (rn.ssq != nullptr && grp != cur_grp) {
            // 1/rms of this group's rows: warp w sums rows w, w+4, ... ;
            // lane-strided partials then a fixed xor butterfly
            const int nt = K >> 4;
            for (int c = warp; c < cols; c += kConsumers) {
                const float* sr = rn.ssq + (int64_t)min(r0 + c, m - 1) * nt;
                float s = 0.f;
                for (int i = lane; i < nt; i += 32) s += sr[i];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) inv[c] = 1.0f / sqrtf(s / (float)K + rn.eps);
            }
            cur_grp = grp;
            // visibility of inv[] to all consumers is ensured by the
            // consumers_sync() preceding the epilogue
        }
        float acc[NB][4];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.f;
        // activation rows >= mr were not copied: read row mr-1 instead
        // (columns are independent inside the MMA; those outputs are dropped)
        uint32_t xoff[NB];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) xoff[nb] = kWBytes + min(nb * 8 + g, mr - 1) * kXPitch + t * 16;
        const uint32_t wa = g * (KS * 2), wb = (g + 8) * (KS * 2);

        for (int ks = 0; ks < nks; ++ks, ++q) {
            const int slot = q % kStages;
            const uint32_t par = (q / kStages) & 1;
            mbar_wait(&wfull[slot], par);
            mbar_wait(&xfull[slot], par);
            const uint32_t st = ring_u32 + slot * sbytes;
#pragma unroll
            for (int i = 0; i < KS / 32 / kConsumers; ++i) {
                const int kb = warp + i * kConsumers;
                const uint32_t sw = (uint32_t)(((kb * 4 + t) ^ g) * 16);  // swizzled chunk
                const uint4 a = lds16(st + wa + sw);
                const uint4 b = lds16(st + wb + sw);
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const uint4 x = lds16(st + xoff[nb] + kb * 64);
                    mma_16816(acc[nb], a.x, b.x, a.y, b.y, x.x, x.y);
                    mma_16816(acc[nb], a.z, b.z, a.w, b.w, x.z, x.w);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
        // cross-warp reduction in fixed warp order, then the epilogue
        float* rw = red + warp * kRows * kMaxCols;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            rw[g * kMaxCols + nb * 8 + 2 * t] = acc[nb][0];
            rw[g * kMaxCols + nb * 8 + 2 * t + 1] = acc[nb][1];
            rw[(g + 8) * kMaxCols + nb * 8 + 2 * t] = acc[nb][2];
            rw[(g + 8) * kMaxCols + nb * 8 + 2 * t + 1] = acc[nb][3];
        }
        consumers_sync();
        epi.tile(red, n0, r0, N, m, cols, rn.ssq != nullptr ? inv : nullptr);
        consumers_sync();
    }
    epi.finish();
    EE_TMAX(tslot + 1);
}

}  // namespace tma_gemv
