// Multi-row (prefill) backbone GEMM on tcgen05 for weights in the TILED
// layout (pack.cu), replacing the GEMV when a pass carries many rows (the
// prompt prefill of `generate_kv_recompute` / `generate_pipeline`,
// eepipe/inference.py:331-334: every prompt row through every layer).
//
//   part[s][r][n] = sum_{k in split s} W[n, k] x[r, k]        (swap-AB GEMM)
//
// * A = 128 weight rows x 64 k per stage, read straight from the tiled
//   layout by a 5-D TMA box {64 k, 1 segment, 16 rows, 1 stage, 8 tiles}:
//   the packer's in-row chunk permutation (c ^ (row & 7)) IS the 128-byte
//   swizzle of a K-major UMMA operand, so the box lands in shared memory in
//   the canonical SW128 layout with SWIZZLE_NONE and no repacking.
// * B = 64 activation rows x 64 k (bf16 row-major, SW128 TMA box).
// * tcgen05.mma.cta_group::1.kind::f16, M = 128 (weights) x N = 64 (rows),
//   fp32 accumulators in TMEM (two 64-column buffers), warp-specialised
//   (TMA producer / single-thread MMA issuer / 4 epilogue warps), 6-stage
//   ring, persistent over (weight tile, row group, k split) work items.
// * Split-K fills the SMs for the narrow matrices (Wo, W2: 32 weight tiles).
//   The epilogue writes fp32 partials; k_prefill_apply then reduces the
//   splits in fixed order and applies the layer epilogue (1/rms of the
//   folded RMSNorm, GELU, residual + row statistics, q / K / V cache
//   writes), so the result is deterministic.
// Rows of a prefill pass only ever go through this kernel (in both
// inference modes), so the GEMV's row-stability contract is unaffected.
#include <cuda.h>

#include "tc_gemm.cuh"

namespace {

constexpr int PBM = 128;  // weight rows per tile
constexpr int PBN = 64;   // activation rows per tile
constexpr int PBK = 64;
constexpr int kPStages = 6;
constexpr int kPABytes = PBM * PBK * 2;  // 16 KB
constexpr int kPBBytes = PBN * PBK * 2;  // 8 KB
constexpr int kPStageBytes = kPABytes + kPBBytes;
constexpr int kPThreads = 6 * 32;  // producer, MMA, 4 epilogue warps
constexpr size_t kPSmem = (size_t)kPStages * kPStageBytes + 1024 + 256;
constexpr int kPTmemCols = 2 * PBN;

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(tc::su32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(tc::su32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kPThreads, 1)
k_prefill_gemm(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
               int N, int m, int K, int splits, float* __restrict__ part) {
    using namespace tc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = tc::align1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes);
    uint64_t* empty = full + kPStages;
    uint64_t* tfull = empty + kPStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = (N + PBM - 1) / PBM;
    const int groups = (m + PBN - 1) / PBN;
    const int items = tiles * groups * splits;
    const int nkb = K / PBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mb_init(&tfull[b], 1);
            mb_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(tmem_slot)),
                     "n"(kPTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger_dev();

    // work item -> (weight tile, row group, split); splits fastest, then
    // groups, so concurrent CTAs share weight tiles in L2
    auto decode = [&](int it, int& tile, int& grp, int& sp) {
        sp = it % splits;
        grp = (it / splits) % groups;
        tile = it / (splits * groups);
    };
    auto krange = [&](int sp, int& k0, int& k1) {
        k0 = (int)((int64_t)nkb * sp / splits);
        k1 = (int)((int64_t)nkb * (sp + 1) / splits);
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tw) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tx) : "memory");
            pdl_wait_dev();  // activations come from the previous kernel
            int s = 0;
            uint32_t ph = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                int tile, grp, sp, k0, k1;
                decode(it, tile, grp, sp);
                krange(sp, k0, k1);
                for (int kb = k0; kb < k1; ++kb) {
                    mb_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * kPStageBytes;
                    mb_expect_tx(&full[s], kPStageBytes);
                    tma_load_5d(st, &tw, 0, kb & 7, 0, kb >> 3, tile * (PBM / 16), &full[s]);
                    tma_load_2d(st + kPABytes, &tx, kb * PBK, grp * PBN, &full[s]);
                    if (++s == kPStages) {
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
            constexpr uint32_t idesc = idesc_bf16(PBM, PBN, false, false);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                int tile, grp, sp, k0, k1;
                decode(it, tile, grp, sp);
                krange(sp, k0, k1);
                mb_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * PBN;
                for (int kb = k0; kb < k1; ++kb) {
                    mb_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = su32(smem + s * kPStageBytes);
                    const uint32_t b0 = a0 + kPABytes;
#pragma unroll
                    for (int k = 0; k < PBK / 16; ++k)
                        if (leader)
                            tc_mma(d, op_desc<false>(a0, k), op_desc<false>(b0, k), idesc,
                                   (kb > k0 || k > 0) ? 1u : 0u);
                    if (leader) tc_commit(&empty[s]);
                    if (++s == kPStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (leader) tc_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> fp32 partials ----------------
        const int quarter = warp & 3;
        int acc = 0;
        uint32_t aph = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int tile, grp, sp;
            decode(it, tile, grp, sp);
            mb_wait(&tfull[acc], aph);
            tc_fence_after();
            const int n = tile * PBM + quarter * 32 + lane;
            const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16) + acc * PBN;
            float* dst = part + (int64_t)sp * m * N;
#pragma unroll 1
            for (int c = 0; c < PBN; c += 16) {
                float v[16];
                tmem_ld16(base + c, v);
                const int r0 = grp * PBN + c;
                if (n < N) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (r0 + j < m) dst[(int64_t)(r0 + j) * N + n] = v[j];
                }
            }
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
                     "n"(kPTmemCols));
    }
}

// ---- reduce the splits in order + the layer epilogue ---------------------------
enum PrefillEpi { kEpiQKV = 0, kEpiGelu = 1, kEpiResidual = 2 };

struct ApplyArgs {
    const float* part;
    int splits, m, N, K;
    const float* ssq_in;  // folded-norm row statistics (K/16 per row) or null
    float eps;
    // epilogue outputs
    float* q;
    bf16* kc;
    bf16* vc;
    const int32_t* pos;
    int h;
    bf16* out_bf16;  // GELU output (m x N)
    float* x;        // residual rows (m x N), updated in place
    bf16* xb;        // bf16 copy of x
    float* ssq_out;  // new row statistics (N/16 per row)
};

// one CTA per (row, 4096-column chunk); 256 threads x 16 consecutive columns
template <int EPI>
__global__ void __launch_bounds__(256) k_prefill_apply(ApplyArgs a) {
    const int r = blockIdx.y;
    const int lane = threadIdx.x & 31;
    __shared__ float s_inv;
    pdl_wait_dev();
    pdl_trigger_dev();
    if (EPI != kEpiResidual) {
        if (threadIdx.x < 32) {
            float s = 0.f;
            if (a.ssq_in) {
                const int nt = a.K >> 4;
                const float* sr = a.ssq_in + (int64_t)r * nt;
                for (int i = lane; i < nt; i += 32) s += sr[i];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            }
            if (lane == 0) s_inv = a.ssq_in ? 1.0f / sqrtf(s / (float)a.K + a.eps) : 1.0f;
        }
        __syncthreads();
    }
    const float inv = EPI != kEpiResidual ? s_inv : 1.0f;
    const int n0 = (blockIdx.x * 256 + threadIdx.x) * 16;
    if (n0 >= a.N) return;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.f;
    for (int sp = 0; sp < a.splits; ++sp) {
        const float4* p = reinterpret_cast<const float4*>(a.part + ((int64_t)sp * a.m + r) * a.N + n0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4 f = p[j];
            v[4 * j] += f.x;
            v[4 * j + 1] += f.y;
            v[4 * j + 2] += f.z;
            v[4 * j + 3] += f.w;
        }
    }
    if (EPI == kEpiQKV) {
        const int h = a.h;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int n = n0 + j;
            const float y = v[j] * inv;
            if (n < h) a.q[(int64_t)r * h + n] = y;
            else if (n < 2 * h) a.kc[(int64_t)a.pos[r] * h + (n - h)] = __float2bfloat16_rn(y);
            else a.vc[(int64_t)a.pos[r] * h + (n - 2 * h)] = __float2bfloat16_rn(y);
        }
    } else if (EPI == kEpiGelu) {
        bf16* o = a.out_bf16 + (int64_t)r * a.N + n0;
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = __float2bfloat16_rn(gelu_erf(v[j] * inv));
    } else {
        float* xr = a.x + (int64_t)r * a.N + n0;
        bf16* xbr = a.xb + (int64_t)r * a.N + n0;
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float nv = xr[j] + v[j];
            xr[j] = nv;
            xbr[j] = __float2bfloat16_rn(nv);
            s = fmaf(nv, nv, s);  // the 16 squares in ascending column order
        }
        a.ssq_out[(int64_t)r * (a.N >> 4) + (n0 >> 4)] = s;
    }
}

int make_tmap_tiled_w(CUtensorMap* map, const void* W, int64_t N, int64_t K) {
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return ee_fail(EE_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        encode = (EncodeFn)fn;
    }
    const int64_t nks = K / kTiledKS, ntiles = (N + 15) / 16;
    // dims (innermost first): 64 k | 8 segments | 16 rows | k-stages | 16-row tiles
    cuuint64_t dims[5] = {64, 8, 16, (cuuint64_t)nks, (cuuint64_t)ntiles};
    cuuint64_t strides[4] = {128, 1024, 16384, (cuuint64_t)nks * 16384};
    cuuint32_t box[5] = {64, 1, 16, 1, PBM / 16};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, (void*)W, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EE_REQUIRE(r == CUDA_SUCCESS, EE_ECUDA, "cuTensorMapEncodeTiled (tiled weights) failed (%d)",
               (int)r);
    return EE_OK;
}

}  // namespace

size_t prefill_ws_bytes(int64_t m, int64_t N_max) {
    return (size_t)4 * (size_t)m * (size_t)N_max * sizeof(float);  // up to 4 splits
}

// Swap-AB tcgen05 GEMM over tiled weights + ordered split reduction + epilogue.
int launch_prefill_tiled(const bf16* x, int64_t m, int64_t K, const void* W, int64_t N, int epi,
                         const float* ssq_in, float eps, float* q, void* kc, void* vc,
                         const int32_t* pos, int64_t h, void* out, float* xres, bf16* xb,
                         float* ssq_out, void* ws, size_t ws_bytes, cudaStream_t s) {
    EE_REQUIRE(K % kTiledKS == 0 && N % 16 == 0 && m > 0, EE_ESHAPE,
               "prefill gemm: need K %% 512 == 0, N %% 16 == 0 (K=%lld N=%lld)", (long long)K,
               (long long)N);
    const int tiles = (int)((N + PBM - 1) / PBM);
    const int groups = (int)((m + PBN - 1) / PBN);
    const int sms = ee_sm_count();
    int splits = 1;
    while (splits < 4 && tiles * groups * splits * 2 <= sms && (K / PBK) >= 8 * splits * 2)
        splits *= 2;
    EE_REQUIRE(ws && ws_bytes >= (size_t)splits * m * N * sizeof(float), EE_ESHAPE,
               "prefill gemm: workspace too small");
    CUtensorMap tw, tx;
    int rc;
    if ((rc = make_tmap_tiled_w(&tw, W, N, K))) return rc;
    if ((rc = tc::make_tmap_bf16(&tx, x, m, K, PBN))) return rc;
    static bool configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 15]) {
        cudaFuncSetAttribute(k_prefill_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPSmem);
        configured[dev & 15] = true;
    }
    const int items = tiles * groups * splits;
    const unsigned grid = (unsigned)(items < sms ? items : sms);
    float* part = (float*)ws;
    cudaError_t e = launch_ex(k_prefill_gemm, dim3(grid), dim3(kPThreads), kPSmem, s, tw, tx,
                              (int)N, (int)m, (int)K, splits, part);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "prefill gemm launch: %s", cudaGetErrorString(e));
    ApplyArgs a{part, splits, (int)m, (int)N, (int)K, ssq_in, eps, q, (bf16*)kc, (bf16*)vc, pos,
                (int)h, (bf16*)out, xres, xb, ssq_out};
    const dim3 ag((unsigned)((N / 16 + 255) / 256), (unsigned)m);
    if (epi == kEpiQKV) e = launch_ex(k_prefill_apply<kEpiQKV>, ag, dim3(256), 0, s, a);
    else if (epi == kEpiGelu) e = launch_ex(k_prefill_apply<kEpiGelu>, ag, dim3(256), 0, s, a);
    else e = launch_ex(k_prefill_apply<kEpiResidual>, ag, dim3(256), 0, s, a);
    if (e != cudaSuccess) return ee_fail(EE_ECUDA, "prefill apply launch: %s", cudaGetErrorString(e));
    return EE_OK;
}
