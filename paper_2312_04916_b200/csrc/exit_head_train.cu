// Fused training exit head: weighted cross-entropy of one exit and its
// gradients on tcgen05 tensor cores, without the (n, V) LOGITS ever being
// written to HBM.
//
// Restates `run_head` (x @ out^T, eepipe/model.py:219-230) + `cross_entropy`
// (eepipe/autodiff.py:301-323, _pykernels.py:64-85) + the matmul backward
// (eepipe/autodiff.py:170-177):
//   S = X W^T,  lse_i = log sum_v exp S_iv,  loss = w/n sum_i (lse_i - S_i,t_i)
//   G = w/n (softmax(S) - onehot(t)),  dX = G W,  dW += G^T X
// as three tcgen05 GEMMs (tc_gemm.cuh) plus one streaming pass:
//   K1  S = X W^T          two-pass epilogue per (row, 128-column part):
//                          part max m_p and target logit, then
//                          P~ = exp(S - m_p) (bf16, into G's buffer) and
//                          its sum s_p.  The logits stay in TMEM.
//   F   per row: merge (m_p, s_p) in fixed part order -> lse, row loss;
//       G = w/n (P~ exp(m_p - lse) - [v == t])  in place (bf16)
//   K3  dX  = G  W    A = G K-major, B = W read MN-major   (K = V)
//   K4  dW += G^T X   A = G read MN-major, B = X MN-major  (K = n)
// MN-major operands are consumed in place through the UMMA descriptor (no
// transposed copies).  Only part-normalised probabilities and then the logit
// GRADIENT G (bf16) reach HBM (the two backward GEMMs contract G along
// different axes, so it must exist); the logits themselves, the softmax and
// the reference's cached (n, V) float64 probs (_ckernels.pyx:130-151) never
// do.  Executed FLOPs = the algorithmic 6 n h V: S is computed
// once.
#include <cuda.h>

#include <mutex>

#include "tc_gemm.cuh"

namespace {

constexpr int kBN = 256;
constexpr int kParts = 2;  // per-row softmax partials per 256-column tile (epilogue halves)

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct TrainWs {
    bf16* g;
    float *pmax, *psum, *tgt, *lse, *rowloss;
    int* flags;  // ordered split-K flags of the dX GEMM
};

constexpr size_t kFlagBytes = 64 * 1024;  // up to 1024 cluster tiles x 16 regions

TrainWs carve(void* ws, int64_t n, int64_t V) {
    TrainWs w;
    char* p = (char*)ws;
    const int64_t ntn = kParts * ((V + kBN - 1) / kBN);
    w.pmax = (float*)p; p += al((size_t)n * ntn * 4);
    w.psum = (float*)p; p += al((size_t)n * ntn * 4);
    w.tgt = (float*)p; p += al((size_t)n * 4);
    w.lse = (float*)p; p += al((size_t)n * 4);
    w.rowloss = (float*)p; p += al((size_t)n * 4);
    w.flags = (int*)p; p += kFlagBytes;
    w.g = (bf16*)p;
    return w;
}

size_t carve_bytes(int64_t n, int64_t V) {
    const int64_t ntn = kParts * ((V + kBN - 1) / kBN);
    return 2 * al((size_t)n * ntn * 4) + 3 * al((size_t)n * 4) + kFlagBytes + al((size_t)n * V * 2);
}

// ---- epilogues ----------------------------------------------------------------
// K1: pass 1 = part max + target logit, pass 2 = P~ = exp(S - m) in bf16
// (row-major n x V, G's buffer) and its sum.  A part with no valid column
// keeps (m, s) = (-inf, 0), which the merge skips.
struct EpiProb {
    static constexpr bool kTwoPass = true;
    static constexpr bool kSplitK = false;
    static constexpr bool kStreamK = false;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = false;
    const int64_t* targets;
    float *pmax, *psum, *tgt;
    bf16* g;
    int ntn, N;
    float m, s;
    int t;  // target id of the row (V < 2^31), -1 for padding rows
    __device__ void begin_tile(int row, int, int, bool valid) {
        m = -INFINITY;
        s = 0.f;
        t = valid ? (int)targets[row] : -1;
    }
    __device__ void pre(int row, int col, const float* v, int nvalid) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < nvalid) m = fmaxf(m, v[j]);
        const int d = t - col;
        if ((unsigned)d < (unsigned)nvalid) {  // rare: the target is in this chunk
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j == d) tgt[row] = v[j];  // register-indexed (no local copy)
        }
    }
    __device__ void chunk(int row, int col, const float* v, int nvalid) {
        float e[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            e[j] = j < nvalid ? __expf(v[j] - m) : 0.f;
            s += e[j];
        }
        bf16* gr = g + (int64_t)row * N + col;
        if (nvalid == 16) {
            uint32_t w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                __nv_bfloat162 b = __floats2bfloat162_rn(e[2 * j], e[2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&b);
            }
            reinterpret_cast<uint4*>(gr)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(gr)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) gr[j] = __float2bfloat16_rn(e[j]);
        }
    }
    __device__ void end_tile(int row, int, int part, bool valid) {
        if (valid) {
            pmax[(int64_t)row * ntn + part] = m;
            psum[(int64_t)row * ntn + part] = s;
        }
    }
};

template <bool ACCUM>
struct EpiF32 {  // K3 store / K4 accumulate, optionally scaled by *gs (device)
    static constexpr bool kTwoPass = false;
    static constexpr bool kSplitK = false;
    static constexpr bool kStreamK = true;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = true;   // TMA-stored output boxes (tc_gemm.cuh)
    static constexpr bool kReduceAdd = ACCUM;  // accumulate: TMA reduce-add in L2
    using OutT = float;
    float* out;
    int ldo;
    const float* gs = nullptr;
    float g = 1.f;
    int out_map(CUtensorMap* m, int M, int N) const { return tc::make_tmap_out(m, out, 4, M, N, ldo); }
    __device__ void stage(int, int, const float* v, int, float* o) {
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = gs ? v[j] * g : v[j];
    }
    __device__ void begin_tile(int, int, int, bool) {
        if (gs) g = __ldg(gs);
    }
    __device__ void chunk(int row, int col, const float* v0, int nvalid) {
        float* o = out + (int64_t)row * ldo + col;
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = gs ? v0[j] * g : v0[j];
        if (nvalid == 16) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
                float4 c = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                if (ACCUM) {
                    const float4 p = *reinterpret_cast<const float4*>(o + j);
                    c.x += p.x;
                    c.y += p.y;
                    c.z += p.z;
                    c.w += p.w;
                }
                *reinterpret_cast<float4*>(o + j) = c;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) o[j] = ACCUM ? o[j] + v[j] : v[j];
        }
    }
    __device__ void end_tile(int, int, int, bool) {}
};

// K3 with ORDERED split-K: split s of tile t adds its partial into dx after
// split s-1 of the same (tile, warp region) has written (per-region flags,
// acquire / release), so dx = ((p0 + p1) + p2) + ... in split order —
// deterministic, with the read-modify-write traffic inside the tensor-bound
// GEMM instead of a separate reduction pass.  Items run split-major, and a
// cluster only ever waits for an item of a lower index, so the persistent
// grid cannot deadlock.  The flags are zero at rest (the last split resets
// them; the host also clears them per call).
struct EpiF32Ordered {
    static constexpr bool kTwoPass = false;
    static constexpr bool kSplitK = true;
    static constexpr bool kStreamK = false;  // stream-K tail allowed (tc_gemm.cuh)
    static constexpr bool kStaged = false;
    float* out;
    int ldo;
    int* flags;  // [tiles][16 regions]
    int splits;
    const float* gs = nullptr;  // optional device scale of every partial
    int s = 0;
    int* flag = nullptr;
    __device__ void set_split(int sp, int t) {
        s = sp;
        const int region = (int)tc::cluster_rank() * tc::kEpiWarps + ((int)(threadIdx.x >> 5) - 2);
        flag = flags + t * 2 * tc::kEpiWarps + region;
    }
    float g = 1.f;
    __device__ void begin_tile(int, int, int, bool) {
        if (gs) g = __ldg(gs);
        if (s > 0) {
            if ((threadIdx.x & 31) == 0) {
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                } while (v < s);
            }
            __syncwarp();
        }
    }
    __device__ void chunk(int row, int col, const float* v0, int nvalid) {
        float* o = out + (int64_t)row * ldo + col;
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = gs ? v0[j] * g : v0[j];
        if (nvalid == 16) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
                float4 c = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                if (s > 0) {
                    const float4 p = __ldcg(reinterpret_cast<const float4*>(o + j));
                    c.x = p.x + c.x;
                    c.y = p.y + c.y;
                    c.z = p.z + c.z;
                    c.w = p.w + c.w;
                }
                *reinterpret_cast<float4*>(o + j) = c;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < nvalid) o[j] = s > 0 ? __ldcg(o + j) + v[j] : v[j];
        }
    }
    __device__ void end_tile(int, int, int, bool) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
            __threadfence();
            const int nv = (s == splits - 1) ? 0 : s + 1;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(nv) : "memory");
        }
    }
};

// split count for a GEMM of `tiles` cluster tiles and nk k-blocks on
// `pairs` clusters: the smallest S <= 4 whose last wave is >= 95% full
// (else the best of 1..4), keeping >= 64 k-blocks per split
static int pick_splits(int tiles, int nk, int pairs) {
    int best = 1;
    double best_eff = 0.0;
    for (int S = 1; S <= 4; ++S) {
        if (S > 1 && nk / S < 64) break;
        const int items = tiles * S;
        const int waves = (items + pairs - 1) / pairs;
        const double eff = (double)items / ((double)waves * pairs);
        if (eff >= 0.95) return S;
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = S;
        }
    }
    return best;
}

// ---- small kernels ---------------------------------------------------------
// per-row merge of the tile partials in ascending (tile, half) order: one
// warp per row, lane-strided partial merges then a fixed xor butterfly
__device__ __forceinline__ void lse_combine(float& m1, float& s1, float m2, float s2) {
    if (s2 == 0.f) return;
    if (s1 == 0.f) {
        m1 = m2;
        s1 = s2;
        return;
    }
    const float M = fmaxf(m1, m2);
    s1 = s1 * expf(m1 - M) + s2 * expf(m2 - M);
    m1 = M;
}
// F: one CTA per row.  Warp 0 merges the row's part partials in ascending
// part order (lane-strided, then a fixed xor butterfly) -> lse and the row
// loss; then all threads rescale the row's P~ in place to the bf16 logit
// gradient G = scale (P~ exp(m_p - lse) - [v == t]), 16 bytes at a time
// (a 16-byte vector never straddles a 128-column part).
constexpr int kFixThreads = 256;
constexpr int kPartCols = kBN / kParts;
__global__ void __launch_bounds__(kFixThreads)
k_grad_fixup(const float* __restrict__ pmax, const float* __restrict__ psum,
             const float* __restrict__ tgt, const int64_t* __restrict__ targets, int ntn, int V,
             float scale, bf16* __restrict__ g, float* __restrict__ lse_out,
             float* __restrict__ rowloss) {
    extern __shared__ float fac[];  // ntn part factors
    __shared__ float sh_lse;
    const int i = blockIdx.x, lane = threadIdx.x & 31;
    const float* pm = pmax + (int64_t)i * ntn;
    const float* ps = psum + (int64_t)i * ntn;
    if (threadIdx.x < 32) {
        float M = -INFINITY, S = 0.f;
        for (int b = lane; b < ntn; b += 32) lse_combine(M, S, pm[b], ps[b]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, M, o);
            const float s2 = __shfl_xor_sync(0xffffffffu, S, o);
            // symmetric combine so both lanes of a pair hold identical values
            const float Mx = fmaxf(M, m2);
            const float a = (S == 0.f) ? 0.f : S * expf(M - Mx);
            const float c = (s2 == 0.f) ? 0.f : s2 * expf(m2 - Mx);
            S = (lane & o) ? (c + a) : (a + c);
            M = Mx;
        }
        if (lane == 0) {
            const float l = M + logf(S);
            sh_lse = l;
            lse_out[i] = l;
            rowloss[i] = l - tgt[i];
        }
    }
    __syncthreads();
    const float l = sh_lse;
    for (int b = threadIdx.x; b < ntn; b += kFixThreads)
        fac[b] = ps[b] == 0.f ? 0.f : scale * __expf(pm[b] - l);
    __syncthreads();
    const int64_t t = targets[i];
    bf16* gr = g + (int64_t)i * V;
    for (int c = threadIdx.x * 8; c < V; c += kFixThreads * 8) {
        const float f = fac[c / kPartCols];
        uint4 u = *reinterpret_cast<const uint4*>(gr + c);
        uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w[j]);
            float2 p = __bfloat1622float2(b);
            p.x = p.x * f - ((int64_t)(c + 2 * j) == t ? scale : 0.f);
            p.y = p.y * f - ((int64_t)(c + 2 * j + 1) == t ? scale : 0.f);
            b = __floats2bfloat162_rn(p.x, p.y);
            w[j] = *reinterpret_cast<uint32_t*>(&b);
        }
        *reinterpret_cast<uint4*>(gr + c) = u;
    }
}

// fixed-shape tree sum of the per-row losses -> weight/n * sum (one CTA)
__global__ void k_loss_sum(const float* __restrict__ rowloss, int n, float scale,
                           float* __restrict__ loss) {
    __shared__ float sh[1024];
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += 1024) s += rowloss[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = sh[0] * scale;
}

}  // namespace

namespace tc {
bool sk_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("EE_GEMM_STREAMK");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

SkWs* sk_workspace(cudaStream_t s, size_t ws_bytes, int nflags) {
    static SkWs table[32];
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    SkWs* w = nullptr;
    for (auto& e : table)
        if (e.dev == dev && e.stream == s) {
            w = &e;
            break;
        }
    if (!w)
        for (auto& e : table)
            if (e.dev < 0) {
                w = &e;
                w->dev = dev;
                w->stream = s;
                break;
            }
    if (!w) return nullptr;
    if (w->ws_bytes < ws_bytes) {
        // grow: the stream's earlier launches may still read the old slots
        if (w->ws) {
            cudaStreamSynchronize(s);
            cudaFree(w->ws);
        }
        w->ws = nullptr;
        w->ws_bytes = 0;
        if (cudaMalloc(&w->ws, ws_bytes) != cudaSuccess) {
            cudaGetLastError();
            w->ws = nullptr;
            return nullptr;
        }
        w->ws_bytes = ws_bytes;
    }
    if (w->nflags < nflags) {
        if (w->flags) {
            cudaStreamSynchronize(s);
            cudaFree(w->flags);
        }
        w->flags = nullptr;
        w->nflags = 0;
        if (cudaMalloc(&w->flags, nflags * sizeof(uint32_t)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        cudaMemsetAsync(w->flags, 0, nflags * sizeof(uint32_t), s);
        w->nflags = nflags;
        w->epoch = 0;
    }
    return w;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    return make_tmap_bf16_ld(map, base, rows, cols, cols, box_rows);
}

namespace {
int encode_2d(CUtensorMap* map, const void* base, bool f32, int64_t rows, int64_t cols, int64_t ld,
              int box_cols, int box_rows);
}
int make_tmap_bf16_ld(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                      int box_rows) {
    EE_REQUIRE(((uintptr_t)base & 15) == 0 && cols % 8 == 0 && ld % 8 == 0 && ld >= cols,
               EE_ESHAPE, "tensor map: base must be 16-B aligned, cols and ld multiples of 8");
    return encode_2d(map, base, false, rows, cols, ld, BK, box_rows);
}

int make_tmap_out(CUtensorMap* map, const void* base, int elem_bytes, int64_t rows, int64_t cols,
                  int64_t ld) {
    const int per16 = 16 / elem_bytes;
    EE_REQUIRE(((uintptr_t)base & 15) == 0 && cols % per16 == 0 && ld % per16 == 0 && ld >= cols,
               EE_ESHAPE, "output tensor map: base 16-B aligned, cols and ld 16-B multiples");
    return encode_2d(map, base, elem_bytes == 4, rows, cols, ld, 128 / elem_bytes, 32);
}

namespace {
int encode_2d(CUtensorMap* map, const void* base, bool f32, int64_t rows, int64_t cols, int64_t ld,
              int box_cols, int box_rows) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * (f32 ? 4 : 2)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    // resolved through the runtime so libee.so does not link libcuda (the
    // build container has no driver; the GPU box does)
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
    CUresult r = encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        2, (void*)base, dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EE_REQUIRE(r == CUDA_SUCCESS, EE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return EE_OK;
}
}  // namespace
}  // namespace tc

size_t exit_head_train_ws_bytes(int64_t n, int64_t /*h*/, int64_t V) { return carve_bytes(n, V); }

namespace {

int check_head_shape(int64_t n, int64_t h, int64_t V, size_t ws_bytes, const void* ws) {
    // h and V set row strides of TMA-read matrices (16-byte multiples);
    // any n works (out-of-range rows / k-blocks are zero-filled by TMA)
    EE_REQUIRE(n > 0 && h > 0 && V > 0 && h % 8 == 0 && V % 8 == 0, EE_ESHAPE,
               "exit_head_train: h and V must be positive multiples of 8 (n=%lld h=%lld V=%lld)",
               (long long)n, (long long)h, (long long)V);
    EE_REQUIRE(n < (1ll << 31) && V < (1ll << 31), EE_ESHAPE, "exit_head_train: too large");
    EE_REQUIRE(ws && ws_bytes >= carve_bytes(n, V), EE_ESHAPE,
               "exit_head_train: workspace too small (%zu < %zu)", ws_bytes, carve_bytes(n, V));
    return EE_OK;
}

// K1 + F + loss: G (n x V bf16) = w/n (softmax - onehot), loss = w/n sum CE
int head_forward(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                 const int64_t* targets, float weight, float* loss, bf16* G, TrainWs& w,
                 cudaStream_t s) {
    const int ntn = (int)(kParts * ((V + kBN - 1) / kBN));
    const float scale = weight / (float)n;
    int rc;
    // K1: S = X W^T -> part max / sum, target logits, P~ into G's buffer
    if ((rc = tc::launch_tc_gemm2<kBN, false, false, false>(
             x, W, (int)n, (int)V, (int)h,
             EpiProb{targets, w.pmax, w.psum, w.tgt, G, ntn, (int)V, 0.f, 0.f, 0}, s)))
        return rc;
    // F: lse, row losses, P~ -> G in place
    k_grad_fixup<<<(unsigned)n, kFixThreads, ntn * sizeof(float), s>>>(
        w.pmax, w.psum, w.tgt, targets, ntn, (int)V, scale, G, w.lse, w.rowloss);
    if ((rc = ee_check_launch("grad_fixup"))) return rc;
    k_loss_sum<<<1, 1024, 0, s>>>(w.rowloss, (int)n, scale, loss);
    return ee_check_launch("loss_sum");
}

// K3 + K4: dx = g G W, dw_acc += g G^T X (g: optional device scalar)
int head_backward(const void* x, int64_t n, int64_t h, const void* W, int64_t V, const bf16* G,
                  const float* gs, float* dx, float* dw_acc, TrainWs& w, cudaStream_t s) {
    int rc;
    // K3: dX = G W     (W (V x h) is the MN-major B operand, K = V); long
    // tiles, few of them: ordered split-K fills the last wave
    {
        const int tiles = (int)(((n + 255) / 256) * ((h + kBN - 1) / kBN));
        const bool fits = (size_t)tiles * 2 * tc::kEpiWarps * sizeof(int) <= kFlagBytes;
        const int S = fits ? pick_splits(tiles, (int)((V + tc::BK - 1) / tc::BK), ee_sm_count() / 2)
                           : 1;
        if (S == 1) {
            if ((rc = tc::launch_tc_gemm2<kBN, false, true, false>(
                     G, W, (int)n, (int)h, (int)V, EpiF32<false>{dx, (int)h, gs}, s)))
                return rc;
        } else {
            const size_t fbytes = (size_t)tiles * 2 * tc::kEpiWarps * sizeof(int);
            cudaMemsetAsync(w.flags, 0, fbytes, s);
            if ((rc = tc::launch_tc_gemm2<kBN, false, true, false>(
                     G, W, (int)n, (int)h, (int)V, EpiF32Ordered{dx, (int)h, w.flags, S, gs}, s,
                     S)))
                return rc;
        }
    }
    // K4: dW += G^T X  (G and X both MN-major, K = n); N-fastest tile order so
    // concurrent CTAs share each G column block
    return tc::launch_tc_gemm2<kBN, true, true, true>(G, x, (int)V, (int)h, (int)n,
                                                     EpiF32<true>{dw_acc, (int)h, gs}, s);
}

}  // namespace

extern "C" int ee_exit_head_train(const void* x, int64_t n, int64_t h, const void* W, int64_t V,
                                  const int64_t* targets, float weight, float* loss, float* dx,
                                  float* dw_acc, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if ((rc = check_head_shape(n, h, V, ws_bytes, ws))) return rc;
    cudaStream_t s = as_stream(stream);
    TrainWs w = carve(ws, n, V);
    if ((rc = head_forward(x, n, h, W, V, targets, weight, loss, w.g, w, s))) return rc;
    return head_backward(x, n, h, W, V, w.g, nullptr, dx, dw_acc, w, s);
}

// The same head split at the autograd boundary: the forward leaves G in a
// caller buffer; the backward scales by the incoming gradient read from
// device memory (no host synchronisation) and accumulates dW straight into
// the caller's float32 gradient sum.
extern "C" int ee_exit_head_train_fwd(const void* x, int64_t n, int64_t h, const void* W,
                                      int64_t V, const int64_t* targets, float weight, float* loss,
                                      void* G, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if ((rc = check_head_shape(n, h, V, ws_bytes, ws))) return rc;
    EE_REQUIRE(G != nullptr, EE_ESHAPE, "exit_head_train_fwd: null G");
    TrainWs w = carve(ws, n, V);
    return head_forward(x, n, h, W, V, targets, weight, loss, (bf16*)G, w, as_stream(stream));
}

extern "C" int ee_exit_head_train_bwd(const void* x, int64_t n, int64_t h, const void* W,
                                      int64_t V, const void* G, const float* grad, float* dx,
                                      float* dw_acc, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if ((rc = check_head_shape(n, h, V, ws_bytes, ws))) return rc;
    EE_REQUIRE(G != nullptr && dx != nullptr && dw_acc != nullptr, EE_ESHAPE,
               "exit_head_train_bwd: null argument");
    TrainWs w = carve(ws, n, V);
    return head_backward(x, n, h, W, V, (const bf16*)G, grad, dx, dw_acc, w, as_stream(stream));
}

// Weight gradient of a bf16 linear layer accumulated straight into a float32
// buffer: dW (in x out) += X^T dY with X (T x in) and dY (T x out) bf16
// row-major (both read MN-major by the UMMA descriptors; no transposes) —
// the backbone's "gradient-accumulation fusion": no bf16 weight gradient, no
// separate accumulation pass.  in, out multiples of 8; any T.
extern "C" int ee_wgrad_accum(const void* X, const void* dY, int64_t T, int64_t in, int64_t out,
                              float* dW, void* stream) {
    EE_REQUIRE(T > 0 && in > 0 && out > 0 && in % 8 == 0 && out % 8 == 0, EE_ESHAPE,
               "wgrad_accum: in and out must be positive multiples of 8 (T=%lld in=%lld out=%lld)",
               (long long)T, (long long)in, (long long)out);
    EE_REQUIRE(T < (1ll << 31) && in < (1ll << 31) && out < (1ll << 31), EE_ESHAPE,
               "wgrad_accum: too large");
    return tc::launch_tc_gemm2<kBN, true, true, true>(X, dY, (int)in, (int)out, (int)T,
                                                     EpiF32<true>{dW, (int)out}, as_stream(stream));
}

// Weight gradients of `parts` adjacent (in, out) matrices in one GEMM:
// dW_j += X^T dY[:, j out : (j + 1) out], dW_j = dW + j in out (the float32
// sums of q / k / v are adjacent in the flat gradient buffer): the output is
// stored stacked (tc_gemm.cuh, osub), dY is one (T, parts out) matrix.
extern "C" int ee_wgrad_accum_stacked(const void* X, const void* dY, int64_t T, int64_t in,
                                      int64_t out, int64_t parts, float* dW, void* stream) {
    EE_REQUIRE(T > 0 && parts >= 1 && in % 128 == 0 && out % 128 == 0, EE_ESHAPE,
               "wgrad_accum_stacked: in and out must be multiples of 128 (T=%lld in=%lld out=%lld)",
               (long long)T, (long long)in, (long long)out);
    EE_REQUIRE(T < (1ll << 31) && in * parts < (1ll << 31) && out * parts < (1ll << 31), EE_ESHAPE,
               "wgrad_accum_stacked: too large");
    return tc::launch_tc_gemm2<kBN, true, true, true>(X, dY, (int)in, (int)(out * parts), (int)T,
                                                     EpiF32<true>{dW, (int)out}, as_stream(stream),
                                                     1, 0, (int)out);
}
