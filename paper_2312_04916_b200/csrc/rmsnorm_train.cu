// Training RMSNorm forward / backward on bf16 activations — the reference's
// `rmsnorm_fwd` / `rmsnorm_bwd` boundary kernels (eepipe/_pykernels.py:36-49,
// eepipe/_ckernels.pyx:46-89) for the (n, h) training backbone:
//
//   fwd:  inv_i = (mean_j x_ij^2 + eps)^-1/2,   y_ij = x_ij inv_i w_j
//   bwd:  gw_j  = sum_i g_ij x_ij inv_i
//         gx_ij = g_ij w_j inv_i - x_ij inv_i^3 (sum_k g_ik w_k x_ik) / h
//
// One warp per row (16-byte vectors, h % 8 == 0), float32 statistics.  The
// weight gradient is reduced deterministically: each CTA writes one float32
// partial row (its rows summed in order) and k_gw_reduce adds the partials in
// CTA order — no atomics, so repeated runs give identical bits.
#include "ee_common.cuh"

namespace {

constexpr int kWarps = 8;               // rows per CTA
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 t = __bfloat1622float2(b[k]);
        f[2 * k] = t.x;
        f[2 * k + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
    uint4 u;
    __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
    return u;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void load_w8(const float* w, int c, float* ww) {
    const float4 w0 = reinterpret_cast<const float4*>(w)[2 * c];
    const float4 w1 = reinterpret_cast<const float4*>(w)[2 * c + 1];
    ww[0] = w0.x; ww[1] = w0.y; ww[2] = w0.z; ww[3] = w0.w;
    ww[4] = w1.x; ww[5] = w1.y; ww[6] = w1.z; ww[7] = w1.w;
}

// One warp per row.  Rows up to kHeld * 256 columns are loaded once into
// registers (all 16-byte loads of the row in flight together); wider rows take
// two sweeps, the second re-reading the row from L1 / L2.
constexpr int kHeld = 8;  // 16-byte chunks per lane held in registers (h <= 2048)
__global__ void __launch_bounds__(kThreads)
k_rms_fwd(const bf16* __restrict__ x, const float* __restrict__ w, int64_t n, int h, float eps,
          bf16* __restrict__ y, float* __restrict__ inv_out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (row >= n) return;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
    uint4* yr = reinterpret_cast<uint4*>(y + row * h);
    const int nvec = h / 8;
    float ss = 0.f;
    if (nvec <= 32 * kHeld) {
        uint4 xs[kHeld];
#pragma unroll
        for (int u = 0; u < kHeld; ++u)
            if (u * 32 + lane < nvec) xs[u] = xr[u * 32 + lane];
#pragma unroll
        for (int u = 0; u < kHeld; ++u)
            if (u * 32 + lane < nvec) {
                float v[8];
                unpack8(xs[u], v);
#pragma unroll
                for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
            }
        ss = warp_sum(ss);
        const float inv = rsqrtf(ss / (float)h + eps);
#pragma unroll
        for (int u = 0; u < kHeld; ++u) {
            const int c = u * 32 + lane;
            if (c < nvec) {
                float v[8], ww[8], o[8];
                unpack8(xs[u], v);
                load_w8(w, c, ww);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] = v[k] * inv * ww[k];
                yr[c] = pack8(o);
            }
        }
        if (lane == 0) inv_out[row] = inv;
        return;
    }
    for (int c = lane; c < nvec; c += 32) {
        float v[8];
        unpack8(xr[c], v);
#pragma unroll
        for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / (float)h + eps);
    for (int c = lane; c < nvec; c += 32) {
        float v[8], ww[8], o[8];
        unpack8(xr[c], v);
        load_w8(w, c, ww);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = v[k] * inv * ww[k];
        yr[c] = pack8(o);
    }
    if (lane == 0) inv_out[row] = inv;
}

// Backward: a grid of about one wave, each warp taking `rpw` consecutive rows.
// Per row: x, g (and gres, a second incoming gradient of x -- the residual
// branch of a pre-norm block -- added to gx in the same pass) are loaded with
// every 16-byte load of the row in flight, the row's weight-gradient terms
// g x inv are added into the warp's own float32 row of shared memory (no
// synchronisation inside the row loop), and gx is written.  At the end the
// CTA sums its warps' rows in warp order into its partial; k_gw_reduce adds
// the partials in CTA order -- no atomics, repeated runs give identical bits.
constexpr int kBwdWarps = 4;
constexpr int kBwdThreads = kBwdWarps * 32;
__device__ __forceinline__ void acc_gw8(float* a, const float* gv, const float* xv, float inv) {
    float4* p = reinterpret_cast<float4*>(a);
    float4 u0 = p[0], u1 = p[1];
    u0.x += gv[0] * xv[0] * inv; u0.y += gv[1] * xv[1] * inv;
    u0.z += gv[2] * xv[2] * inv; u0.w += gv[3] * xv[3] * inv;
    u1.x += gv[4] * xv[4] * inv; u1.y += gv[5] * xv[5] * inv;
    u1.z += gv[6] * xv[6] * inv; u1.w += gv[7] * xv[7] * inv;
    p[0] = u0;
    p[1] = u1;
}
#ifndef EE_RMS_SW
#define EE_RMS_SW 1
#endif
#ifndef EE_RMS_BWD_MINB
#define EE_RMS_BWD_MINB 1
#endif
__global__ void __launch_bounds__(kBwdThreads, EE_RMS_BWD_MINB)
k_rms_bwd(const bf16* __restrict__ x, const float* w, const float* __restrict__ inv_in,
          const bf16* __restrict__ g, const bf16* __restrict__ gres, int64_t n, int h, int rpw,
          bf16* __restrict__ gx, float* __restrict__ gw_part) {
    extern __shared__ float4 acc_raw[];
    float* acc = reinterpret_cast<float*>(acc_raw);  // [kBwdWarps][h], then w (h)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nvec = h / 8;
    float* my = acc + (size_t)warp * h;
    for (int c = lane; c < nvec; c += 32) {
        reinterpret_cast<float4*>(my)[2 * c] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(my)[2 * c + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#if EE_RMS_SW
    // the norm weight once per CTA in shared memory: the row loops read it
    // with shared loads instead of a dependent global load per chunk
    float* sw = acc + (size_t)kBwdWarps * h;
    for (int j4 = threadIdx.x; j4 < h / 4; j4 += kBwdThreads)
        reinterpret_cast<float4*>(sw)[j4] = reinterpret_cast<const float4*>(w)[j4];
    __syncthreads();
    w = sw;
#endif
    const bool held = nvec <= 32 * kHeld;
    const int64_t r0 = ((int64_t)blockIdx.x * kBwdWarps + warp) * rpw;
    for (int i = 0; i < rpw; ++i) {
        const int64_t row = r0 + i;
        if (row >= n) break;
        const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
        const uint4* gr = reinterpret_cast<const uint4*>(g + row * h);
        const uint4* rr = gres ? reinterpret_cast<const uint4*>(gres + row * h) : nullptr;
        uint4* gxr = reinterpret_cast<uint4*>(gx + row * h);
        const float inv = inv_in[row];
        float dot = 0.f;
        if (held) {
            uint4 xs[kHeld], gs[kHeld], rs[kHeld];
#pragma unroll
            for (int u = 0; u < kHeld; ++u) {
                const int c = u * 32 + lane;
                if (c < nvec) {
                    xs[u] = xr[c];
                    gs[u] = gr[c];
                    if (rr) rs[u] = rr[c];
                }
            }
#pragma unroll
            for (int u = 0; u < kHeld; ++u) {
                const int c = u * 32 + lane;
                if (c < nvec) {
                    float xv[8], gv[8], ww[8];
                    unpack8(xs[u], xv);
                    unpack8(gs[u], gv);
                    load_w8(w, c, ww);
#pragma unroll
                    for (int k = 0; k < 8; ++k) dot += gv[k] * ww[k] * xv[k];
                    acc_gw8(my + 8 * c, gv, xv, inv);
                }
            }
            dot = warp_sum(dot);
            const float coef = inv * inv * inv * dot / (float)h;
#pragma unroll
            for (int u = 0; u < kHeld; ++u) {
                const int c = u * 32 + lane;
                if (c < nvec) {
                    float xv[8], gv[8], ww[8], o[8];
                    unpack8(xs[u], xv);
                    unpack8(gs[u], gv);
                    load_w8(w, c, ww);
#pragma unroll
                    for (int k = 0; k < 8; ++k) o[k] = gv[k] * ww[k] * inv - xv[k] * coef;
                    if (rr) {
                        float rv[8];
                        unpack8(rs[u], rv);
#pragma unroll
                        for (int k = 0; k < 8; ++k) o[k] += rv[k];
                    }
                    gxr[c] = pack8(o);
                }
            }
        } else {
            for (int c0 = 0; c0 < nvec; c0 += 32 * kHeld) {
                uint4 xs[kHeld], gs[kHeld];
#pragma unroll
                for (int u = 0; u < kHeld; ++u) {
                    const int c = c0 + u * 32 + lane;
                    if (c < nvec) {
                        xs[u] = xr[c];
                        gs[u] = gr[c];
                    }
                }
#pragma unroll
                for (int u = 0; u < kHeld; ++u) {
                    const int c = c0 + u * 32 + lane;
                    if (c < nvec) {
                        float xv[8], gv[8], ww[8];
                        unpack8(xs[u], xv);
                        unpack8(gs[u], gv);
                        load_w8(w, c, ww);
#pragma unroll
                        for (int k = 0; k < 8; ++k) dot += gv[k] * ww[k] * xv[k];
                        acc_gw8(my + 8 * c, gv, xv, inv);
                    }
                }
            }
            dot = warp_sum(dot);
            const float coef = inv * inv * inv * dot / (float)h;
            for (int c0 = 0; c0 < nvec; c0 += 32 * kHeld) {
                uint4 xs[kHeld], gs[kHeld], rs[kHeld];
#pragma unroll
                for (int u = 0; u < kHeld; ++u) {
                    const int c = c0 + u * 32 + lane;
                    if (c < nvec) {
                        xs[u] = xr[c];
                        gs[u] = gr[c];
                        if (rr) rs[u] = rr[c];
                    }
                }
#pragma unroll
                for (int u = 0; u < kHeld; ++u) {
                    const int c = c0 + u * 32 + lane;
                    if (c < nvec) {
                        float xv[8], gv[8], ww[8], o[8];
                        unpack8(xs[u], xv);
                        unpack8(gs[u], gv);
                        load_w8(w, c, ww);
#pragma unroll
                        for (int k = 0; k < 8; ++k) o[k] = gv[k] * ww[k] * inv - xv[k] * coef;
                        if (rr) {
                            float rv[8];
                            unpack8(rs[u], rv);
#pragma unroll
                            for (int k = 0; k < 8; ++k) o[k] += rv[k];
                        }
                        gxr[c] = pack8(o);
                    }
                }
            }
        }
    }
    __syncthreads();
    // this CTA's partial: the warps' rows summed in warp order
    for (int j4 = threadIdx.x; j4 < h / 4; j4 += kBwdThreads) {
        float4 s4 = reinterpret_cast<const float4*>(acc)[j4];
#pragma unroll
        for (int r = 1; r < kBwdWarps; ++r) {
            const float4 t = reinterpret_cast<const float4*>(acc + (size_t)r * h)[j4];
            s4.x += t.x; s4.y += t.y; s4.z += t.z; s4.w += t.w;
        }
        reinterpret_cast<float4*>(gw_part + (size_t)blockIdx.x * h)[j4] = s4;
    }
}

// gw_j (+)= sum over the CTA partials in CTA order (deterministic): a CTA per
// 32 columns, warp v sums partials v, v + W, v + 2W, ... (lane = column; W =
// kRedWarps), then the W warp sums are added in warp order
#ifndef EE_RED_WARPS
#define EE_RED_WARPS 32
#endif
constexpr int kRedWarps = EE_RED_WARPS;  // 32: ~9 partials per warp (latency-bound sums)
__global__ void __launch_bounds__(kRedWarps * 32)
k_gw_reduce(const float* __restrict__ part, int nparts, int h, int accumulate,
            float* __restrict__ gw) {
    __shared__ float red[kRedWarps][32];
    const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + lane;
    float s = 0.f;
    if (j < h) {
        float s4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent chains, combined in order
        int p = v;
        // unrolled: 16 partial loads in flight per thread (same per-chain order)
#pragma unroll 4
        for (; p + 3 * kRedWarps < nparts; p += 4 * kRedWarps) {
#pragma unroll
            for (int k = 0; k < 4; ++k) s4[k] += part[(int64_t)(p + k * kRedWarps) * h + j];
        }
        for (; p < nparts; p += kRedWarps) s4[0] += part[(int64_t)p * h + j];
        s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    red[v][lane] = s;
    __syncthreads();
    if (v == 0 && j < h) {
        float t = red[0][lane];
#pragma unroll
        for (int r = 1; r < kRedWarps; ++r) t += red[r][lane];
        gw[j] = accumulate ? gw[j] + t : t;
    }
}

}  // namespace

// backward grid: about one wave of CTAs (occupancy-limited by the per-warp
// shared rows), never more CTAs than warps' worth of rows
struct BwdGrid {
    int ctas, rpw;
    size_t smem;
};
BwdGrid bwd_grid(int64_t n, int64_t h) {
    BwdGrid gr;
    gr.smem = (size_t)(kBwdWarps + (EE_RMS_SW ? 1 : 0)) * h * sizeof(float);
    static int64_t cached_h = -1;  // occupancy of the last width asked for
    static int cached_per_sm = 1;
    int per_sm = cached_per_sm;
    if (h != cached_h) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_rms_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr = true;
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rms_bwd, kBwdThreads,
                                                          gr.smem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        cached_h = h;
        cached_per_sm = per_sm;
    }
    const int64_t warps_needed = n;  // at most one row per warp
    int64_t ctas = (int64_t)ee_sm_count() * per_sm;
    const int64_t max_ctas = (warps_needed + kBwdWarps - 1) / kBwdWarps;
    if (ctas > max_ctas) ctas = max_ctas;
    if (ctas < 1) ctas = 1;
    gr.rpw = (int)((n + ctas * kBwdWarps - 1) / (ctas * kBwdWarps));
    if (gr.rpw < 1) gr.rpw = 1;
    gr.ctas = (int)((n + (int64_t)gr.rpw * kBwdWarps - 1) / ((int64_t)gr.rpw * kBwdWarps));
    return gr;
}

size_t rmsnorm_train_ws_bytes(int64_t n, int64_t h) {
    // partials: at most one per kBwdWarps rows
    return (size_t)((n + kBwdWarps - 1) / kBwdWarps) * (size_t)h * sizeof(float);
}

extern "C" int ee_rmsnorm_fwd(const void* x, int64_t n, int64_t h, const float* w, float eps,
                              void* y, float* inv_rms, void* stream) {
    EE_REQUIRE(n >= 0 && h > 0 && h % 8 == 0, EE_ESHAPE, "rmsnorm_fwd: need h %% 8 == 0 (h=%lld)",
               (long long)h);
    if (n == 0) return EE_OK;
    cudaStream_t s = as_stream(stream);
    const unsigned grid = (unsigned)((n + kWarps - 1) / kWarps);
    k_rms_fwd<<<grid, kThreads, 0, s>>>((const bf16*)x, w, n, (int)h, eps, (bf16*)y, inv_rms);
    return ee_check_launch("rmsnorm_fwd");
}

extern "C" int ee_rmsnorm_bwd(const void* x, const float* w, const float* inv_rms, const void* gy,
                              const void* gres, int64_t n, int64_t h, void* gx, float* gw,
                              int accumulate_gw, void* ws, size_t ws_bytes, void* stream) {
    EE_REQUIRE(n >= 0 && h > 0 && h % 8 == 0, EE_ESHAPE, "rmsnorm_bwd: need h %% 8 == 0 (h=%lld)",
               (long long)h);
    EE_REQUIRE(ws_bytes >= rmsnorm_train_ws_bytes(n, h), EE_ESHAPE,
               "rmsnorm_bwd: workspace too small");
    EE_REQUIRE((size_t)(kBwdWarps + 1) * h * sizeof(float) <= 227 * 1024, EE_ESHAPE,
               "rmsnorm_bwd: h too large (%lld)", (long long)h);
    cudaStream_t s = as_stream(stream);
    int nparts = 0;
    if (n > 0) {
        const BwdGrid gr = bwd_grid(n, h);
        nparts = gr.ctas;
        k_rms_bwd<<<gr.ctas, kBwdThreads, gr.smem, s>>>((const bf16*)x, w, inv_rms, (const bf16*)gy,
                                                        (const bf16*)gres, n, (int)h, gr.rpw,
                                                        (bf16*)gx, (float*)ws);
        int rc;
        if ((rc = ee_check_launch("rmsnorm_bwd"))) return rc;
    }
    k_gw_reduce<<<(unsigned)((h + 31) / 32), kRedWarps * 32, 0, s>>>((const float*)ws, nparts, (int)h,
                                                                    accumulate_gw, gw);
    return ee_check_launch("rmsnorm_gw_reduce");
}
