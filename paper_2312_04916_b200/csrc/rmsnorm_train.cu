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

// two sweeps over the row (the second re-reads it from L1)
__global__ void __launch_bounds__(kThreads)
k_rms_fwd(const bf16* __restrict__ x, const float* __restrict__ w, int64_t n, int h, float eps,
          bf16* __restrict__ y, float* __restrict__ inv_out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (row >= n) return;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
    const int nvec = h / 8;
    float ss = 0.f;
    for (int c = lane; c < nvec; c += 32) {
        float v[8];
        unpack8(xr[c], v);
#pragma unroll
        for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / (float)h + eps);
    uint4* yr = reinterpret_cast<uint4*>(y + row * h);
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

// One warp per row.  The row's x and g chunks are loaded 8 per lane at a time
// (8 independent 16-byte loads in flight) and kept in registers for the
// second sweep when the row fits (h <= 2048); gres (optional) is a second
// incoming gradient of x added to gx in the same pass (the residual branch of
// a pre-norm block), so no separate element-wise add reads / writes (n, h).
constexpr int kChunkRegs = 8;  // 16-byte chunks per lane held in registers
__global__ void __launch_bounds__(kThreads)
k_rms_bwd(const bf16* __restrict__ x, const float* __restrict__ w, const float* __restrict__ inv_in,
          const bf16* __restrict__ g, const bf16* __restrict__ gres, int64_t n, int h,
          bf16* __restrict__ gx, float* __restrict__ gw_part) {
    __shared__ float part[kWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
    const bool valid = row < n;
    const int nvec = h / 8;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
    const uint4* gr = reinterpret_cast<const uint4*>(g + row * h);
    const bool held = nvec <= 32 * kChunkRegs;  // whole row in registers
    uint4 xs[kChunkRegs], gs[kChunkRegs];
    float dot = 0.f, inv = 0.f;
    if (valid) {
        inv = inv_in[row];
        for (int c0 = 0; c0 < nvec; c0 += 32 * kChunkRegs) {
#pragma unroll
            for (int u = 0; u < kChunkRegs; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < nvec) {
                    xs[u] = xr[c];
                    gs[u] = gr[c];
                }
            }
#pragma unroll
            for (int u = 0; u < kChunkRegs; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < nvec) {
                    float xv[8], gv[8], ww[8];
                    unpack8(xs[u], xv);
                    unpack8(gs[u], gv);
                    load_w8(w, c, ww);
#pragma unroll
                    for (int k = 0; k < 8; ++k) dot += gv[k] * ww[k] * xv[k];
                }
            }
        }
        dot = warp_sum(dot);
    }
    const float coef = inv * inv * inv * dot / (float)h;
    uint4* gxr = reinterpret_cast<uint4*>(gx + row * h);
    const uint4* rr = gres ? reinterpret_cast<const uint4*>(gres + row * h) : nullptr;
    // second sweep, 256 columns per step for the whole CTA: gx, and this
    // CTA's weight-gradient partial (rows summed in warp order)
    for (int c0 = 0; c0 < nvec; c0 += 32) {
        const int c = c0 + lane;
        float gwv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (valid && c < nvec) {
            float xv[8], gv[8], ww[8], o[8];
            const int u = c0 / 32;
            if (held) {
                // u < kChunkRegs: register-resident chunk (indices unrolled below)
                uint4 xu = xs[0], gu = gs[0];
#pragma unroll
                for (int q = 1; q < kChunkRegs; ++q)
                    if (q == u) {
                        xu = xs[q];
                        gu = gs[q];
                    }
                unpack8(xu, xv);
                unpack8(gu, gv);
            } else {
                unpack8(xr[c], xv);
                unpack8(gr[c], gv);
            }
            load_w8(w, c, ww);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                o[k] = gv[k] * ww[k] * inv - xv[k] * coef;
                gwv[k] = gv[k] * xv[k] * inv;
            }
            if (rr) {
                float rv[8];
                unpack8(rr[c], rv);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] += rv[k];
            }
            gxr[c] = pack8(o);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) part[warp][lane * 8 + k] = gwv[k];
        __syncthreads();
        const int j = c0 * 8 + threadIdx.x;
        if (j < h) {
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < kWarps; ++r) acc += part[r][threadIdx.x];
            gw_part[(int64_t)blockIdx.x * h + j] = acc;
        }
        __syncthreads();
    }
}

// gw_j (+)= sum over CTA partials in CTA order (deterministic), two levels:
// k_gw_reduce1 sums consecutive groups of partials (grid.y groups) into
// level-2 partials, k_gw_reduce2 sums those in group order
constexpr int kGroups = 32;
__global__ void k_gw_reduce1(const float* __restrict__ part, int nparts, int h,
                             float* __restrict__ part2) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= h) return;
    const int g = blockIdx.y;
    const int p0 = (int)((int64_t)nparts * g / kGroups), p1 = (int)((int64_t)nparts * (g + 1) / kGroups);
    float s = 0.f;
    for (int p = p0; p < p1; ++p) s += part[(int64_t)p * h + j];
    part2[(int64_t)g * h + j] = s;
}
__global__ void k_gw_reduce2(const float* __restrict__ part2, int h, int accumulate,
                             float* __restrict__ gw) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= h) return;
    float s = 0.f;
#pragma unroll 8
    for (int g = 0; g < kGroups; ++g) s += part2[(int64_t)g * h + j];
    gw[j] = accumulate ? gw[j] + s : s;
}

}  // namespace

size_t rmsnorm_train_ws_bytes(int64_t n, int64_t h) {
    return ((size_t)((n + kWarps - 1) / kWarps) + kGroups) * (size_t)h * sizeof(float);
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
    cudaStream_t s = as_stream(stream);
    const int nparts = (int)((n + kWarps - 1) / kWarps);
    if (n > 0) {
        k_rms_bwd<<<nparts, kThreads, 0, s>>>((const bf16*)x, w, inv_rms, (const bf16*)gy,
                                              (const bf16*)gres, n, (int)h, (bf16*)gx, (float*)ws);
        int rc;
        if ((rc = ee_check_launch("rmsnorm_bwd"))) return rc;
    }
    float* part2 = (float*)ws + (size_t)nparts * h;
    k_gw_reduce1<<<dim3((unsigned)((h + 255) / 256), kGroups), 256, 0, s>>>((const float*)ws, nparts,
                                                                           (int)h, part2);
    int rc;
    if ((rc = ee_check_launch("rmsnorm_gw_reduce1"))) return rc;
    k_gw_reduce2<<<(unsigned)((h + 255) / 256), 256, 0, s>>>(part2, (int)h, accumulate_gw, gw);
    return ee_check_launch("rmsnorm_gw_reduce2");
}
