// The decode-layer chain and the layer-range launcher used by KV
// recomputation.  Host-side C++ issues the kernels so a whole span of layers
// costs one ABI call (and is CUDA-graph capturable from the caller).
//
// Perf mode (EE_BF16_TILED): 5 PDL-chained kernels per layer.  The RMSNorms
// are folded: attn_norm / mlp_norm were multiplied into the columns of
// Wqkv / W1 at pack time, the GEMVs read the raw bf16 copy of the residual
// rows (xb) and scale their outputs by 1/rms computed from the per-16-column
// sum-of-squares partials (ssq) that the residual epilogues (and
// ee_row_stats) maintain next to x:
//   QKV(xb, ssq) + KV write -> attention -> wo + residual(x, xb, ssq)
//   -> W1(xb, ssq) + GELU -> W2 + residual(x, xb, ssq)
// Parity mode (EE_F32) and row-major bf16: 7 kernels with explicit norms:
//   xn <- rmsnorm(x) -> QKV -> attention -> wo + residual -> attn <-
//   rmsnorm(x) -> W1 + GELU -> xn -> W2 + residual.
#include <stdlib.h>

#include "ee_common.cuh"

// kernels ee_decode_layer launches for a pass of m rows (the launch count a
// caller reports)
int decode_layer_launches(const ee_decoder_t* D, int64_t m) {
    if (m == 0) return 0;
    if (D->dtype != EE_BF16_TILED) return 7;
    const bool prefill = m >= kPrefillMinRows && D->pf_ws &&
                         D->pf_ws_bytes >= (size_t)4 * m * 4 * D->h * sizeof(float);
    return prefill ? 9 : 5;  // 4 x (GEMM + apply) + attention, or 4 GEMVs + attention
}

// profiling stand-in for the attention (EE_ABLATE bit 2): PDL trigger + wait only
__global__ void k_null_pdl() {
    pdl_trigger_dev();
    pdl_wait_dev();
}

extern "C" int ee_decode_layer(const ee_decoder_t* D, const ee_layer_t* L, int64_t row0, int64_t m,
                               const int32_t* pos, int32_t max_pos, void* stream) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(D && L && D->x && pos, EE_ESHAPE, "decode_layer: null argument");
    EE_REQUIRE(row0 >= 0 && row0 + m <= D->max_rows, EE_ESHAPE,
               "decode_layer: rows [%lld, %lld) exceed scratch capacity %lld", (long long)row0,
               (long long)(row0 + m), (long long)D->max_rows);
    cudaStream_t s = as_stream(stream);
    const int64_t h = D->h;
    const int dt = D->dtype;
    float* x = D->x + row0 * h;
    // EE_ABLATE (profiling only; wrong results): bit 0 skips the explicit
    // RMSNorm launches, bit 1 the attention, bit 2 replaces the attention by
    // an empty PDL kernel.
    static const int ablate = getenv("EE_ABLATE") ? atoi(getenv("EE_ABLATE")) : 0;
    // EE_PDL_SKIP (debug): bit k launches kernel k of the tiled decode layer
    // (QKV, attention, wo, w1, w2) without PDL
    static const int pdl_skip = getenv("EE_PDL_SKIP") ? atoi(getenv("EE_PDL_SKIP")) : 0;
    int rc;
    if (dt == EE_BF16_TILED) {
        EE_REQUIRE(D->xb && D->ssq, EE_ESHAPE, "decode_layer: tiled mode needs xb and ssq");
        bf16* xb = (bf16*)D->xb + row0 * h;
        float* ssq = D->ssq + row0 * (h / 16);
        const GemvNorm folded{ssq, D->eps, nullptr, nullptr};
        const GemvNorm stats{nullptr, 0.f, xb, ssq};
        if (m >= kPrefillMinRows && D->pf_ws &&
            D->pf_ws_bytes >= (size_t)4 * m * 4 * h * sizeof(float)) {
            // many rows (prompt prefill): tcgen05 GEMMs instead of GEMVs
            void* pw = D->pf_ws;
            const size_t pb = D->pf_ws_bytes;
            if ((rc = launch_prefill_tiled(xb, m, h, L->wqkv, 3 * h, 0, ssq, D->eps, D->q,
                                           L->kcache, L->vcache, pos, h, nullptr, nullptr, nullptr,
                                           nullptr, pw, pb, s)))
                return rc;
            if ((rc = launch_attention(D->q, m, pos, max_pos, L->kcache, L->vcache, D->nh,
                                       h / D->nh, dt, D->attn, D->ws, D->ws_bytes, s)))
                return rc;
            if ((rc = launch_prefill_tiled((const bf16*)D->attn, m, h, L->wo, h, 2, nullptr, 0.f,
                                           nullptr, nullptr, nullptr, nullptr, h, nullptr, x, xb,
                                           ssq, pw, pb, s)))
                return rc;
            if ((rc = launch_prefill_tiled(xb, m, h, L->w1, 4 * h, 1, ssq, D->eps, nullptr, nullptr,
                                           nullptr, nullptr, h, D->xn, nullptr, nullptr, nullptr, pw,
                                           pb, s)))
                return rc;
            return launch_prefill_tiled((const bf16*)D->xn, m, 4 * h, L->w2, h, 2, nullptr, 0.f,
                                        nullptr, nullptr, nullptr, nullptr, h, nullptr, x, xb, ssq,
                                        pw, pb, s);
        }
        g_pdl_off = pdl_skip & 1;
        if ((rc = launch_qkv_tiled(xb, m, h, L->wqkv, folded, D->q, L->kcache, L->vcache, pos, s)))
            return rc;
        g_pdl_off = pdl_skip & 2;
        if (ablate & 4) {
            if (launch_ex(k_null_pdl, dim3((unsigned)D->nh), dim3(256), 0, s) != cudaSuccess)
                return ee_fail(EE_ECUDA, "null launch");
        } else if (!(ablate & 2) &&
                   (rc = launch_attention(D->q, m, pos, max_pos, L->kcache, L->vcache, D->nh,
                                          h / D->nh, dt, D->attn, D->ws, D->ws_bytes, s)))
            return rc;
        g_pdl_off = pdl_skip & 4;
        if ((rc = launch_gemv_tiled((const bf16*)D->attn, m, h, L->wo, h, EE_EPI_RESIDUAL, x, h,
                                    stats, s)))
            return rc;
        g_pdl_off = pdl_skip & 8;
        if ((rc = launch_gemv_tiled(xb, m, h, L->w1, 4 * h, EE_EPI_GELU, D->xn, 4 * h, folded, s)))
            return rc;
        g_pdl_off = pdl_skip & 16;
        rc = launch_gemv_tiled((const bf16*)D->xn, m, 4 * h, L->w2, h, EE_EPI_RESIDUAL, x, h,
                               stats, s);
        g_pdl_off = pdl_skip & 32;  // whatever follows the layer (next layer, heads)
        return rc;
    }
    if (!(ablate & 1) &&
        (rc = launch_rmsnorm_rows(x, h, nullptr, m, h, L->attn_norm, D->eps, D->xn, dt, s)))
        return rc;
    if ((rc = launch_qkv(D->xn, m, h, L->wqkv, dt, D->q, L->kcache, L->vcache, pos, s))) return rc;
    if (!(ablate & 2) &&
        (rc = launch_attention(D->q, m, pos, max_pos, L->kcache, L->vcache, D->nh, h / D->nh, dt,
                               D->attn, D->ws, D->ws_bytes, s)))
        return rc;
    if ((rc = launch_gemv(D->attn, m, h, L->wo, h, dt, EE_EPI_RESIDUAL, x, h, s))) return rc;
    if (!(ablate & 1) &&
        (rc = launch_rmsnorm_rows(x, h, nullptr, m, h, L->mlp_norm, D->eps, D->attn, dt, s)))
        return rc;
    if ((rc = launch_gemv(D->attn, m, h, L->w1, 4 * h, dt, EE_EPI_GELU, D->xn, 4 * h, s))) return rc;
    return launch_gemv(D->xn, m, 4 * h, L->w2, h, dt, EE_EPI_RESIDUAL, x, h, s);
}

extern "C" int ee_decode_layers(const ee_decoder_t* D, const ee_layer_t* layers, int32_t n_layers,
                                int64_t n_rows, const int32_t* m_active, const int32_t* pos,
                                int32_t max_pos, void* stream) {
    EE_REQUIRE(n_layers >= 0 && (n_layers == 0 || (layers && m_active)), EE_ESHAPE,
               "decode_layers: bad arguments");
    for (int32_t i = 0; i < n_layers; ++i) {
        const int64_t m = m_active[i];
        EE_REQUIRE(m >= 0 && m <= n_rows, EE_ESHAPE, "decode_layers: m_active[%d]=%lld > n_rows",
                   i, (long long)m);
        const int64_t r0 = n_rows - m;
        int rc = ee_decode_layer(D, &layers[i], r0, m, pos + r0, max_pos, stream);
        if (rc) return rc;
    }
    return EE_OK;
}
