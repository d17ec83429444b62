// The decode-layer chain and the layer-range launcher used by KV
// recomputation.  Host-side C++ issues the kernels so a whole span of layers
// costs one ABI call (and is CUDA-graph capturable from the caller).
//
// Scratch use per layer (dec->xn is (rows, 4h), dec->attn is (rows, h)):
//   xn[:, :h] <- rmsnorm(x, attn_norm)        -> QKV GEMV (+ KV write) -> q
//   attn      <- attention(q)                 -> wo GEMV, residual into x
//   attn      <- rmsnorm(x, mlp_norm)         -> w1 GEMV + GELU -> xn (4h)
//   xn        -> w2 GEMV, residual into x
#include "ee_common.cuh"

extern "C" int ee_decode_layer(const ee_decoder_t* D, const ee_layer_t* L, float* x, int64_t m,
                               const int32_t* pos, int32_t max_pos, void* stream) {
    if (m == 0) return EE_OK;
    EE_REQUIRE(D && L && x && pos, EE_ESHAPE, "decode_layer: null argument");
    EE_REQUIRE(m <= D->max_rows, EE_ESHAPE, "decode_layer: %lld rows > scratch capacity %lld",
               (long long)m, (long long)D->max_rows);
    cudaStream_t s = as_stream(stream);
    const int64_t h = D->h;
    const int dt = D->dtype;
    int rc;
    // 7 PDL-chained kernels; the TMA GEMVs prefetch their weights while the
    // preceding (small) kernel runs
    if ((rc = launch_rmsnorm_rows(x, h, nullptr, m, h, L->attn_norm, D->eps, D->xn, dt, s))) return rc;
    if ((rc = launch_qkv(D->xn, m, h, L->wqkv, dt, D->q, L->kcache, L->vcache, pos, s))) return rc;
    if ((rc = launch_attention(D->q, m, pos, max_pos, L->kcache, L->vcache, D->nh, h / D->nh, dt,
                               D->attn, D->ws, D->ws_bytes, s)))
        return rc;
    if ((rc = launch_gemv(D->attn, m, h, L->wo, h, dt, EE_EPI_RESIDUAL, x, h, s))) return rc;
    if ((rc = launch_rmsnorm_rows(x, h, nullptr, m, h, L->mlp_norm, D->eps, D->attn, dt, s))) return rc;
    if ((rc = launch_gemv(D->attn, m, h, L->w1, 4 * h, dt, EE_EPI_GELU, D->xn, 4 * h, s))) return rc;
    return launch_gemv(D->xn, m, 4 * h, L->w2, h, dt, EE_EPI_RESIDUAL, x, h, s);
}

extern "C" int ee_decode_layers(const ee_decoder_t* D, const ee_layer_t* layers, int32_t n_layers,
                                int64_t n_rows, const int32_t* m_active, float* x,
                                const int32_t* pos, int32_t max_pos, void* stream) {
    EE_REQUIRE(n_layers >= 0 && (n_layers == 0 || (layers && m_active)), EE_ESHAPE,
               "decode_layers: bad arguments");
    for (int32_t i = 0; i < n_layers; ++i) {
        const int64_t m = m_active[i];
        EE_REQUIRE(m >= 0 && m <= n_rows, EE_ESHAPE, "decode_layers: m_active[%d]=%lld > n_rows",
                   i, (long long)m);
        const int64_t r0 = n_rows - m;
        int rc = ee_decode_layer(D, &layers[i], x + r0 * D->h, m, pos + r0, max_pos, stream);
        if (rc) return rc;
    }
    return EE_OK;
}
