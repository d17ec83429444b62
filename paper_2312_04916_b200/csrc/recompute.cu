// The KV-recomputation decode loop of `generate_kv_recompute`
// (eepipe/inference.py:256-381, run_pass 283-327) as ONE native call: the
// host side of every pass (control block, gather lists, layer segments,
// head evaluations, exit decisions, deferred-token bookkeeping, KV fill
// discipline) runs in C++ with the GIL released, so the GPU is idle only for
// the unavoidable decision round trip at an exit tap or at the end of a
// pass (~microseconds of host work instead of Python's ~100 µs per token).
//
// Semantics follow the reference line by line (see inference.py's Python
// restatement `_PassRunner` / `_kv_recompute`, which this replaces):
//   * rows of a pass are ordered by entry depth DESCENDING (deferred tokens,
//     then the new one); layer l advances the rows with entry < l (a suffix);
//   * a head at tap t is evaluated for row r iff (t > entry_r or (t == 0 and
//     entry_r == 0)) and (r is the decide row or entry_r > 0);
//   * the first firing head at the decide row's shallowest tap decides, the
//     final head decides otherwise; an unforced pass stops at that tap;
//   * a pass is forced (full depth) when max_deferred rows are deferred;
//     after a shallow pass every row is re-deferred at max(entry, depth);
//   * a final flush pass completes the deferred KV (no decide row);
//   * KV at (layer, position) is written exactly once and read only after it
//     was written (KVCache.fill / view, inference.py:58-70).
#include <chrono>
#include <cmath>
#include <cstring>
#include <atomic>
#include <vector>

#include "ee_common.cuh"

namespace {

struct Slot {
    int head;   // index into heads
    int off;    // ctrl offset of the chunk's row list
    int count;  // rows in the chunk
    int row0;   // index of the chunk's first row in the tap's row list
    int tap;    // layer index of the head
};

struct Runner {
    const ee_generate_args_t* A;
    const ee_engine_t* E;
    cudaStream_t s;
    int L, h;
    std::vector<int> taps;                 // distinct head taps, ascending
    std::vector<std::vector<int>> at_tap;  // head indices per tap
    std::vector<uint8_t> kv;               // [L][s_max] fill mask
    int stage = 0;                         // alternating host staging half
    bool mapped = false;                   // result slots in host-mapped memory (res == res_host)
    std::chrono::steady_clock::time_point t_start;

    int64_t launches = 0, h2d = 0, d2h = 0;

    int32_t* host_half() { return E->ctrl_host + (int64_t)stage * E->ctrl_cap; }

    int upload(const int32_t* src, int64_t n) {
        EE_REQUIRE(n <= E->ctrl_cap, EE_ESHAPE, "recompute: control block overflow (%lld > %lld)",
                   (long long)n, (long long)E->ctrl_cap);
        h2d += 4 * n;
        return ee_copy_h2d(E->ctrl, src, (size_t)n * 4, E->stream);
    }

    int eval_head(int hi, const int32_t* rows_dev, int m, int slot) {
        const ee_head_t& hd = E->heads[hi];
        const float* xsrc = E->dec->x;
        const int32_t* rows = rows_dev;
        int rc;
        if (hd.kind == 2) {  // mlp+embed: x' = x + GELU(RMSNorm(x; pre_norm) W1) W2
            if ((rc = ee_rmsnorm_rows(E->dec->x, h, rows, m, h, nullptr, E->eps, E->head_x, EE_F32,
                                      E->stream)))
                return rc;
            if ((rc = ee_rmsnorm_rows((const float*)E->head_x, h, nullptr, m, h, hd.pre_norm, E->eps,
                                      E->head_xn, E->dcode, E->stream)))
                return rc;
            if ((rc = ee_gemv(E->head_xn, m, h, hd.w1t, 4 * (int64_t)h, E->dcode, EE_EPI_GELU,
                              E->head_mid, 4 * (int64_t)h, E->stream)))
                return rc;
            if ((rc = ee_gemv(E->head_mid, m, 4 * (int64_t)h, hd.w2t, h, E->dcode, EE_EPI_RESIDUAL,
                              E->head_x, h, E->stream)))
                return rc;
            xsrc = (const float*)E->head_x;
            rows = nullptr;
            launches += 4;
        }
        launches += 2;  // row gather + norm, then the head GEMV
        uint8_t* r = E->res + (int64_t)slot * E->res_stride;
        if (mapped)  // host-mapped result slot: arm its completion word
            *(volatile int32_t*)(E->res_host + (int64_t)slot * E->res_stride + E->off_bad) = -1;
        return ee_exit_head_infer(xsrc, h, rows, m, h, hd.norm, E->eps, hd.W, hd.V, E->wcode,
                                  A->threshold, (int32_t*)(r + E->off_tok), (float*)(r + E->off_conf),
                                  r + E->off_fire, (int32_t*)(r + E->off_bad), nullptr, E->head_ws,
                                  E->head_ws_bytes, E->stream);
    }

    int mark_written(int la, int lb, const int32_t* pos, int n_act) {
        // layers la..lb (1-based) wrote K/V at pos[0..n_act); each of those
        // rows then read [0, pos] (eepipe/inference.py:58-70)
        int maxp = 0;
        for (int i = 0; i < n_act; ++i) maxp = pos[i] > maxp ? pos[i] : maxp;
        for (int l = la; l <= lb; ++l) {
            uint8_t* mrow = kv.data() + (int64_t)(l - 1) * A->s_max;
            for (int i = 0; i < n_act; ++i) {
                EE_REQUIRE(!mrow[pos[i]], EE_ECONFIG, "KV at layer %d, position %d already filled", l,
                           pos[i]);
                mrow[pos[i]] = 1;
            }
            for (int p = 0; p <= maxp; ++p)
                EE_REQUIRE(mrow[p], EE_ECONFIG, "reading unfilled KV at layer %d below %d", l,
                           maxp + 1);
        }
        return EE_OK;
    }

    // one run_pass; decide_row < 0: flush pass.  embed_tok >= 0: embed the
    // new token into row n-1 first.  Returns rc; decision in (*tok, *layer),
    // *has = 0 if no decision; *depth.
    const ee_decoder_t* dec = nullptr;  // decoder used by the current pass

    int pass(int n, const int32_t* pos, const int32_t* entry, int decide_row, bool forced,
             int embed_tok, int embed_pos, int* tok, int* layer, int* has, int* depth) {
        int rc;
        // control block: positions | per-tap gather lists | new token id, position
        stage ^= 1;
        int32_t* c = host_half();
        int64_t len = 0;
        for (int r = 0; r < n; ++r) c[len++] = pos[r];
        std::vector<int> list_off(taps.size(), -1), list_len(taps.size(), 0);
        for (size_t ti = 0; ti < taps.size(); ++ti) {
            const int tap = taps[ti];
            const int64_t start = len;
            for (int r = 0; r < n; ++r)
                if ((tap > entry[r] || (tap == 0 && entry[r] == 0)) &&
                    (r == decide_row || entry[r] > 0))
                    c[len++] = r;
            if (len > start) {
                list_off[ti] = (int)start;
                list_len[ti] = (int)(len - start);
            }
        }
        int64_t emb_off = -1;
        if (embed_tok >= 0) {
            emb_off = len;
            c[len++] = embed_tok;
            c[len++] = embed_pos;
        }
        if ((rc = upload(c, len))) return rc;
        const ee_decoder_t* D = dec ? dec : E->dec;
        if (embed_tok >= 0) {
            const bool tiled = D->dtype == EE_BF16_TILED;
            launches += tiled ? 2 : 1;
            if ((rc = ee_embed_stats(E->ctrl + emb_off, E->ctrl + emb_off + 1, 1, E->tok_emb,
                                     E->pos_emb, h, E->dcode, D->x + (int64_t)(n - 1) * h,
                                     tiled ? (char*)D->xb + 2 * (int64_t)(n - 1) * h : nullptr,
                                     tiled ? D->ssq + (int64_t)(n - 1) * (h / 16) : nullptr,
                                     E->stream)))
                return rc;
        }
        int max_pos = 0;
        for (int r = 0; r < n; ++r) max_pos = pos[r] > max_pos ? pos[r] : max_pos;

        std::vector<Slot> slots;
        int checked = 0;
        *has = 0;
        *depth = L;
        auto eval_tap = [&](int tap, bool* gates) -> int {
            *gates = false;
            size_t ti = 0;
            while (ti < taps.size() && taps[ti] != tap) ++ti;
            if (ti == taps.size() || list_off[ti] < 0) return EE_OK;
            const int off = list_off[ti], cnt = list_len[ti];
            for (int hi : at_tap[ti]) {
                for (int c0 = 0; c0 < cnt; c0 += A->head_max_rows) {
                    const int m = cnt - c0 < A->head_max_rows ? cnt - c0 : A->head_max_rows;
                    const int slot = (int)slots.size();
                    EE_REQUIRE(slot < E->max_slots, EE_ECONFIG, "too many head evaluations in one pass");
                    int rc2 = eval_head(hi, E->ctrl + off + c0, m, slot);
                    if (rc2) return rc2;
                    slots.push_back(Slot{hi, off, m, c0, tap});
                    for (int j = 0; j < m; ++j)
                        if (c[off + c0 + j] == decide_row) *gates = true;
                }
            }
            return EE_OK;
        };
        auto decide_from = [&]() -> int {
            const int upto = (int)slots.size();
            if (upto == checked) return EE_OK;
            const size_t nb = (size_t)upto * E->res_stride;
            d2h += nb;
            if (mapped) {
                // the heads write straight into host memory; the word each
                // writes last (nonfinite flag) was armed to -1 at launch
                for (int k = checked; k < upto; ++k) {
                    const volatile int32_t* done =
                        (const volatile int32_t*)(E->res_host + (int64_t)k * E->res_stride + E->off_bad);
                    long spins = 0;
                    while (*done == -1) {
                        if ((++spins & 0xFFFF) == 0) {  // surface a failed launch
                            const cudaError_t q = cudaStreamQuery(s);
                            EE_REQUIRE(q == cudaSuccess || q == cudaErrorNotReady, EE_ECUDA,
                                       "pass sync: %s", cudaGetErrorString(q));
                            if (q == cudaSuccess && *done == -1)
                                return ee_fail(EE_ECUDA, "exit head result never arrived");
                        }
                    }
                }
                std::atomic_thread_fence(std::memory_order_acquire);
            } else {
                cudaError_t e = cudaMemcpyAsync(E->res_host, E->res, nb, cudaMemcpyDeviceToHost, s);
                EE_REQUIRE(e == cudaSuccess, EE_ECUDA, "result copy: %s", cudaGetErrorString(e));
                e = cudaStreamSynchronize(s);
                EE_REQUIRE(e == cudaSuccess, EE_ECUDA, "pass sync: %s", cudaGetErrorString(e));
            }
            for (int k = 0; k < upto; ++k) {
                const uint8_t* r = E->res_host + (int64_t)k * E->res_stride;
                EE_REQUIRE(*(const int32_t*)(r + E->off_bad) == 0, EE_ENONFINITE,
                           "non-finite exit logits");
            }
            for (int k = checked; k < upto; ++k) {
                const Slot& sl = slots[k];
                const ee_head_t& hd = E->heads[sl.head];
                const uint8_t* r = E->res_host + (int64_t)k * E->res_stride;
                for (int j = 0; j < sl.count; ++j) {
                    const int row = c[sl.off + sl.row0 + j];
                    if (row == decide_row && !*has) {
                        const int t = ((const int32_t*)(r + E->off_tok))[j];
                        if (hd.is_final) {
                            *tok = t;
                            *layer = L;
                            *has = 1;
                        } else if ((r + E->off_fire)[j]) {
                            *tok = t;
                            *layer = hd.tap;
                            *has = 1;
                        }
                    }
                }
            }
            checked = upto;
            return EE_OK;
        };
        auto log = [&]() {
            for (size_t k = 0; k < slots.size(); ++k) {
                const Slot& sl = slots[k];
                const uint8_t* r = E->res_host + (int64_t)k * E->res_stride;
                for (int j = 0; j < sl.count; ++j) {
                    const int row = c[sl.off + sl.row0 + j];
                    A->conf[(int64_t)pos[row] * A->n_heads + sl.head] =
                        ((const float*)(r + E->off_conf))[j];
                }
            }
        };

        bool gates;
        if ((rc = eval_tap(0, &gates))) return rc;
        if (gates && !forced && (A->threshold < 1.0f || L == 0)) {
            if ((rc = decide_from())) return rc;
            if (*has && *layer == 0) {
                log();
                *depth = 0;
                return EE_OK;
            }
        }
        std::vector<int> stops;
        for (int t : taps)
            if (t >= 1) stops.push_back(t);
        if (stops.empty() || stops.back() != L) stops.push_back(L);
        std::vector<int32_t> m_act_arr(L + 1);
        int la = 1;
        for (int tap : stops) {
            int l = la;
            while (l <= tap) {
                auto active = [&](int layer) {
                    int m = 0;
                    for (int r = 0; r < n; ++r) m += entry[r] < layer;
                    return m;
                };
                const int m_act = active(l);
                int l2 = l;
                while (l2 + 1 <= tap && active(l2 + 1) == m_act) ++l2;
                if (m_act) {
                    for (int i = 0; i <= l2 - l; ++i) m_act_arr[i] = m_act;
                    launches += (int64_t)decode_layer_launches(D, m_act) * (l2 - l + 1);
                    if ((rc = ee_decode_layers(D, E->layers + (l - 1), l2 - l + 1, n,
                                               m_act_arr.data(), E->ctrl, max_pos, E->stream)))
                        return rc;
                    if ((rc = mark_written(l, l2, pos + (n - m_act), m_act))) return rc;
                }
                l = l2 + 1;
            }
            la = tap + 1;
            if ((rc = eval_tap(tap, &gates))) return rc;
            if (gates && !forced && !*has && (A->threshold < 1.0f || tap == L)) {
                if ((rc = decide_from())) return rc;
                if (*has && !forced && *layer == tap && tap < L) {
                    *depth = tap;
                    break;
                }
            }
        }
        if (checked < (int)slots.size())
            if ((rc = decide_from())) return rc;
        log();
        return EE_OK;
    }
};

}  // namespace

extern "C" int ee_generate_kv_recompute(ee_generate_args_t* A) {
    EE_REQUIRE(A && A->engine && A->engine->dec, EE_ESHAPE, "recompute: null argument");
    const ee_engine_t* E = A->engine;
    EE_REQUIRE(A->prompt_len >= 1, EE_ECONFIG, "prompt must be non-empty");
    EE_REQUIRE(A->max_deferred >= 1, EE_ECONFIG, "max_deferred must be at least 1");
    EE_REQUIRE(A->threshold > 0.f && A->threshold <= 1.f, EE_ECONFIG, "threshold must lie in (0, 1]");
    EE_REQUIRE(A->prompt_len + A->max_new <= A->s_max, EE_ETOKEN,
               "context of %d positions exceeds max_seq_len %d", A->prompt_len + A->max_new, A->s_max);
    EE_REQUIRE(E->dec->max_rows >= A->prompt_len && E->dec->max_rows >= A->max_deferred + 1,
               EE_ESHAPE, "recompute: decoder scratch too small");
    Runner R;
    R.A = A;
    R.E = E;
    R.s = as_stream(E->stream);
    R.L = E->n_layers;
    R.h = (int)E->dec->h;
    R.mapped = E->res == E->res_host;
    for (int i = 0; i < E->n_heads; ++i) {
        const int t = E->heads[i].tap;
        if (R.taps.empty() || R.taps.back() != t) {
            R.taps.push_back(t);
            R.at_tap.emplace_back();
        }
        R.at_tap.back().push_back(i);
    }
    R.kv.assign((size_t)R.L * A->s_max, 0);
    R.t_start = std::chrono::steady_clock::now();
    auto now_s = [&]() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - R.t_start).count();
    };
    int rc;
    const int L = R.L;
    const int t0 = A->prompt_len;
    // prefill: every prompt row at full depth, its last row decides token 1
    {
        R.stage ^= 1;
        int32_t* c = R.host_half();
        for (int i = 0; i < t0; ++i) {
            c[i] = A->prompt[i];
            c[t0 + i] = i;
        }
        if ((rc = R.upload(c, 2 * (int64_t)t0))) return rc;
        const ee_decoder_t* D = E->dec;
        const bool tiled = D->dtype == EE_BF16_TILED;
        R.launches += tiled ? 2 : 1;
        if ((rc = ee_embed_stats(E->ctrl, E->ctrl + t0, t0, E->tok_emb, E->pos_emb, R.h, E->dcode,
                                 D->x, tiled ? D->xb : nullptr, tiled ? D->ssq : nullptr,
                                 E->stream)))
            return rc;
    }
    std::vector<int32_t> pos(t0), ent(t0, 0);
    for (int i = 0; i < t0; ++i) pos[i] = i;
    int tok = 0, layer = L, has = 0, depth = L;
    // the prefill pass (and only it) may take the multi-row tcgen05 GEMM
    ee_decoder_t dec_prefill = *E->dec;
    dec_prefill.pf_ws = E->pf_ws;
    dec_prefill.pf_ws_bytes = E->pf_ws_bytes;
    R.dec = &dec_prefill;
    rc = R.pass(t0, pos.data(), ent.data(), t0 - 1, true, -1, 0, &tok, &layer, &has, &depth);
    R.dec = nullptr;
    if (rc) return rc;
    EE_REQUIRE(has, EE_ECUDA, "recompute: prefill produced no decision");
    A->pass_depths[0] = L;
    std::vector<int32_t> dpos, dent;  // deferred tokens: rows 0..k-1, entry descending
    int position = t0 - 1;
    int gen = 0;
    double t_last = 0.0;
    for (int i = 0; i < A->max_new; ++i) {
        A->tokens[i] = tok;
        A->exit_layers[i] = layer;
        const double t = now_s();
        A->latency_s[i] = t - t_last;
        t_last = t;
        gen = i + 1;
        if (i == A->max_new - 1) break;
        ++position;
        const bool forced = (int)dpos.size() >= A->max_deferred;
        const int n = (int)dpos.size() + 1;
        pos.assign(dpos.begin(), dpos.end());
        pos.push_back(position);
        ent.assign(dent.begin(), dent.end());
        ent.push_back(0);
        if ((rc = R.pass(n, pos.data(), ent.data(), n - 1, forced, tok, position, &tok, &layer, &has,
                         &depth)))
            return rc;
        EE_REQUIRE(has, EE_ECUDA, "recompute: pass produced no decision");
        A->pass_depths[i + 1] = depth;
        if (depth < L) {
            for (auto& e : dent) e = e > depth ? e : depth;
            dpos.push_back(position);
            dent.push_back(depth);
        } else {
            dpos.clear();
            dent.clear();
        }
        EE_REQUIRE((int)dpos.size() <= A->max_deferred, EE_ECUDA, "deferred list overflow");
    }
    A->n_generated = gen;
    A->flushed = 0;
    if (!dpos.empty()) {  // complete the remaining KV entries and deep-exit confidences
        int dummy_tok, dummy_layer, dummy_has, dummy_depth;
        if ((rc = R.pass((int)dpos.size(), dpos.data(), dent.data(), -1, true, -1, 0, &dummy_tok,
                         &dummy_layer, &dummy_has, &dummy_depth)))
            return rc;
        A->flushed = 1;
    }
    const cudaError_t e = cudaStreamSynchronize(R.s);
    EE_REQUIRE(e == cudaSuccess, EE_ECUDA, "recompute: final sync: %s", cudaGetErrorString(e));
    A->total_s = now_s();
    // KV must be complete for every position < t0 + gen - 1 (inference.py:373-374)
    for (int l = 0; l < L; ++l)
        for (int p = 0; p < t0 + gen - 1; ++p)
            EE_REQUIRE(R.kv[(size_t)l * A->s_max + p], EE_ECONFIG,
                       "KV fill mask incomplete after generation");
    if (A->kv_mask) std::memcpy(A->kv_mask, R.kv.data(), R.kv.size());
    A->launches = R.launches;
    A->h2d_bytes = R.h2d;
    A->d2h_bytes = R.d2h;
    return EE_OK;
}
