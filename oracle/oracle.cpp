// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY. Not part of the product path.
//
// Plain, slow, obviously-correct CPU oracle for the READ-ME (arXiv 2410.19123) pre-gated MoE layer.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
// this library. It shares no code, header, table or helper with paper_2410_19123_b200/ (the CUDA
// path), and the CUDA path never calls it.
//
// Arithmetic: every input is widened exactly to double (bf16 -> double and f32 -> double are exact);
// every intermediate is double; nothing is rounded; no SIMD intrinsics; build with -O2, no fast-math.
// Parallelism: std::thread over independent tokens/rows only, so results are bitwise identical for any
// thread count.
//
// Citations are PAPER.md line numbers (section / equation) in the paper's LaTeX source, plus SPEC.md
// where the desk-scale spec fixes a convention. Readings of the paper (Q1..Q14) are listed in DESIGN.md.
//
// Pins (what keeps this honest, see tests/test_oracle_pins.py):
//   oracle_route        : P3 invariants, P6 SPEC worked examples, brute-force rank definition (P5)
//   oracle_dispatch     : P3 bijection + bit copy
//   oracle_expert_ffn   : P1 full-FFN expert == dense FFN, P2 partition identity, P7 closed forms, P8 ReLU
//                         SPEC examples, P9 zero input, P10 power-of-two scaling
//   oracle_combine      : P7(iii) hand combination, SPEC.md:162 (0.75, 3.75)
//   oracle_moe_layer    : P4 permutation equivariance, P5 brute force, P11 route-once
//   oracle_bruteforce   : independent Eq. 2 evaluation from the DENSE weights (no sort/scan/buffers)
//   oracle_ep_sim       : P12 == oracle_moe_layer exactly
// Parity unpinned: realism of the synthetic activations/weights/logits (no checkpoint exists here).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ---- exact widening of the three storage dtypes -------------------------------------------------
enum Dt : int32_t { DT_F64 = 0, DT_F32 = 1, DT_BF16 = 2 };

inline double load(const void* p, int32_t dt, int64_t i) {
    if (dt == DT_F64) return static_cast<const double*>(p)[i];
    if (dt == DT_F32) return static_cast<double>(static_cast<const float*>(p)[i]);
    // bf16: the upper 16 bits of an IEEE binary32.
    uint32_t bits = static_cast<uint32_t>(static_cast<const uint16_t*>(p)[i]) << 16;
    float f;
    std::memcpy(&f, &bits, 4);
    return static_cast<double>(f);
}

inline bool dt_ok(int32_t dt) { return dt == DT_F64 || dt == DT_F32 || dt == DT_BF16; }

template <class F>
void parallel_for(int64_t n, int32_t nthreads, F&& f) {
    if (nthreads <= 1 || n < 2) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    if (nthreads > n) nthreads = static_cast<int32_t>(n);
    std::vector<std::thread> pool;
    for (int32_t w = 0; w < nthreads; ++w) {
        pool.emplace_back([&, w]() {
            for (int64_t i = w; i < n; i += nthreads) f(i);
        });
    }
    for (auto& th : pool) th.join();
}

// SiLU as the Llama-2 SwiGLU FFN uses it: silu(z) = z / (1 + e^{-z}) (PAPER.md:159 with sigma = SwiGLU, Q4).
inline double silu(double z) { return z / (1.0 + std::exp(-z)); }

// One expert FFN on one row: F_i(x) = W_2 M_i^T sigma(M_i W_1 x), with the mask already
// applied (the expert's own stacked weights). act 0: SwiGLU h = silu(Wg x) * (Wu x).
// act 1: the paper's literal two-layer form with sigma = ReLU, h = relu(Wg x) (Wu unused) — used only to
// check SPEC's hand examples verbatim.
void ffn_row(const void* xrow, int32_t xdt, int64_t xoff, int32_t H, int32_t d, const void* wg,
             const void* wu, const void* wd, int32_t wdt, int64_t wg_off, int64_t wd_off, int32_t act,
             std::vector<double>& h, double* yrow) {
    for (int32_t n = 0; n < d; ++n) {
        double g = 0.0, u = 0.0;
        for (int32_t c = 0; c < H; ++c) {
            const double xc = load(xrow, xdt, xoff + c);
            g += load(wg, wdt, wg_off + static_cast<int64_t>(n) * H + c) * xc;
            if (act == 0) u += load(wu, wdt, wg_off + static_cast<int64_t>(n) * H + c) * xc;
        }
        h[n] = (act == 0) ? silu(g) * u : (g > 0.0 ? g : 0.0);
    }
    for (int32_t c = 0; c < H; ++c) {
        double acc = 0.0;
        for (int32_t n = 0; n < d; ++n) acc += load(wd, wdt, wd_off + static_cast<int64_t>(c) * d + n) * h[n];
        yrow[c] = acc;
    }
}

}  // namespace

extern "C" {

// Status codes of the oracle (its own; unrelated to the product's readme_status).
enum { ORACLE_OK = 0, ORACLE_BAD_ARG = 1, ORACLE_NONFINITE = 2 };

int oracle_version(void) { return 1; }

// ---- a1-a4: top-K selection, gate weights, histogram, exclusive scan, stable permutation ------------
// Eq. 2: expert i is selected for token t iff |{j : G_j >= G_i}| <= K. Read with Q2
// (exactly K experts, ties -> lower id), the indicator becomes a rank:
//     rank_i = #{j : G_j > G_i} + #{j < i : G_j == G_i};   selected iff rank_i < K,
// and rank_i is the output position (descending logit, then ascending id).
// Weights (Q1): softmax over the selected logits, w_j = exp(l_j - m) / sum exp(l_j' - m).
// Grouping (Alg. 1 ReqQueueByExpert): counts[e] = #{(t,j): idx[t][j] = e};
// offsets[0] = 0, offsets[e+1] = offsets[e] + counts[e]; for flat slot s = t*K + j in ascending order
// (FIFO queues, Q7), dest[s] = offsets[e] + (number of earlier slots with the same expert); src = dest^-1.
int oracle_route(const void* logits, int32_t logits_dt, int64_t T, int32_t E, int32_t K, int32_t* idx,
                 double* w, int32_t* counts, int32_t* offsets, int32_t* dest, int32_t* src) {
    if (T < 0 || E < 1 || K < 1 || K > E || !dt_ok(logits_dt)) return ORACLE_BAD_ARG;
    for (int64_t i = 0; i < T * E; ++i)
        if (!std::isfinite(load(logits, logits_dt, i))) return ORACLE_NONFINITE;  // SPEC.md:167, Q3
    std::vector<double> sel(K);
    for (int64_t t = 0; t < T; ++t) {
        for (int32_t i = 0; i < E; ++i) {
            const double gi = load(logits, logits_dt, t * E + i);
            int32_t rank = 0;
            for (int32_t j = 0; j < E; ++j) {
                const double gj = load(logits, logits_dt, t * E + j);
                if (gj > gi || (gj == gi && j < i)) ++rank;
            }
            if (rank < K) {
                idx[t * K + rank] = i;
                sel[rank] = gi;
            }
        }
        const double m = sel[0];
        double z = 0.0;
        for (int32_t j = 0; j < K; ++j) z += std::exp(sel[j] - m);
        for (int32_t j = 0; j < K; ++j) w[t * K + j] = std::exp(sel[j] - m) / z;
    }
    for (int32_t e = 0; e < E; ++e) counts[e] = 0;
    for (int64_t s = 0; s < T * K; ++s) counts[idx[s]] += 1;
    offsets[0] = 0;
    for (int32_t e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + counts[e];
    std::vector<int32_t> fill(E, 0);
    for (int64_t s = 0; s < T * K; ++s) {
        const int32_t e = idx[s];
        dest[s] = offsets[e] + fill[e]++;
        if (src) src[dest[s]] = static_cast<int32_t>(s);
    }
    return ORACLE_OK;
}

// ---- a5: dispatch, x_sorted[dest[s]] = x[s / K] (tokens grouped by their expert) -----
int oracle_dispatch(const void* x, int32_t xdt, int64_t T, int32_t H, int32_t K, const int32_t* dest,
                    double* x_sorted) {
    if (T < 0 || H < 1 || K < 1 || !dt_ok(xdt)) return ORACLE_BAD_ARG;
    for (int64_t s = 0; s < T * K; ++s) {
        const int64_t t = s / K;
        if (dest[s] < 0 || dest[s] >= T * K) return ORACLE_BAD_ARG;
        for (int32_t c = 0; c < H; ++c) x_sorted[static_cast<int64_t>(dest[s]) * H + c] = load(x, xdt, t * H + c);
    }
    return ORACLE_OK;
}

// ---- a6+a7: per-expert FFN over expert-contiguous rows ----------------------------------------------
// Segment g covers rows [offsets[g], offsets[g+1]); its expert is g % E (n_src source groups of E
// segments each; n_src = 1 on one GPU, n_src = G for the expert-parallel receive buffer).
// Weights: w_gate/w_up [E][d][H] (rows = the expert's neurons S_e of W_1), w_down [E][H][d] (columns).
int oracle_expert_ffn(const void* x_sorted, int32_t xdt, int64_t rows, int32_t H, int32_t E, int32_t d,
                      int32_t n_src, const int32_t* offsets, const void* w_gate, const void* w_up,
                      const void* w_down, int32_t wdt, int32_t act, double* y_sorted, int32_t nthreads) {
    if (rows < 0 || H < 1 || E < 1 || d < 1 || n_src < 1 || !dt_ok(xdt) || !dt_ok(wdt)) return ORACLE_BAD_ARG;
    const int64_t nseg = static_cast<int64_t>(n_src) * E;
    if (offsets[0] != 0 || offsets[nseg] != rows) return ORACLE_BAD_ARG;
    std::vector<int32_t> seg_of(rows);
    for (int64_t g = 0; g < nseg; ++g) {
        if (offsets[g + 1] < offsets[g]) return ORACLE_BAD_ARG;
        for (int64_t r = offsets[g]; r < offsets[g + 1]; ++r) seg_of[r] = static_cast<int32_t>(g);
    }
    parallel_for(rows, nthreads, [&](int64_t r) {
        std::vector<double> h(d);
        const int64_t e = seg_of[r] % E;
        ffn_row(x_sorted, xdt, r * H, H, d, w_gate, w_up, w_down, wdt, e * d * H, e * H * d, act, h,
                y_sorted + r * H);
    });
    return ORACLE_OK;
}

// ---- RMSNorm for the MoE-only pre-norm stack (reading Q10 in DESIGN.md; Llama-2's RMSNorm with weight 1):
// y[t] = x[t] / sqrt(mean_c x[t][c]^2 + eps).
int oracle_rmsnorm(const void* x, int32_t xdt, int64_t T, int32_t H, double eps, double* y) {
    if (T < 0 || H < 1 || eps < 0 || !dt_ok(xdt)) return ORACLE_BAD_ARG;
    for (int64_t t = 0; t < T; ++t) {
        double ss = 0.0;
        for (int32_t c = 0; c < H; ++c) {
            const double v = load(x, xdt, t * H + c);
            ss += v * v;
        }
        const double r = 1.0 / std::sqrt(ss / H + eps);
        for (int32_t c = 0; c < H; ++c) y[t * H + c] = load(x, xdt, t * H + c) * r;
    }
    return ORACLE_OK;
}

// ---- a6 alone: h_r = silu(W_gate,e x_r) * (W_up,e x_r) (the hidden activation of expert e's SwiGLU FFN,
// PAPER.md:159 with sigma = SwiGLU). h [rows][d] double.
int oracle_expert_hidden(const void* x_sorted, int32_t xdt, int64_t rows, int32_t H, int32_t E, int32_t d,
                         int32_t n_src, const int32_t* offsets, const void* w_gate, const void* w_up, int32_t wdt,
                         double* h, int32_t nthreads) {
    if (rows < 0 || H < 1 || E < 1 || d < 1 || n_src < 1 || !dt_ok(xdt) || !dt_ok(wdt)) return ORACLE_BAD_ARG;
    const int64_t nseg = static_cast<int64_t>(n_src) * E;
    if (offsets[0] != 0 || offsets[nseg] != rows) return ORACLE_BAD_ARG;
    std::vector<int32_t> seg_of(rows);
    for (int64_t g = 0; g < nseg; ++g) {
        if (offsets[g + 1] < offsets[g]) return ORACLE_BAD_ARG;
        for (int64_t r = offsets[g]; r < offsets[g + 1]; ++r) seg_of[r] = static_cast<int32_t>(g);
    }
    parallel_for(rows, nthreads, [&](int64_t r) {
        const int64_t e = seg_of[r] % E;
        for (int32_t n = 0; n < d; ++n) {
            double g = 0.0, u = 0.0;
            for (int32_t c = 0; c < H; ++c) {
                const double xc = load(x_sorted, xdt, r * H + c);
                g += load(w_gate, wdt, (e * d + n) * static_cast<int64_t>(H) + c) * xc;
                u += load(w_up, wdt, (e * d + n) * static_cast<int64_t>(H) + c) * xc;
            }
            h[r * d + n] = silu(g) * u;
        }
    });
    return ORACLE_OK;
}

// ---- a7 alone: y_r = W_down,e h_r (the W_2 M_i^T factor). y [rows][H] double.
int oracle_expert_down(const void* h, int32_t hdt, int64_t rows, int32_t H, int32_t E, int32_t d, int32_t n_src,
                       const int32_t* offsets, const void* w_down, int32_t wdt, double* y, int32_t nthreads) {
    if (rows < 0 || H < 1 || E < 1 || d < 1 || n_src < 1 || !dt_ok(hdt) || !dt_ok(wdt)) return ORACLE_BAD_ARG;
    const int64_t nseg = static_cast<int64_t>(n_src) * E;
    if (offsets[0] != 0 || offsets[nseg] != rows) return ORACLE_BAD_ARG;
    std::vector<int32_t> seg_of(rows);
    for (int64_t g = 0; g < nseg; ++g) {
        if (offsets[g + 1] < offsets[g]) return ORACLE_BAD_ARG;
        for (int64_t r = offsets[g]; r < offsets[g + 1]; ++r) seg_of[r] = static_cast<int32_t>(g);
    }
    parallel_for(rows, nthreads, [&](int64_t r) {
        const int64_t e = seg_of[r] % E;
        for (int32_t c = 0; c < H; ++c) {
            double acc = 0.0;
            for (int32_t n = 0; n < d; ++n)
                acc += load(w_down, wdt, (e * H + c) * static_cast<int64_t>(d) + n) * load(h, hdt, r * d + n);
            y[r * H + c] = acc;
        }
    });
    return ORACLE_OK;
}

// ---- a8: combine, y[t] = res[t] + sum_{j<K} w[t][j] * y_sorted[dest[t*K+j]] (Eq. 2's weighted sum,
// PAPER.md:137; j ascending, Q8). residual may be null.
int oracle_combine(const double* y_sorted, int64_t T, int32_t H, int32_t K, const int32_t* dest,
                   const double* w, const void* residual, int32_t rdt, double* y) {
    if (T < 0 || H < 1 || K < 1 || (residual && !dt_ok(rdt))) return ORACLE_BAD_ARG;
    for (int64_t t = 0; t < T; ++t) {
        for (int32_t c = 0; c < H; ++c) {
            double acc = residual ? load(residual, rdt, t * H + c) : 0.0;
            for (int32_t j = 0; j < K; ++j) acc += w[t * K + j] * y_sorted[static_cast<int64_t>(dest[t * K + j]) * H + c];
            y[t * H + c] = acc;
        }
    }
    return ORACLE_OK;
}

// ---- the whole layer: a1..a8 composed (Eq. 2). Outputs the routing plan too. --------------------------
int oracle_moe_layer(const void* x, int32_t xdt, int64_t T, int32_t H, const void* logits, int32_t ldt,
                     int32_t E, int32_t K, int32_t d, const void* w_gate, const void* w_up,
                     const void* w_down, int32_t wdt, int32_t act, const void* residual, int32_t rdt,
                     double* y, int32_t* idx, double* w, int32_t* counts, int32_t* offsets, int32_t* dest,
                     int32_t* src, int32_t nthreads) {
    int rc = oracle_route(logits, ldt, T, E, K, idx, w, counts, offsets, dest, src);
    if (rc) return rc;
    std::vector<double> xs(static_cast<size_t>(T * K) * H), ys(static_cast<size_t>(T * K) * H);
    rc = oracle_dispatch(x, xdt, T, H, K, dest, xs.data());
    if (rc) return rc;
    rc = oracle_expert_ffn(xs.data(), DT_F64, T * K, H, E, d, 1, offsets, w_gate, w_up, w_down, wdt, act,
                           ys.data(), nthreads);
    if (rc) return rc;
    return oracle_combine(ys.data(), T, H, K, dest, w, residual, rdt, y);
}

// ---- the dense FFN F_0(x) = W_2 sigma(W_1 x), SwiGLU form, written separately ----------
// dense_w_gate/up [D][H], dense_w_down [H][D].
int oracle_dense_ffn(const void* x, int32_t xdt, int64_t T, int32_t H, int32_t D, const void* wg,
                     const void* wu, const void* wd, int32_t wdt, int32_t act, double* y, int32_t nthreads) {
    if (T < 0 || H < 1 || D < 1 || !dt_ok(xdt) || !dt_ok(wdt)) return ORACLE_BAD_ARG;
    parallel_for(T, nthreads, [&](int64_t t) {
        std::vector<double> h(D);
        for (int32_t n = 0; n < D; ++n) {
            double g = 0.0, u = 0.0;
            for (int32_t c = 0; c < H; ++c) {
                const double xc = load(x, xdt, t * H + c);
                g += load(wg, wdt, static_cast<int64_t>(n) * H + c) * xc;
                if (act == 0) u += load(wu, wdt, static_cast<int64_t>(n) * H + c) * xc;
            }
            h[n] = (act == 0) ? silu(g) * u : (g > 0.0 ? g : 0.0);
        }
        for (int32_t c = 0; c < H; ++c) {
            double acc = 0.0;
            for (int32_t n = 0; n < D; ++n) acc += load(wd, wdt, static_cast<int64_t>(c) * D + n) * h[n];
            y[t * H + c] = acc;
        }
    });
    return ORACLE_OK;
}

// ---- expert slicing (setup row of §8(a)): W_gate,e = W_gate[S_e,:], W_up,e = W_up[S_e,:],
// W_down,e = W_down[:,S_e] (M_i a selection matrix without replacement).
// Outputs are double copies (exact).
int oracle_build_experts(const void* wg, const void* wu, const void* wd, int32_t wdt, int32_t D, int32_t H,
                         int32_t E, int32_t d, const int32_t* neuron_idx, double* eg, double* eu, double* ed) {
    if (D < 1 || H < 1 || E < 1 || d < 1 || d > D || !dt_ok(wdt)) return ORACLE_BAD_ARG;
    for (int32_t e = 0; e < E; ++e) {
        for (int32_t n = 0; n < d; ++n) {
            const int32_t src = neuron_idx[e * d + n];
            if (src < 0 || src >= D || (n > 0 && src <= neuron_idx[e * d + n - 1])) return ORACLE_BAD_ARG;
            for (int32_t c = 0; c < H; ++c) {
                eg[(static_cast<int64_t>(e) * d + n) * H + c] = load(wg, wdt, static_cast<int64_t>(src) * H + c);
                eu[(static_cast<int64_t>(e) * d + n) * H + c] = load(wu, wdt, static_cast<int64_t>(src) * H + c);
            }
            for (int32_t c = 0; c < H; ++c)
                ed[(static_cast<int64_t>(e) * H + c) * d + n] = load(wd, wdt, static_cast<int64_t>(c) * D + src);
        }
    }
    return ORACLE_OK;
}

// ---- brute force: Eq. 2 evaluated literally per token, with no sort, scan, permutation or stacked
// expert buffers. For each expert i the indicator is evaluated by counting (Q2 tie rule), the weight is
// the softmax over the selected logits, and F_i(x_t) is computed straight from the DENSE weights through
// the expert's neuron list S_i (W_2 M_i^T sigma(M_i W_1 x)). Sum over i ascending.
int oracle_bruteforce(const void* x, int32_t xdt, int64_t T, int32_t H, const void* logits, int32_t ldt,
                      int32_t E, int32_t K, int32_t D, int32_t d, const void* wg, const void* wu,
                      const void* wd, int32_t wdt, const int32_t* neuron_idx, int32_t act, double* y) {
    if (T < 0 || H < 1 || E < 1 || K < 1 || K > E || d < 1 || d > D) return ORACLE_BAD_ARG;
    std::vector<double> h(d);
    for (int64_t t = 0; t < T; ++t) {
        std::vector<char> on(E, 0);
        double m = -INFINITY;
        for (int32_t i = 0; i < E; ++i) {
            const double gi = load(logits, ldt, t * E + i);
            if (!std::isfinite(gi)) return ORACLE_NONFINITE;
            int32_t ge = 0;  // |{j : G_j >= G_i}| with ties broken towards the lower id (Q2)
            for (int32_t j = 0; j < E; ++j) {
                const double gj = load(logits, ldt, t * E + j);
                if (gj > gi || (gj == gi && j < i)) ++ge;
            }
            on[i] = (ge < K);
            if (on[i] && gi > m) m = gi;
        }
        double z = 0.0;
        for (int32_t i = 0; i < E; ++i)
            if (on[i]) z += std::exp(load(logits, ldt, t * E + i) - m);
        for (int32_t c = 0; c < H; ++c) y[t * H + c] = 0.0;
        for (int32_t i = 0; i < E; ++i) {
            if (!on[i]) continue;
            const double wi = std::exp(load(logits, ldt, t * E + i) - m) / z;
            const int32_t* S = neuron_idx + static_cast<int64_t>(i) * d;
            for (int32_t n = 0; n < d; ++n) {
                double g = 0.0, u = 0.0;
                for (int32_t c = 0; c < H; ++c) {
                    const double xc = load(x, xdt, t * H + c);
                    g += load(wg, wdt, static_cast<int64_t>(S[n]) * H + c) * xc;
                    if (act == 0) u += load(wu, wdt, static_cast<int64_t>(S[n]) * H + c) * xc;
                }
                h[n] = (act == 0) ? silu(g) * u : (g > 0.0 ? g : 0.0);
            }
            for (int32_t c = 0; c < H; ++c) {
                double acc = 0.0;
                for (int32_t n = 0; n < d; ++n) acc += load(wd, wdt, static_cast<int64_t>(c) * D + S[n]) * h[n];
                y[t * H + c] += wi * acc;
            }
        }
    }
    return ORACLE_OK;
}

// ---- expert-parallel simulation: G simulated ranks, tokens split contiguously
// (rank r holds tokens [r*T/G, (r+1)*T/G)), experts split contiguously (rank q owns experts
// [q*E/G, (q+1)*E/G)). Each rank routes its own tokens with the same pre-gating logits, sends the rows of
// each expert to its owner (all-to-all, rows received in source-rank order), the owner evaluates its
// experts, the rows go back (reverse all-to-all) and each rank combines locally. Everything is in one
// address space; the "network" is memcpy of doubles. Must equal oracle_moe_layer exactly (P12).
int oracle_ep_sim(int32_t G, const void* x, int32_t xdt, int64_t T, int32_t H, const void* logits,
                  int32_t ldt, int32_t E, int32_t K, int32_t d, const void* w_gate, const void* w_up,
                  const void* w_down, int32_t wdt, int32_t act, double* y, int32_t nthreads) {
    if (G < 1 || T % G != 0 || E % G != 0) return ORACLE_BAD_ARG;
    const int64_t Tl = T / G;
    const int32_t El = E / G;
    // Per rank: local routing plan and local expert-sorted rows.
    std::vector<std::vector<int32_t>> idx(G), offs(G), dst(G);
    std::vector<std::vector<double>> wts(G), xs(G), ys(G);
    for (int32_t r = 0; r < G; ++r) {
        idx[r].resize(Tl * K);
        wts[r].resize(Tl * K);
        offs[r].resize(E + 1);
        dst[r].resize(Tl * K);
        std::vector<int32_t> cnt(E), srcv(Tl * K);
        const size_t lsz = ldt == DT_F64 ? 8 : (ldt == DT_F32 ? 4 : 2);
        const size_t xsz = xdt == DT_F64 ? 8 : (xdt == DT_F32 ? 4 : 2);
        const void* lr = static_cast<const char*>(logits) + static_cast<size_t>(r * Tl * E) * lsz;
        const void* xr = static_cast<const char*>(x) + static_cast<size_t>(r * Tl * H) * xsz;
        int rc = oracle_route(lr, ldt, Tl, E, K, idx[r].data(), wts[r].data(), cnt.data(), offs[r].data(),
                              dst[r].data(), srcv.data());
        if (rc) return rc;
        xs[r].resize(static_cast<size_t>(Tl * K) * H);
        rc = oracle_dispatch(xr, xdt, Tl, H, K, dst[r].data(), xs[r].data());
        if (rc) return rc;
        ys[r].resize(xs[r].size());
    }
    // Owner q receives, from each source p in ascending order, p's rows for experts [q*El, (q+1)*El).
    for (int32_t q = 0; q < G; ++q) {
        std::vector<int32_t> seg_off(static_cast<size_t>(G) * El + 1, 0);
        std::vector<double> recv;
        for (int32_t p = 0; p < G; ++p) {
            for (int32_t el = 0; el < El; ++el) {
                const int32_t e = q * El + el;
                const int32_t g = p * El + el;
                seg_off[g + 1] = seg_off[g] + (offs[p][e + 1] - offs[p][e]);
            }
            const int64_t b = offs[p][q * El], n = offs[p][(q + 1) * El] - b;
            recv.insert(recv.end(), xs[p].begin() + b * H, xs[p].begin() + (b + n) * H);
        }
        const int64_t rows = seg_off[static_cast<size_t>(G) * El];
        std::vector<double> out(static_cast<size_t>(rows) * H);
        // expert of segment g is g % El on the owner, i.e. global expert q*El + g % El.
        const size_t wsz = wdt == DT_F64 ? 8 : (wdt == DT_F32 ? 4 : 2);
        const void* wgq = static_cast<const char*>(w_gate) + static_cast<size_t>(q) * El * d * H * wsz;
        const void* wuq = static_cast<const char*>(w_up) + static_cast<size_t>(q) * El * d * H * wsz;
        const void* wdq = static_cast<const char*>(w_down) + static_cast<size_t>(q) * El * H * d * wsz;
        int rc = oracle_expert_ffn(recv.data(), DT_F64, rows, H, El, d, G, seg_off.data(), wgq, wuq, wdq, wdt,
                                   act, out.data(), nthreads);
        if (rc) return rc;
        // Reverse all-to-all: rows go back to their source rank, in the order they came.
        int64_t cur = 0;
        for (int32_t p = 0; p < G; ++p) {
            const int64_t b = offs[p][q * El], n = offs[p][(q + 1) * El] - b;
            std::memcpy(ys[p].data() + b * H, out.data() + cur * H, static_cast<size_t>(n * H) * sizeof(double));
            cur += n;
        }
    }
    for (int32_t r = 0; r < G; ++r) {
        int rc = oracle_combine(ys[r].data(), Tl, H, K, dst[r].data(), wts[r].data(), nullptr, 0,
                                y + r * Tl * H);
        if (rc) return rc;
    }
    return ORACLE_OK;
}

}  // extern "C"
