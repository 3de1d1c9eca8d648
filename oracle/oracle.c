/*
 * oracle.c — plain, slow, obviously-correct CPU forward pass.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this.  The product path (paper_2306_03622_b200/) never does.
 *
 * What it computes: swapping and pipelining change WHEN
 * bytes arrive, not WHAT is computed — "This approach does not affect the execution
 * order, and thus can still ensure the correctness of the model inference"
 * (§"Asynchronous API redirection"); inference "is typically executed
 * layer by layer" (§"Model swapping and pipeline execution").  So the
 * oracle is the plain definition of the forward pass: the layer table executed in
 * order, every op written out from its textbook definition, in IEEE double precision,
 * over the caller's bf16/f32 weight bytes (upcast exactly).  There is no blocking,
 * fusion or reordering; each output element is accumulated sequentially in index
 * order, so results do not depend on the OpenMP thread count.
 *
 * Shares no code with the CUDA path: its own structs (or_*), its own bf16 decode,
 * its own op definitions.  Its only contact with the product is the byte format of
 * the caller's weight blob and the layer-table vocabulary (op / act / rule numbers),
 * which it restates here.
 *
 * Pins: tests/test_oracle_*.py (closed forms, textbook constants, brute force,
 * torch float64 / HF transformers reference modules).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* Thread control for the timed CPU baseline (bench.py): torchrun pins OMP_NUM_THREADS=1 per rank, so
 * the thread count is set explicitly; the result does not depend on it (each output element is
 * accumulated sequentially by one thread). */
int oracle_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}

/* ---- table vocabulary (restated; see synth/models.py and include/fsw.h) ---- */
enum { OR_EMBED = 1, OR_LAYERNORM = 2, OR_LINEAR = 3, OR_ATTENTION = 4,
       OR_CONV2D = 5, OR_MAXPOOL = 6, OR_AVGPOOL = 7 };
enum { OR_ACT_NONE = 0, OR_ACT_RELU = 1, OR_ACT_GELU_ERF = 2, OR_ACT_GELU_TANH = 3, OR_ACT_TANH = 4 };
enum { OR_RULE_IDS = 0, OR_RULE_POSITION = 1, OR_RULE_ZERO = 2 };
enum { OR_BF16 = 0, OR_F32 = 1, OR_I32 = 2 };

typedef struct { uint64_t offset, bytes; uint32_t dtype, rank; uint32_t shape[4]; } or_tensor;
typedef struct { uint32_t dtype, rank; uint32_t shape[4]; } or_slot;
typedef struct { uint32_t op, first_ref, n_refs; int32_t in0, in1, out; int32_t attr[8]; } or_layer;

typedef struct {
    const uint8_t* w;
    const or_tensor* tensors;
    const uint32_t* refs;
    const or_slot* slots;
    double* const* buf;      /* one float64 buffer per slot, caller-allocated */
} or_model;

/* ---- scalar definitions ---- */
static double bf16_to_f64(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* element i of tensor t as double (bf16 or f32 storage) */
static double tval(const or_model* m, uint32_t t, uint64_t i) {
    const or_tensor* T = &m->tensors[t];
    if (T->dtype == OR_BF16) {
        uint16_t b;
        memcpy(&b, m->w + T->offset + 2 * i, 2);
        return bf16_to_f64(b);
    }
    float f;
    memcpy(&f, m->w + T->offset + 4 * i, 4);
    return (double)f;
}

static uint64_t slot_numel(const or_slot* s) {
    uint64_t n = 1;
    for (uint32_t i = 0; i < s->rank; ++i) n *= s->shape[i];
    return n;
}

/* GELU(x) = x·Φ(x) (Hendrycks & Gimpel), erf form (BERT, MLP) — SURVEY §8c reading #4 */
double or_gelu_erf(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }
/* GELU tanh approximation used by GPT-2 */
double or_gelu_tanh(double x) {
    return 0.5 * x * (1.0 + tanh(sqrt(2.0 / M_PI) * (x + 0.044715 * x * x * x)));
}

static double act(int a, double x) {
    switch (a) {
        case OR_ACT_RELU: return x > 0.0 ? x : 0.0;
        case OR_ACT_GELU_ERF: return or_gelu_erf(x);
        case OR_ACT_GELU_TANH: return or_gelu_tanh(x);
        case OR_ACT_TANH: return tanh(x);
        default: return x;
    }
}

static float attr_f32(int32_t a) { float f; memcpy(&f, &a, 4); return f; }

/* ---- ops ---- */

/* EMBED: out[t][c] = Σ_j table_j[row_j(t)][c]   (BERT word+position+type; GPT wte+wpe) */
static int op_embed(const or_model* m, const or_layer* L) {
    const or_slot* so = &m->slots[L->out];
    const uint32_t T = so->shape[0], C = so->shape[1];
    const double* ids = m->buf[L->in0];
    double* out = m->buf[L->out];
    int nt = L->attr[0];
    for (uint32_t t = 0; t < T; ++t) {
        for (uint32_t c = 0; c < C; ++c) {
            double s = 0.0;
            for (int j = 0; j < nt; ++j) {
                uint32_t tid = m->refs[L->first_ref + j];
                uint64_t row;
                if (L->attr[1 + j] == OR_RULE_IDS) row = (uint64_t)ids[t];
                else if (L->attr[1 + j] == OR_RULE_POSITION) row = t;
                else row = 0;
                if (row >= m->tensors[tid].shape[0]) return -1;
                s += tval(m, tid, row * C + c);
            }
            out[(uint64_t)t * C + c] = s;
        }
    }
    return 0;
}

/* LAYERNORM over the last dim: y = (x − μ)/sqrt(σ² + eps)·γ + β, σ² the biased variance */
static int op_layernorm(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const uint32_t C = si->shape[si->rank - 1];
    const uint64_t R = slot_numel(si) / C;
    const double eps = (double)attr_f32(L->attr[0]);
    const uint32_t tg = m->refs[L->first_ref], tb = m->refs[L->first_ref + 1];
    const double* x = m->buf[L->in0];
    double* y = m->buf[L->out];
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)R; ++r) {
        const double* xr = x + r * C;
        double mu = 0.0, var = 0.0;
        for (uint32_t c = 0; c < C; ++c) mu += xr[c];
        mu /= C;
        for (uint32_t c = 0; c < C; ++c) var += (xr[c] - mu) * (xr[c] - mu);
        var /= C;
        const double inv = 1.0 / sqrt(var + eps);
        for (uint32_t c = 0; c < C; ++c)
            y[r * C + c] = (xr[c] - mu) * inv * tval(m, tg, c) + tval(m, tb, c);
    }
    return 0;
}

/* LINEAR: y[i][o] = act( Σ_k x[r0+i][k]·W[o][k] + b[o] + res[i][o] ),  W stored [out][in] */
static int op_linear(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const or_slot* so = &m->slots[L->out];
    const uint32_t K = si->shape[si->rank - 1];
    const uint64_t Rin = slot_numel(si) / K;
    const uint32_t tw = m->refs[L->first_ref];
    const uint32_t N = m->tensors[tw].shape[0];
    if (m->tensors[tw].shape[1] != K) return -1;
    const int has_b = L->n_refs > 1;
    const uint32_t tbias = has_b ? m->refs[L->first_ref + 1] : 0;
    const uint64_t r0 = (uint64_t)L->attr[1];
    const uint64_t R = L->attr[2] > 0 ? (uint64_t)L->attr[2] : Rin;
    if (r0 + R > Rin || slot_numel(so) != R * N) return -1;
    const double* x = m->buf[L->in0];
    const double* res = L->in1 >= 0 ? m->buf[L->in1] : NULL;
    double* y = m->buf[L->out];
    const int a = L->attr[0];
#pragma omp parallel
    {
        double* wrow = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(static)
        for (int64_t o = 0; o < (int64_t)N; ++o) {
            for (uint32_t k = 0; k < K; ++k) wrow[k] = tval(m, tw, (uint64_t)o * K + k);
            const double b = has_b ? tval(m, tbias, o) : 0.0;
            for (uint64_t i = 0; i < R; ++i) {
                const double* xr = x + (r0 + i) * K;
                double s = 0.0;
                for (uint32_t k = 0; k < K; ++k) s += xr[k] * wrow[k];
                s += b;
                if (res) s += res[i * N + o];
                y[i * N + o] = act(a, s);
            }
        }
        free(wrow);
    }
    return 0;
}

/* ATTENTION (core of multi-head self-attention): qkv row t = [q | k | v], each H·dh wide,
 * head h = columns h·dh … h·dh+dh−1.  S = q kᵀ/√dh, causal mask j > t, P = softmax(S),
 * ctx[t][h·dh + d] = Σ_j P[t][j]·v[j][h·dh + d]. */
static int op_attention(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const uint32_t T = si->shape[0], W3 = si->shape[1];
    const int H = L->attr[0], dh = L->attr[1], causal = L->attr[2];
    const uint32_t D = (uint32_t)(H * dh);
    if (W3 != 3 * D) return -1;
    const double* qkv = m->buf[L->in0];
    double* ctx = m->buf[L->out];
    const double scale = 1.0 / sqrt((double)dh);
#pragma omp parallel
    {
        double* p = (double*)malloc(sizeof(double) * T);
#pragma omp for collapse(2) schedule(static)
        for (int h = 0; h < H; ++h) {
            for (int64_t t = 0; t < (int64_t)T; ++t) {
                const double* q = qkv + t * W3 + (uint64_t)h * dh;
                const uint32_t jmax = causal ? (uint32_t)t + 1 : T;
                double mx = -INFINITY;
                for (uint32_t j = 0; j < jmax; ++j) {
                    const double* k = qkv + (uint64_t)j * W3 + D + (uint64_t)h * dh;
                    double s = 0.0;
                    for (int d = 0; d < dh; ++d) s += q[d] * k[d];
                    p[j] = s * scale;
                    if (p[j] > mx) mx = p[j];
                }
                double z = 0.0;
                for (uint32_t j = 0; j < jmax; ++j) { p[j] = exp(p[j] - mx); z += p[j]; }
                for (int d = 0; d < dh; ++d) {
                    double s = 0.0;
                    for (uint32_t j = 0; j < jmax; ++j)
                        s += p[j] * qkv[(uint64_t)j * W3 + 2 * D + (uint64_t)h * dh + d];
                    ctx[t * D + (uint64_t)h * dh + d] = s / z;
                }
            }
        }
        free(p);
    }
    return 0;
}

/* CONV2D, NHWC activations [H][W][C], weights KRSC [Cout][R][S][Cin], batch 1, square kernel:
 * out[p][q][co] = act( Σ_{r,s,ci} in[p·st−pad+r][q·st−pad+s][ci]·W[co][r][s][ci] + b[co] + res[p][q][co] ),
 * zero padding outside the image. */
static int op_conv2d(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const or_slot* so = &m->slots[L->out];
    const uint32_t Hi = si->shape[0], Wi = si->shape[1], Ci = si->shape[2];
    const uint32_t Ho = so->shape[0], Wo = so->shape[1], Co = so->shape[2];
    const uint32_t tw = m->refs[L->first_ref], tb = m->refs[L->first_ref + 1];
    const or_tensor* Tw = &m->tensors[tw];
    const uint32_t R = Tw->shape[1], S = Tw->shape[2];
    if (Tw->shape[0] != Co || Tw->shape[3] != Ci) return -1;
    const int a = L->attr[0], st = L->attr[1], pad = L->attr[2];
    const double* x = m->buf[L->in0];
    const double* res = L->in1 >= 0 ? m->buf[L->in1] : NULL;
    double* y = m->buf[L->out];
#pragma omp parallel for schedule(static)
    for (int64_t co = 0; co < (int64_t)Co; ++co) {
        for (uint32_t p = 0; p < Ho; ++p) {
            for (uint32_t q = 0; q < Wo; ++q) {
                double s = 0.0;
                for (uint32_t r = 0; r < R; ++r) {
                    const int ih = (int)(p * st) - pad + (int)r;
                    if (ih < 0 || ih >= (int)Hi) continue;
                    for (uint32_t c = 0; c < S; ++c) {
                        const int iw = (int)(q * st) - pad + (int)c;
                        if (iw < 0 || iw >= (int)Wi) continue;
                        const double* xp = x + ((uint64_t)ih * Wi + iw) * Ci;
                        const uint64_t wb = (((uint64_t)co * R + r) * S + c) * Ci;
                        for (uint32_t ci = 0; ci < Ci; ++ci) s += xp[ci] * tval(m, tw, wb + ci);
                    }
                }
                s += tval(m, tb, co);
                const uint64_t oi = ((uint64_t)p * Wo + q) * Co + co;
                if (res) s += res[oi];
                y[oi] = act(a, s);
            }
        }
    }
    return 0;
}

/* MAXPOOL k×k / stride, padding counts as −∞ */
static int op_maxpool(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const or_slot* so = &m->slots[L->out];
    const uint32_t Hi = si->shape[0], Wi = si->shape[1], C = si->shape[2];
    const uint32_t Ho = so->shape[0], Wo = so->shape[1];
    const int k = L->attr[0], st = L->attr[1], pad = L->attr[2];
    const double* x = m->buf[L->in0];
    double* y = m->buf[L->out];
    for (uint32_t p = 0; p < Ho; ++p)
        for (uint32_t q = 0; q < Wo; ++q)
            for (uint32_t c = 0; c < C; ++c) {
                double mx = -INFINITY;
                for (int r = 0; r < k; ++r)
                    for (int s = 0; s < k; ++s) {
                        const int ih = (int)(p * st) - pad + r, iw = (int)(q * st) - pad + s;
                        if (ih < 0 || iw < 0 || ih >= (int)Hi || iw >= (int)Wi) continue;
                        const double v = x[((uint64_t)ih * Wi + iw) * C + c];
                        if (v > mx) mx = v;
                    }
                y[((uint64_t)p * Wo + q) * C + c] = mx;
            }
    return 0;
}

/* AVGPOOL (global): y[c] = (1/(H·W)) Σ_{h,w} x[h][w][c] */
static int op_avgpool(const or_model* m, const or_layer* L) {
    const or_slot* si = &m->slots[L->in0];
    const uint32_t HW = si->shape[0] * si->shape[1], C = si->shape[2];
    const double* x = m->buf[L->in0];
    double* y = m->buf[L->out];
    for (uint32_t c = 0; c < C; ++c) {
        double s = 0.0;
        for (uint32_t i = 0; i < HW; ++i) s += x[(uint64_t)i * C + c];
        y[c] = s / HW;
    }
    return 0;
}

/* Decode the request input into its float64 slot. */
int oracle_load_input(const or_slot* s, const uint8_t* in, double* buf) {
    const uint64_t n = slot_numel(s);
    for (uint64_t i = 0; i < n; ++i) {
        if (s->dtype == OR_I32) { int32_t v; memcpy(&v, in + 4 * i, 4); buf[i] = v; }
        else if (s->dtype == OR_F32) { float v; memcpy(&v, in + 4 * i, 4); buf[i] = v; }
        else { uint16_t v; memcpy(&v, in + 2 * i, 2); buf[i] = bf16_to_f64(v); }
    }
    return 0;
}

/* Run layers [first, last) of the table in order.  Returns 0, or −(index+1) of a bad layer. */
int oracle_run(const uint8_t* weights, const or_tensor* tensors, const uint32_t* refs,
               const or_slot* slots, const or_layer* layers, uint32_t first, uint32_t last,
               double* const* slot_bufs) {
    or_model m = { weights, tensors, refs, slots, slot_bufs };
    for (uint32_t i = first; i < last; ++i) {
        const or_layer* L = &layers[i];
        int rc;
        switch (L->op) {
            case OR_EMBED: rc = op_embed(&m, L); break;
            case OR_LAYERNORM: rc = op_layernorm(&m, L); break;
            case OR_LINEAR: rc = op_linear(&m, L); break;
            case OR_ATTENTION: rc = op_attention(&m, L); break;
            case OR_CONV2D: rc = op_conv2d(&m, L); break;
            case OR_MAXPOOL: rc = op_maxpool(&m, L); break;
            case OR_AVGPOOL: rc = op_avgpool(&m, L); break;
            default: rc = -1;
        }
        if (rc != 0) return -(int)(i + 1);
    }
    return 0;
}
