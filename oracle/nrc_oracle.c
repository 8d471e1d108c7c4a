/*
 * nrc_oracle.c -- plain, slow, fp64 CPU ORACLE for the Neural Radiance Caching
 * hot path (Mueller, Rousselle, Novak, Keller, "Real-time Neural Radiance
 * Caching for Path Tracing", arXiv 2106.12372).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2106_12372_b200/, libnrc.so) never links, imports
 * or calls anything in oracle/; the two share no code, headers, tables or
 * constant generators.  Inputs reach both sides only through nrc_inputs/
 * (seeded generators, no method arithmetic).
 *
 * Citations: "P:L<n>" = /root/reference/PAPER.md line n; "S:L<n>" = SPEC.md
 * line n; numbered readings (R1..R20) are listed in DESIGN.md section 3.
 *
 * Every function is the plain definition written out, in the paper's order
 * and notation: no blocking, fusion or reordering.  fp64 throughout, except
 * the position normalisation step (R3), which both sides fix to fp32 so the
 * integer floor parts of the triangle wave are bit-identical.
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   orc_tri, orc_quartic, orc_one_blob, orc_sph, orc_freq ... pinned (closed
 *       forms, SPEC worked examples, periodicity, integral of quartic = 1)
 *   orc_encode ............................................. pinned (golden
 *       vector tests/golden/encode_c0.txt, structural invariants)
 *   orc_*_d (depth nh, N4) ................................... pinned (nh = 5
 *       equals the pinned width functions; identity-layer extensions of a
 *       net compute the same function and gradients; finite differences)
 *   orc_grad_batch_exact (N4 training) ..................... pinned (central
 *       finite differences through the exact encodings)
 *   orc_freq_sin / orc_gauss / orc_encode_exact (N4) ....... pinned (sin at
 *       dyadic points, Gaussian closed forms, layout shared with orc_encode)
 *   orc_query_accumulate ................................... pinned (unit
 *       throughput + identity pixels = query, permutation, accumulation)
 *   orc_assemble_targets ................................... pinned (one-vertex
 *       closed form, unbiased flag, hand-evaluated 3-vertex path, linearity)
 *   orc_forward_w / orc_query_batch_w / orc_init_weights_w . pinned (width
 *       embedding into the 64 net, numpy matmul chain, Glorot moments)
 *   orc_backward_w / orc_grad_batch_w / orc_train_step_w ... pinned (exact
 *       zero-padding embeddings 32 -> 64 and 64 -> 128 against the pinned
 *       width-64 functions, central finite differences at hw = 32 and 128)
 *   orc_forward / orc_query ................................ pinned (zero net,
 *       constant net via pad channel, linear chain, homogeneity, permutation)
 *   orc_loss ............................................... pinned (S:L193-195
 *       values 0.2493766 and 33.333, FD with frozen luminance)
 *   orc_backward / orc_grad_batch .......................... pinned (central
 *       finite differences, zero-gradient, 1-layer outer product)
 *   orc_adam ............................................... pinned (zero grad,
 *       first-step |dw| = lr|g|/(|g|+eps), monotonicity)
 *   orc_ema ................................................ pinned (t=1,
 *       constant stream 1e4 steps, a=0, linearity, printed-form 0.5124*C)
 *   orc_lcg_* .............................................. pinned (S:L274
 *       example [3,0,1,2], bijection for many n)
 *   orc_init_weights ....................................... pinned (Glorot
 *       bound, moments of the uniform distribution)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---- architecture (reading R1: 6 weight matrices) ------------ */
#define ORC_IN 64     /* 62 encoded dims padded to 64            */
#define ORC_HID 64    /* "five hidden layers have 64 neurons each"  */
#define ORC_OUT 3     /* "reduces the 64 dimensions to three RGB values"     */
#define ORC_NMAT 6
/* logical parameter layout: W0..W4 (64x64), W5 (3x64), row-major [out][in] */
#define ORC_NPARAM (5 * 64 * 64 + 3 * 64)

static const int64_t orc_mat_off[ORC_NMAT + 1] = {0, 4096, 8192, 12288, 16384, 20480, 20672};
static const int orc_mat_rows[ORC_NMAT] = {64, 64, 64, 64, 64, 3};

int64_t orc_param_count(void) { return ORC_NPARAM; }

/* ---- cheap primitives, fig:cheap_primitives ------------------ */

/* tri(x) := 2 | x mod 2 - 1 | - 1 with floored modulo. */
double orc_tri(double x)
{
    double m = x - 2.0 * floor(x / 2.0); /* x mod 2 in [0, 2) */
    return 2.0 * fabs(m - 1.0) - 1.0;
}

/* quartic(x) := 15/16 (1 - x^2)^2 on |x| <= 1, else 0. */
double orc_quartic(double x)
{
    if (fabs(x) > 1.0) return 0.0;
    double t = 1.0 - x * x;
    return 15.0 / 16.0 * t * t;
}

/* One-blob encoding with k evenly spaced kernels (k=4 P:L588).
 * Reading R6: centres (i+1/2)/k, width 1/k, input clamped to [0,1]. */
void orc_one_blob(double s, int k, double* out)
{
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
    for (int i = 0; i < k; ++i) {
        double c = (i + 0.5) / k;
        out[i] = orc_quartic((s - c) * k);
    }
}

/* sph(u): conversion to spherical coordinates normalised to [0,1]^2
 * (Table 1 caption).  Reading R7: theta' = acos(z)/pi,
 * phi' = (atan2(y,x)+pi)/(2 pi), order (theta', phi'); zero vector -> (0,0,1).
 * Returns 1 if the input was the zero vector (counted by callers). */
int orc_sph(const double* u_in, double* out)
{
    double x = u_in[0], y = u_in[1], z = u_in[2];
    double len = sqrt(x * x + y * y + z * z);
    int degenerate = 0;
    if (!(len > 0.0)) {
        x = 0.0; y = 0.0; z = 1.0;
        degenerate = 1;
    } else {
        x /= len; y /= len; z /= len;
    }
    if (z > 1.0) z = 1.0;
    if (z < -1.0) z = -1.0;
    out[0] = acos(z) / M_PI;
    out[1] = (atan2(y, x) + M_PI) / (2.0 * M_PI);
    return degenerate;
}

/* Frequency encoding with 12 triangle waves of frequency 2^d, d = 0..11,
 * cosine terms omitted (tri replaces sin).
 * Reading R4: entry d = tri(2^d v). */
void orc_freq(double v, double* out12)
{
    for (int d = 0; d < 12; ++d) out12[d] = orc_tri(ldexp(v, d));
}

/* Position normalisation (reading R3): v = fp32(fp32(p - lo) * inv),
 * inv = fp32(1 / fp32(hi - lo)), no clamp, no FMA contraction. */
float orc_normalize_pos(float p, float lo, float hi)
{
    volatile float ext = hi - lo;
    volatile float inv = 1.0f / ext;
    volatile float d = p - lo;
    volatile float v = d * inv;
    return v;
}

/* Input encoding, Table 1 + padding.
 * record layout (nrc_inputs, 16 floats): pos[3] dir[3] normal[3] roughness
 * diffuse[3] specular[3].  Output e[64] (readings R4-R6, R19):
 *   e[12a+d]  = tri(2^d v_a)           a = x,y,z; d = 0..11   (36)
 *   e[36..39] = ob(theta'(omega)), e[40..43] = ob(phi'(omega))   (8)
 *   e[44..47] = ob(theta'(n)),     e[48..51] = ob(phi'(n))       (8)
 *   e[52..55] = ob(1 - exp(-r))                                  (4)
 *   e[56..58] = alpha, e[59..61] = beta (identity)       (6)
 *   e[62] = e[63] = 1 (pad with a value of 1)            (2)
 * Returns the number of degenerate (zero) direction vectors. */
int orc_encode(const float* rec, const float* aabb_lo, const float* aabb_hi, double* e)
{
    int degenerate = 0;
    for (int a = 0; a < 3; ++a) {
        float v = orc_normalize_pos(rec[a], aabb_lo[a], aabb_hi[a]);
        orc_freq((double)v, e + 12 * a);
    }
    double u[3], sp[2];
    u[0] = rec[3]; u[1] = rec[4]; u[2] = rec[5];
    degenerate += orc_sph(u, sp);
    orc_one_blob(sp[0], 4, e + 36);
    orc_one_blob(sp[1], 4, e + 40);
    u[0] = rec[6]; u[1] = rec[7]; u[2] = rec[8];
    degenerate += orc_sph(u, sp);
    orc_one_blob(sp[0], 4, e + 44);
    orc_one_blob(sp[1], 4, e + 48);
    double r = rec[9];
    if (r < 0.0) r = 0.0;
    orc_one_blob(1.0 - exp(-r), 4, e + 52); /* ob(1 - e^{-r}) */
    for (int c = 0; c < 3; ++c) e[56 + c] = rec[10 + c];
    for (int c = 0; c < 3; ++c) e[59 + c] = rec[13 + c];
    e[62] = 1.0;
    e[63] = 1.0;
    return degenerate;
}

/* ---- exact encodings: the primitives the cheap ones replace
 * (fig:cheap_primitives).  Reading R21: the frequency
 * entry d is sin(pi 2^d v) (NeRF's form, the paper's "12 sine functions, each
 * with frequency 2^d").  Reading R22: the one-blob kernel is the
 * Gaussian of the one-blob encoding [Mueller et al. 2019] with sigma = 1/k,
 * i.e. sigma = 1 in bin units: g(x) = exp(-x^2/2) / sqrt(2 pi), evaluated at
 * the bin centres, no truncation. */
double orc_gauss(double x) { return exp(-0.5 * x * x) / sqrt(2.0 * M_PI); }

void orc_freq_sin(double v, double* out12)
{
    for (int d = 0; d < 12; ++d) out12[d] = sin(M_PI * ldexp(v, d));
}

void orc_one_blob_gauss(double s, int k, double* out)
{
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
    for (int i = 0; i < k; ++i) out[i] = orc_gauss((s - (i + 0.5) / k) * k);
}

/* orc_encode with the exact primitives (same layout, readings R3-R7). */
int orc_encode_exact(const float* rec, const float* aabb_lo, const float* aabb_hi, double* e)
{
    int degenerate = 0;
    for (int a = 0; a < 3; ++a) {
        float v = orc_normalize_pos(rec[a], aabb_lo[a], aabb_hi[a]);
        orc_freq_sin((double)v, e + 12 * a);
    }
    double u[3], sp[2];
    u[0] = rec[3]; u[1] = rec[4]; u[2] = rec[5];
    degenerate += orc_sph(u, sp);
    orc_one_blob_gauss(sp[0], 4, e + 36);
    orc_one_blob_gauss(sp[1], 4, e + 40);
    u[0] = rec[6]; u[1] = rec[7]; u[2] = rec[8];
    degenerate += orc_sph(u, sp);
    orc_one_blob_gauss(sp[0], 4, e + 44);
    orc_one_blob_gauss(sp[1], 4, e + 48);
    double r = rec[9];
    if (r < 0.0) r = 0.0;
    orc_one_blob_gauss(1.0 - exp(-r), 4, e + 52);
    for (int c = 0; c < 3; ++c) e[56 + c] = rec[10 + c];
    for (int c = 0; c < 3; ++c) e[59 + c] = rec[13 + c];
    e[62] = 1.0;
    e[63] = 1.0;
    return degenerate;
}

void orc_encode_batch_exact(const float* recs, int64_t n, const float* lo, const float* hi, double* E)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) orc_encode_exact(recs + 16 * i, lo, hi, E + 64 * i);
}

void orc_encode_batch(const float* recs, int64_t n, const float* lo, const float* hi, double* E)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) orc_encode(recs + 16 * i, lo, hi, E + 64 * i);
}

/* ---- network (fig:fully-fused-illustration (a) P:L545) -------
 * H[0] = e; H[i+1] = ReLU(W_i H[i]), i = 0..4; y = W_5 H[5] (linear output,
 * reading R2).  W in the logical layout (row-major [out][in]). */
void orc_forward(const double* W, const double* e, double* H /* 6*64 */, double* y /* 3 */)
{
    for (int k = 0; k < ORC_IN; ++k) H[k] = e[k];
    for (int i = 0; i < 5; ++i) {
        const double* Wi = W + orc_mat_off[i];
        const double* hin = H + 64 * i;
        double* hout = H + 64 * (i + 1);
        for (int o = 0; o < 64; ++o) {
            double acc = 0.0;
            for (int k = 0; k < 64; ++k) acc += Wi[64 * o + k] * hin[k];
            hout[o] = acc > 0.0 ? acc : 0.0;
        }
    }
    const double* W5 = W + orc_mat_off[5];
    for (int o = 0; o < 3; ++o) {
        double acc = 0.0;
        for (int k = 0; k < 64; ++k) acc += W5[64 * o + k] * H[64 * 5 + k];
        y[o] = acc;
    }
}

/* flags shared in meaning (not in code) with include/nrc.h */
#define ORC_FACTORIZE 1u
#define ORC_CLAMP_QUERY 2u

/* Cache query (P:L874-878 reflectance factorisation; clamp reading R2):
 * q = max(0, y * (alpha + beta)).  W is the set being evaluated (EMA weights
 * for queries, P:L355 -- the caller chooses). */
void orc_query_batch(const double* W, const float* recs, int64_t n, const float* lo, const float* hi,
                     unsigned flags, double* q)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double e[64], H[6 * 64], y[3];
        const float* rec = recs + 16 * i;
        orc_encode(rec, lo, hi, e);
        orc_forward(W, e, H, y);
        for (int c = 0; c < 3; ++c) {
            double v = y[c];
            if (flags & ORC_FACTORIZE) v *= (double)rec[10 + c] + (double)rec[13 + c];
            if ((flags & ORC_CLAMP_QUERY) && v < 0.0) v = 0.0;
            q[3 * i + c] = v;
        }
    }
}

/* ---- width ablation (BASELINE.json configs[3]): the same network
 * with hidden width hw in {32, 64, 128} instead of 64 (the input stays the
 * 64-dim encoding; the depth stays 5 hidden layers).
 * Logical layout: W0 [hw][64], W1..W4 [hw][hw], W5 [3][hw], row-major
 * [out][in]; P(hw) = 64 hw + 4 hw^2 + 3 hw parameters.  Plain definition:
 * H0 = e; H_{i+1} = ReLU(W_i H_i), i = 0..4; y = W5 H5. */
int64_t orc_param_count_w(int hw) { return 64 * (int64_t)hw + 4 * (int64_t)hw * hw + 3 * (int64_t)hw; }

static int64_t orc_mat_off_w(int hw, int i)
{
    if (i == 0) return 0;
    return 64 * (int64_t)hw + (int64_t)(i - 1) * hw * hw;
}

void orc_forward_w(int hw, const double* W, const double* e, double* y)
{
    double h[128], hn[128];
    for (int o = 0; o < hw; ++o) {
        double acc = 0.0;
        for (int k = 0; k < ORC_IN; ++k) acc += W[orc_mat_off_w(hw, 0) + ORC_IN * o + k] * e[k];
        h[o] = acc > 0.0 ? acc : 0.0;
    }
    for (int i = 1; i < 5; ++i) {
        const double* Wi = W + orc_mat_off_w(hw, i);
        for (int o = 0; o < hw; ++o) {
            double acc = 0.0;
            for (int k = 0; k < hw; ++k) acc += Wi[hw * o + k] * h[k];
            hn[o] = acc > 0.0 ? acc : 0.0;
        }
        for (int o = 0; o < hw; ++o) h[o] = hn[o];
    }
    const double* W5 = W + orc_mat_off_w(hw, 5);
    for (int o = 0; o < 3; ++o) {
        double acc = 0.0;
        for (int k = 0; k < hw; ++k) acc += W5[hw * o + k] * h[k];
        y[o] = acc;
    }
}

void orc_query_batch_w(int hw, const double* W, const float* recs, int64_t n, const float* lo, const float* hi,
                       unsigned flags, double* q)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double e[64], y[3];
        const float* rec = recs + 16 * i;
        orc_encode(rec, lo, hi, e);
        orc_forward_w(hw, W, e, y);
        for (int c = 0; c < 3; ++c) {
            double v = y[c];
            if (flags & ORC_FACTORIZE) v *= (double)rec[10 + c] + (double)rec[13 + c];
            if ((flags & ORC_CLAMP_QUERY) && v < 0.0) v = 0.0;
            q[3 * i + c] = v;
        }
    }
}

/* orc_query_batch with the exact encoding (N4). */
void orc_query_batch_exact(const double* W, const float* recs, int64_t n, const float* lo, const float* hi,
                           unsigned flags, double* q)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double e[64], H[6 * 64], y[3];
        const float* rec = recs + 16 * i;
        orc_encode_exact(rec, lo, hi, e);
        orc_forward(W, e, H, y);
        for (int c = 0; c < 3; ++c) {
            double v = y[c];
            if (flags & ORC_FACTORIZE) v *= (double)rec[10 + c] + (double)rec[13 + c];
            if ((flags & ORC_CLAMP_QUERY) && v < 0.0) v = 0.0;
            q[3 * i + c] = v;
        }
    }
}

/* Pixel reconstruction from the cache: the
 * rendering path of pixel pix[i] ends in cache query i; its radiance reaches
 * the pixel through the path throughput T_i:  image[pix[i]] += T_i (.) q_i,
 * q = orc_query_batch.  Sequential in i (the order of the adds is fixed). */
void orc_query_accumulate(const double* W, const float* recs, int64_t n, const float* lo, const float* hi,
                          unsigned flags, const uint32_t* pix, const float* thr, double* image)
{
    double* q = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    orc_query_batch(W, recs, n, lo, hi, flags, q);
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) image[3 * (int64_t)pix[i] + c] += (double)thr[3 * i + c] * q[3 * i + c];
    free(q);
}

/* ---- relative L2 loss, Eq.(5) ---------------------------------
 * l = (1/3) sum_c (yhat_c - t_c)^2 / (sg(lambda)^2 + eps), where lambda is the
 * Rec.709 luminance of the prediction (readings R8, R9, R10).
 * dl/dyhat_c = 2 (yhat_c - t_c) / (3 (lambda^2 + eps)), lambda held constant
 * (stop-gradient sg).  Returns l; writes dl/dyhat if dyhat != NULL. */
double orc_loss(const double* yhat, const double* t, double eps, double* dyhat)
{
    double lam = 0.2126 * yhat[0] + 0.7152 * yhat[1] + 0.0722 * yhat[2];
    double den = lam * lam + eps;
    double l = 0.0;
    for (int c = 0; c < 3; ++c) {
        double r = yhat[c] - t[c];
        l += r * r / den;
        if (dyhat) dyhat[c] = 2.0 * r / (3.0 * den);
    }
    return l / 3.0;
}

/* Same loss with an externally frozen denominator luminance (used by the
 * finite-difference pin, which needs sg(.) held at the base point). */
double orc_loss_frozen(const double* yhat, const double* t, double eps, double lam)
{
    double den = lam * lam + eps;
    double l = 0.0;
    for (int c = 0; c < 3; ++c) {
        double r = yhat[c] - t[c];
        l += r * r / den;
    }
    return l / 3.0;
}

/* ---- backward pass: reverse-mode through the 6 layers --------
 * dy = dl/dy (3).  G += outer products:  G5 += dy h5^T;  delta5 = W5^T dy;
 * for i = 4..0: g = delta_{i+1} * 1[h_{i+1} > 0] (ReLU'(0) = 0, reading R17);
 * G_i += g h_i^T;  delta_i = W_i^T g. */
void orc_backward(const double* W, const double* H, const double* dy, double* G)
{
    double delta[64], g[64];
    const double* W5 = W + orc_mat_off[5];
    double* G5 = G + orc_mat_off[5];
    for (int o = 0; o < 3; ++o)
        for (int k = 0; k < 64; ++k) G5[64 * o + k] += dy[o] * H[64 * 5 + k];
    for (int k = 0; k < 64; ++k) {
        double acc = 0.0;
        for (int o = 0; o < 3; ++o) acc += W5[64 * o + k] * dy[o];
        delta[k] = acc;
    }
    for (int i = 4; i >= 0; --i) {
        const double* Wi = W + orc_mat_off[i];
        double* Gi = G + orc_mat_off[i];
        const double* hout = H + 64 * (i + 1);
        const double* hin = H + 64 * i;
        for (int o = 0; o < 64; ++o) g[o] = hout[o] > 0.0 ? delta[o] : 0.0;
        for (int o = 0; o < 64; ++o)
            for (int k = 0; k < 64; ++k) Gi[64 * o + k] += g[o] * hin[k];
        if (i > 0) {
            for (int k = 0; k < 64; ++k) {
                double acc = 0.0;
                for (int o = 0; o < 64; ++o) acc += Wi[64 * o + k] * g[o];
                delta[k] = acc;
            }
        }
    }
}

/* Per-record loss and gradient over a batch: writes the UN-normalised sums
 * G = sum_records dl/dW (the 1/N of the batch mean is applied by the caller;
 * reading R13) and loss_sum = sum_records l.  The loss sees the factored,
 * unclamped prediction yhat = y * (alpha + beta) (readings R2, R9).  Records
 * with a non-finite target are masked (no loss, no gradient) and counted
 * (S:L262).  Deterministic for any thread count: the batch is cut into a
 * fixed number of contiguous chunks, each summed in index order, and the
 * chunk sums are added in chunk order. */
#define ORC_CHUNKS 64
static void orc_grad_batch_enc(const double* W, const float* recs, const float* tgts, int64_t n, const float* lo,
                               const float* hi, double eps, unsigned flags, double* G, double* loss_sum,
                               int64_t* n_bad_targets, int exact)
{
    double* Gc = (double*)calloc((size_t)ORC_CHUNKS * ORC_NPARAM, sizeof(double));
    double lc[ORC_CHUNKS];
    int64_t bc[ORC_CHUNKS];
#pragma omp parallel for schedule(dynamic, 1)
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        int64_t i0 = n * ch / ORC_CHUNKS, i1 = n * (ch + 1) / ORC_CHUNKS;
        double* Gk = Gc + (size_t)ch * ORC_NPARAM;
        double lsum = 0.0;
        int64_t nbad = 0;
        for (int64_t i = i0; i < i1; ++i) {
            const float* rec = recs + 16 * i;
            const float* tg = tgts + 3 * i;
            if (!(isfinite(tg[0]) && isfinite(tg[1]) && isfinite(tg[2]))) {
                ++nbad;
                continue;
            }
            double e[64], H[6 * 64], y[3], yhat[3], t[3], dyhat[3], dy[3];
            if (exact) orc_encode_exact(rec, lo, hi, e); else orc_encode(rec, lo, hi, e);
            orc_forward(W, e, H, y);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                yhat[c] = y[c] * f;
                t[c] = tg[c];
            }
            lsum += orc_loss(yhat, t, eps, dyhat);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                dy[c] = dyhat[c] * f; /* chain rule through yhat = y * (alpha+beta) */
            }
            orc_backward(W, H, dy, Gk);
        }
        lc[ch] = lsum;
        bc[ch] = nbad;
    }
    memset(G, 0, sizeof(double) * ORC_NPARAM);
    double lsum = 0.0;
    int64_t nbad = 0;
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        const double* Gk = Gc + (size_t)ch * ORC_NPARAM;
        for (int64_t j = 0; j < ORC_NPARAM; ++j) G[j] += Gk[j];
        lsum += lc[ch];
        nbad += bc[ch];
    }
    free(Gc);
    if (loss_sum) *loss_sum = lsum;
    if (n_bad_targets) *n_bad_targets = nbad;
}

void orc_grad_batch(const double* W, const float* recs, const float* tgts, int64_t n, const float* lo,
                    const float* hi, double eps, unsigned flags, double* G, double* loss_sum,
                    int64_t* n_bad_targets)
{
    orc_grad_batch_enc(W, recs, tgts, n, lo, hi, eps, flags, G, loss_sum, n_bad_targets, 0);
}

/* orc_grad_batch with the exact encoding (N4: sin frequency + Gaussian
 * one-blob, orc_encode_exact) -- the training counterpart of
 * orc_query_batch_exact. */
void orc_grad_batch_exact(const double* W, const float* recs, const float* tgts, int64_t n, const float* lo,
                          const float* hi, double eps, unsigned flags, double* G, double* loss_sum,
                          int64_t* n_bad_targets)
{
    orc_grad_batch_enc(W, recs, tgts, n, lo, hi, eps, flags, G, loss_sum, n_bad_targets, 1);
}

/* ---- Adam (reading R11: lr, beta1, beta2, eps outside sqrt,
 * standard bias correction, t starting at 1).  Non-finite gradient entries
 * are zeroed and counted. Returns the count. */
int64_t orc_adam(double* w, double* m, double* v, const double* g_in, int64_t P, int64_t t, double lr,
                 double b1, double b2, double eps)
{
    int64_t bad = 0;
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t j = 0; j < P; ++j) {
        double g = g_in[j];
        if (!isfinite(g)) {
            g = 0.0;
            ++bad;
        }
        m[j] = b1 * m[j] + (1.0 - b1) * g;
        v[j] = b2 * v[j] + (1.0 - b2) * g * g;
        double mhat = m[j] / bc1;
        double vhat = v[j] / bc2;
        w[j] -= lr * mhat / (sqrt(vhat) + eps);
    }
    return bad;
}

/* ---- EMA of the weights, Eq.(2) --------------------------------
 * eta_t = 1 - a^t.  Reading R12 (constant-preserving form):
 *   Wbar_t = [(1-a) W_t + a eta_{t-1} Wbar_{t-1}] / eta_t.
 * printed_form != 0 evaluates Eq.(2) exactly as printed:
 *   Wbar_t = (1-a)/eta_t W_t + a eta_{t-1} Wbar_{t-1}. */
void orc_ema(double* wbar, const double* w, int64_t P, int64_t t, double a, int printed_form)
{
    double eta_t = 1.0 - pow(a, (double)t);
    double eta_p = 1.0 - pow(a, (double)(t - 1));
    for (int64_t j = 0; j < P; ++j) {
        if (printed_form)
            wbar[j] = (1.0 - a) / eta_t * w[j] + a * eta_p * wbar[j];
        else
            wbar[j] = ((1.0 - a) * w[j] + a * eta_p * wbar[j]) / eta_t;
    }
}

/* ---- LCG shuffle into s batches of l records ------------------
 * Reading R15.  splitmix64 stream of the shuffle seed gives (a, c);
 * m = 2^ceil(log2 n); f(i) = (a i + c) mod m; perm(i) = f iterated until < n. */
static uint64_t orc_splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void orc_lcg_params(uint64_t n, uint64_t seed, uint64_t* a, uint64_t* c, uint64_t* m)
{
    uint64_t mm = 1;
    while (mm < n) mm <<= 1;
    uint64_t x0 = orc_splitmix64(seed);
    uint64_t x1 = orc_splitmix64(seed + 0x9E3779B97F4A7C15ull);
    uint64_t aa = ((x0 & (mm - 1)) & ~(uint64_t)3) | 1;
    if (mm >= 8 && aa == 1) aa = 5;
    *a = aa;
    *c = (x1 & (mm - 1)) | 1;
    *m = mm;
}

uint64_t orc_lcg_perm(uint64_t i, uint64_t n, uint64_t a, uint64_t c, uint64_t m)
{
    uint64_t x = i;
    do {
        x = (a * x + c) & (m - 1);
    } while (x >= n);
    return x;
}

void orc_lcg_permute(uint64_t n, uint64_t a, uint64_t c, uint64_t m, uint64_t* out)
{
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_lcg_perm(i, n, a, c, m);
}

/* ---- self-training targets.
 * A training path has vertices v_0 .. v_{m-1} (camera side first).  Per vertex:
 * emitted radiance E_i, next-event estimate N_i and the path throughput T_i
 * (BSDF * cos / pdf) from v_i towards v_{i+1}, each RGB, stored as 9 floats
 * [E N T].  The path's tail radiance L_tail is the cache's prediction at the
 * terminal vertex (self-training) or 0 for the unbiased fraction
 * u = 1/16 of paths terminated by Russian roulette only (flag bit
 * 0).  The target of each vertex is the radiance transported back to it:
 *   target(v_{m-1}) = E + N + T (.) L_tail
 *   target(v_i)     = E_i + N_i + T_i (.) target(v_{i+1}),   i = m-2 .. 0. */
void orc_assemble_targets(const uint32_t* first, const uint32_t* len, const uint32_t* flags, int64_t n_paths,
                          const float* vert, const float* tail, double* targets)
{
    for (int64_t p = 0; p < n_paths; ++p) {
        double acc[3];
        for (int c = 0; c < 3; ++c) acc[c] = (flags[p] & 1u) ? 0.0 : (double)tail[3 * p + c];
        for (int64_t k = (int64_t)len[p] - 1; k >= 0; --k) {
            const int64_t v = (int64_t)first[p] + k;
            const float* x = vert + 9 * v;
            for (int c = 0; c < 3; ++c) {
                acc[c] = (double)x[c] + (double)x[3 + c] + (double)x[6 + c] * acc[c];
                targets[3 * v + c] = acc[c];
            }
        }
    }
}

/* ---- initialisation (reading R16): Glorot-uniform from a
 * counter-based splitmix64 stream: u = (splitmix64(seed ^ (i<<32 | r*in+c))
 * >> 11) * 2^-53;  w = fp32((2u - 1) sqrt(6 / (fan_in + fan_out))). */
void orc_init_weights(uint64_t seed, float* W32)
{
    for (int i = 0; i < ORC_NMAT; ++i) {
        int rows = orc_mat_rows[i];
        double bound = sqrt(6.0 / (64.0 + (double)rows));
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < 64; ++c) {
                uint64_t ctr = ((uint64_t)i << 32) | (uint64_t)(r * 64 + c);
                double u = (double)(orc_splitmix64(seed ^ ctr) >> 11) * (1.0 / 9007199254740992.0);
                W32[orc_mat_off[i] + 64 * r + c] = (float)((2.0 * u - 1.0) * bound);
            }
    }
}

/* Reading R16 at hidden width hw: the same Glorot-uniform counter stream,
 * fan_in = 64 (W0) or hw, fan_out = hw (W0..W4) or 3 (W5); counter
 * (i << 32 | r * fan_in + c).  At hw = 64 this is orc_init_weights. */
void orc_init_weights_w(int hw, uint64_t seed, float* W32)
{
    for (int i = 0; i < ORC_NMAT; ++i) {
        int rows = i < 5 ? hw : 3, cols = i == 0 ? ORC_IN : hw;
        double bound = sqrt(6.0 / ((double)cols + (double)rows));
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                uint64_t ctr = ((uint64_t)i << 32) | (uint64_t)(r * cols + c);
                double u = (double)(orc_splitmix64(seed ^ ctr) >> 11) * (1.0 / 9007199254740992.0);
                W32[orc_mat_off_w(hw, i) + (int64_t)cols * r + c] = (float)((2.0 * u - 1.0) * bound);
            }
    }
}

/* ---- one optimisation step: gradient of the batch mean
 * loss, Adam, EMA.  w, m, v, wbar are fp64 arrays of ORC_NPARAM.  Returns the
 * batch-mean loss. */
double orc_train_step(double* w, double* m, double* v, double* wbar, int64_t t, const float* recs,
                      const float* tgts, int64_t n, const float* lo, const float* hi, double loss_eps,
                      unsigned flags, double lr, double b1, double b2, double adam_eps, double ema_a,
                      int ema_printed, double* G_out, int64_t* bad_grads, int64_t* bad_targets)
{
    double G[ORC_NPARAM];
    double lsum = 0.0;
    if (n <= 0) return 0.0; /* empty batch: no-op */
    orc_grad_batch(w, recs, tgts, n, lo, hi, loss_eps, flags, G, &lsum, bad_targets);
    for (int64_t j = 0; j < ORC_NPARAM; ++j) G[j] /= (double)n; /* batch mean (R10, R13) */
    if (G_out) memcpy(G_out, G, sizeof(G));
    int64_t bad = orc_adam(w, m, v, G, ORC_NPARAM, t, lr, b1, b2, adam_eps);
    if (bad_grads) *bad_grads = bad;
    orc_ema(wbar, w, ORC_NPARAM, t, ema_a, ema_printed);
    return lsum / (double)n;
}

/* ---- width ablation, training (BASELINE.json configs[3]: "32/64/128-neuron
 * hidden layers at 1080p query+train").  The same definitions as
 * orc_forward / orc_backward / orc_grad_batch / orc_train_step (P:L662-667,
 * Eq.(5), Eq.(2)) with hidden width hw: logical layout
 * of orc_forward_w, P(hw) = orc_param_count_w(hw) parameters.
 * H holds h_0 (64 values, the encoding) then h_1..h_5 (hw values each). */
void orc_forward_stash_w(int hw, const double* W, const double* e, double* H, double* y)
{
    for (int k = 0; k < ORC_IN; ++k) H[k] = e[k];
    for (int i = 0; i < 5; ++i) {
        const int in = i == 0 ? ORC_IN : hw;
        const double* Wi = W + orc_mat_off_w(hw, i);
        const double* hin = i == 0 ? H : H + ORC_IN + (int64_t)(i - 1) * hw;
        double* hout = H + ORC_IN + (int64_t)i * hw;
        for (int o = 0; o < hw; ++o) {
            double acc = 0.0;
            for (int k = 0; k < in; ++k) acc += Wi[(int64_t)in * o + k] * hin[k];
            hout[o] = acc > 0.0 ? acc : 0.0;
        }
    }
    const double* W5 = W + orc_mat_off_w(hw, 5);
    const double* h5 = H + ORC_IN + 4 * (int64_t)hw;
    for (int o = 0; o < 3; ++o) {
        double acc = 0.0;
        for (int k = 0; k < hw; ++k) acc += W5[(int64_t)hw * o + k] * h5[k];
        y[o] = acc;
    }
}

/* Reverse mode at width hw (cf. orc_backward): G5 += dy h5^T; delta5 = W5^T dy;
 * for i = 4..0: g = delta_{i+1} * 1[h_{i+1} > 0] (R17); G_i += g h_i^T;
 * delta_i = W_i^T g (i > 0). */
void orc_backward_w(int hw, const double* W, const double* H, const double* dy, double* G)
{
    double delta[128], g[128];
    const double* W5 = W + orc_mat_off_w(hw, 5);
    double* G5 = G + orc_mat_off_w(hw, 5);
    const double* h5 = H + ORC_IN + 4 * (int64_t)hw;
    for (int o = 0; o < 3; ++o)
        for (int k = 0; k < hw; ++k) G5[(int64_t)hw * o + k] += dy[o] * h5[k];
    for (int k = 0; k < hw; ++k) {
        double acc = 0.0;
        for (int o = 0; o < 3; ++o) acc += W5[(int64_t)hw * o + k] * dy[o];
        delta[k] = acc;
    }
    for (int i = 4; i >= 0; --i) {
        const int in = i == 0 ? ORC_IN : hw;
        const double* Wi = W + orc_mat_off_w(hw, i);
        double* Gi = G + orc_mat_off_w(hw, i);
        const double* hout = H + ORC_IN + (int64_t)i * hw;
        const double* hin = i == 0 ? H : H + ORC_IN + (int64_t)(i - 1) * hw;
        for (int o = 0; o < hw; ++o) g[o] = hout[o] > 0.0 ? delta[o] : 0.0;
        for (int o = 0; o < hw; ++o)
            for (int k = 0; k < in; ++k) Gi[(int64_t)in * o + k] += g[o] * hin[k];
        if (i > 0) {
            for (int k = 0; k < in; ++k) {
                double acc = 0.0;
                for (int o = 0; o < hw; ++o) acc += Wi[(int64_t)in * o + k] * g[o];
                delta[k] = acc;
            }
        }
    }
}

/* orc_grad_batch at width hw: un-normalised gradient sum, loss sum, masked
 * non-finite targets; the same fixed chunking (deterministic). */
void orc_grad_batch_w(int hw, const double* W, const float* recs, const float* tgts, int64_t n, const float* lo,
                      const float* hi, double eps, unsigned flags, double* G, double* loss_sum,
                      int64_t* n_bad_targets)
{
    const int64_t P = orc_param_count_w(hw);
    double* Gc = (double*)calloc((size_t)ORC_CHUNKS * (size_t)P, sizeof(double));
    double lc[ORC_CHUNKS];
    int64_t bc[ORC_CHUNKS];
#pragma omp parallel for schedule(dynamic, 1)
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        int64_t i0 = n * ch / ORC_CHUNKS, i1 = n * (ch + 1) / ORC_CHUNKS;
        double* Gk = Gc + (size_t)ch * (size_t)P;
        double lsum = 0.0;
        int64_t nbad = 0;
        for (int64_t i = i0; i < i1; ++i) {
            const float* rec = recs + 16 * i;
            const float* tg = tgts + 3 * i;
            if (!(isfinite(tg[0]) && isfinite(tg[1]) && isfinite(tg[2]))) {
                ++nbad;
                continue;
            }
            double e[64], H[64 + 5 * 128], y[3], yhat[3], t[3], dyhat[3], dy[3];
            orc_encode(rec, lo, hi, e);
            orc_forward_stash_w(hw, W, e, H, y);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                yhat[c] = y[c] * f;
                t[c] = tg[c];
            }
            lsum += orc_loss(yhat, t, eps, dyhat);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                dy[c] = dyhat[c] * f;
            }
            orc_backward_w(hw, W, H, dy, Gk);
        }
        lc[ch] = lsum;
        bc[ch] = nbad;
    }
    memset(G, 0, sizeof(double) * (size_t)P);
    double lsum = 0.0;
    int64_t nbad = 0;
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        const double* Gk = Gc + (size_t)ch * (size_t)P;
        for (int64_t j = 0; j < P; ++j) G[j] += Gk[j];
        lsum += lc[ch];
        nbad += bc[ch];
    }
    free(Gc);
    if (loss_sum) *loss_sum = lsum;
    if (n_bad_targets) *n_bad_targets = nbad;
}

/* orc_train_step at width hw (w, m, v, wbar: fp64 arrays of P(hw)). */
double orc_train_step_w(int hw, double* w, double* m, double* v, double* wbar, int64_t t, const float* recs,
                        const float* tgts, int64_t n, const float* lo, const float* hi, double loss_eps,
                        unsigned flags, double lr, double b1, double b2, double adam_eps, double ema_a,
                        int ema_printed, double* G_out, int64_t* bad_grads, int64_t* bad_targets)
{
    const int64_t P = orc_param_count_w(hw);
    double lsum = 0.0;
    if (n <= 0) return 0.0;
    double* G = (double*)malloc(sizeof(double) * (size_t)P);
    orc_grad_batch_w(hw, w, recs, tgts, n, lo, hi, loss_eps, flags, G, &lsum, bad_targets);
    for (int64_t j = 0; j < P; ++j) G[j] /= (double)n;
    if (G_out) memcpy(G_out, G, sizeof(double) * (size_t)P);
    int64_t bad = orc_adam(w, m, v, G, P, t, lr, b1, b2, adam_eps);
    if (bad_grads) *bad_grads = bad;
    orc_ema(wbar, w, P, t, ema_a, ema_printed);
    free(G);
    return lsum / (double)n;
}

/* ---- depth variants ("depth other than 5"): the network of
 * orc_forward_w with nh hidden layers instead of five (P:L694 fixes five; the
 * variant keeps the 64-dim input, hidden width hw, ReLU, linear 3-output
 * layer).  Logical layout: W0 [hw][64], W1..W_{nh-1} [hw][hw], W_nh [3][hw]
 * (the output layer), row-major [out][in]; P = 64 hw + (nh-1) hw^2 + 3 hw.
 * H holds h_0 (64 values) then h_1..h_nh (hw each). */
int64_t orc_param_count_d(int hw, int nh) { return 64 * (int64_t)hw + (int64_t)(nh - 1) * hw * hw + 3 * (int64_t)hw; }

static int64_t orc_mat_off_d(int hw, int nh, int i)
{
    (void)nh;
    if (i == 0) return 0;
    return 64 * (int64_t)hw + (int64_t)(i - 1) * hw * hw; /* i = nh: the output layer */
}

void orc_forward_stash_d(int hw, int nh, const double* W, const double* e, double* H, double* y)
{
    for (int k = 0; k < ORC_IN; ++k) H[k] = e[k];
    for (int i = 0; i < nh; ++i) {
        const int in = i == 0 ? ORC_IN : hw;
        const double* Wi = W + orc_mat_off_d(hw, nh, i);
        const double* hin = i == 0 ? H : H + ORC_IN + (int64_t)(i - 1) * hw;
        double* hout = H + ORC_IN + (int64_t)i * hw;
        for (int o = 0; o < hw; ++o) {
            double acc = 0.0;
            for (int k = 0; k < in; ++k) acc += Wi[(int64_t)in * o + k] * hin[k];
            hout[o] = acc > 0.0 ? acc : 0.0;
        }
    }
    const double* Wo = W + orc_mat_off_d(hw, nh, nh);
    const double* hl = H + ORC_IN + (int64_t)(nh - 1) * hw;
    for (int o = 0; o < 3; ++o) {
        double acc = 0.0;
        for (int k = 0; k < hw; ++k) acc += Wo[(int64_t)hw * o + k] * hl[k];
        y[o] = acc;
    }
}

/* Reverse mode (cf. orc_backward_w): G_nh += dy h_nh^T; delta = W_nh^T dy;
 * for i = nh-1..0: g = delta * 1[h_{i+1} > 0] (R17); G_i += g h_i^T;
 * delta = W_i^T g (i > 0). */
void orc_backward_d(int hw, int nh, const double* W, const double* H, const double* dy, double* G)
{
    double delta[128], g[128];
    const double* Wo = W + orc_mat_off_d(hw, nh, nh);
    double* Go = G + orc_mat_off_d(hw, nh, nh);
    const double* hl = H + ORC_IN + (int64_t)(nh - 1) * hw;
    for (int o = 0; o < 3; ++o)
        for (int k = 0; k < hw; ++k) Go[(int64_t)hw * o + k] += dy[o] * hl[k];
    for (int k = 0; k < hw; ++k) {
        double acc = 0.0;
        for (int o = 0; o < 3; ++o) acc += Wo[(int64_t)hw * o + k] * dy[o];
        delta[k] = acc;
    }
    for (int i = nh - 1; i >= 0; --i) {
        const int in = i == 0 ? ORC_IN : hw;
        const double* Wi = W + orc_mat_off_d(hw, nh, i);
        double* Gi = G + orc_mat_off_d(hw, nh, i);
        const double* hout = H + ORC_IN + (int64_t)i * hw;
        const double* hin = i == 0 ? H : H + ORC_IN + (int64_t)(i - 1) * hw;
        for (int o = 0; o < hw; ++o) g[o] = hout[o] > 0.0 ? delta[o] : 0.0;
        for (int o = 0; o < hw; ++o)
            for (int k = 0; k < in; ++k) Gi[(int64_t)in * o + k] += g[o] * hin[k];
        if (i > 0) {
            for (int k = 0; k < in; ++k) {
                double acc = 0.0;
                for (int o = 0; o < hw; ++o) acc += Wi[(int64_t)in * o + k] * g[o];
                delta[k] = acc;
            }
        }
    }
}

void orc_query_batch_d(int hw, int nh, const double* W, const float* recs, int64_t n, const float* lo,
                       const float* hi, unsigned flags, double* q)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double e[64], H[64 + 16 * 128], y[3];
        const float* rec = recs + 16 * i;
        orc_encode(rec, lo, hi, e);
        orc_forward_stash_d(hw, nh, W, e, H, y);
        for (int c = 0; c < 3; ++c) {
            double v = y[c];
            if (flags & ORC_FACTORIZE) v *= (double)rec[10 + c] + (double)rec[13 + c];
            if ((flags & ORC_CLAMP_QUERY) && v < 0.0) v = 0.0;
            q[3 * i + c] = v;
        }
    }
}

/* orc_grad_batch at width hw and depth nh (same fixed chunking). */
void orc_grad_batch_d(int hw, int nh, const double* W, const float* recs, const float* tgts, int64_t n,
                      const float* lo, const float* hi, double eps, unsigned flags, double* G, double* loss_sum,
                      int64_t* n_bad_targets)
{
    const int64_t P = orc_param_count_d(hw, nh);
    double* Gc = (double*)calloc((size_t)ORC_CHUNKS * (size_t)P, sizeof(double));
    double lc[ORC_CHUNKS];
    int64_t bc[ORC_CHUNKS];
#pragma omp parallel for schedule(dynamic, 1)
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        int64_t i0 = n * ch / ORC_CHUNKS, i1 = n * (ch + 1) / ORC_CHUNKS;
        double* Gk = Gc + (size_t)ch * (size_t)P;
        double lsum = 0.0;
        int64_t nbad = 0;
        for (int64_t i = i0; i < i1; ++i) {
            const float* rec = recs + 16 * i;
            const float* tg = tgts + 3 * i;
            if (!(isfinite(tg[0]) && isfinite(tg[1]) && isfinite(tg[2]))) {
                ++nbad;
                continue;
            }
            double e[64], H[64 + 16 * 128], y[3], yhat[3], t[3], dyhat[3], dy[3];
            orc_encode(rec, lo, hi, e);
            orc_forward_stash_d(hw, nh, W, e, H, y);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                yhat[c] = y[c] * f;
                t[c] = tg[c];
            }
            lsum += orc_loss(yhat, t, eps, dyhat);
            for (int c = 0; c < 3; ++c) {
                double f = (flags & ORC_FACTORIZE) ? (double)rec[10 + c] + (double)rec[13 + c] : 1.0;
                dy[c] = dyhat[c] * f;
            }
            orc_backward_d(hw, nh, W, H, dy, Gk);
        }
        lc[ch] = lsum;
        bc[ch] = nbad;
    }
    memset(G, 0, sizeof(double) * (size_t)P);
    double lsum = 0.0;
    int64_t nbad = 0;
    for (int ch = 0; ch < ORC_CHUNKS; ++ch) {
        const double* Gk = Gc + (size_t)ch * (size_t)P;
        for (int64_t j = 0; j < P; ++j) G[j] += Gk[j];
        lsum += lc[ch];
        nbad += bc[ch];
    }
    free(Gc);
    if (loss_sum) *loss_sum = lsum;
    if (n_bad_targets) *n_bad_targets = nbad;
}

/* Reading R16 at width hw and depth nh: counter (i << 32 | r fan_in + c),
 * layer index i = 0..nh (the output layer is i = nh; at nh = 5 this is
 * orc_init_weights_w). */
void orc_init_weights_d(int hw, int nh, uint64_t seed, float* W32)
{
    for (int i = 0; i <= nh; ++i) {
        int rows = i < nh ? hw : 3, cols = i == 0 ? ORC_IN : hw;
        double bound = sqrt(6.0 / ((double)cols + (double)rows));
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                uint64_t ctr = ((uint64_t)i << 32) | (uint64_t)(r * cols + c);
                double u = (double)(orc_splitmix64(seed ^ ctr) >> 11) * (1.0 / 9007199254740992.0);
                W32[orc_mat_off_d(hw, nh, i) + (int64_t)cols * r + c] = (float)((2.0 * u - 1.0) * bound);
            }
    }
}

/* orc_train_step at width hw and depth nh. */
double orc_train_step_d(int hw, int nh, double* w, double* m, double* v, double* wbar, int64_t t, const float* recs,
                        const float* tgts, int64_t n, const float* lo, const float* hi, double loss_eps,
                        unsigned flags, double lr, double b1, double b2, double adam_eps, double ema_a,
                        int ema_printed, double* G_out, int64_t* bad_grads, int64_t* bad_targets)
{
    const int64_t P = orc_param_count_d(hw, nh);
    double lsum = 0.0;
    if (n <= 0) return 0.0;
    double* G = (double*)malloc(sizeof(double) * (size_t)P);
    orc_grad_batch_d(hw, nh, w, recs, tgts, n, lo, hi, loss_eps, flags, G, &lsum, bad_targets);
    for (int64_t j = 0; j < P; ++j) G[j] /= (double)n;
    if (G_out) memcpy(G_out, G, sizeof(double) * (size_t)P);
    int64_t bad = orc_adam(w, m, v, G, P, t, lr, b1, b2, adam_eps);
    if (bad_grads) *bad_grads = bad;
    orc_ema(wbar, w, P, t, ema_a, ema_printed);
    free(G);
    return lsum / (double)n;
}
