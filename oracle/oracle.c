/*
 * oracle.c -- fp64 CPU oracle for DreamZero block-causal chunk attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2602_15922_b200/), and neither side includes or links the other.
 *
 * What it computes is the plain definition, written out in fp64 on inputs
 * that the caller has already rounded to the bf16 values the GPU sees
 * (reading A18).  No blocking, no fusion, no online softmax.
 *
 *   1. per-head RMSNorm   x^_i = x_i / sqrt(mean_j x_j^2 + eps) * g_{h,i}
 *        BASELINE.json north_star (BJ:5) "per-head RMSNorm on Q/K"; readings
 *        A1 (per head, over D), A2 (eps inside the root), A3 (gain [H, D]).
 *   2. 3D RoPE over (t, h, w)  BJ:5 "3D (frame, height, width) RoPE", split
 *        (d_t, d_h, d_w) from BJ:7/BJ:8.  Readings A4 (norm, then RoPE),
 *        A5 (theta 1e4), A6 (interleaved pairs (2i, 2i+1) inside each axis
 *        slice, slices in order t|h|w), A7 (omega_i = theta^(-2i/d_a)).
 *   3. visibility (Fig. 10; Alg. 2 l.558-607):
 *        a NOISY query of chunk k sees CLEAN keys of chunk < k and every key
 *        of its own span; a CLEAN query of chunk j sees CLEAN keys of chunk
 *        <= j.  Nothing else.
 *   4. attention  O_s = sum_j softmax_j(<q^_s, k^_j> * scale) v_j over the
 *        visible j, scale = 1/sqrt(D) (BJ:7 "softmax scale 1/sqrt(64)").
 *   5. tile classifier: SKIP / PARTIAL / FULL per (q-tile, kv-tile) of a
 *        given (BM, BN) (BJ:5 "bit-exactly on mask and tile-skip decisions").
 *
 * Pins (tests/test_oracle_pins.py) tie every function to something other
 * than itself: closed forms, invariants, a pure-Python fsum brute force,
 * mpmath at 50 digits, torch float64 SDPA, and the Fig. 10 worked example.
 *
 * Layouts: row-major, token-major.  x[n][H][D]; pos[n][3] int32 (t, h, w);
 * tags: chunk[n], kind[n] (0 CLEAN, 1 NOISY), span[n] int32.
 * Return value: 0 on success, -1 on invalid arguments.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_CLEAN 0
#define ORACLE_NOISY 1

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Step 1: per-head RMSNorm (BJ:5; readings A1-A3). out may alias x. */
int oracle_rmsnorm(const double *x, const double *gain, int64_t n, int32_t H, int32_t D,
                   double eps, double *out) {
    if (!x || !gain || !out || n < 0 || H <= 0 || D <= 0) return -1;
    for (int64_t t = 0; t < n; ++t) {
        for (int32_t h = 0; h < H; ++h) {
            const double *row = x + (t * H + h) * D;
            double *dst = out + (t * H + h) * D;
            double ss = 0.0;
            for (int32_t i = 0; i < D; ++i) ss += row[i] * row[i];
            double inv = 1.0 / sqrt(ss / (double)D + eps);
            for (int32_t i = 0; i < D; ++i) dst[i] = row[i] * inv * gain[h * D + i];
        }
    }
    return 0;
}

/* Step 2: 3D RoPE (BJ:5, BJ:7-8; readings A5-A7).  In place on x[n][H][D].
 * For axis a in (t, h, w) with slice offset o_a and width d_a, pair i < d_a/2:
 *   omega = theta^(-2i/d_a), phi = p_a * omega,
 *   (u, w) = (x[o_a+2i], x[o_a+2i+1]) -> (u cos phi - w sin phi, u sin phi + w cos phi). */
int oracle_rope3d(double *x, const int32_t *pos, int64_t n, int32_t H, int32_t D,
                  const int32_t *rope_dims, double theta) {
    if (!x || !pos || !rope_dims || n < 0 || H <= 0 || D <= 0) return -1;
    int32_t sum = 0;
    for (int a = 0; a < 3; ++a) {
        if (rope_dims[a] < 0 || rope_dims[a] % 2) return -1;
        sum += rope_dims[a];
    }
    if (sum != D) return -1;
    for (int64_t t = 0; t < n; ++t) {
        int32_t off = 0;
        for (int a = 0; a < 3; ++a) {
            const int32_t da = rope_dims[a];
            const double p = (double)pos[t * 3 + a];
            for (int32_t i = 0; i < da / 2; ++i) {
                const double omega = pow(theta, -2.0 * (double)i / (double)da);
                const double phi = p * omega;
                const double c = cos(phi), s = sin(phi);
                for (int32_t h = 0; h < H; ++h) {
                    double *row = x + (t * H + h) * D + off;
                    const double u = row[2 * i], w = row[2 * i + 1];
                    row[2 * i] = u * c - w * s;
                    row[2 * i + 1] = u * s + w * c;
                }
            }
            off += da;
        }
    }
    return 0;
}

/* Steps 1+2 on one tensor: out = RoPE(RMSNorm(x)) (reading A4: norm first). */
int oracle_prologue(const double *x, const double *gain, const int32_t *pos, int64_t n,
                    int32_t H, int32_t D, const int32_t *rope_dims, double theta, double eps,
                    double *out) {
    int rc = oracle_rmsnorm(x, gain, n, H, D, eps, out);
    if (rc) return rc;
    return oracle_rope3d(out, pos, n, H, D, rope_dims, theta);
}

/* Step 3: the Fig. 10 rule (S:208 rules (b)-(e)). */
int oracle_visible(int32_t q_chunk, int32_t q_kind, int32_t q_span,
                   int32_t k_chunk, int32_t k_kind, int32_t k_span) {
    if (q_span == k_span) return 1;                       /* own span, bidirectional */
    if (k_kind != ORACLE_CLEAN) return 0;                 /* never another noisy span */
    if (q_kind == ORACLE_NOISY) return k_chunk < q_chunk; /* noisy k sees clean < k   */
    return k_chunk <= q_chunk;                            /* clean j sees clean <= j  */
}

/* Step 4: masked softmax attention for one batch element.
 * q[nq][H][D], k[nk][H][D], v[nk][H][D] are the post-prologue values (k, v as
 * stored in the cache).  out[nq][H][D]; lse[nq][H] = log sum_j exp(score_j)
 * (natural log, -inf for an empty visible set, reading A15; then O = 0). */
int oracle_attention(const double *q, const double *k, const double *v, int64_t nq, int64_t nk,
                     int32_t H, int32_t D, double scale,
                     const int32_t *q_chunk, const int32_t *q_kind, const int32_t *q_span,
                     const int32_t *k_chunk, const int32_t *k_kind, const int32_t *k_span,
                     double *out, double *lse) {
    if (!q || !k || !v || !out || nq < 0 || nk < 0 || H <= 0 || D <= 0) return -1;
    if (!q_chunk || !q_kind || !q_span || !k_chunk || !k_kind || !k_span) return -1;
    const int64_t total = nq * (int64_t)H;
    int err = 0;
#pragma omp parallel
    {
        double *score = (double *)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
        if (!score) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t idx = 0; idx < total; ++idx) {
            if (!score) continue;
            const int64_t s = idx / H;
            const int32_t h = (int32_t)(idx % H);
            const double *qs = q + (s * H + h) * D;
            double *os = out + (s * H + h) * D;
            double m = -INFINITY;
            for (int64_t j = 0; j < nk; ++j) {
                if (!oracle_visible(q_chunk[s], q_kind[s], q_span[s], k_chunk[j], k_kind[j], k_span[j])) {
                    score[j] = -INFINITY;
                    continue;
                }
                const double *kj = k + (j * H + h) * D;
                double dot = 0.0;
                for (int32_t i = 0; i < D; ++i) dot += qs[i] * kj[i];
                score[j] = dot * scale;
                if (score[j] > m) m = score[j];
            }
            for (int32_t i = 0; i < D; ++i) os[i] = 0.0;
            if (m == -INFINITY) {
                if (lse) lse[s * H + h] = -INFINITY;
                continue;
            }
            double denom = 0.0;
            for (int64_t j = 0; j < nk; ++j) {
                if (score[j] == -INFINITY) continue;
                const double p = exp(score[j] - m);
                denom += p;
                const double *vj = v + (j * H + h) * D;
                for (int32_t i = 0; i < D; ++i) os[i] += p * vj[i];
            }
            for (int32_t i = 0; i < D; ++i) os[i] /= denom;
            if (lse) lse[s * H + h] = m + log(denom);
        }
        free(score);
    }
    return err ? -1 : 0;
}

/* Step 5: tile classifier.  map[qt * n_kt + kt] = 0 SKIP (no visible pair),
 * 2 FULL (all BM x BN pairs in bounds and visible), 1 PARTIAL otherwise.
 * Out-of-bounds rows/columns count as not visible. */
int oracle_tile_map(int64_t nq, int64_t nk, int32_t BM, int32_t BN,
                    const int32_t *q_chunk, const int32_t *q_kind, const int32_t *q_span,
                    const int32_t *k_chunk, const int32_t *k_kind, const int32_t *k_span,
                    uint8_t *map) {
    if (BM <= 0 || BN <= 0 || nq < 0 || nk < 0 || !map) return -1;
    const int64_t n_qt = (nq + BM - 1) / BM, n_kt = (nk + BN - 1) / BN;
    for (int64_t qt = 0; qt < n_qt; ++qt) {
        for (int64_t kt = 0; kt < n_kt; ++kt) {
            int64_t vis = 0;
            for (int64_t s = qt * BM; s < (qt + 1) * BM; ++s) {
                for (int64_t j = kt * BN; j < (kt + 1) * BN; ++j) {
                    if (s >= nq || j >= nk) continue;
                    vis += oracle_visible(q_chunk[s], q_kind[s], q_span[s], k_chunk[j], k_kind[j], k_span[j]);
                }
            }
            map[qt * n_kt + kt] = vis == 0 ? 0 : (vis == (int64_t)BM * BN ? 2 : 1);
        }
    }
    return 0;
}
