/*
 * ORACLE — test infrastructure only. Nothing in the product path links this.
 *
 * Plain-C restatement of the sketch-hash stream used by the reference's
 * build_sparse_embedding (/root/reference/pkg/src/skipm/sketching.py:93-119):
 *   rng = Generator(Philox(seed))                          sketching.py:104
 *   cols = rng.integers(0, w, size=(n, s))                 sketching.py:109
 *   duplicate rows redrawn in ascending row order           sketching.py:110-115
 *   signs = rng.integers(0, 2, size=(n, s)) * 2.0 - 1.0    sketching.py:116
 * and of the ADW summation order of apply_sketch (sketching.py:154,160).
 *
 * The arithmetic lives in numpy 2.3.5 (third-party, not under /root/reference):
 *   - Philox4x64-10 (Random123 round function, numpy/random/src/philox),
 *     counter incremented before each 4-word block, key from SeedSequence
 *     (computed by the caller on the host);
 *   - next_uint32: low half of a 64-bit output, then its buffered high half;
 *   - bounded integers below 2^32: Lemire's multiply-shift with rejection
 *     threshold (2^32 - w) mod w (numpy random_bounded_uint64_fill ->
 *     buffered_bounded_lemire_uint32).
 * Pinned against numpy / the live reference by tests/golden (make_golden.py).
 *
 * Word addressing: 32-bit word q of the stream is half (q & 1) of 64-bit
 * output k = q >> 1, which is lane (k & 3) of Philox block ctr = (k >> 2) + 1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static inline uint64_t mulhi64(uint64_t a, uint64_t b) {
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
}

void oracle_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
        uint64_t h0 = mulhi64(0xD2E7470EE14C6C93ULL, c0), l0 = 0xD2E7470EE14C6C93ULL * c0;
        uint64_t h1 = mulhi64(0xCA5A826395121157ULL, c2), l1 = 0xCA5A826395121157ULL * c2;
        uint64_t n0 = h1 ^ c1 ^ k0, n1 = l1, n2 = h0 ^ c3 ^ k1, n3 = l0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 64-bit output number k (0-based) of a fresh Philox(key). */
uint64_t oracle_out64(uint64_t k0, uint64_t k1, uint64_t k) {
    uint64_t ctr[4] = {(k >> 2) + 1, 0, 0, 0}, key[2] = {k0, k1}, o[4];
    oracle_philox4x64_10(ctr, key, o);
    return o[k & 3];
}

static inline uint32_t word32(uint64_t k0, uint64_t k1, uint64_t q) {
    uint64_t v = oracle_out64(k0, k1, q >> 1);
    return (q & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
}

/* Draw cnt bounded integers in [0, w) starting at stream word *pos (advanced). */
void oracle_lemire_draw(uint64_t k0, uint64_t k1, uint64_t *pos, uint32_t w,
                        int64_t cnt, int64_t *out) {
    uint32_t thr = (uint32_t)((0x100000000ULL - w) % w);
    uint64_t q = *pos;
    for (int64_t i = 0; i < cnt; ++i) {
        uint64_t m;
        for (;;) {
            m = (uint64_t)word32(k0, k1, q++) * (uint64_t)w;
            if ((uint32_t)m >= thr) break;
        }
        out[i] = (int64_t)(m >> 32);
    }
    *pos = q;
}

static int row_has_dup(const int64_t *row, int s) {
    for (int a = 0; a < s; ++a)
        for (int b = a + 1; b < s; ++b)
            if (row[a] == row[b]) return 1;
    return 0;
}

/*
 * Full sparse embedding for the 2s < w branch. cols: n*s int64 row-major,
 * vals: n*s doubles. Returns the number of stream words consumed.
 */
uint64_t oracle_sparse_embedding(uint64_t k0, uint64_t k1, int64_t n, int32_t w, int32_t s,
                                 int64_t *cols, double *vals) {
    uint64_t pos = 0;
    oracle_lemire_draw(k0, k1, &pos, (uint32_t)w, n * s, cols);
    int64_t *dup = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * s > 0 ? n * s : 1));
    for (;;) {
        int64_t nd = 0;
        for (int64_t j = 0; j < n; ++j)
            if (row_has_dup(cols + j * s, s)) dup[nd++] = j;
        if (!nd) break;
        oracle_lemire_draw(k0, k1, &pos, (uint32_t)w, nd * s, tmp);
        for (int64_t r = 0; r < nd; ++r)
            memcpy(cols + dup[r] * s, tmp + r * s, sizeof(int64_t) * (size_t)s);
    }
    double rs = sqrt((double)s);
    for (int64_t i = 0; i < n * s; ++i) {
        uint32_t wd = word32(k0, k1, pos++);
        double sign = (double)(wd >> 31) * 2.0 - 1.0;
        vals[i] = sign / rs;
    }
    free(dup);
    free(tmp);
    return pos;
}

/*
 * ADW[i, b] for dense row-major A (m x n), scaling d (n), embedding cols/vals
 * (n x s). Sum over (j, k) with cols[j,k] == b in ascending j then k of
 * fl(fl(A_ij * d_j) * val_jk), separate multiply and add (scipy csr_matmat
 * order after A.multiply(d).tocsr(), sketching.py:154,160). out: m x w row-major.
 * volatile keeps gcc from contracting into FMA.
 */
void oracle_adw_dense(const double *A, int64_t m, int64_t n, const double *d,
                      const int64_t *cols, const double *vals, int32_t s, int32_t w,
                      double *out) {
    memset(out, 0, sizeof(double) * (size_t)(m * w));
    for (int64_t i = 0; i < m; ++i) {
        double *row = out + i * w;
        for (int64_t j = 0; j < n; ++j) {
            volatile double ad = A[i * n + j] * d[j];
            for (int k = 0; k < s; ++k) {
                volatile double t = ad * vals[j * s + k];
                row[cols[j * s + k]] = row[cols[j * s + k]] + t;
            }
        }
    }
}
