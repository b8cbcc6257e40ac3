/*
 * TEST INFRASTRUCTURE ONLY — CPU checker for the B200 engine; never linked
 * into the product library.
 *
 * Sequential restatement of the reference's stack-based pool-adjacent-
 * violators sweep for the top-k weighted Huber isotonic problem,
 * /root/reference/pkg/src/l0cert/prox.py:46-98 (`_pava_topk_huber`):
 *
 *   minimise  sum_j (v_j - xs_j)^2 / 2 + rho * H_M(v_j) * [j < k]
 *   s.t.      v non-increasing,   xs sorted non-increasing.
 *
 * Each element enters as a singleton pool with value hprox(x, w, M)
 * (prox.py:70-73); a newer pool merges into the older one while its value is
 * STRICTLY larger (prox.py:80); a merged pool with weight sum P, magnitude
 * sum S and count N takes the value hprox(S/N, P/N, M) (prox.py:86-91).
 * Arithmetic is plain IEEE double in the same operation order as the
 * reference (compile with -ffp-contract=off so no FMA contraction happens),
 * so the values are bit-identical to the numba kernel.
 *
 * l0o_pava additionally reports every pool boundary (the `last` stack of the
 * reference) so tests can compare PAVA pool boundaries with the GPU kernel.
 */
#include <stdint.h>
#include <stdlib.h>

static double hprox_scalar(double x, double w, double M) {
    /* prox.py:42 — x/(1+w) inside the quadratic zone, x - w*M outside */
    if (x <= M * (1.0 + w)) return x / (1.0 + w);
    return x - w * M;
}

/*
 * xs[p]   sorted magnitudes (non-increasing)
 * out[p]  pooled values
 * ends    optional (may be NULL): inclusive end index of every pool, length p
 * returns the number of pools (or -1 on allocation failure)
 */
int64_t l0o_pava(const double* xs, int64_t p, int64_t k, double rho, double M,
                 double* out, int64_t* ends) {
    if (p <= 0) return 0;
    double* wsum = (double*)malloc(sizeof(double) * (size_t)p);
    double* msum = (double*)malloc(sizeof(double) * (size_t)p);
    double* cnt = (double*)malloc(sizeof(double) * (size_t)p);
    double* val = (double*)malloc(sizeof(double) * (size_t)p);
    int64_t* last = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    if (!wsum || !msum || !cnt || !val || !last) {
        free(wsum); free(msum); free(cnt); free(val); free(last);
        return -1;
    }
    int64_t top = -1; /* index of the newest pool on the stack */
    for (int64_t j = 0; j < p; ++j) {
        double w = (j < k) ? rho : 0.0;
        double x = xs[j];
        ++top;
        wsum[top] = w;
        msum[top] = x;
        cnt[top] = 1.0;
        val[top] = hprox_scalar(x, w, M);
        last[top] = j;
        while (top > 0 && val[top] > val[top - 1]) {
            /* fold the newer pool into the older one, older-first sums */
            wsum[top - 1] += wsum[top];
            msum[top - 1] += msum[top];
            cnt[top - 1] += cnt[top];
            last[top - 1] = last[top];
            --top;
            double mean = msum[top] / cnt[top];
            double wavg = wsum[top] / cnt[top];
            val[top] = hprox_scalar(mean, wavg, M);
        }
    }
    int64_t start = 0;
    for (int64_t b = 0; b <= top; ++b) {
        for (int64_t j = start; j <= last[b]; ++j) out[j] = val[b];
        if (ends) ends[b] = last[b];
        start = last[b] + 1;
    }
    free(wsum); free(msum); free(cnt); free(val); free(last);
    return top + 1;
}
