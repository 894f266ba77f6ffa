/* Host twin of potr::exp_neg (paper_2601_14821_b200/csrc/common.cuh): the same
 * sequence of IEEE operations (fma() == DFMA), used by tests/test_exp.py to
 * bound its error against long-double expl over the rasterizer's domain.
 * TEST INFRASTRUCTURE ONLY. */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../paper_2601_14821_b200/csrc/exp_table.h"

static const double POTR_EXP_TABLE[64][2] = POTR_EXP_TABLE_INIT;

static double exp_neg(double x) {
    double t = fma(x, POTR_EXP_INV_STEP, POTR_EXP_SHIFT);
    double k = t - POTR_EXP_SHIFT;
    uint64_t tb;
    memcpy(&tb, &t, 8);
    int32_t ki = (int32_t)(uint32_t)tb;
    double r = fma(k, -POTR_EXP_STEP_HI, x);
    r = fma(k, -POTR_EXP_STEP_LO, r);
    double r2 = r * r;
    double a = fma(r, POTR_EXP_C3, POTR_EXP_C2);
    double b = fma(r, POTR_EXP_C5, POTR_EXP_C4);
    double q = fma(r2, b, a);
    double p = fma(r2, q, r);
    int j = ki & 63, m = ki >> 6;
    double res = fma(POTR_EXP_TABLE[j][0], p, POTR_EXP_TABLE[j][1]) + POTR_EXP_TABLE[j][0];
    uint64_t rb;
    memcpy(&rb, &res, 8);
    rb += (uint64_t)((int64_t)m << 52);
    memcpy(&res, &rb, 8);
    return res;
}

/* max |error| in ulps over n points evenly spread on [lo, hi]; also the count
 * of results that differ from glibc exp(). */
double exp_twin_max_ulp(double lo, double hi, int64_t n, int64_t *n_diff_glibc) {
    double worst = 0.0;
    int64_t nd = 0;
    for (int64_t i = 0; i < n; i++) {
        double x = lo + (hi - lo) * ((double)i / (double)(n - 1));
        double got = exp_neg(x);
        long double ref = expl((long double)x);
        double ulp = nextafter(got, INFINITY) - got;
        double err = (double)fabsl(((long double)got - ref) / (long double)ulp);
        if (err > worst) worst = err;
        if (got != exp(x)) nd++;
    }
    *n_diff_glibc = nd;
    return worst;
}

double exp_twin(double x) { return exp_neg(x); }
