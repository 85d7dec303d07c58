/* A plain C caller of the drop-in boundary (include/mltune_b200.h): no
 * Python, no torch. Builds a small space and a deterministic ensemble, asks
 * the library for the top-m (mlt_top_m, the C entry point under
 * tuner.top_m_predicted, tuner.py:95-131) and prints the result as JSON for
 * tests/test_c_abi.py to compare with the oracle; the same on a slice
 * through the resident-plan API.
 *
 *   gcc -std=c99 -I include tests/c/abi_topm.c -L paper_1506_00842_b200 \
 *       -lmltune_b200 -Wl,-rpath,<dir> -lm -o abi_topm && ./abi_topm        */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

#include "mltune_b200.h"

#define P 4
#define K 3
#define H 30
#define M 12

static int check(int rc, const char* what) {
  if (rc != MLT_OK) {
    fprintf(stderr, "%s failed: %d (%s)\n", what, rc, mlt_last_error());
    exit(1);
  }
  return rc;
}

int main(void) {
  /* space: 16 x 64 x 8 x 128 = 1,048,576 configurations, one max-product rule */
  const int32_t radix[P] = {16, 64, 8, 128};
  int64_t values[16 + 64 + 8 + 128];
  int at = 0;
  for (int p = 0; p < P; ++p)
    for (int v = 0; v < radix[p]; ++v) values[at++] = (int64_t)(v + 1) * (p + 1);
  const int32_t kind[1] = {MLT_RULE_MAX_PRODUCT}, nops[1] = {2}, pos[2] = {0, 2};
  const int64_t coeff[2] = {1, 1}, bound[1] = {200};
  mlt_space sp = {P, radix, values, 1, kind, nops, pos, coeff, bound};

  /* ensemble: deterministic weights */
  static double w1[K * H * P], b1[K * H], w2[K * H];
  double b2[K], mean[K], sd[K];
  for (int i = 0; i < K * H * P; ++i) w1[i] = 1.5 * sin(0.37 * i + 0.1);
  for (int i = 0; i < K * H; ++i) {
    b1[i] = 0.8 * cos(0.53 * i);
    w2[i] = 0.6 * sin(1.7 * i + 0.3);
  }
  for (int m = 0; m < K; ++m) {
    b2[m] = 0.1 * m - 0.05;
    mean[m] = -3.0 + 0.2 * m;
    sd[m] = 0.5 + 0.1 * m;
  }
  mlt_ensemble en = {K, P, H, radix, w1, b1, w2, b2, mean, sd};

  if (mlt_abi_version() != MLT_ABI_VERSION) {
    fprintf(stderr, "ABI version mismatch\n");
    return 1;
  }
  mlt_ctx* ctx = NULL;
  check(mlt_ctx_create(0, &ctx), "mlt_ctx_create");

  int64_t card = 1;
  for (int p = 0; p < P; ++p) card *= radix[p];
  int64_t idx[M], n = 0;
  double pred[M];
  mlt_sweep_stats st;
  check(mlt_top_m(ctx, &sp, &en, M, 0, card, NULL, 0, idx, pred, &n, &st), "mlt_top_m");

  /* the same through a resident plan, on a slice */
  mlt_plan* plan = NULL;
  check(mlt_plan_create(ctx, &sp, &en, &plan), "mlt_plan_create");
  int64_t sidx[M], sn = 0;
  double spred[M];
  check(mlt_plan_top_m(plan, M, card / 4, card / 2, sidx, spred, &sn, NULL), "mlt_plan_top_m");
  check(mlt_plan_destroy(plan), "mlt_plan_destroy");

  printf("{\"card\": %lld, \"path\": %d, \"n\": %lld, \"idx\": [", (long long)card, st.path, (long long)n);
  for (int64_t t = 0; t < n; ++t) printf("%s%lld", t ? ", " : "", (long long)idx[t]);
  printf("], \"pred\": [");
  for (int64_t t = 0; t < n; ++t) printf("%s%.17g", t ? ", " : "", pred[t]);
  printf("], \"slice_idx\": [");
  for (int64_t t = 0; t < sn; ++t) printf("%s%lld", t ? ", " : "", (long long)sidx[t]);
  printf("]}\n");
  check(mlt_ctx_destroy(ctx), "mlt_ctx_destroy");
  return 0;
}
