/* A plain C caller of the staging session (include/ddm_b200.h): stage a stack
 * once, run the whole map and a cutoff / lag subset from it, check the C-ABI error contract.
 * Compiled as C (not C++) by tests/test_cpp_api.py: the boundary carries no C++ types. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ddm_b200.h"

#define W 64
#define H 64
#define N 700

static int fail(const char* what) {
    printf("FAIL %s: %s\n", what, ddm_b200_last_error());
    return 1;
}

int main(void) {
    const int64_t plane = (int64_t)H * (W / 2 + 1);
    uint16_t* px = malloc(sizeof(uint16_t) * W * H * N);
    for (int64_t i = 0; i < (int64_t)W * H * N; ++i) px[i] = (uint16_t)((i * 2654435761u) >> 20);
    double* full = malloc(sizeof(double) * plane * N);
    double* sub = malloc(sizeof(double) * plane * 3);
    ddm_b200* s = NULL;
    if (ddm_b200_create(W, H, N, 0, 0, &s) != DDM_B200_OK) return fail("create");
    /* two pieces, second first */
    if (ddm_b200_stage_frames(s, px + (int64_t)W * H * 400, 400, N - 400) != DDM_B200_OK) return fail("stage b");
    /* not every frame staged yet: an input error */
    if (ddm_b200_run_with_ft(s, NULL, 0, NULL, 0, full, plane * N, NULL, NULL) != DDM_B200_E_INPUT)
        return fail("unstaged run");
    if (ddm_b200_stage_frames(s, px, 0, 400) != DDM_B200_OK) return fail("stage a");
    ddm_b200_counters c;
    ddm_b200_timing t;
    if (ddm_b200_run_with_ft(s, NULL, 0, NULL, 0, full, plane * N, &c, &t) != DDM_B200_OK) return fail("run");
    if (c.spatial_ffts != N || c.temporal_ffts != 2u * (uint64_t)plane) { printf("FAIL counters\n"); return 1; }
    for (int64_t q = 0; q < plane; ++q)
        if (full[q] != 0.0) { printf("FAIL d(0)\n"); return 1; }
    /* wave vectors 5, 40, 100 and lags {3, 1, 650}: equal to the whole-map entries */
    const int64_t wv[3] = {5, 40, 100};
    const int64_t lags[3] = {3, 1, 650};
    if (ddm_b200_run_with_ft(s, wv, 3, lags, 3, sub, plane * 3, NULL, NULL) != DDM_B200_OK) return fail("subset");
    const int64_t sorted[3] = {1, 3, 650};
    for (int li = 0; li < 3; ++li)
        for (int64_t q = 0; q < plane; ++q) {
            const double want = (q == 5 || q == 40 || q == 100) ? full[sorted[li] * plane + q] : 0.0;
            if (sub[li * plane + q] != want) { printf("FAIL subset value\n"); return 1; }
        }
    /* errors: status codes and a message, nothing thrown across the boundary */
    if (ddm_b200_run_with_ft(s, wv, 3, lags, 3, sub, 10, NULL, NULL) != DDM_B200_E_INPUT) return fail("capacity");
    if (ddm_b200_last_error()[0] == '\0') { printf("FAIL empty message\n"); return 1; }
    if (ddm_b200_stage_frames(NULL, px, 0, 1) != DDM_B200_E_INPUT) return fail("null session");
    if (ddm_b200_destroy(s) != DDM_B200_OK) return fail("destroy");
    printf("OK session C caller: %lld wave vectors x %d lags, step1 %.3f ms step2 %.3f ms\n",
           (long long)plane, N, t.step1 * 1e3, t.step2 * 1e3);
    free(px);
    free(full);
    free(sub);
    return 0;
}
