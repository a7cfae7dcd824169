/* Plain-C use of the C ABI (include/rtm.h), no Python: BASELINE.json configs[0] (C1: 64^3,
 * dx = 10 m, dt = 1 ms, v = 2000 m/s, 100 steps, a Ricker 15 Hz source at the centre).
 *
 *   cc -O2 -I include examples/rtm_c1.c -L paper_1310_8232_b200 -lrtm_b200 \
 *      -Wl,-rpath,$PWD/paper_1310_8232_b200 -lm -o rtm_c1 && ./rtm_c1
 *
 * Prints max|u| and a checksum of u^100; every error path prints rtm_last_error(). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "rtm.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_ != RTM_OK) {                                                         \
            fprintf(stderr, "%s -> %d: %s\n", #call, rc_, rtm_last_error());         \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void) {
    const int n = 64, steps = 100;
    const float dx = 10.0f, dt = 1e-3f, v0 = 2000.0f, f0 = 15.0f;
    /* c0..c5: the 10th-order central 2nd-derivative weights (BASELINE.json configs[0]) */
    const float coeffs[6] = {-5269.0f / 1800.0f, 5.0f / 3.0f, -5.0f / 21.0f, 5.0f / 126.0f,
                             -5.0f / 1008.0f, 1.0f / 3150.0f};
    rtm_ctx* ctx = rtm_create(n, n, n, dx, dt, coeffs);
    if (!ctx) {
        fprintf(stderr, "rtm_create: %s\n", rtm_last_error());
        return 1;
    }
    const size_t pts = (size_t)n * n * n;
    float* v = (float*)malloc(pts * sizeof(float));
    float* u = (float*)malloc(pts * sizeof(float));
    float w[100];
    for (size_t i = 0; i < pts; ++i) v[i] = v0;
    for (int k = 0; k < steps; ++k) { /* w[k] = (v dt)^2 ricker(k dt), t0 = 1/f0 (DESIGN R4, R5) */
        const double a = pow(M_PI * f0 * (k * (double)dt - 1.0 / f0), 2.0);
        w[k] = (float)(pow((double)v0 * dt, 2.0) * (1.0 - 2.0 * a) * exp(-a));
    }
    CHECK(rtm_set_velocity(ctx, v));
    CHECK(rtm_inject_source(ctx, n / 2, n / 2, n / 2, w, steps));
    CHECK(rtm_step(ctx, steps));
    CHECK(rtm_read_field(ctx, u));
    double m = 0.0, sum = 0.0;
    for (size_t i = 0; i < pts; ++i) {
        m = fmax(m, fabs((double)u[i]));
        sum += u[i];
    }
    printf("C1 after %d steps: max|u| = %.6e, sum(u) = %.6e, %.3f ms per rtm_step\n", steps, m, sum,
           (double)rtm_last_elapsed_ms(ctx));
    rtm_destroy(ctx);
    free(v);
    free(u);
    return 0;
}
