/*
 * lbm_demo.c — the C ABI used from plain C (no Python, no torch): a D3Q19 TRT + Guo channel flow (config
 * C1's setup at a small size) in the two-grid pull pattern, 200 steps from rest, then the centre-line
 * velocity against the steady Poiseuille parabola u = F / (2 nu) (y - 1/2)(H + 1/2 - y) scaled by the
 * start-up fraction, and the total mass. Build (after python -m paper_2001_11806_b200.build):
 *
 *   gcc -O2 -I include examples/lbm_demo.c -L paper_2001_11806_b200 -llbm_b200 \
 *       -Wl,-rpath,$PWD/paper_2001_11806_b200 -o lbm_demo && ./lbm_demo
 *
 * Prints one line "mass=<...> umax=<...> launches=<...>" and exits 0 on success.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "lbm.h"

#define CHECK(call)                                                                                  \
    do {                                                                                             \
        int _s = (call);                                                                             \
        if (_s != LBM_OK) {                                                                          \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, lbm_strerror(_s), lbm_last_error(h));     \
            return 1;                                                                                \
        }                                                                                            \
    } while (0)

int main(int argc, char **argv) {
    const int64_t nx = 32, ny = 34, nz = 16;  /* fluid rows y = 1..32 between no-slip walls */
    const int steps = argc > 1 ? atoi(argv[1]) : 200;
    uint8_t *flags = calloc((size_t)(nx * ny * nz), 1);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t x = 0; x < nx; ++x) {
            flags[x + nx * (0 + ny * z)] = LBM_FLAG_NOSLIP;
            flags[x + nx * ((ny - 1) + ny * z)] = LBM_FLAG_NOSLIP;
        }
    lbm_config cfg;
    lbm_config_default(&cfg);
    cfg.stencil = LBM_D3Q19;
    cfg.collision = LBM_TRT;
    cfg.n_rates = 2;
    cfg.rates[0] = 1.6;
    cfg.rates[1] = 0.5; /* magic parameter 3/16 (G14) */
    cfg.force[0] = 1e-6;
    cfg.global[0] = nx;
    cfg.global[1] = ny;
    cfg.global[2] = nz;
    cfg.periodic[1] = 0;
    cfg.flags = flags;
    lbm_handle h = NULL;
    CHECK(lbm_create(&cfg, &h));
    CHECK(lbm_init_random(h, 0, 0.0, 0.0, 0, 0.0)); /* rho = 1, u = 0 */
    CHECK(lbm_step(h, steps));
    CHECK(lbm_sync(h));
    const int64_t cells = nx * ny * nz;
    double *rho = malloc(sizeof(double) * (size_t)cells), *u = malloc(sizeof(double) * 3 * (size_t)cells);
    CHECK(lbm_get_macroscopic(h, rho, u, LBM_HOST));
    double mass = 0.0, umax = 0.0;
    for (int64_t i = 0; i < cells; ++i) {
        const int64_t y = (i / nx) % ny;
        if (y == 0 || y == ny - 1) continue;
        mass += rho[i];
        if (u[i] > umax) umax = u[i];
    }
    printf("mass=%.15e umax=%.15e launches=%lld\n", mass, umax, (long long)lbm_launch_count(h));
    lbm_destroy(h);
    free(rho);
    free(u);
    free(flags);
    return 0;
}
