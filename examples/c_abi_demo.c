/* Plain-C consumer of the C ABI: decomposes the reference's known-answer matrix
 * [[1,2],[3,4]] (proj/tests/test_decompose.cpp:69-77) through the host-buffer entry points.
 * Build: gcc -std=c11 -Iinclude examples/c_abi_demo.c -Lpaper_2401_16378_b200 -lpd_b200 \
 *        -Wl,-rpath,$PWD/paper_2401_16378_b200 -o c_abi_demo */
#include <stdio.h>

#include "pd_api.h"

int main(void) {
    pd_ctx* ctx = NULL;
    int rc = pd_ctx_create(0, &ctx);
    if (rc != PD_OK) {
        fprintf(stderr, "pd_ctx_create: %d %s\n", rc, pd_last_error());
        return 2;
    }
    const double g[8] = {1, 0, 2, 0, 3, 0, 4, 0};
    double c[8];
    rc = pd_decompose(ctx, 1, g, c, PD_PATH_GRAY);
    if (rc != PD_OK) {
        fprintf(stderr, "pd_decompose: %s\n", pd_last_error());
        return 1;
    }
    printf("%g%+gi %g%+gi %g%+gi %g%+gi\n", c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
    /* contract violation: n >= 4^N is std::invalid_argument in the reference */
    double one[2];
    rc = pd_coeff(ctx, 1, g, 4, 0, one);
    printf("out-of-range n -> %d (%s)\n", rc, pd_last_error());
    /* batched single strings: Y and Z of the same matrix */
    const uint64_t ns[2] = {2, 3};
    double two[4];
    int rc2 = pd_coeff_batch(ctx, 1, g, ns, 2, two);
    printf("batch: %g%+gi %g%+gi (rc=%d)\n", two[0], two[1], two[2], two[3], rc2);
    printf("launches=%llu\n", (unsigned long long)pd_launch_count());
    pd_ctx_destroy(ctx);
    return (c[0] == 2.5 && c[2] == 2.5 && c[5] == -0.5 && c[6] == -1.5 && rc == PD_EINVAL && rc2 == PD_OK &&
            two[1] == -0.5 && two[2] == -1.5) ? 0 : 1;
}
