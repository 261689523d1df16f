// check_glibc_log.c -- compare rsim_log.h's restated glibc_log() with the C library's log()
// on the inputs expovariate feeds it (1 - k * 2^-53, k uniform 53-bit) plus random normal
// doubles in (2^-20, 2^20). Build: gcc -O2 -ffp-contract=off -o check check_glibc_log.c -lm
// Usage: check N [seed]   -> prints "mismatches M of N" (exit 1 if M > 0)
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include "../paper_2603_15202_b200/csrc/rsim_log.h"

static const double TAB[256] = RSIM_LOG_TAB_INIT;

int main(int argc, char **argv) {
    long n = argc > 1 ? atol(argv[1]) : 1000000;
    uint64_t s = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
    long bad = 0;
    for (long i = 0; i < n; i++) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        double x;
        if (i & 1) x = 1.0 - (double)(s >> 11) * 0x1p-53;
        else x = ldexp(1.0 + (double)(s >> 12) * 0x1p-52, (int)((s >> 3) % 41) - 20);
        volatile double a = log(x);
        double b = glibc_log(x, TAB);
        if (memcmp((const void *)&a, &b, 8) != 0) {
            if (bad < 5) printf("x=%a libm=%a restated=%a\n", x, (double)a, b);
            bad++;
        }
    }
    printf("mismatches %ld of %ld\n", bad, n);
    return bad != 0;
}
