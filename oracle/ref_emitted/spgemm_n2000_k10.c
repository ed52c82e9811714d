/* generated kernel source; compile with: cc -O3 -ffp-contract=off */
#include <math.h>

/* level 0, 191004 instance(s), 1 result(s) each */
static void k0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 47751; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[0 + i]];
            const double x1 = x[p[191004 + i]];
            x[40000 + i] = x0*x1;
        }
    }
}

/* level 0, 4396 instance(s), 1 result(s) each */
static void k1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1099; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[382008 + i]];
            const double x1 = x[p[386404 + i]];
            const double x2 = x[p[390800 + i]];
            const double x3 = x[p[395196 + i]];
            x[231004 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 68 instance(s), 1 result(s) each */
static void k2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 17; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[399592 + i]];
            const double x1 = x[p[399660 + i]];
            const double x2 = x[p[399728 + i]];
            const double x3 = x[p[399796 + i]];
            const double x4 = x[p[399864 + i]];
            const double x5 = x[p[399932 + i]];
            x[235400 + i] = x0*x1 + x2*x3 + x4*x5;
        }
    }
}

void sg_run(double* x, const double* c, const unsigned* p) {
    k0(x, c, p);
    k1(x, c, p);
    k2(x, c, p);
}
