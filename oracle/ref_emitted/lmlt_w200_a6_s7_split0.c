/* generated kernel source; compile with: cc -O3 -ffp-contract=off */
#include <math.h>

/* level 3, 40000 instance(s), 4 result(s) each */
static void face_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[0 + i]];
            const double x1 = x[p[0 + i] + 1];
            const double x2 = x[p[0 + i] + 2];
            const double x3 = x[p[0 + i] + 3];
            const double x4 = x[p[0 + i] + 4];
            const double x5 = x[p[0 + i] + 5];
            const double x6 = x[p[0 + i] + 603];
            const double x7 = x[p[0 + i] + 604];
            const double x8 = x[p[0 + i] + 605];
            x[360000 + i] = (-(x3 - x0)*(x0 - x6) + -(x4 - x1)*(x1 - x7) + -(x5 - x2)*(x2 - x8))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[400000 + i] = (-(x6 - x3)*(x3 - x0) + -(x7 - x4)*(x4 - x1) + -(x8 - x5)*(x5 - x2))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[440000 + i] = (-(x0 - x6)*(x6 - x3) + -(x1 - x7)*(x7 - x4) + -(x2 - x8)*(x8 - x5))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[480000 + i] = sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)))*0.16666666666666666;
        }
    }
}

/* level 3, 40000 instance(s), 4 result(s) each */
static void face_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[40000 + i]];
            const double x1 = x[p[40000 + i] + 1];
            const double x2 = x[p[40000 + i] + 2];
            const double x3 = x[p[40000 + i] + 603];
            const double x4 = x[p[40000 + i] + 604];
            const double x5 = x[p[40000 + i] + 605];
            const double x6 = x[p[40000 + i] + 600];
            const double x7 = x[p[40000 + i] + 601];
            const double x8 = x[p[40000 + i] + 602];
            x[520408 + i] = (-(x3 - x0)*(x0 - x6) + -(x4 - x1)*(x1 - x7) + -(x5 - x2)*(x2 - x8))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[560408 + i] = (-(x6 - x3)*(x3 - x0) + -(x7 - x4)*(x4 - x1) + -(x8 - x5)*(x5 - x2))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[600408 + i] = (-(x0 - x6)*(x6 - x3) + -(x1 - x7)*(x7 - x4) + -(x2 - x8)*(x8 - x5))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[640408 + i] = sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)))*0.16666666666666666;
        }
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void ldiag2_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[80000 + i]];
        const double x1 = x[p[80002 + i]];
        x[680816 + i] = x0 + x1;
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void ldiag4_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[80004 + i]];
        const double x1 = x[p[80004 + i] + 40000];
        const double x2 = x[p[80004 + i] + 160408];
        const double x3 = x[p[80006 + i]];
        x[680820 + i] = x0 + x1 + x2 + x3;
    }
}

/* level 2, 792 instance(s), 1 result(s) each */
static void ldiag6_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 198; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[80008 + i]];
            const double x1 = x[p[80800 + i]];
            const double x2 = x[p[81592 + i]];
            const double x3 = x[p[82384 + i]];
            const double x4 = x[p[83176 + i]];
            const double x5 = x[p[83968 + i]];
            x[680824 + i] = x0 + x1 + x2 + x3 + x4 + x5;
        }
    }
}

/* level 2, 40000 instance(s), 1 result(s) each */
static void ldiag12_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[84760 + i]];
            const double x1 = x[p[84760 + i] + 40000];
            const double x2 = x[p[84760 + i] + 160408];
            const double x3 = x[p[84760 + i] + 240408];
            const double x4 = x[p[84760 + i] + 160409];
            const double x5 = x[p[84760 + i] + 200409];
            const double x6 = x[p[84760 + i] + 200];
            const double x7 = x[p[84760 + i] + 80200];
            const double x8 = x[p[84760 + i] + 40201];
            const double x9 = x[p[84760 + i] + 80201];
            const double x10 = x[p[84760 + i] + 200609];
            const double x11 = x[p[84760 + i] + 240609];
            x[681616 + i] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + x8 + x9 + x10 + x11;
        }
    }
}

/* level 2, 796 instance(s), 1 result(s) each */
static void loff1_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 199; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[124760 + i]];
            x[722024 + i] = -x0;
        }
    }
}

/* level 2, 40000 instance(s), 1 result(s) each */
static void loff2_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[125556 + i]];
            const double x1 = x[p[125556 + i] + 200409];
            x[722820 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 40000 instance(s), 1 result(s) each */
static void loff2_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[165556 + i]];
            const double x1 = x[p[165556 + i] + 200408];
            x[763228 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 40000 instance(s), 1 result(s) each */
static void loff2_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[205556 + i]];
            const double x1 = x[p[205556 + i] - 80208];
            x[803636 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void mdiag2_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[245556 + i]];
        const double x1 = x[p[245556 + i] + 160408];
        x[844044 + i] = x0 + x1;
    }
}

/* level 2, 792 instance(s), 1 result(s) each */
static void mdiag3_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 198; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[245558 + i]];
            const double x1 = x[p[246350 + i]];
            const double x2 = x[p[247142 + i]];
            x[844048 + i] = x0 + x1 + x2;
        }
    }
}

/* level 2, 40000 instance(s), 1 result(s) each */
static void mdiag6_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[247934 + i]];
            const double x1 = x[p[247934 + i] + 160408];
            const double x2 = x[p[247934 + i] + 160409];
            const double x3 = x[p[247934 + i] + 200];
            const double x4 = x[p[247934 + i] + 201];
            const double x5 = x[p[247934 + i] + 160609];
            x[844840 + i] = x0 + x1 + x2 + x3 + x4 + x5;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[287934 + i]];
            const double x1 = x[p[287934 + i] + 41205];
            x[885248 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[327934 + i]];
            const double x1 = x[p[327934 + i] + 122220];
            x[925656 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[367934 + i]];
            const double x1 = x[p[367934 + i] + 41204];
            x[966064 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[407934 + i]];
            const double x1 = x[p[407934 + i] + 81612];
            x[1006472 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[447934 + i]];
            const double x1 = x[p[447934 + i] + 163224];
            x[1046880 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[487934 + i]];
            const double x1 = x[p[487934 + i] + 122020];
            x[1087288 + i] = x0*x1;
        }
    }
}

/* level 1, 40000 instance(s), 1 result(s) each */
static void lm_s6(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[527934 + i]];
            const double x1 = x[p[527934 + i] + 81813];
            x[1127696 + i] = x0*x1;
        }
    }
}

/* level 1, 3974 instance(s), 1 result(s) each */
static void lm_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 993; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[567934 + i]];
            const double x1 = x[p[571908 + i]];
            x[1168104 + i] = x0*x1;
        }
    }
    for (long i = 3972; i < 3974; ++i) {
        const double x0 = x[p[567934 + i]];
        const double x1 = x[p[571908 + i]];
        x[1168104 + i] = x0*x1;
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[575882 + i]];
            const double x1 = x[p[575882 + i] - 202636];
            x[1172080 + i] = x0*x1;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[615882 + i]];
            const double x1 = x[p[615882 + i] - 364868];
            x[1212080 + i] = x0*x1;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[655882 + i]];
            const double x1 = x[p[655882 + i] - 364267];
            x[1252080 + i] = x0*x1;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[695882 + i]];
            const double x1 = x[p[695882 + i] - 81611];
            x[1292080 + i] = x0*x1;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[735882 + i]];
            const double x1 = x[p[735882 + i] - 243646];
            x[1332080 + i] = x0*x1;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out1_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[775882 + i]];
            const double x1 = x[p[775882 + i] - 162430];
            x[1372080 + i] = x0*x1;
        }
    }
}

/* level 0, 1584 instance(s), 1 result(s) each */
static void out1_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 396; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[815882 + i]];
            const double x1 = x[p[817466 + i]];
            x[1412080 + i] = x0*x1;
        }
    }
}

/* level 0, 32 instance(s), 1 result(s) each */
static void out1a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 8; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[819050 + i]];
            const double x1 = x[p[819082 + i]];
            const double x2 = x[p[819114 + i]];
            x[1413664 + i] = x0*x1 + x2;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[819146 + i]];
            const double x1 = x[p[819146 + i] - 283852];
            const double x2 = x[p[819146 + i] - 202040];
            const double x3 = x[p[819146 + i] - 364667];
            x[1413696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[859146 + i]];
            const double x1 = x[p[859146 + i] - 284053];
            const double x2 = x[p[859146 + i] + 80816];
            const double x3 = x[p[859146 + i] - 243645];
            x[1453696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[899146 + i]];
            const double x1 = x[p[899146 + i] - 203038];
            const double x2 = x[p[899146 + i] - 40408];
            const double x3 = x[p[899146 + i] - 243446];
            x[1493696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[939146 + i]];
            const double x1 = x[p[939146 + i] - 162228];
            const double x2 = x[p[939146 + i] + 202040];
            const double x3 = x[p[939146 + i] - 202635];
            x[1533696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[979146 + i]];
            const double x1 = x[p[979146 + i] - 122019];
            const double x2 = x[p[979146 + i] + 242448];
            const double x3 = x[p[979146 + i] - 81411];
            x[1573696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out2_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1019146 + i]];
            const double x1 = x[p[1019146 + i] - 243245];
            const double x2 = x[p[1019146 + i] - 40408];
            const double x3 = x[p[1019146 + i] - 162229];
            x[1613696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 3168 instance(s), 1 result(s) each */
static void out2_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 792; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1059146 + i]];
            const double x1 = x[p[1062314 + i]];
            const double x2 = x[p[1065482 + i]];
            const double x3 = x[p[1068650 + i]];
            x[1653696 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 38 instance(s), 1 result(s) each */
static void out2a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 9; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1071818 + i]];
            const double x1 = x[p[1071856 + i]];
            const double x2 = x[p[1071894 + i]];
            const double x3 = x[p[1071932 + i]];
            const double x4 = x[p[1071970 + i]];
            x[1656864 + i] = x0*x1 + x2*x3 + x4;
        }
    }
    for (long i = 36; i < 38; ++i) {
        const double x0 = x[p[1071818 + i]];
        const double x1 = x[p[1071856 + i]];
        const double x2 = x[p[1071894 + i]];
        const double x3 = x[p[1071932 + i]];
        const double x4 = x[p[1071970 + i]];
        x[1656864 + i] = x0*x1 + x2*x3 + x4;
    }
}

/* level 0, 1594 instance(s), 1 result(s) each */
static void out3_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 398; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1072008 + i]];
            const double x1 = x[p[1073602 + i]];
            const double x2 = x[p[1075196 + i]];
            const double x3 = x[p[1076790 + i]];
            const double x4 = x[p[1078384 + i]];
            const double x5 = x[p[1079978 + i]];
            x[1656904 + i] = x0*x1 + x2*x3 + x4*x5;
        }
    }
    for (long i = 1592; i < 1594; ++i) {
        const double x0 = x[p[1072008 + i]];
        const double x1 = x[p[1073602 + i]];
        const double x2 = x[p[1075196 + i]];
        const double x3 = x[p[1076790 + i]];
        const double x4 = x[p[1078384 + i]];
        const double x5 = x[p[1079978 + i]];
        x[1656904 + i] = x0*x1 + x2*x3 + x4*x5;
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1081572 + i]];
            const double x1 = x[p[1081572 + i] - 283853];
            const double x2 = x[p[1081572 + i] - 121224];
            const double x3 = x[p[1081572 + i] - 364669];
            const double x4 = x[p[1081572 + i] - 40408];
            const double x5 = x[p[1081572 + i] - 324261];
            const double x6 = x[p[1081572 + i] - 80816];
            const double x7 = x[p[1081572 + i] - 405873];
            x[1658500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1121572 + i]];
            const double x1 = x[p[1121572 + i] - 162427];
            const double x2 = x[p[1121572 + i] + 40408];
            const double x3 = x[p[1121572 + i] - 81412];
            const double x4 = x[p[1121572 + i] + 161632];
            const double x5 = x[p[1121572 + i] - 122020];
            const double x6 = x[p[1121572 + i] + 242448];
            const double x7 = x[p[1121572 + i] - 203431];
            x[1698500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1161572 + i]];
            const double x1 = x[p[1161572 + i] - 324260];
            const double x2 = x[p[1161572 + i] + 40408];
            const double x3 = x[p[1161572 + i] - 364467];
            const double x4 = x[p[1161572 + i] - 40408];
            const double x5 = x[p[1161572 + i] - 283652];
            const double x6 = x[p[1161572 + i] - 202040];
            const double x7 = x[p[1161572 + i] - 405671];
            x[1738500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1201572 + i]];
            const double x1 = x[p[1201572 + i] - 283853];
            const double x2 = x[p[1201572 + i] - 80816];
            const double x3 = x[p[1201572 + i] - 243245];
            const double x4 = x[p[1201572 + i] + 40408];
            const double x5 = x[p[1201572 + i] - 202837];
            const double x6 = x[p[1201572 + i] - 40408];
            const double x7 = x[p[1201572 + i] - 324857];
            x[1778500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1241572 + i]];
            const double x1 = x[p[1241572 + i] - 203037];
            const double x2 = x[p[1241572 + i] - 121224];
            const double x3 = x[p[1241572 + i] - 243444];
            const double x4 = x[p[1241572 + i] + 40408];
            const double x5 = x[p[1241572 + i] - 283852];
            const double x6 = x[p[1241572 + i] + 80816];
            const double x7 = x[p[1241572 + i] - 325056];
            x[1818500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out4_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1281572 + i]];
            const double x1 = x[p[1281572 + i] - 202837];
            const double x2 = x[p[1281572 + i] + 161632];
            const double x3 = x[p[1281572 + i] - 162228];
            const double x4 = x[p[1281572 + i] + 80816];
            const double x5 = x[p[1281572 + i] - 243244];
            const double x6 = x[p[1281572 + i] - 40408];
            const double x7 = x[p[1281572 + i] - 284248];
            x[1858500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 4746 instance(s), 1 result(s) each */
static void out4_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1186; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1321572 + i]];
            const double x1 = x[p[1326318 + i]];
            const double x2 = x[p[1331064 + i]];
            const double x3 = x[p[1335810 + i]];
            const double x4 = x[p[1340556 + i]];
            const double x5 = x[p[1345302 + i]];
            const double x6 = x[p[1350048 + i]];
            const double x7 = x[p[1354794 + i]];
            x[1898500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
    for (long i = 4744; i < 4746; ++i) {
        const double x0 = x[p[1321572 + i]];
        const double x1 = x[p[1326318 + i]];
        const double x2 = x[p[1331064 + i]];
        const double x3 = x[p[1335810 + i]];
        const double x4 = x[p[1340556 + i]];
        const double x5 = x[p[1345302 + i]];
        const double x6 = x[p[1350048 + i]];
        const double x7 = x[p[1354794 + i]];
        x[1898500 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
    }
}

/* level 0, 35 instance(s), 1 result(s) each */
static void out4a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 8; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1359540 + i]];
            const double x1 = x[p[1359575 + i]];
            const double x2 = x[p[1359610 + i]];
            const double x3 = x[p[1359645 + i]];
            const double x4 = x[p[1359680 + i]];
            const double x5 = x[p[1359715 + i]];
            const double x6 = x[p[1359750 + i]];
            const double x7 = x[p[1359785 + i]];
            const double x8 = x[p[1359820 + i]];
            x[1903248 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8;
        }
    }
    for (long i = 32; i < 35; ++i) {
        const double x0 = x[p[1359540 + i]];
        const double x1 = x[p[1359575 + i]];
        const double x2 = x[p[1359610 + i]];
        const double x3 = x[p[1359645 + i]];
        const double x4 = x[p[1359680 + i]];
        const double x5 = x[p[1359715 + i]];
        const double x6 = x[p[1359750 + i]];
        const double x7 = x[p[1359785 + i]];
        const double x8 = x[p[1359820 + i]];
        x[1903248 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8;
    }
}

/* level 0, 792 instance(s), 1 result(s) each */
static void out5_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 198; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1359855 + i]];
            const double x1 = x[p[1360647 + i]];
            const double x2 = x[p[1361439 + i]];
            const double x3 = x[p[1362231 + i]];
            const double x4 = x[p[1363023 + i]];
            const double x5 = x[p[1363815 + i]];
            const double x6 = x[p[1364607 + i]];
            const double x7 = x[p[1365399 + i]];
            const double x8 = x[p[1366191 + i]];
            const double x9 = x[p[1366983 + i]];
            x[1903284 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9;
        }
    }
}

/* level 0, 40000 instance(s), 1 result(s) each */
static void out7_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1367775 + i]];
            const double x1 = x[p[1367775 + i] - 365264];
            const double x2 = x[p[1367775 + i] - 40408];
            const double x3 = x[p[1367775 + i] - 283853];
            const double x4 = x[p[1367775 + i] + 40408];
            const double x5 = x[p[1367775 + i] - 324260];
            const double x6 = x[p[1367775 + i] - 80816];
            const double x7 = x[p[1367775 + i] - 243245];
            const double x8 = x[p[1367775 + i] - 161632];
            const double x9 = x[p[1367775 + i] - 243244];
            const double x10 = x[p[1367775 + i] - 121224];
            const double x11 = x[p[1367775 + i] - 324060];
            const double x12 = x[p[1367775 + i] + 80816];
            const double x13 = x[p[1367775 + i] - 283652];
            x[1904076 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13;
        }
    }
}

/* level 0, 788 instance(s), 1 result(s) each */
static void out7_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 197; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1407775 + i]];
            const double x1 = x[p[1408563 + i]];
            const double x2 = x[p[1409351 + i]];
            const double x3 = x[p[1410139 + i]];
            const double x4 = x[p[1410927 + i]];
            const double x5 = x[p[1411715 + i]];
            const double x6 = x[p[1412503 + i]];
            const double x7 = x[p[1413291 + i]];
            const double x8 = x[p[1414079 + i]];
            const double x9 = x[p[1414867 + i]];
            const double x10 = x[p[1415655 + i]];
            const double x11 = x[p[1416443 + i]];
            const double x12 = x[p[1417231 + i]];
            const double x13 = x[p[1418019 + i]];
            x[1944076 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13;
        }
    }
}

/* level 0, 3 instance(s), 1 result(s) each */
static void out7a_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 3; ++i) {
        const double x0 = x[p[1418807 + i]];
        const double x1 = x[p[1418807 + i] - 365264];
        const double x2 = x[p[1418807 + i] - 40408];
        const double x3 = x[p[1418807 + i] - 283853];
        const double x4 = x[p[1418807 + i] + 40408];
        const double x5 = x[p[1418807 + i] - 324260];
        const double x6 = x[p[1418807 + i] - 80816];
        const double x7 = x[p[1418807 + i] - 243245];
        const double x8 = x[p[1418807 + i] - 161632];
        const double x9 = x[p[1418807 + i] - 243244];
        const double x10 = x[p[1418807 + i] - 121224];
        const double x11 = x[p[1418807 + i] - 324060];
        const double x12 = x[p[1418807 + i] + 80816];
        const double x13 = x[p[1418807 + i] - 283652];
        const double x14 = x[p[1418810 + i]];
        x[1944864 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13 + x14;
    }
}

void sg_run(double* x, const double* c, const unsigned* p) {
    face_s0(x, c, p);
    face_s1(x, c, p);
    ldiag2_b(x, c, p);
    ldiag4_b(x, c, p);
    ldiag6_b(x, c, p);
    ldiag12_s0(x, c, p);
    loff1_b(x, c, p);
    loff2_s0(x, c, p);
    loff2_s1(x, c, p);
    loff2_s2(x, c, p);
    mdiag2_b(x, c, p);
    mdiag3_b(x, c, p);
    mdiag6_s0(x, c, p);
    lm_s0(x, c, p);
    lm_s1(x, c, p);
    lm_s2(x, c, p);
    lm_s3(x, c, p);
    lm_s4(x, c, p);
    lm_s5(x, c, p);
    lm_s6(x, c, p);
    lm_b(x, c, p);
    out1_s0(x, c, p);
    out1_s1(x, c, p);
    out1_s2(x, c, p);
    out1_s3(x, c, p);
    out1_s4(x, c, p);
    out1_s5(x, c, p);
    out1_b(x, c, p);
    out1a_b(x, c, p);
    out2_s0(x, c, p);
    out2_s1(x, c, p);
    out2_s2(x, c, p);
    out2_s3(x, c, p);
    out2_s4(x, c, p);
    out2_s5(x, c, p);
    out2_b(x, c, p);
    out2a_b(x, c, p);
    out3_b(x, c, p);
    out4_s0(x, c, p);
    out4_s1(x, c, p);
    out4_s2(x, c, p);
    out4_s3(x, c, p);
    out4_s4(x, c, p);
    out4_s5(x, c, p);
    out4_b(x, c, p);
    out4a_b(x, c, p);
    out5_b(x, c, p);
    out7_s0(x, c, p);
    out7_b(x, c, p);
    out7a_b(x, c, p);
}
