/* generated kernel source; compile with: cc -O3 -ffp-contract=off */
#include <math.h>

/* level 3, 1000000 instance(s), 4 result(s) each */
static void face_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[0 + i]];
            const double x1 = x[p[0 + i] + 1];
            const double x2 = x[p[0 + i] + 2];
            const double x3 = x[p[0 + i] + 3003];
            const double x4 = x[p[0 + i] + 3004];
            const double x5 = x[p[0 + i] + 3005];
            const double x6 = x[p[0 + i] + 3000];
            const double x7 = x[p[0 + i] + 3001];
            const double x8 = x[p[0 + i] + 3002];
            x[9000000 + i] = (-(x3 - x0)*(x0 - x6) + -(x4 - x1)*(x1 - x7) + -(x5 - x2)*(x2 - x8))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[10000000 + i] = (-(x6 - x3)*(x3 - x0) + -(x7 - x4)*(x4 - x1) + -(x8 - x5)*(x5 - x2))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[11000000 + i] = (-(x0 - x6)*(x6 - x3) + -(x1 - x7)*(x7 - x4) + -(x2 - x8)*(x8 - x5))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[12000000 + i] = sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)))*0.16666666666666666;
        }
    }
}

/* level 3, 1000000 instance(s), 4 result(s) each */
static void face_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[1000000 + i]];
            const double x1 = x[p[1000000 + i] + 1];
            const double x2 = x[p[1000000 + i] + 2];
            const double x3 = x[p[1000000 + i] + 3];
            const double x4 = x[p[1000000 + i] + 4];
            const double x5 = x[p[1000000 + i] + 5];
            const double x6 = x[p[1000000 + i] + 3003];
            const double x7 = x[p[1000000 + i] + 3004];
            const double x8 = x[p[1000000 + i] + 3005];
            x[13002008 + i] = (-(x3 - x0)*(x0 - x6) + -(x4 - x1)*(x1 - x7) + -(x5 - x2)*(x2 - x8))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[14002008 + i] = (-(x6 - x3)*(x3 - x0) + -(x7 - x4)*(x4 - x1) + -(x8 - x5)*(x5 - x2))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[15002008 + i] = (-(x0 - x6)*(x6 - x3) + -(x1 - x7)*(x7 - x4) + -(x2 - x8)*(x8 - x5))*0.5/sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)));
            x[16002008 + i] = sqrt(((x3 - x0)*(x3 - x0) + (x4 - x1)*(x4 - x1) + (x5 - x2)*(x5 - x2))*(-(x0 - x6)*-(x0 - x6) + -(x1 - x7)*-(x1 - x7) + -(x2 - x8)*-(x2 - x8)) - ((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8))*((x3 - x0)*-(x0 - x6) + (x4 - x1)*-(x1 - x7) + (x5 - x2)*-(x2 - x8)))*0.16666666666666666;
        }
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void ldiag2_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[2000000 + i]];
        const double x1 = x[p[2000002 + i]];
        x[17004016 + i] = x0 + x1;
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void ldiag4_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[2000004 + i]];
        const double x1 = x[p[2000004 + i] + 1000000];
        const double x2 = x[p[2000004 + i] - 4002008];
        const double x3 = x[p[2000006 + i]];
        x[17004020 + i] = x0 + x1 + x2 + x3;
    }
}

/* level 2, 3992 instance(s), 1 result(s) each */
static void ldiag6_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 998; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[2000008 + i]];
            const double x1 = x[p[2004000 + i]];
            const double x2 = x[p[2007992 + i]];
            const double x3 = x[p[2011984 + i]];
            const double x4 = x[p[2015976 + i]];
            const double x5 = x[p[2019968 + i]];
            x[17004024 + i] = x0 + x1 + x2 + x3 + x4 + x5;
        }
    }
}

/* level 2, 1000000 instance(s), 1 result(s) each */
static void ldiag12_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[2023960 + i]];
            const double x1 = x[p[2023960 + i] + 1000000];
            const double x2 = x[p[2023960 + i] - 4002008];
            const double x3 = x[p[2023960 + i] - 2002008];
            const double x4 = x[p[2023960 + i] - 4002007];
            const double x5 = x[p[2023960 + i] - 3002007];
            const double x6 = x[p[2023960 + i] + 1000];
            const double x7 = x[p[2023960 + i] + 2001000];
            const double x8 = x[p[2023960 + i] + 1001001];
            const double x9 = x[p[2023960 + i] + 2001001];
            const double x10 = x[p[2023960 + i] - 3001007];
            const double x11 = x[p[2023960 + i] - 2001007];
            x[17008016 + i] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + x8 + x9 + x10 + x11;
        }
    }
}

/* level 2, 3996 instance(s), 1 result(s) each */
static void loff1_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 999; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[3023960 + i]];
            x[18010024 + i] = -x0;
        }
    }
}

/* level 2, 1000000 instance(s), 1 result(s) each */
static void loff2_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[3027956 + i]];
            const double x1 = x[p[3027956 + i] - 3002008];
            x[18014020 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 1000000 instance(s), 1 result(s) each */
static void loff2_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[4027956 + i]];
            const double x1 = x[p[4027956 + i] + 6003008];
            x[19016028 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 1000000 instance(s), 1 result(s) each */
static void loff2_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[5027956 + i]];
            const double x1 = x[p[5027956 + i] - 3002007];
            x[20018036 + i] = -x0 + -x1;
        }
    }
}

/* level 2, 2 instance(s), 1 result(s) each */
static void mdiag2_b(double* x, const double* c, const unsigned* p) {
    for (long i = 0; i < 2; ++i) {
        const double x0 = x[p[6027956 + i]];
        const double x1 = x[p[6027956 + i] - 4002008];
        x[21020044 + i] = x0 + x1;
    }
}

/* level 2, 3992 instance(s), 1 result(s) each */
static void mdiag3_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 998; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[6027958 + i]];
            const double x1 = x[p[6031950 + i]];
            const double x2 = x[p[6035942 + i]];
            x[21020048 + i] = x0 + x1 + x2;
        }
    }
}

/* level 2, 1000000 instance(s), 1 result(s) each */
static void mdiag6_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[6039934 + i]];
            const double x1 = x[p[6039934 + i] - 4002008];
            const double x2 = x[p[6039934 + i] - 4002007];
            const double x3 = x[p[6039934 + i] + 1000];
            const double x4 = x[p[6039934 + i] + 1001];
            const double x5 = x[p[6039934 + i] - 4001007];
            x[21024040 + i] = x0 + x1 + x2 + x3 + x4 + x5;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[7039934 + i]];
            const double x1 = x[p[7039934 + i] + 3011021];
            x[22026048 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[8039934 + i]];
            const double x1 = x[p[8039934 + i] + 2008012];
            x[23028056 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[9039934 + i]];
            const double x1 = x[p[9039934 + i] + 1006004];
            x[24030064 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[10039934 + i]];
            const double x1 = x[p[10039934 + i] + 1007004];
            x[25032072 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[11039934 + i]];
            const double x1 = x[p[11039934 + i] + 4016024];
            x[26034080 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[12039934 + i]];
            const double x1 = x[p[12039934 + i] + 3010020];
            x[27036088 + i] = x0*x1;
        }
    }
}

/* level 1, 1000000 instance(s), 1 result(s) each */
static void lm_s6(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[13039934 + i]];
            const double x1 = x[p[13039934 + i] + 2008013];
            x[28038096 + i] = x0*x1;
        }
    }
}

/* level 1, 19974 instance(s), 1 result(s) each */
static void lm_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 4993; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[14039934 + i]];
            const double x1 = x[p[14059908 + i]];
            x[29040104 + i] = x0*x1;
        }
    }
    for (long i = 19972; i < 19974; ++i) {
        const double x0 = x[p[14039934 + i]];
        const double x1 = x[p[14059908 + i]];
        x[29040104 + i] = x0*x1;
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[14079882 + i]];
            const double x1 = x[p[14079882 + i] - 5013036];
            x[29060080 + i] = x0*x1;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[15079882 + i]];
            const double x1 = x[p[15079882 + i] - 4011027];
            x[30060080 + i] = x0*x1;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[16079882 + i]];
            const double x1 = x[p[16079882 + i] - 4012030];
            x[31060080 + i] = x0*x1;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[17079882 + i]];
            const double x1 = x[p[17079882 + i] - 9022067];
            x[32060080 + i] = x0*x1;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[18079882 + i]];
            const double x1 = x[p[18079882 + i] - 4014028];
            x[33060080 + i] = x0*x1;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out1_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[19079882 + i]];
            const double x1 = x[p[19079882 + i] - 9024070];
            x[34060080 + i] = x0*x1;
        }
    }
}

/* level 0, 7984 instance(s), 1 result(s) each */
static void out1_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1996; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[20079882 + i]];
            const double x1 = x[p[20087866 + i]];
            x[35060080 + i] = x0*x1;
        }
    }
}

/* level 0, 35 instance(s), 1 result(s) each */
static void out1a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 8; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[20095850 + i]];
            const double x1 = x[p[20095885 + i]];
            const double x2 = x[p[20095920 + i]];
            x[35068064 + i] = x0*x1 + x2;
        }
    }
    for (long i = 32; i < 35; ++i) {
        const double x0 = x[p[20095850 + i]];
        const double x1 = x[p[20095885 + i]];
        const double x2 = x[p[20095920 + i]];
        x[35068064 + i] = x0*x1 + x2;
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[20095955 + i]];
            const double x1 = x[p[20095955 + i] - 5015036];
            const double x2 = x[p[20095955 + i] + 4008032];
            const double x3 = x[p[20095955 + i] - 4013027];
            x[35068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[21095955 + i]];
            const double x1 = x[p[21095955 + i] - 10024075];
            const double x2 = x[p[21095955 + i] - 6012048];
            const double x3 = x[p[21095955 + i] - 9021067];
            x[36068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[22095955 + i]];
            const double x1 = x[p[22095955 + i] - 7017052];
            const double x2 = x[p[22095955 + i] - 3006024];
            const double x3 = x[p[22095955 + i] - 5013035];
            x[37068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[23095955 + i]];
            const double x1 = x[p[23095955 + i] - 8021062];
            const double x2 = x[p[23095955 + i] - 4008032];
            const double x3 = x[p[23095955 + i] - 9023070];
            x[38068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[24095955 + i]];
            const double x1 = x[p[24095955 + i] - 7020053];
            const double x2 = x[p[24095955 + i] - 3006024];
            const double x3 = x[p[24095955 + i] - 9024069];
            x[39068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out2_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[25095955 + i]];
            const double x1 = x[p[25095955 + i] - 3010021];
            const double x2 = x[p[25095955 + i] + 2004016];
            const double x3 = x[p[25095955 + i] - 4011029];
            x[40068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 15968 instance(s), 1 result(s) each */
static void out2_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 3992; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[26095955 + i]];
            const double x1 = x[p[26111923 + i]];
            const double x2 = x[p[26127891 + i]];
            const double x3 = x[p[26143859 + i]];
            x[41068100 + i] = x0*x1 + x2*x3;
        }
    }
}

/* level 0, 41 instance(s), 1 result(s) each */
static void out2a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 10; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[26159827 + i]];
            const double x1 = x[p[26159868 + i]];
            const double x2 = x[p[26159909 + i]];
            const double x3 = x[p[26159950 + i]];
            const double x4 = x[p[26159991 + i]];
            x[41084068 + i] = x0*x1 + x2*x3 + x4;
        }
    }
    for (long i = 40; i < 41; ++i) {
        const double x0 = x[p[26159827 + i]];
        const double x1 = x[p[26159868 + i]];
        const double x2 = x[p[26159909 + i]];
        const double x3 = x[p[26159950 + i]];
        const double x4 = x[p[26159991 + i]];
        x[41084068 + i] = x0*x1 + x2*x3 + x4;
    }
}

/* level 0, 7994 instance(s), 1 result(s) each */
static void out3_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 1998; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[26160032 + i]];
            const double x1 = x[p[26168026 + i]];
            const double x2 = x[p[26176020 + i]];
            const double x3 = x[p[26184014 + i]];
            const double x4 = x[p[26192008 + i]];
            const double x5 = x[p[26200002 + i]];
            x[41084112 + i] = x0*x1 + x2*x3 + x4*x5;
        }
    }
    for (long i = 7992; i < 7994; ++i) {
        const double x0 = x[p[26160032 + i]];
        const double x1 = x[p[26168026 + i]];
        const double x2 = x[p[26176020 + i]];
        const double x3 = x[p[26184014 + i]];
        const double x4 = x[p[26192008 + i]];
        const double x5 = x[p[26200002 + i]];
        x[41084112 + i] = x0*x1 + x2*x3 + x4*x5;
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[26207996 + i]];
            const double x1 = x[p[26207996 + i] - 7019053];
            const double x2 = x[p[26207996 + i] - 2004016];
            const double x3 = x[p[26207996 + i] - 9022069];
            const double x4 = x[p[26207996 + i] - 1002008];
            const double x5 = x[p[26207996 + i] - 8020061];
            const double x6 = x[p[26207996 + i] - 4008032];
            const double x7 = x[p[26207996 + i] - 10028073];
            x[41092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s1(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[27207996 + i]];
            const double x1 = x[p[27207996 + i] - 5015037];
            const double x2 = x[p[27207996 + i] - 1002008];
            const double x3 = x[p[27207996 + i] - 4013029];
            const double x4 = x[p[27207996 + i] + 2004016];
            const double x5 = x[p[27207996 + i] - 6017045];
            const double x6 = x[p[27207996 + i] + 3006024];
            const double x7 = x[p[27207996 + i] - 7023049];
            x[42092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s2(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[28207996 + i]];
            const double x1 = x[p[28207996 + i] - 6017044];
            const double x2 = x[p[28207996 + i] - 2004016];
            const double x3 = x[p[28207996 + i] - 4012027];
            const double x4 = x[p[28207996 + i] + 2004016];
            const double x5 = x[p[28207996 + i] - 5014036];
            const double x6 = x[p[28207996 + i] + 4008032];
            const double x7 = x[p[28207996 + i] - 7022047];
            x[43092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s3(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[29207996 + i]];
            const double x1 = x[p[29207996 + i] - 5014037];
            const double x2 = x[p[29207996 + i] - 1002008];
            const double x3 = x[p[29207996 + i] - 4011028];
            const double x4 = x[p[29207996 + i] + 3006024];
            const double x5 = x[p[29207996 + i] - 3010020];
            const double x6 = x[p[29207996 + i] + 2004016];
            const double x7 = x[p[29207996 + i] - 6019040];
            x[44092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s4(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[30207996 + i]];
            const double x1 = x[p[30207996 + i] - 8020059];
            const double x2 = x[p[30207996 + i] - 3006024];
            const double x3 = x[p[30207996 + i] - 9021068];
            const double x4 = x[p[30207996 + i] - 2004016];
            const double x5 = x[p[30207996 + i] - 10024076];
            const double x6 = x[p[30207996 + i] - 6012048];
            const double x7 = x[p[30207996 + i] - 11029079];
            x[45092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out4_s5(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[31207996 + i]];
            const double x1 = x[p[31207996 + i] - 8021061];
            const double x2 = x[p[31207996 + i] + 1002008];
            const double x3 = x[p[31207996 + i] - 9023068];
            const double x4 = x[p[31207996 + i] - 1002008];
            const double x5 = x[p[31207996 + i] - 7019052];
            const double x6 = x[p[31207996 + i] - 3006024];
            const double x7 = x[p[31207996 + i] - 10029072];
            x[46092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
}

/* level 0, 23946 instance(s), 1 result(s) each */
static void out4_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 5986; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[32207996 + i]];
            const double x1 = x[p[32231942 + i]];
            const double x2 = x[p[32255888 + i]];
            const double x3 = x[p[32279834 + i]];
            const double x4 = x[p[32303780 + i]];
            const double x5 = x[p[32327726 + i]];
            const double x6 = x[p[32351672 + i]];
            const double x7 = x[p[32375618 + i]];
            x[47092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
        }
    }
    for (long i = 23944; i < 23946; ++i) {
        const double x0 = x[p[32207996 + i]];
        const double x1 = x[p[32231942 + i]];
        const double x2 = x[p[32255888 + i]];
        const double x3 = x[p[32279834 + i]];
        const double x4 = x[p[32303780 + i]];
        const double x5 = x[p[32327726 + i]];
        const double x6 = x[p[32351672 + i]];
        const double x7 = x[p[32375618 + i]];
        x[47092108 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7;
    }
}

/* level 0, 28 instance(s), 1 result(s) each */
static void out4a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 7; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[32399564 + i]];
            const double x1 = x[p[32399592 + i]];
            const double x2 = x[p[32399620 + i]];
            const double x3 = x[p[32399648 + i]];
            const double x4 = x[p[32399676 + i]];
            const double x5 = x[p[32399704 + i]];
            const double x6 = x[p[32399732 + i]];
            const double x7 = x[p[32399760 + i]];
            const double x8 = x[p[32399788 + i]];
            x[47116056 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8;
        }
    }
}

/* level 0, 3992 instance(s), 1 result(s) each */
static void out5_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 998; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[32399816 + i]];
            const double x1 = x[p[32403808 + i]];
            const double x2 = x[p[32407800 + i]];
            const double x3 = x[p[32411792 + i]];
            const double x4 = x[p[32415784 + i]];
            const double x5 = x[p[32419776 + i]];
            const double x6 = x[p[32423768 + i]];
            const double x7 = x[p[32427760 + i]];
            const double x8 = x[p[32431752 + i]];
            const double x9 = x[p[32435744 + i]];
            x[47116084 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9;
        }
    }
}

/* level 0, 1000000 instance(s), 1 result(s) each */
static void out7_s0(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 250000; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[32439736 + i]];
            const double x1 = x[p[32439736 + i] - 9026064];
            const double x2 = x[p[32439736 + i] + 1002008];
            const double x3 = x[p[32439736 + i] - 8021061];
            const double x4 = x[p[32439736 + i] - 2004016];
            const double x5 = x[p[32439736 + i] - 6017044];
            const double x6 = x[p[32439736 + i] - 3006024];
            const double x7 = x[p[32439736 + i] - 7018053];
            const double x8 = x[p[32439736 + i] + 2004016];
            const double x9 = x[p[32439736 + i] - 7018052];
            const double x10 = x[p[32439736 + i] - 1002008];
            const double x11 = x[p[32439736 + i] - 6016044];
            const double x12 = x[p[32439736 + i] - 4008032];
            const double x13 = x[p[32439736 + i] - 8020060];
            x[47120076 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13;
        }
    }
}

/* level 0, 3988 instance(s), 1 result(s) each */
static void out7_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 997; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[33439736 + i]];
            const double x1 = x[p[33443724 + i]];
            const double x2 = x[p[33447712 + i]];
            const double x3 = x[p[33451700 + i]];
            const double x4 = x[p[33455688 + i]];
            const double x5 = x[p[33459676 + i]];
            const double x6 = x[p[33463664 + i]];
            const double x7 = x[p[33467652 + i]];
            const double x8 = x[p[33471640 + i]];
            const double x9 = x[p[33475628 + i]];
            const double x10 = x[p[33479616 + i]];
            const double x11 = x[p[33483604 + i]];
            const double x12 = x[p[33487592 + i]];
            const double x13 = x[p[33491580 + i]];
            x[48120076 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13;
        }
    }
}

/* level 0, 11 instance(s), 1 result(s) each */
static void out7a_b(double* x, const double* c, const unsigned* p) {
    #pragma omp parallel for
    for (long ii = 0; ii < 2; ++ii) {
        #pragma omp simd
        for (long j = 0; j < 4; ++j) {
            const long i = ii*4 + j;
            const double x0 = x[p[33495568 + i]];
            const double x1 = x[p[33495568 + i] - 9026064];
            const double x2 = x[p[33495568 + i] + 1002008];
            const double x3 = x[p[33495568 + i] - 8021061];
            const double x4 = x[p[33495568 + i] - 2004016];
            const double x5 = x[p[33495568 + i] - 6017044];
            const double x6 = x[p[33495568 + i] - 3006024];
            const double x7 = x[p[33495568 + i] - 7018053];
            const double x8 = x[p[33495568 + i] + 2004016];
            const double x9 = x[p[33495568 + i] - 7018052];
            const double x10 = x[p[33495568 + i] - 1002008];
            const double x11 = x[p[33495568 + i] - 6016044];
            const double x12 = x[p[33495568 + i] - 4008032];
            const double x13 = x[p[33495568 + i] - 8020060];
            const double x14 = x[p[33495579 + i]];
            x[48124064 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13 + x14;
        }
    }
    for (long i = 8; i < 11; ++i) {
        const double x0 = x[p[33495568 + i]];
        const double x1 = x[p[33495568 + i] - 9026064];
        const double x2 = x[p[33495568 + i] + 1002008];
        const double x3 = x[p[33495568 + i] - 8021061];
        const double x4 = x[p[33495568 + i] - 2004016];
        const double x5 = x[p[33495568 + i] - 6017044];
        const double x6 = x[p[33495568 + i] - 3006024];
        const double x7 = x[p[33495568 + i] - 7018053];
        const double x8 = x[p[33495568 + i] + 2004016];
        const double x9 = x[p[33495568 + i] - 7018052];
        const double x10 = x[p[33495568 + i] - 1002008];
        const double x11 = x[p[33495568 + i] - 6016044];
        const double x12 = x[p[33495568 + i] - 4008032];
        const double x13 = x[p[33495568 + i] - 8020060];
        const double x14 = x[p[33495579 + i]];
        x[48124064 + i] = x0*x1 + x2*x3 + x4*x5 + x6*x7 + x8*x9 + x10*x11 + x12*x13 + x14;
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
