/* philox_gauss.h — the counter-based Gaussian generator that defines the KRP
 * sketch factors Omega_k in "philox" mode. Shared, byte-for-byte, by the CUDA
 * kernels (paper_2511_03598_b200/csrc/sketch.cu) and the CPU oracle
 * (oracle/ttr_oracle.cpp) so both sides draw the SAME Omega.
 *
 * Replaces the reference's sequential stream for the sketch factors:
 *   GaussianStream::next / ::matrix     proj/core/src/rng.cpp:34-67
 *   draw_gaussian_factors               proj/core/src/sketch.cpp:44-56
 *   append_gaussian_columns / appends   proj/core/src/sketch.cpp:58-65,
 *                                       proj/core/src/round_rand.cpp:87-90
 * The reference draws Omega_t..Omega_d column-major from ONE xoshiro256++
 * stream, so entry values depend on draw history. Here every entry is a pure
 * function of (seed, mode k, global column c, row i):
 *
 *   ctr  = (floor(i/2), c, k, tag)   key = (lo32(seed), hi32(seed))
 *   x    = Philox4x32-10(ctr, key)                (Salmon et al., SC'11)
 *   u1   = ((x1:x0 >> 11) + 1) * 2^-53   in (0, 1]
 *   u2   =  (x3:x2 >> 11)      * 2^-53   in [0, 1)
 *   rho  = sqrt(-2 log u1)
 *   Omega_k(i, c) = rho * cos(2 pi u2)  (i even)
 *                 = rho * sin(2 pi u2)  (i odd)
 *
 * Because a column's values never depend on how many columns were drawn
 * before it, adaptive appends equal a one-shot draw of the wider factor.
 *
 * Bit-exactness across host and device: log, sin and cos are evaluated with
 * the fdlibm polynomials (argument reduction in "turns", so no large-argument
 * reduction is needed) using only IEEE-754 round-to-nearest +, -, *, /, sqrt
 * and fused multiply-add, each spelled through the TTR_* macros below. On the
 * device they map to the __d*_rn / __fma_rn intrinsics, which nvcc never
 * contracts; on the host the translation unit must be compiled with
 * -ffp-contract=off (oracle/Makefile does this) and fma maps to std::fma.
 */
#ifndef TTR_PHILOX_GAUSS_H
#define TTR_PHILOX_GAUSS_H

#include <stdint.h>

#if defined(__CUDACC__)
#define TTR_HD __host__ __device__ __forceinline__
#else
#define TTR_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define TTR_ADD(a, b) __dadd_rn((a), (b))
#define TTR_SUB(a, b) __dsub_rn((a), (b))
#define TTR_MUL(a, b) __dmul_rn((a), (b))
#define TTR_DIV(a, b) __ddiv_rn((a), (b))
#define TTR_FMA(a, b, c) __fma_rn((a), (b), (c))
#define TTR_SQRT(a) __dsqrt_rn((a))
#define TTR_MULHI32(a, b) __umulhi((a), (b))
#define TTR_AS_U64(x) ((uint64_t)__double_as_longlong(x))
#define TTR_AS_F64(u) __longlong_as_double((long long)(u))
#else
#include <math.h>
#include <string.h>
#define TTR_ADD(a, b) ((a) + (b))
#define TTR_SUB(a, b) ((a) - (b))
#define TTR_MUL(a, b) ((a) * (b))
#define TTR_DIV(a, b) ((a) / (b))
#define TTR_FMA(a, b, c) fma((a), (b), (c))
#define TTR_SQRT(a) sqrt((a))
#define TTR_MULHI32(a, b) ((uint32_t)(((uint64_t)(a) * (uint64_t)(b)) >> 32))
static inline uint64_t ttr_as_u64_host(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double ttr_as_f64_host(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define TTR_AS_U64(x) ttr_as_u64_host(x)
#define TTR_AS_F64(u) ttr_as_f64_host(u)
#endif

#define TTR_PHILOX_TAG_KRP 0u /* tag used for the KRP factors Omega_k */

typedef struct { uint32_t v[4]; } ttr_u32x4;

/* Philox4x32 with 10 rounds (Random123 constants). */
TTR_HD ttr_u32x4 ttr_philox4x32_10(ttr_u32x4 ctr, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = M0 * ctr.v[0], hi0 = TTR_MULHI32(M0, ctr.v[0]);
        const uint32_t lo1 = M1 * ctr.v[2], hi1 = TTR_MULHI32(M1, ctr.v[2]);
        ttr_u32x4 n;
        n.v[0] = hi1 ^ ctr.v[1] ^ k0;
        n.v[1] = lo1;
        n.v[2] = hi0 ^ ctr.v[3] ^ k1;
        n.v[3] = lo0;
        ctr = n;
        k0 += W0;
        k1 += W1;
    }
    return ctr;
}

/* log(u) for u in [2^-53, 1]: fdlibm e_log.c reduction and polynomial. */
TTR_HD double ttr_log_unit(double u) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                 Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                 Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                 Lg7 = 1.479819860511658591e-01;
    const uint64_t bits = TTR_AS_U64(u);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    uint64_t mbits = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull; /* m in [1,2) */
    if (mbits > 0x3ff6a09e667f3bcdull) { /* m > sqrt(2): halve it (exact) */
        mbits -= 0x0010000000000000ull;
        e += 1;
    }
    const double m = TTR_AS_F64(mbits);
    const double f = TTR_SUB(m, 1.0); /* exact (Sterbenz) */
    const double s = TTR_DIV(f, TTR_ADD(2.0, f));
    const double z = TTR_MUL(s, s);
    const double w = TTR_MUL(z, z);
    const double t1 = TTR_MUL(w, TTR_FMA(w, TTR_FMA(w, Lg6, Lg4), Lg2));
    const double t2 = TTR_MUL(z, TTR_FMA(w, TTR_FMA(w, TTR_FMA(w, Lg7, Lg5), Lg3), Lg1));
    const double R = TTR_ADD(t2, t1);
    const double hfsq = TTR_MUL(TTR_MUL(0.5, f), f);
    const double de = (double)e;
    /* log(1+f) = f - (hfsq - (s*(hfsq+R) + e*ln2_lo)) + e*ln2_hi */
    const double corr = TTR_FMA(s, TTR_ADD(hfsq, R), TTR_MUL(de, ln2_lo));
    return TTR_FMA(de, ln2_hi, TTR_SUB(f, TTR_SUB(hfsq, corr)));
}

/* sin and cos of x in [-pi/4, pi/4]: fdlibm k_sin.c / k_cos.c (y = 0). */
TTR_HD double ttr_kernel_sin(double x) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    const double z = TTR_MUL(x, x);
    const double v = TTR_MUL(z, x);
    const double r = TTR_FMA(z, TTR_FMA(z, TTR_FMA(z, TTR_FMA(z, S6, S5), S4), S3), S2);
    return TTR_FMA(v, TTR_FMA(z, r, S1), x);
}

TTR_HD double ttr_kernel_cos(double x) {
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    const double z = TTR_MUL(x, x);
    const double r = TTR_MUL(z, TTR_FMA(z, TTR_FMA(z, TTR_FMA(z, TTR_FMA(z, TTR_FMA(z, C6, C5), C4), C3), C2), C1));
    const double hz = TTR_MUL(0.5, z);
    const double w = TTR_SUB(1.0, hz);
    return TTR_ADD(w, TTR_FMA(z, r, TTR_SUB(TTR_SUB(1.0, w), hz)));
}

/* (cos(2 pi t), sin(2 pi t)) for t in [0, 1), reduced in quarter turns. */
TTR_HD void ttr_sincos_turns(double t, double* c, double* s) {
    const double pio2_hi = 1.57079632679489655800e+00, pio2_lo = 6.12323399573676603587e-17;
    const double q4 = TTR_MUL(4.0, t);          /* exact */
    const double q = (double)(int)TTR_ADD(q4, 0.5); /* nearest quadrant, q4 >= 0 */
    const double r = TTR_SUB(q4, q);            /* exact, |r| <= 1/2 */
    const double x = TTR_FMA(r, pio2_hi, TTR_MUL(r, pio2_lo));
    const double cx = ttr_kernel_cos(x), sx = ttr_kernel_sin(x);
    switch (((int)q) & 3) {
    case 0: *c = cx; *s = sx; break;
    case 1: *c = -sx; *s = cx; break;
    case 2: *c = -cx; *s = -sx; break;
    default: *c = sx; *s = -cx; break;
    }
}

/* Box-Muller pair for rows (2p, 2p+1) of column c of Omega_k. */
TTR_HD void ttr_philox_gauss_pair(uint64_t seed, uint32_t mode, uint32_t col, uint32_t pair,
                                  uint32_t tag, double* even, double* odd) {
    ttr_u32x4 ctr;
    ctr.v[0] = pair;
    ctr.v[1] = col;
    ctr.v[2] = mode;
    ctr.v[3] = tag;
    const ttr_u32x4 x = ttr_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t w1 = ((uint64_t)x.v[1] << 32) | x.v[0];
    const uint64_t w2 = ((uint64_t)x.v[3] << 32) | x.v[2];
    const double u1 = TTR_MUL((double)((w1 >> 11) + 1), 1.1102230246251565404e-16); /* 2^-53 */
    const double u2 = TTR_MUL((double)(w2 >> 11), 1.1102230246251565404e-16);
    const double rho = TTR_SQRT(TTR_MUL(-2.0, ttr_log_unit(u1)));
    double c, s;
    ttr_sincos_turns(u2, &c, &s);
    *even = TTR_MUL(rho, c);
    *odd = TTR_MUL(rho, s);
}

/* Single entry Omega_k(row, col) (mode is the 1-based TT mode index). */
TTR_HD double ttr_philox_omega(uint64_t seed, uint32_t mode, uint32_t col, uint32_t row) {
    double e, o;
    ttr_philox_gauss_pair(seed, mode, col, row >> 1, TTR_PHILOX_TAG_KRP, &e, &o);
    return (row & 1u) ? o : e;
}

#endif /* TTR_PHILOX_GAUSS_H */
