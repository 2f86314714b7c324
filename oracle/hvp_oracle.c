/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference algorithm.
 *
 * See hvp_oracle.h.  This file restates, in plain C, the parts of the reference
 * (/root/reference/proj, "hvp") that the B200 engine replaces.  It is the checker
 * for the CUDA path; it is never linked into, or called by, the product.
 * Compiled with -ffp-contract=off (oracle/Makefile) so the double-precision FFT
 * restated from fft.hpp/fft.cpp reproduces the reference built with the same flag
 * bit-for-bit (pinned by tests/test_oracle_pin.py).
 */
#include "hvp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg)
{
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------- */
/* Counters (counters.hpp:11-28, incremented at ops.cpp:610,653,683,718,916)  */

static _Atomic uint64_t g_cnt[5]; /* cmux, blindRotate, iks, pks, cb */

void orc_counters(uint64_t* out)
{
    for (int i = 0; i < 5; i++)
        out[i] = atomic_load(&g_cnt[i]);
}

void orc_counters_reset(void)
{
    for (int i = 0; i < 5; i++)
        atomic_store(&g_cnt[i], 0);
}

/* ------------------------------------------------------------------------- */
/* ChaCha20 CSPRNG (rng.cpp:16-191)                                           */

typedef struct {
    uint32_t state[16], block[16];
    int pos;
} rng_t;

static uint32_t rotl32(uint32_t x, int k) { return (x << k) | (x >> (32 - k)); }

#define QR(a, b, c, d)                \
    do {                              \
        a += b;                       \
        d = rotl32(d ^ a, 16);        \
        c += d;                       \
        b = rotl32(b ^ c, 12);        \
        a += b;                       \
        d = rotl32(d ^ a, 8);         \
        c += d;                       \
        b = rotl32(b ^ c, 7);         \
    } while (0)

static void chacha_block(const uint32_t* in, uint32_t* out) /* rng.cpp:28-44 */
{
    memcpy(out, in, 64);
    for (int r = 0; r < 10; r++) {
        QR(out[0], out[4], out[8], out[12]);
        QR(out[1], out[5], out[9], out[13]);
        QR(out[2], out[6], out[10], out[14]);
        QR(out[3], out[7], out[11], out[15]);
        QR(out[0], out[5], out[10], out[15]);
        QR(out[1], out[6], out[11], out[12]);
        QR(out[2], out[7], out[8], out[13]);
        QR(out[3], out[4], out[9], out[14]);
    }
    for (int i = 0; i < 16; i++)
        out[i] += in[i];
}

static uint64_t splitmix64(uint64_t* x) /* rng.cpp:46-53 */
{
    *x += 0x9e3779b97f4a7c15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static void rng_seed(rng_t* r, uint64_t seed) /* rng.cpp:57-70, 81-91 */
{
    uint32_t key[8];
    uint64_t s = seed;
    for (int i = 0; i < 4; i++) {
        uint64_t v = splitmix64(&s);
        key[2 * i] = (uint32_t)v;
        key[2 * i + 1] = (uint32_t)(v >> 32);
    }
    r->state[0] = 0x61707865;
    r->state[1] = 0x3320646e;
    r->state[2] = 0x79622d32;
    r->state[3] = 0x6b206574;
    for (int i = 0; i < 8; i++)
        r->state[4 + i] = key[i];
    r->state[12] = r->state[13] = r->state[14] = r->state[15] = 0;
    r->pos = 16;
}

static uint32_t rng_next(rng_t* r) /* rng.hpp:29-34, rng.cpp:93-99 */
{
    if (r->pos == 16) {
        chacha_block(r->state, r->block);
        r->pos = 0;
        if (++r->state[12] == 0)
            ++r->state[13];
    }
    return r->block[r->pos++];
}

static uint64_t rng_u64(rng_t* r) /* rng.hpp:36-41 */
{
    uint64_t lo = rng_next(r);
    uint64_t hi = rng_next(r);
    return lo | (hi << 32);
}

/* std::generate_canonical<double, 53>(Csprng) as implemented by libstdc++
 * (bits/random.tcc): two 32-bit draws, sum in double, divide by 2^64. */
static double gen_canonical(rng_t* r)
{
    double sum = 0.0, tmp = 1.0;
    for (int k = 0; k < 2; k++) {
        sum += (double)rng_next(r) * tmp;
        tmp *= 4294967296.0;
    }
    double ret = sum / tmp;
    if (ret >= 1.0)
        ret = nextafter(1.0, 0.0);
    return ret;
}

/* std::normal_distribution<double>(0, sigma)(rng) on a FRESH distribution object
 * (rng.cpp:209-223 constructs one per call): libstdc++'s Marsaglia polar method,
 * returning y * mult (the saved x * mult is discarded with the object). */
static double normal_sample(rng_t* r, double sigma)
{
    double x, y, r2;
    do {
        x = 2.0 * gen_canonical(r) - 1.0;
        y = 2.0 * gen_canonical(r) - 1.0;
        r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2 * log(r2) / r2);
    double ret = y * mult;
    return ret * sigma + 0.0;
}

static uint32_t double_to_torus32(double d) /* rng.cpp:101-105 */
{
    return (uint32_t)(int64_t)llround((d - floor(d)) * 4294967296.0);
}

static uint64_t double_to_torus64(double d) /* rng.cpp:107-115 */
{
    double frac = d - floor(d);
    double hi = floor(frac * 4294967296.0);
    double lo = (frac * 4294967296.0 - hi) * 4294967296.0;
    return ((uint64_t)hi << 32) + (uint64_t)(int64_t)llround(lo);
}

static uint32_t noise32(rng_t* r, double sigma) /* rng.cpp:117-123 */
{
    if (sigma == 0.0)
        return 0;
    return double_to_torus32(normal_sample(r, sigma));
}

static uint64_t noise64(rng_t* r, double sigma) /* rng.cpp:125-131 */
{
    if (sigma == 0.0)
        return 0;
    return double_to_torus64(normal_sample(r, sigma));
}

/* ------------------------------------------------------------------------- */
/* Parameter sets (params.cpp:31-86)                                          */

typedef struct {
    char name[16];
    uint32_t n;
    double alpha0;
    uint32_t N1, l1, Bg1Bits;
    double alpha1;
    uint32_t N2, l2, Bg2Bits;
    double alpha2;
    uint32_t ksBaseBits, ksLen, pksBaseBits, pksLen;
    double alphaPks;
    int fft;
} params_t;

static const uint32_t kMu32 = 1u << 29; /* params.hpp:12 */

static int params_by_name(const char* name, params_t* p)
{
    memset(p, 0, sizeof *p);
    if (strcmp(name, "tfhe-80") == 0) { /* params.cpp:31-56 */
        strcpy(p->name, "tfhe-80");
        p->n = 500;
        p->alpha0 = 2.44e-5;
        p->N1 = 1024;
        p->l1 = 2;
        p->Bg1Bits = 10;
        p->alpha1 = 3.73e-9;
        p->N2 = 2048;
        p->l2 = 4;
        p->Bg2Bits = 9;
        p->alpha2 = pow(2.0, -44);
        p->ksBaseBits = 2;
        p->ksLen = 8;
        p->pksBaseBits = 3;
        p->pksLen = 10;
        p->alphaPks = pow(2.0, -31);
        p->fft = 1;
        return 0;
    }
    if (strcmp(name, "test-det") == 0) { /* params.cpp:58-86 */
        strcpy(p->name, "test-det");
        p->n = 16;
        p->N1 = 64;
        p->l1 = 2;
        p->Bg1Bits = 16;
        p->N2 = 128;
        p->l2 = 4;
        p->Bg2Bits = 16;
        p->ksBaseBits = 4;
        p->ksLen = 8;
        p->pksBaseBits = 4;
        p->pksLen = 8;
        p->fft = 0;
        return 0;
    }
    return fail("unknown parameter set");
}

/* ------------------------------------------------------------------------- */
/* Negacyclic FFT (fft.hpp:15-97, fft.cpp:10-85)                              */

typedef struct {
    size_t N, M;
    double *twRe, *twIm, *twistRe, *twistIm;
} plan_t;

static void plan_init(plan_t* pl, size_t N) /* fft.cpp:10-31 */
{
    const double pi = 3.141592653589793; /* std::numbers::pi */
    pl->N = N;
    pl->M = N / 2;
    pl->twRe = malloc(sizeof(double) * pl->M / 2);
    pl->twIm = malloc(sizeof(double) * pl->M / 2);
    pl->twistRe = malloc(sizeof(double) * pl->M);
    pl->twistIm = malloc(sizeof(double) * pl->M);
    for (size_t j = 0; j < pl->M / 2; j++) {
        const double ang = -2.0 * pi * (double)j / (double)pl->M;
        pl->twRe[j] = cos(ang);
        pl->twIm[j] = sin(ang);
    }
    for (size_t j = 0; j < pl->M; j++) {
        const double ang = pi * (double)j / (double)N;
        pl->twistRe[j] = cos(ang);
        pl->twistIm[j] = sin(ang);
    }
}

static void plan_free(plan_t* pl)
{
    free(pl->twRe);
    free(pl->twIm);
    free(pl->twistRe);
    free(pl->twistIm);
}

static void fft_dif(const plan_t* pl, double* re, double* im) /* fft.cpp:33-55 */
{
    const size_t M = pl->M;
    for (size_t len = M >> 1; len > 0; len >>= 1) {
        const size_t stride = M / (len << 1);
        for (size_t base = 0; base < M; base += len << 1) {
            for (size_t k = 0; k < len; k++) {
                const double wr = pl->twRe[k * stride];
                const double wi = pl->twIm[k * stride];
                const size_t i0 = base + k, i1 = i0 + len;
                const double ur = re[i0], ui = im[i0];
                const double vr = re[i1], vi = im[i1];
                re[i0] = ur + vr;
                im[i0] = ui + vi;
                const double dr = ur - vr;
                const double di = ui - vi;
                re[i1] = dr * wr - di * wi;
                im[i1] = dr * wi + di * wr;
            }
        }
    }
}

static void ifft_dit(const plan_t* pl, double* re, double* im) /* fft.cpp:58-76 */
{
    const size_t M = pl->M;
    for (size_t len = 1; len < M; len <<= 1) {
        const size_t stride = M / (len << 1);
        for (size_t base = 0; base < M; base += len << 1) {
            for (size_t k = 0; k < len; k++) {
                const double wr = pl->twRe[k * stride];
                const double wi = -pl->twIm[k * stride];
                const size_t i0 = base + k, i1 = i0 + len;
                const double tr = re[i1] * wr - im[i1] * wi;
                const double ti = re[i1] * wi + im[i1] * wr;
                re[i1] = re[i0] - tr;
                im[i1] = im[i0] - ti;
                re[i0] += tr;
                im[i0] += ti;
            }
        }
    }
}

/* FftPlan::forward with the signed interpretation of the input (fft.hpp:64-75). */
static void fft_forward_i32(const plan_t* pl, double* re, double* im, const int32_t* p)
{
    for (size_t j = 0; j < pl->M; j++) {
        const double x = (double)p[j], y = (double)p[j + pl->M];
        re[j] = x * pl->twistRe[j] - y * pl->twistIm[j];
        im[j] = x * pl->twistIm[j] + y * pl->twistRe[j];
    }
    fft_dif(pl, re, im);
}

static void fft_forward_u32(const plan_t* pl, double* re, double* im, const uint32_t* p)
{
    for (size_t j = 0; j < pl->M; j++) {
        const double x = (double)(int32_t)p[j], y = (double)(int32_t)p[j + pl->M];
        re[j] = x * pl->twistRe[j] - y * pl->twistIm[j];
        im[j] = x * pl->twistIm[j] + y * pl->twistRe[j];
    }
    fft_dif(pl, re, im);
}

static void fft_forward_u64(const plan_t* pl, double* re, double* im, const uint64_t* p)
{
    for (size_t j = 0; j < pl->M; j++) {
        const double x = (double)(int64_t)p[j], y = (double)(int64_t)p[j + pl->M];
        re[j] = x * pl->twistRe[j] - y * pl->twistIm[j];
        im[j] = x * pl->twistIm[j] + y * pl->twistRe[j];
    }
    fft_dif(pl, re, im);
}

static uint32_t torus_from_double32(double x) /* fft.hpp:47-50 */
{
    return (uint32_t)(int64_t)llrint(x);
}

static uint64_t torus_from_double64(double x) /* fft.hpp:52-62 */
{
    const double kTwo64 = 18446744073709551616.0;
    const double kTwo63 = 9223372036854775808.0;
    x -= kTwo64 * nearbyint(x / kTwo64);
    if (x >= kTwo63)
        x -= kTwo64;
    if (x < -kTwo63)
        x += kTwo64;
    return (uint64_t)(int64_t)llrint(x);
}

/* FftPlan::inverseToTorus (fft.hpp:77-97) */
static void fft_inverse_u32(const plan_t* pl, uint32_t* out, double* re, double* im)
{
    ifft_dit(pl, re, im);
    const double scale = 1.0 / (double)pl->M;
    for (size_t j = 0; j < pl->M; j++) {
        const double x = re[j] * scale, y = im[j] * scale;
        const double cr = x * pl->twistRe[j] + y * pl->twistIm[j];
        const double ci = y * pl->twistRe[j] - x * pl->twistIm[j];
        out[j] = torus_from_double32(cr);
        out[j + pl->M] = torus_from_double32(ci);
    }
}

static void fft_inverse_u64(const plan_t* pl, uint64_t* out, double* re, double* im)
{
    ifft_dit(pl, re, im);
    const double scale = 1.0 / (double)pl->M;
    for (size_t j = 0; j < pl->M; j++) {
        const double x = re[j] * scale, y = im[j] * scale;
        const double cr = x * pl->twistRe[j] + y * pl->twistIm[j];
        const double ci = y * pl->twistRe[j] - x * pl->twistIm[j];
        out[j] = torus_from_double64(cr);
        out[j + pl->M] = torus_from_double64(ci);
    }
}

/* ------------------------------------------------------------------------- */
/* Polynomial arithmetic (poly.hpp)                                           */

/* polyMulAccExact (poly.hpp:15-29) */
static void poly_mul_acc_exact32(uint32_t* acc, const int32_t* digits, const uint32_t* poly,
                                 size_t N)
{
    for (size_t i = 0; i < N; i++) {
        const uint32_t d = (uint32_t)digits[i];
        if (d == 0)
            continue;
        size_t j = 0;
        for (; j < N - i; j++)
            acc[i + j] += d * poly[j];
        for (; j < N; j++)
            acc[i + j - N] -= d * poly[j];
    }
}

/* Full product out[0..2n) = a * b over Z/2^64 by Karatsuba (ring arithmetic only, so it
 * equals the schoolbook sum word for word).  scratch: 4n words. */
static void kara64(const uint64_t* a, const uint64_t* b, size_t n, uint64_t* out,
                   uint64_t* scratch)
{
    if (n <= 32) {
        memset(out, 0, 8 * 2 * n);
        for (size_t i = 0; i < n; i++) {
            const uint64_t x = a[i];
            if (x == 0)
                continue;
            for (size_t j = 0; j < n; j++)
                out[i + j] += x * b[j];
        }
        return;
    }
    const size_t h = n / 2;
    uint64_t *sa = scratch, *sb = scratch + h, *z1 = scratch + 2 * h, *rest = scratch + 4 * h;
    kara64(a, b, h, out, rest);              /* z0 -> out[0, n) */
    kara64(a + h, b + h, h, out + n, rest);  /* z2 -> out[n, 2n) */
    for (size_t i = 0; i < h; i++) {
        sa[i] = a[i] + a[h + i];
        sb[i] = b[i] + b[h + i];
    }
    kara64(sa, sb, h, z1, rest);             /* (a0 + a1)(b0 + b1) */
    for (size_t i = 0; i < n; i++)
        z1[i] -= out[i] + out[n + i];
    for (size_t i = 0; i < n; i++)
        out[h + i] += z1[i];
}

/* polyMulAccExact (poly.hpp:15-29) at 64 bits: acc += digits * poly mod (X^N + 1).  Large N
 * goes through Karatsuba + the negacyclic fold -- the same exact integers mod 2^64 as the
 * schoolbook loop, fast enough for full-size level-2 blind rotations in the tests. */
static void poly_mul_acc_exact64(uint64_t* acc, const int32_t* digits, const uint64_t* poly,
                                 size_t N)
{
    if (N >= 256 && (N & (N - 1)) == 0) {
        uint64_t* buf = malloc(8 * (N + 2 * N + 8 * N));
        uint64_t *a = buf, *prod = buf + N, *scratch = buf + 3 * N;
        for (size_t i = 0; i < N; i++)
            a[i] = (uint64_t)(int64_t)digits[i];
        kara64(a, poly, N, prod, scratch);
        for (size_t i = 0; i < N; i++)
            acc[i] += prod[i] - prod[N + i];
        free(buf);
        return;
    }
    for (size_t i = 0; i < N; i++) {
        const uint64_t d = (uint64_t)(int64_t)digits[i];
        if (d == 0)
            continue;
        size_t j = 0;
        for (; j < N - i; j++)
            acc[i + j] += d * poly[j];
        for (; j < N; j++)
            acc[i + j - N] -= d * poly[j];
    }
}

/* polyRotate (poly.hpp:32-48) */
static void poly_rotate32(uint32_t* out, const uint32_t* p, size_t N, uint32_t k)
{
    if (k < N) {
        for (size_t i = 0; i < k; i++)
            out[i] = 0u - p[i + N - k];
        for (size_t i = k; i < N; i++)
            out[i] = p[i - k];
    }
    else {
        const uint32_t kk = k - (uint32_t)N;
        for (size_t i = 0; i < kk; i++)
            out[i] = p[i + N - kk];
        for (size_t i = kk; i < N; i++)
            out[i] = 0u - p[i - kk];
    }
}

static void poly_rotate64(uint64_t* out, const uint64_t* p, size_t N, uint32_t k)
{
    if (k < N) {
        for (size_t i = 0; i < k; i++)
            out[i] = 0ull - p[i + N - k];
        for (size_t i = k; i < N; i++)
            out[i] = p[i - k];
    }
    else {
        const uint32_t kk = k - (uint32_t)N;
        for (size_t i = 0; i < kk; i++)
            out[i] = p[i + N - kk];
        for (size_t i = kk; i < N; i++)
            out[i] = 0ull - p[i - kk];
    }
}

/* polyMulBinary (poly.hpp:61-75) */
static void poly_mul_binary32(uint32_t* out, const uint32_t* torus, const uint32_t* bits,
                              size_t N)
{
    memset(out, 0, N * sizeof *out);
    for (size_t i = 0; i < N; i++) {
        if (!bits[i])
            continue;
        size_t j = 0;
        for (; j < N - i; j++)
            out[i + j] += torus[j];
        for (; j < N; j++)
            out[i + j - N] -= torus[j];
    }
}

static void poly_mul_binary64(uint64_t* out, const uint64_t* torus, const uint32_t* bits,
                              size_t N)
{
    memset(out, 0, N * sizeof *out);
    for (size_t i = 0; i < N; i++) {
        if (!bits[i])
            continue;
        size_t j = 0;
        for (; j < N - i; j++)
            out[i + j] += torus[j];
        for (; j < N; j++)
            out[i + j - N] -= torus[j];
    }
}

/* decomposePoly (poly.hpp:79-97): signed digits, NO final rounding bit. */
static void decompose32(int32_t* out, const uint32_t* p, size_t N, uint32_t l,
                        uint32_t bgBits)
{
    const uint32_t halfBg = 1u << (bgBits - 1);
    const uint32_t mask = (bgBits == 32) ? 0xffffffffu : ((1u << bgBits) - 1);
    uint32_t offset = 0;
    for (uint32_t i = 1; i <= l; i++)
        offset += halfBg << (32 - i * bgBits);
    for (size_t j = 0; j < N; j++) {
        const uint32_t v = p[j] + offset;
        for (uint32_t i = 0; i < l; i++) {
            const uint32_t digit = ((v >> (32 - (i + 1) * bgBits)) & mask) - halfBg;
            out[i * N + j] = (int32_t)digit;
        }
    }
}

static void decompose64(int32_t* out, const uint64_t* p, size_t N, uint32_t l,
                        uint32_t bgBits)
{
    const uint64_t halfBg = 1ull << (bgBits - 1);
    const uint64_t mask = (1ull << bgBits) - 1;
    uint64_t offset = 0;
    for (uint32_t i = 1; i <= l; i++)
        offset += halfBg << (64 - i * bgBits);
    for (size_t j = 0; j < N; j++) {
        const uint64_t v = p[j] + offset;
        for (uint32_t i = 0; i < l; i++) {
            const uint64_t digit = ((v >> (64 - (i + 1) * bgBits)) & mask) - halfBg;
            out[i * N + j] = (int32_t)(int64_t)digit;
        }
    }
}

/* modSwitch (ops.cpp:49-55) */
static uint32_t mod_switch(uint32_t m, uint32_t phase)
{
    const uint64_t interval = ((1ull << 63) / m) * 2;
    const uint64_t half = interval / 2;
    return (uint32_t)((((uint64_t)phase << 32) + half) / interval);
}

/* ------------------------------------------------------------------------- */
/* Context: parameters + keys                                                 */

struct orc_ctx {
    params_t p;
    rng_t rng;
    uint32_t *lv0, *lv1, *lv2;
    int has_bk, has_cb, exact;
    uint32_t* bk1;   /* n x 2l1 x 2 x N1 */
    uint64_t* bk2;   /* n x 2l2 x 2 x N2 */
    double* bk1fd;   /* prepared (ops.cpp:520-546): n x [2l1 rows x 2 polys x (re M, im M)] */
    double* bk2fd;
    uint32_t* ksk;   /* N1 x t x (2^b-1) x (n+1) (ops.hpp:18-29) */
    uint32_t *pksNegS, *pksId; /* (N2+1) x t x (2^b-1) x 2N1 (ops.hpp:32-42) */
    plan_t plan1, plan2;
};

static size_t ksk_words_p(const params_t* p)
{
    return (size_t)p->N1 * p->ksLen * (((size_t)1 << p->ksBaseBits) - 1) * (p->n + 1);
}

static size_t pks_words_p(const params_t* p)
{
    return ((size_t)p->N2 + 1) * p->pksLen * (((size_t)1 << p->pksBaseBits) - 1) * 2 *
           p->N1;
}

orc_ctx* orc_ctx_new(const char* name, uint32_t n_override, uint64_t seed)
{
    orc_ctx* c = calloc(1, sizeof *c);
    if (params_by_name(name, &c->p) != 0) {
        free(c);
        return NULL;
    }
    if (n_override)
        c->p.n = n_override;
    rng_seed(&c->rng, seed);
    /* genSecretKey (ops.cpp:264-279) */
    c->lv0 = malloc(4 * c->p.n);
    c->lv1 = malloc(4 * c->p.N1);
    c->lv2 = malloc(4 * c->p.N2);
    for (uint32_t i = 0; i < c->p.n; i++)
        c->lv0[i] = rng_next(&c->rng) & 1;
    for (uint32_t i = 0; i < c->p.N1; i++)
        c->lv1[i] = rng_next(&c->rng) & 1;
    for (uint32_t i = 0; i < c->p.N2; i++)
        c->lv2[i] = rng_next(&c->rng) & 1;
    plan_init(&c->plan1, c->p.N1);
    plan_init(&c->plan2, c->p.N2);
    return c;
}

static void free_keys(orc_ctx* c)
{
    free(c->bk1);
    free(c->bk2);
    free(c->bk1fd);
    free(c->bk2fd);
    free(c->ksk);
    free(c->pksNegS);
    free(c->pksId);
    c->bk1 = NULL;
    c->bk2 = NULL;
    c->bk1fd = c->bk2fd = NULL;
    c->ksk = c->pksNegS = c->pksId = NULL;
    c->has_bk = c->has_cb = 0;
}

void orc_ctx_free(orc_ctx* c)
{
    if (!c)
        return;
    free_keys(c);
    free(c->lv0);
    free(c->lv1);
    free(c->lv2);
    plan_free(&c->plan1);
    plan_free(&c->plan2);
    free(c);
}

void orc_set_exact(orc_ctx* c, int exact) { c->exact = exact; }

void orc_params(const orc_ctx* c, uint32_t* o)
{
    const params_t* p = &c->p;
    uint32_t v[14] = {p->n,          p->N1,     p->l1,    p->Bg1Bits, p->N2,
                      p->l2,         p->Bg2Bits, p->ksBaseBits, p->ksLen,
                      p->pksBaseBits, p->pksLen, (uint32_t)p->fft,
                      (uint32_t)c->has_bk, (uint32_t)c->has_cb};
    memcpy(o, v, sizeof v);
}

/* trlweEncryptZero (ops.cpp:161-180) at level 1 / level 2 */
static void trlwe_encrypt_zero32(orc_ctx* c, uint32_t* out, double alpha)
{
    const uint32_t N = c->p.N1;
    uint32_t* a = out;
    uint32_t* b = out + N;
    for (uint32_t i = 0; i < N; i++)
        a[i] = rng_next(&c->rng);
    poly_mul_binary32(b, a, c->lv1, N);
    if (alpha != 0.0)
        for (uint32_t i = 0; i < N; i++)
            b[i] += noise32(&c->rng, alpha);
}

static void trlwe_encrypt_zero64(orc_ctx* c, uint64_t* out, double alpha)
{
    const uint32_t N = c->p.N2;
    uint64_t* a = out;
    uint64_t* b = out + N;
    for (uint32_t i = 0; i < N; i++)
        a[i] = rng_u64(&c->rng);
    poly_mul_binary64(b, a, c->lv2, N);
    if (alpha != 0.0)
        for (uint32_t i = 0; i < N; i++)
            b[i] += noise64(&c->rng, alpha);
}

/* trgswEncryptAtLevel (ops.cpp:182-205) */
static void trgsw_encrypt32(orc_ctx* c, int m, uint32_t* out)
{
    const uint32_t N = c->p.N1, l = c->p.l1;
    for (uint32_t r = 0; r < 2 * l; r++)
        trlwe_encrypt_zero32(c, out + (size_t)r * 2 * N, c->p.alpha1);
    if (m)
        for (uint32_t i = 0; i < l; i++) {
            const uint32_t h = 1u << (32 - (i + 1) * c->p.Bg1Bits);
            out[(size_t)i * 2 * N] += h;
            out[(size_t)(l + i) * 2 * N + N] += h;
        }
}

static void trgsw_encrypt64(orc_ctx* c, int m, uint64_t* out)
{
    const uint32_t N = c->p.N2, l = c->p.l2;
    for (uint32_t r = 0; r < 2 * l; r++)
        trlwe_encrypt_zero64(c, out + (size_t)r * 2 * N, c->p.alpha2);
    if (m)
        for (uint32_t i = 0; i < l; i++) {
            const uint64_t h = 1ull << (64 - (i + 1) * c->p.Bg2Bits);
            out[(size_t)i * 2 * N] += h;
            out[(size_t)(l + i) * 2 * N + N] += h;
        }
}

/* prepareTrgsw, FFT branch (ops.cpp:520-546) */
static void prepare32(orc_ctx* c, const uint32_t* g, double* fd)
{
    const uint32_t N = c->p.N1, M = N / 2;
    for (uint32_t r = 0; r < 2 * c->p.l1; r++)
        for (int poly = 0; poly < 2; poly++) {
            double* o = fd + ((size_t)r * 2 + poly) * N;
            fft_forward_u32(&c->plan1, o, o + M, g + (size_t)r * 2 * N + (size_t)poly * N);
        }
}

static void prepare64(orc_ctx* c, const uint64_t* g, double* fd)
{
    const uint32_t N = c->p.N2, M = N / 2;
    for (uint32_t r = 0; r < 2 * c->p.l2; r++)
        for (int poly = 0; poly < 2; poly++) {
            double* o = fd + ((size_t)r * 2 + poly) * N;
            fft_forward_u64(&c->plan2, o, o + M, g + (size_t)r * 2 * N + (size_t)poly * N);
        }
}

static void prepare_all(orc_ctx* c) /* ops.cpp:404-415 */
{
    const params_t* p = &c->p;
    if (p->fft) {
        const size_t per1 = (size_t)2 * p->l1 * 2 * p->N1;
        c->bk1fd = malloc(sizeof(double) * p->n * per1);
        for (uint32_t i = 0; i < p->n; i++)
            prepare32(c, c->bk1 + i * per1, c->bk1fd + i * per1);
        if (c->has_cb) {
            const size_t per2 = (size_t)2 * p->l2 * 2 * p->N2;
            c->bk2fd = malloc(sizeof(double) * p->n * per2);
            for (uint32_t i = 0; i < p->n; i++)
                prepare64(c, c->bk2 + i * per2, c->bk2fd + i * per2);
        }
    }
}

/* genKeySwitchKey (ops.cpp:283-313) */
static void gen_ksk(orc_ctx* c)
{
    const params_t* p = &c->p;
    const uint32_t perBase = (1u << p->ksBaseBits) - 1;
    c->ksk = malloc(4 * ksk_words_p(p));
    size_t pos = 0;
    for (uint32_t i = 0; i < p->N1; i++)
        for (uint32_t j = 0; j < p->ksLen; j++)
            for (uint32_t u = 0; u < perBase; u++) {
                const uint32_t msg = (c->lv1[i] * (u + 1)) << (32 - (j + 1) * p->ksBaseBits);
                uint32_t b = msg + noise32(&c->rng, p->alpha0);
                for (uint32_t k = 0; k < p->n; k++) {
                    const uint32_t a = rng_next(&c->rng);
                    c->ksk[pos + k] = a;
                    b += a * c->lv0[k];
                }
                c->ksk[pos + p->n] = b;
                pos += p->n + 1;
            }
}

/* genPrivKeySwitchKey (ops.cpp:315-351); func given as int64 per coefficient */
static uint32_t* gen_pks(orc_ctx* c, const int64_t* func)
{
    const params_t* p = &c->p;
    const uint32_t perBase = (1u << p->pksBaseBits) - 1;
    uint32_t* d = malloc(4 * pks_words_p(p));
    uint32_t* row = malloc(4 * 2 * p->N1);
    size_t pos = 0;
    for (uint32_t i = 0; i <= p->N2; i++) {
        const uint32_t factor = i < p->N2 ? c->lv2[i] : (uint32_t)-1;
        for (uint32_t j = 0; j < p->pksLen; j++)
            for (uint32_t u = 0; u < perBase; u++) {
                trlwe_encrypt_zero32(c, row, p->alphaPks);
                const uint32_t scale = ((u + 1) * factor) << (32 - (j + 1) * p->pksBaseBits);
                for (uint32_t k = 0; k < p->N1; k++)
                    row[p->N1 + k] += (uint32_t)func[k] * scale;
                memcpy(d + pos, row, 4 * 2 * p->N1);
                pos += 2 * (size_t)p->N1;
            }
    }
    free(row);
    return d;
}

/* BootstrappingKey::generate (ops.cpp:355-385) */
int orc_keygen(orc_ctx* c, int with_cb)
{
    const params_t* p = &c->p;
    free_keys(c);
    c->has_cb = with_cb;
    const size_t per1 = (size_t)2 * p->l1 * 2 * p->N1;
    c->bk1 = malloc(4 * p->n * per1);
    for (uint32_t i = 0; i < p->n; i++)
        trgsw_encrypt32(c, (int)c->lv0[i], c->bk1 + i * per1);
    if (with_cb) {
        const size_t per2 = (size_t)2 * p->l2 * 2 * p->N2;
        c->bk2 = malloc(8 * p->n * per2);
        for (uint32_t i = 0; i < p->n; i++)
            trgsw_encrypt64(c, (int)c->lv0[i], c->bk2 + i * per2);
    }
    gen_ksk(c);
    if (with_cb) {
        int64_t* negS = calloc(p->N1, sizeof(int64_t));
        int64_t* id = calloc(p->N1, sizeof(int64_t));
        for (uint32_t i = 0; i < p->N1; i++)
            negS[i] = -(int64_t)c->lv1[i];
        id[0] = 1;
        c->pksNegS = gen_pks(c, negS);
        c->pksId = gen_pks(c, id);
        free(negS);
        free(id);
    }
    c->has_bk = 1;
    prepare_all(c);
    return 0;
}

int orc_import_keys(orc_ctx* c, const uint32_t* lv0, const uint32_t* lv1,
                    const uint32_t* lv2, const uint32_t* bk1, const uint64_t* bk2,
                    const uint32_t* ksk, const uint32_t* pks_negs, const uint32_t* pks_id,
                    int has_cb)
{
    const params_t* p = &c->p;
    free_keys(c);
    if (lv0)
        memcpy(c->lv0, lv0, 4 * p->n);
    if (lv1)
        memcpy(c->lv1, lv1, 4 * p->N1);
    if (lv2)
        memcpy(c->lv2, lv2, 4 * p->N2);
    const size_t per1 = (size_t)2 * p->l1 * 2 * p->N1;
    c->bk1 = malloc(4 * p->n * per1);
    memcpy(c->bk1, bk1, 4 * p->n * per1);
    c->ksk = malloc(4 * ksk_words_p(p));
    memcpy(c->ksk, ksk, 4 * ksk_words_p(p));
    c->has_cb = has_cb;
    if (has_cb) {
        const size_t per2 = (size_t)2 * p->l2 * 2 * p->N2;
        c->bk2 = malloc(8 * p->n * per2);
        memcpy(c->bk2, bk2, 8 * p->n * per2);
        if (pks_negs && pks_id) {
            c->pksNegS = malloc(4 * pks_words_p(p));
            c->pksId = malloc(4 * pks_words_p(p));
            memcpy(c->pksNegS, pks_negs, 4 * pks_words_p(p));
            memcpy(c->pksId, pks_id, 4 * pks_words_p(p));
        }
    }
    c->has_bk = 1;
    prepare_all(c);
    return 0;
}

int orc_export_sk(const orc_ctx* c, uint32_t* lv0, uint32_t* lv1, uint32_t* lv2)
{
    memcpy(lv0, c->lv0, 4 * c->p.n);
    memcpy(lv1, c->lv1, 4 * c->p.N1);
    memcpy(lv2, c->lv2, 4 * c->p.N2);
    return 0;
}

int orc_export_bk1(const orc_ctx* c, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    memcpy(out, c->bk1, 4 * (size_t)c->p.n * 2 * c->p.l1 * 2 * c->p.N1);
    return 0;
}

int orc_export_bk2(const orc_ctx* c, uint64_t* out)
{
    if (!c->has_cb)
        return fail("no circuit-bootstrapping material");
    memcpy(out, c->bk2, 8 * (size_t)c->p.n * 2 * c->p.l2 * 2 * c->p.N2);
    return 0;
}

size_t orc_ksk_words(const orc_ctx* c) { return ksk_words_p(&c->p); }

int orc_export_ksk(const orc_ctx* c, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    memcpy(out, c->ksk, 4 * ksk_words_p(&c->p));
    return 0;
}

size_t orc_pks_words(const orc_ctx* c) { return c->has_cb ? pks_words_p(&c->p) : 0; }

int orc_export_pks(const orc_ctx* c, int which, uint32_t* out)
{
    if (!c->has_cb)
        return fail("no circuit-bootstrapping material");
    memcpy(out, which == 0 ? c->pksNegS : c->pksId, 4 * pks_words_p(&c->p));
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Encryption / decryption (ops.cpp:428-515)                                  */

int orc_tlwe_encrypt(orc_ctx* c, int m, uint32_t* out) /* ops.cpp:428-440 */
{
    const uint32_t n = c->p.n;
    uint32_t b = (m ? kMu32 : 0u - kMu32) + noise32(&c->rng, c->p.alpha0);
    for (uint32_t i = 0; i < n; i++) {
        out[i] = rng_next(&c->rng);
        b += out[i] * c->lv0[i];
    }
    out[n] = b;
    return 0;
}

uint32_t orc_tlwe_phase(const orc_ctx* c, const uint32_t* ct, int level) /* 442-450 */
{
    const uint32_t dim = level == 0 ? c->p.n : c->p.N1;
    const uint32_t* key = level == 0 ? c->lv0 : c->lv1;
    uint32_t phase = ct[dim];
    for (uint32_t i = 0; i < dim; i++)
        phase -= ct[i] * key[i];
    return phase;
}

int orc_trlwe_encrypt(orc_ctx* c, const uint32_t* bits, double alpha, uint32_t* out)
{
    /* trlweEncrypt (ops.cpp:458-468) */
    trlwe_encrypt_zero32(c, out, alpha);
    for (uint32_t i = 0; i < c->p.N1; i++)
        out[c->p.N1 + i] += bits[i] ? kMu32 : 0u - kMu32;
    return 0;
}

uint32_t orc_trlwe_phase_at(const orc_ctx* c, const uint32_t* ct, uint32_t k)
{
    /* trlwePhaseAt (ops.cpp:494-505) */
    const uint32_t N = c->p.N1;
    uint32_t acc = 0;
    for (uint32_t j = 0; j <= k; j++)
        acc += ct[k - j] * c->lv1[j];
    for (uint32_t j = k + 1; j < N; j++)
        acc -= ct[k + N - j] * c->lv1[j];
    return ct[N + k] - acc;
}

int orc_trgsw_encrypt(orc_ctx* c, int m, double alpha, uint32_t* out)
{
    (void)alpha; /* trgswEncryptAtLevel uses alpha1 (ops.cpp:195-196) */
    trgsw_encrypt32(c, m, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* External product and CMUX (ops.cpp:553-626)                                */

/* g: raw TRGSW rows (exact) and/or prepared fd (fft) */
static void ext_prod32(const orc_ctx* c, const uint32_t* in, const uint32_t* graw,
                       const double* gfd, uint32_t* out)
{
    const uint32_t N = c->p.N1, l = c->p.l1, M = N / 2;
    int32_t* digits = malloc(sizeof(int32_t) * 2 * l * N);
    decompose32(digits, in, N, l, c->p.Bg1Bits);
    decompose32(digits + (size_t)l * N, in + N, N, l, c->p.Bg1Bits);
    memset(out, 0, 4 * 2 * N);
    if (!c->p.fft || c->exact || !gfd) {
        for (uint32_t r = 0; r < 2 * l; r++) {
            const int32_t* d = digits + (size_t)r * N;
            poly_mul_acc_exact32(out, d, graw + (size_t)r * 2 * N, N);
            poly_mul_acc_exact32(out + N, d, graw + (size_t)r * 2 * N + N, N);
        }
    }
    else {
        double* buf = calloc(6 * (size_t)M, sizeof(double));
        double *re = buf, *im = buf + M, *aR = buf + 2 * M, *aI = buf + 3 * M,
               *bR = buf + 4 * M, *bI = buf + 5 * M;
        for (uint32_t r = 0; r < 2 * l; r++) {
            fft_forward_i32(&c->plan1, re, im, digits + (size_t)r * N);
            const double* ga = gfd + ((size_t)r * 2 + 0) * N;
            const double* gb = gfd + ((size_t)r * 2 + 1) * N;
            for (uint32_t k = 0; k < M; k++) {
                const double xr = re[k], xi = im[k];
                aR[k] += xr * ga[k] - xi * ga[M + k];
                aI[k] += xr * ga[M + k] + xi * ga[k];
                bR[k] += xr * gb[k] - xi * gb[M + k];
                bI[k] += xr * gb[M + k] + xi * gb[k];
            }
        }
        fft_inverse_u32(&c->plan1, out, aR, aI);
        fft_inverse_u32(&c->plan1, out + N, bR, bI);
        free(buf);
    }
    free(digits);
}

static void ext_prod64(const orc_ctx* c, const uint64_t* in, const uint64_t* graw,
                       const double* gfd, uint64_t* out)
{
    const uint32_t N = c->p.N2, l = c->p.l2, M = N / 2;
    int32_t* digits = malloc(sizeof(int32_t) * 2 * l * N);
    decompose64(digits, in, N, l, c->p.Bg2Bits);
    decompose64(digits + (size_t)l * N, in + N, N, l, c->p.Bg2Bits);
    memset(out, 0, 8 * 2 * N);
    if (!c->p.fft || c->exact || !gfd) {
        for (uint32_t r = 0; r < 2 * l; r++) {
            const int32_t* d = digits + (size_t)r * N;
            poly_mul_acc_exact64(out, d, graw + (size_t)r * 2 * N, N);
            poly_mul_acc_exact64(out + N, d, graw + (size_t)r * 2 * N + N, N);
        }
    }
    else {
        double* buf = calloc(6 * (size_t)M, sizeof(double));
        double *re = buf, *im = buf + M, *aR = buf + 2 * M, *aI = buf + 3 * M,
               *bR = buf + 4 * M, *bI = buf + 5 * M;
        for (uint32_t r = 0; r < 2 * l; r++) {
            fft_forward_i32(&c->plan2, re, im, digits + (size_t)r * N);
            const double* ga = gfd + ((size_t)r * 2 + 0) * N;
            const double* gb = gfd + ((size_t)r * 2 + 1) * N;
            for (uint32_t k = 0; k < M; k++) {
                const double xr = re[k], xi = im[k];
                aR[k] += xr * ga[k] - xi * ga[M + k];
                aI[k] += xr * ga[M + k] + xi * ga[k];
                bR[k] += xr * gb[k] - xi * gb[M + k];
                bI[k] += xr * gb[M + k] + xi * gb[k];
            }
        }
        fft_inverse_u64(&c->plan2, out, aR, aI);
        fft_inverse_u64(&c->plan2, out + N, bR, bI);
        free(buf);
    }
    free(digits);
}

int orc_external_product(orc_ctx* c, const uint32_t* trgsw, const uint32_t* trlwe,
                         uint32_t* out)
{
    double* fd = NULL;
    if (c->p.fft && !c->exact) {
        fd = malloc(sizeof(double) * 2 * c->p.l1 * 2 * c->p.N1);
        prepare32(c, trgsw, fd);
    }
    ext_prod32(c, trlwe, trgsw, fd, out);
    free(fd);
    return 0;
}

int orc_external_product_lvl2(orc_ctx* c, const uint64_t* trgsw, const uint64_t* trlwe,
                              uint64_t* out)
{
    double* fd = NULL;
    if (c->p.fft && !c->exact) {
        fd = malloc(sizeof(double) * 2 * c->p.l2 * 2 * c->p.N2);
        prepare64(c, trgsw, fd);
    }
    ext_prod64(c, trlwe, trgsw, fd, out);
    free(fd);
    return 0;
}

/* cmux (ops.cpp:606-614): c0 + ExtProd(c1 - c0, sel) */
static void cmux32(const orc_ctx* c, const uint32_t* selraw, const double* selfd,
                   const uint32_t* c1, const uint32_t* c0, uint32_t* out)
{
    const uint32_t N2x = 2 * c->p.N1;
    uint32_t* diff = malloc(4 * N2x);
    atomic_fetch_add(&g_cnt[0], 1);
    for (uint32_t i = 0; i < N2x; i++)
        diff[i] = c1[i] - c0[i];
    ext_prod32(c, diff, selraw, selfd, out);
    for (uint32_t i = 0; i < N2x; i++)
        out[i] += c0[i];
    free(diff);
}

int orc_cmux(orc_ctx* c, const uint32_t* sel, const uint32_t* c1, const uint32_t* c0,
             uint32_t* out)
{
    double* fd = NULL;
    if (c->p.fft && !c->exact) {
        fd = malloc(sizeof(double) * 2 * c->p.l1 * 2 * c->p.N1);
        prepare32(c, sel, fd);
    }
    cmux32(c, sel, fd, c1, c0, out);
    free(fd);
    return 0;
}

/* sampleExtract (ops.cpp:628-643) */
static void sample_extract32(const uint32_t* ct, size_t N, size_t k, uint32_t* out)
{
    for (size_t i = 0; i <= k; i++)
        out[i] = ct[k - i];
    for (size_t i = k + 1; i < N; i++)
        out[i] = 0u - ct[N + k - i];
    out[N] = ct[N + k];
}

static void sample_extract64(const uint64_t* ct, size_t N, size_t k, uint64_t* out)
{
    for (size_t i = 0; i <= k; i++)
        out[i] = ct[k - i];
    for (size_t i = k + 1; i < N; i++)
        out[i] = 0ull - ct[N + k - i];
    out[N] = ct[N + k];
}

int orc_sample_extract(orc_ctx* c, const uint32_t* trlwe, uint32_t k, uint32_t* out)
{
    if (k >= c->p.N1)
        return fail("sampleExtract: index out of range");
    sample_extract32(trlwe, c->p.N1, k, out);
    return 0;
}

/* identityKeySwitch (ops.cpp:651-679) */
static void iks(const orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    const params_t* p = &c->p;
    const uint32_t baseBits = p->ksBaseBits, t = p->ksLen, n = p->n;
    const uint32_t mask = (1u << baseBits) - 1;
    const uint32_t offset = baseBits * t >= 32 ? 0 : 1u << (32 - (1 + baseBits * t));
    const size_t perBase = ((size_t)1 << baseBits) - 1;
    atomic_fetch_add(&g_cnt[2], 1);
    memset(out, 0, 4 * n);
    out[n] = in[p->N1];
    for (uint32_t i = 0; i < p->N1; i++) {
        const uint32_t v = in[i] + offset;
        for (uint32_t j = 0; j < t; j++) {
            const uint32_t d = (v >> (32 - (j + 1) * baseBits)) & mask;
            if (d == 0)
                continue;
            const uint32_t* row = c->ksk + (((size_t)i * t + j) * perBase + d - 1) * (n + 1);
            for (uint32_t k = 0; k < n; k++)
                out[k] -= row[k];
            out[n] -= row[n];
        }
    }
}

int orc_identity_key_switch(orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    iks(c, in, out);
    return 0;
}

/* privateKeySwitch (ops.cpp:681-708) */
static void pks(const orc_ctx* c, const uint64_t* in, const uint32_t* table, uint32_t* out)
{
    const params_t* p = &c->p;
    const uint32_t baseBits = p->pksBaseBits, t = p->pksLen, N1 = p->N1;
    const uint64_t mask = (1ull << baseBits) - 1;
    const uint64_t offset = baseBits * t >= 64 ? 0 : 1ull << (64 - (1 + baseBits * t));
    const size_t perBase = ((size_t)1 << baseBits) - 1;
    atomic_fetch_add(&g_cnt[3], 1);
    memset(out, 0, 4 * 2 * N1);
    for (uint32_t i = 0; i <= p->N2; i++) {
        const uint64_t v = (i < p->N2 ? in[i] : in[p->N2]) + offset;
        for (uint32_t j = 0; j < t; j++) {
            const uint64_t d = (v >> (64 - (j + 1) * baseBits)) & mask;
            if (d == 0)
                continue;
            const uint32_t* row =
                table + (((size_t)i * t + j) * perBase + (uint32_t)(d - 1)) * 2 * N1;
            for (uint32_t k = 0; k < N1; k++)
                out[k] -= row[k];
            for (uint32_t k = 0; k < N1; k++)
                out[N1 + k] -= row[N1 + k];
        }
    }
}

int orc_private_key_switch(orc_ctx* c, const uint64_t* in, int which, uint32_t* out)
{
    if (!c->has_cb)
        return fail("no circuit-bootstrapping material");
    pks(c, in, which == 0 ? c->pksNegS : c->pksId, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Blind rotation and bootstrapping (ops.cpp:713-762)                         */

static void blind_rotate32(const orc_ctx* c, const uint32_t* ct, const uint32_t* tv,
                           uint32_t* acc)
{
    const params_t* p = &c->p;
    const uint32_t N = p->N1, twoN = 2 * N;
    const size_t per = (size_t)2 * p->l1 * 2 * N;
    uint32_t* diff = malloc(4 * 2 * N);
    uint32_t* ep = malloc(4 * 2 * N);
    atomic_fetch_add(&g_cnt[1], 1);
    const uint32_t rot = (twoN - mod_switch(twoN, ct[p->n])) % twoN;
    poly_rotate32(acc, tv, N, rot);
    poly_rotate32(acc + N, tv + N, N, rot);
    for (uint32_t i = 0; i < p->n; i++) {
        const uint32_t bara = mod_switch(twoN, ct[i]);
        if (bara == 0)
            continue;
        /* polyMulByXkMinusOne (poly.hpp:51-57) */
        poly_rotate32(diff, acc, N, bara);
        poly_rotate32(diff + N, acc + N, N, bara);
        for (uint32_t j = 0; j < 2 * N; j++)
            diff[j] -= acc[j];
        ext_prod32(c, diff, c->bk1 + i * per, c->bk1fd ? c->bk1fd + i * per : NULL, ep);
        for (uint32_t j = 0; j < 2 * N; j++)
            acc[j] += ep[j];
    }
    free(diff);
    free(ep);
}

static void blind_rotate64(const orc_ctx* c, const uint32_t* ct, const uint64_t* tv,
                           uint64_t* acc)
{
    const params_t* p = &c->p;
    const uint32_t N = p->N2, twoN = 2 * N;
    const size_t per = (size_t)2 * p->l2 * 2 * N;
    uint64_t* diff = malloc(8 * 2 * N);
    uint64_t* ep = malloc(8 * 2 * N);
    atomic_fetch_add(&g_cnt[1], 1);
    const uint32_t rot = (twoN - mod_switch(twoN, ct[p->n])) % twoN;
    poly_rotate64(acc, tv, N, rot);
    poly_rotate64(acc + N, tv + N, N, rot);
    for (uint32_t i = 0; i < p->n; i++) {
        const uint32_t bara = mod_switch(twoN, ct[i]);
        if (bara == 0)
            continue;
        poly_rotate64(diff, acc, N, bara);
        poly_rotate64(diff + N, acc + N, N, bara);
        for (uint32_t j = 0; j < 2 * N; j++)
            diff[j] -= acc[j];
        ext_prod64(c, diff, c->bk2 + i * per, c->bk2fd ? c->bk2fd + i * per : NULL, ep);
        for (uint32_t j = 0; j < 2 * N; j++)
            acc[j] += ep[j];
    }
    free(diff);
    free(ep);
}

int orc_blind_rotate_lvl2(orc_ctx* c, const uint32_t* in, const uint64_t* testvec,
                          uint64_t* out)
{
    if (!c->has_cb)
        return fail("no circuit-bootstrapping material");
    blind_rotate64(c, in, testvec, out);
    return 0;
}

/* T level-2 blind rotations (test vector b = h[t]/2 everywhere) on `threads` host threads:
 * the level-2 half of circuitBootstrap (ops.cpp:914-935) for the parity tests. */
typedef struct {
    const orc_ctx* c;
    const uint32_t* in;
    const uint64_t* h;
    uint64_t* out;
    size_t T;
    atomic_size_t next;
} br2_job;

static void* br2_worker(void* arg)
{
    br2_job* j = arg;
    const uint32_t N = j->c->p.N2, n1 = j->c->p.n + 1;
    uint64_t* tv = calloc(2 * (size_t)N, 8);
    for (;;) {
        const size_t t = atomic_fetch_add(&j->next, 1);
        if (t >= j->T)
            break;
        for (uint32_t k = 0; k < N; k++)
            tv[N + k] = j->h[t] / 2;
        blind_rotate64(j->c, j->in + t * n1, tv, j->out + t * 2 * (size_t)N);
    }
    free(tv);
    return NULL;
}

int orc_blind_rotate_lvl2_batch(orc_ctx* c, const uint32_t* in, const uint64_t* h,
                                uint64_t* out, size_t T, unsigned threads)
{
    if (!c->has_cb)
        return fail("no circuit-bootstrapping material");
    if (threads < 1)
        threads = 1;
    br2_job j = {c, in, h, out, T, 0};
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (unsigned i = 0; i < threads; i++)
        pthread_create(&th[i], NULL, br2_worker, &j);
    for (unsigned i = 0; i < threads; i++)
        pthread_join(th[i], NULL);
    free(th);
    return 0;
}

/* bootstrapToTrlwe (ops.cpp:750-757) */
static void bootstrap_to_trlwe(const orc_ctx* c, const uint32_t* ct, uint32_t* out)
{
    const uint32_t N = c->p.N1;
    uint32_t* tv = calloc(2 * N, 4);
    for (uint32_t i = 0; i < N; i++)
        tv[N + i] = kMu32;
    blind_rotate32(c, ct, tv, out);
    free(tv);
}

int orc_bootstrap_to_trlwe(orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    bootstrap_to_trlwe(c, in, out);
    return 0;
}

/* gateBootstrap (ops.cpp:759-762) */
static void gate_bootstrap(const orc_ctx* c, const uint32_t* ct, uint32_t* out)
{
    const uint32_t N = c->p.N1;
    uint32_t* tr = malloc(4 * 2 * N);
    uint32_t* se = malloc(4 * (N + 1));
    bootstrap_to_trlwe(c, ct, tr);
    sample_extract32(tr, N, 0, se);
    iks(c, se, out);
    free(tr);
    free(se);
}

int orc_gate_bootstrap(orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    gate_bootstrap(c, in, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Homomorphic gates (ops.cpp:774-909)                                        */

enum { K_AND, K_ANDNOT, K_MUX, K_NAND, K_NOR, K_NOT, K_OR, K_ORNOT, K_XNOR, K_XOR };

static int gate_arity(int kind) /* ops.hpp:196-206 */
{
    return kind == K_NOT ? 1 : kind == K_MUX ? 3 : 2;
}

/* linComb (ops.cpp:774-806) over two terms */
static void lin_comb2(uint32_t n, int c0, const uint32_t* x, int c1, const uint32_t* y,
                      uint32_t bias, uint32_t* out)
{
    for (uint32_t i = 0; i <= n; i++)
        out[i] = (uint32_t)c0 * x[i] + (uint32_t)c1 * y[i] + (i == n ? bias : 0u);
}

static void hom_gate(const orc_ctx* c, int kind, const uint32_t* in, uint32_t* out)
{
    const uint32_t n = c->p.n, N = c->p.N1;
    const uint32_t negMu = 0u - kMu32;
    const uint32_t* a = in;
    const uint32_t* b = in + (n + 1);
    uint32_t* t = malloc(4 * (n + 1));
    switch (kind) {
    case K_NOT: /* ops.cpp:849-855 */
        for (uint32_t i = 0; i <= n; i++)
            out[i] = 0u - a[i];
        break;
    case K_AND:
        lin_comb2(n, 1, a, 1, b, negMu, t);
        gate_bootstrap(c, t, out);
        break;
    case K_NAND:
        lin_comb2(n, -1, a, -1, b, kMu32, t);
        gate_bootstrap(c, t, out);
        break;
    case K_OR:
        lin_comb2(n, 1, a, 1, b, kMu32, t);
        gate_bootstrap(c, t, out);
        break;
    case K_NOR:
        lin_comb2(n, -1, a, -1, b, negMu, t);
        gate_bootstrap(c, t, out);
        break;
    case K_XOR:
        lin_comb2(n, 2, a, 2, b, 2 * kMu32, t);
        gate_bootstrap(c, t, out);
        break;
    case K_XNOR:
        lin_comb2(n, -2, a, -2, b, 2 * negMu, t);
        gate_bootstrap(c, t, out);
        break;
    case K_ANDNOT:
        lin_comb2(n, 1, a, -1, b, negMu, t);
        gate_bootstrap(c, t, out);
        break;
    case K_ORNOT:
        lin_comb2(n, 1, a, -1, b, kMu32, t);
        gate_bootstrap(c, t, out);
        break;
    case K_MUX: { /* ops.cpp:880-893; in = {sel, a, b} */
        const uint32_t* s = in;
        const uint32_t* x = in + (n + 1);
        const uint32_t* y = in + 2 * (n + 1);
        uint32_t* u = malloc(4 * (n + 1));
        uint32_t* tr = malloc(4 * 2 * N);
        uint32_t* t1 = malloc(4 * (N + 1));
        uint32_t* t2 = malloc(4 * (N + 1));
        lin_comb2(n, 1, s, 1, x, negMu, u);
        lin_comb2(n, -1, s, 1, y, negMu, t);
        bootstrap_to_trlwe(c, u, tr);
        sample_extract32(tr, N, 0, t1);
        bootstrap_to_trlwe(c, t, tr);
        sample_extract32(tr, N, 0, t2);
        for (uint32_t i = 0; i < N; i++)
            t1[i] += t2[i];
        t1[N] = t1[N] + t2[N] + kMu32;
        iks(c, t1, out);
        free(u);
        free(tr);
        free(t1);
        free(t2);
        break;
    }
    }
    free(t);
}

int orc_hom_gate(orc_ctx* c, int kind, const uint32_t* in, int nin, uint32_t* out)
{
    if (kind < 0 || kind > K_XOR)
        return fail("homGate: unknown kind");
    if (nin != gate_arity(kind))
        return fail("homGate: bad arity");
    if (!c->has_bk && kind != K_NOT)
        return fail("no key");
    hom_gate(c, kind, in, out);
    return 0;
}

typedef struct {
    orc_ctx* c;
    const int* kinds;
    const uint32_t* in;
    uint32_t* out;
    size_t G;
    _Atomic size_t next;
} batch_job;

static void* batch_worker(void* arg)
{
    batch_job* j = arg;
    const uint32_t n = j->c->p.n;
    for (;;) {
        size_t g = atomic_fetch_add(&j->next, 1);
        if (g >= j->G)
            break;
        hom_gate(j->c, j->kinds[g], j->in + g * 3 * (n + 1), j->out + g * (n + 1));
    }
    return NULL;
}

int orc_hom_gate_batch(orc_ctx* c, const int* kinds, const uint32_t* in, uint32_t* out,
                       size_t G, unsigned threads)
{
    if (!c->has_bk)
        return fail("no key");
    batch_job j = {c, kinds, in, out, G, 0};
    if (threads < 1)
        threads = 1;
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (unsigned i = 1; i < threads; i++)
        pthread_create(&th[i], NULL, batch_worker, &j);
    batch_worker(&j);
    for (unsigned i = 1; i < threads; i++)
        pthread_join(th[i], NULL);
    free(th);
    return 0;
}

/* homMuxNoSeIks (ops.cpp:898-909) */
static void hom_mux_no_se_iks(const orc_ctx* c, const uint32_t* s, const uint32_t* x,
                              const uint32_t* y, uint32_t* out)
{
    const uint32_t n = c->p.n, N = c->p.N1;
    const uint32_t negMu = 0u - kMu32;
    uint32_t* u = malloc(4 * (n + 1));
    uint32_t* v = malloc(4 * (n + 1));
    uint32_t* t2 = malloc(4 * 2 * N);
    lin_comb2(n, 1, s, 1, x, negMu, u);
    lin_comb2(n, -1, s, 1, y, negMu, v);
    bootstrap_to_trlwe(c, u, out);
    bootstrap_to_trlwe(c, v, t2);
    for (uint32_t i = 0; i < 2 * N; i++)
        out[i] += t2[i];
    out[N] += kMu32;
    free(u);
    free(v);
    free(t2);
}

int orc_hom_mux_no_se_iks(orc_ctx* c, const uint32_t* sel, const uint32_t* a,
                          const uint32_t* b, uint32_t* out)
{
    if (!c->has_bk)
        return fail("no key");
    hom_mux_no_se_iks(c, sel, a, b, out);
    return 0;
}

/* circuitBootstrap (ops.cpp:914-935) */
static void circuit_bootstrap(const orc_ctx* c, const uint32_t* ct, uint32_t* out)
{
    const params_t* p = &c->p;
    const uint32_t l = p->l1, N1 = p->N1, N2 = p->N2;
    uint64_t* tv = calloc(2 * N2, 8);
    uint64_t* acc = malloc(8 * 2 * N2);
    uint64_t* t2 = malloc(8 * (N2 + 1));
    atomic_fetch_add(&g_cnt[4], 1);
    for (uint32_t i = 0; i < l; i++) {
        const uint64_t h = 1ull << (64 - (i + 1) * p->Bg1Bits);
        for (uint32_t k = 0; k < N2; k++)
            tv[N2 + k] = h / 2;
        blind_rotate64(c, ct, tv, acc);
        sample_extract64(acc, N2, 0, t2);
        t2[N2] += h / 2;
        pks(c, t2, c->pksNegS, out + (size_t)i * 2 * N1);
        pks(c, t2, c->pksId, out + (size_t)(l + i) * 2 * N1);
    }
    free(tv);
    free(acc);
    free(t2);
}

int orc_circuit_bootstrap(orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    if (!c->has_cb)
        return fail("bootstrapping key lacks circuit bootstrapping material");
    circuit_bootstrap(c, in, out);
    return 0;
}

/* trgswNot (ops.cpp:937-947) */
static void trgsw_not(const params_t* p, const uint32_t* in, uint32_t* out)
{
    const uint32_t N = p->N1, l = p->l1;
    for (size_t i = 0; i < (size_t)2 * l * 2 * N; i++)
        out[i] = 0u - in[i];
    for (uint32_t i = 0; i < l; i++) {
        const uint32_t h = 1u << (32 - (i + 1) * p->Bg1Bits);
        out[(size_t)i * 2 * N] += h;
        out[(size_t)(l + i) * 2 * N + N] += h;
    }
}

int orc_trgsw_not(orc_ctx* c, const uint32_t* in, uint32_t* out)
{
    trgsw_not(&c->p, in, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* CMUX memory (mem.cpp)                                                      */

typedef struct {
    uint32_t* sel;    /* v raw TRGSW */
    uint32_t* notSel; /* v raw TRGSW */
    double* selfd;    /* prepared (fft params only) */
    double* notfd;
} addr_t;

static size_t trgsw_words(const params_t* p) { return (size_t)2 * p->l1 * 2 * p->N1; }

/* addressToTrgsw + prepareAddress (mem.cpp:21-47) */
static void address_prepare(const orc_ctx* c, const uint32_t* bits, uint32_t v, addr_t* a)
{
    const size_t tw = trgsw_words(&c->p);
    a->sel = malloc(4 * tw * v);
    a->notSel = malloc(4 * tw * v);
    a->selfd = a->notfd = NULL;
    for (uint32_t d = 0; d < v; d++) {
        circuit_bootstrap(c, bits + (size_t)d * (c->p.n + 1), a->sel + d * tw);
        trgsw_not(&c->p, a->sel + d * tw, a->notSel + d * tw);
    }
    if (c->p.fft && !c->exact) {
        a->selfd = malloc(sizeof(double) * tw * v);
        a->notfd = malloc(sizeof(double) * tw * v);
        for (uint32_t d = 0; d < v; d++) {
            prepare32((orc_ctx*)c, a->sel + d * tw, a->selfd + d * tw);
            prepare32((orc_ctx*)c, a->notSel + d * tw, a->notfd + d * tw);
        }
    }
}

static void address_free(addr_t* a)
{
    free(a->sel);
    free(a->notSel);
    free(a->selfd);
    free(a->notfd);
}

#define SELRAW(a, d) ((a)->sel + (size_t)(d) * tw)
#define SELFD(a, d) ((a)->selfd ? (a)->selfd + (size_t)(d) * tw : NULL)
#define NOTRAW(a, d) ((a)->notSel + (size_t)(d) * tw)
#define NOTFD(a, d) ((a)->notfd ? (a)->notfd + (size_t)(d) * tw : NULL)

int orc_ram_cycle(orc_ctx* c, uint32_t v, uint32_t w, uint32_t* ram, const uint32_t* addr,
                  const uint32_t* wflag, const uint32_t* wdata, uint32_t* readout)
{
    if (!c->has_cb)
        return fail("bootstrapping key lacks circuit bootstrapping material");
    const params_t* p = &c->p;
    const uint32_t N = p->N1, n = p->n, words = 1u << v;
    const size_t tw = trgsw_words(p), cw = 2 * (size_t)N;
    addr_t A;
    address_prepare(c, addr, v, &A); /* mem.cpp:122-127 */
    /* ramReadUnit (mem.cpp:49-72) */
    uint32_t* read = malloc(4 * cw * w);
    uint32_t* layer = malloc(4 * cw * words);
    for (uint32_t j = 0; j < w; j++) {
        memcpy(layer, ram + (size_t)j * words * cw, 4 * cw * words);
        size_t size = words;
        for (uint32_t d = 0; d < v; d++) {
            const size_t half = size / 2;
            for (size_t k = 0; k < half; k++) {
                uint32_t* tmp = malloc(4 * cw);
                cmux32(c, SELRAW(&A, d), SELFD(&A, d), layer + (2 * k + 1) * cw,
                       layer + 2 * k * cw, tmp);
                memcpy(layer + k * cw, tmp, 4 * cw);
                free(tmp);
            }
            size = half;
        }
        memcpy(read + (size_t)j * cw, layer, 4 * cw);
    }
    free(layer);
    /* ramControlUnit (mem.cpp:74-90) */
    uint32_t* ctl = malloc(4 * cw * w);
    uint32_t* se = malloc(4 * (N + 1));
    for (uint32_t j = 0; j < w; j++) {
        sample_extract32(read + (size_t)j * cw, N, 0, se);
        iks(c, se, readout + (size_t)j * (n + 1));
        hom_mux_no_se_iks(c, wflag, wdata + (size_t)j * (n + 1), readout + (size_t)j * (n + 1),
                          ctl + (size_t)j * cw);
    }
    /* ramWriteUnit (mem.cpp:92-120) */
    uint32_t* next = malloc(4 * cw * w * words);
    uint32_t* t = malloc(4 * cw);
    uint32_t* t2 = malloc(4 * cw);
    uint32_t* lw = malloc(4 * (n + 1));
    for (size_t idx = 0; idx < (size_t)w * words; idx++) {
        const uint32_t j = (uint32_t)(idx / words), Ad = (uint32_t)(idx % words);
        const uint32_t* old = ram + idx * cw;
        if (Ad & 1)
            cmux32(c, SELRAW(&A, 0), SELFD(&A, 0), ctl + (size_t)j * cw, old, t);
        else
            cmux32(c, NOTRAW(&A, 0), NOTFD(&A, 0), ctl + (size_t)j * cw, old, t);
        for (uint32_t d = 1; d < v; d++) {
            if ((Ad >> d) & 1)
                cmux32(c, SELRAW(&A, d), SELFD(&A, d), t, old, t2);
            else
                cmux32(c, NOTRAW(&A, d), NOTFD(&A, d), t, old, t2);
            memcpy(t, t2, 4 * cw);
        }
        sample_extract32(t, N, 0, se);
        iks(c, se, lw);
        bootstrap_to_trlwe(c, lw, next + idx * cw);
    }
    memcpy(ram, next, 4 * cw * w * words);
    free(next);
    free(t);
    free(t2);
    free(lw);
    free(se);
    free(ctl);
    free(read);
    address_free(&A);
    return 0;
}

static uint32_t ctz32(uint32_t x)
{
    uint32_t r = 0;
    while (x && !(x & 1)) {
        x >>= 1;
        r++;
    }
    return r;
}

uint32_t orc_rom_luts(const orc_ctx* c, uint32_t depth_bytes)
{
    const uint32_t vrom = ctz32(depth_bytes / 4);
    uint32_t low = ctz32(c->p.N1 / 32);
    if (vrom < low)
        low = vrom;
    return 1u << (vrom - low);
}

/* addressToTrgsw + prepareAddress + romRead (mem.cpp:137-177) */
int orc_rom_read(orc_ctx* c, uint32_t depth_bytes, const uint32_t* luts, uint32_t nluts,
                 const uint32_t* addr, uint32_t vrom, uint32_t* out)
{
    if (!c->has_cb)
        return fail("bootstrapping key lacks circuit bootstrapping material");
    const params_t* p = &c->p;
    const uint32_t N = p->N1, n = p->n;
    const size_t tw = trgsw_words(p), cw = 2 * (size_t)N;
    if (ctz32(depth_bytes / 4) != vrom)
        return fail("romRead: address width mismatch");
    uint32_t lowBits = ctz32(N / 32);
    if (vrom < lowBits)
        lowBits = vrom;
    const uint32_t highBits = vrom - lowBits;
    if (nluts != (1u << highBits))
        return fail("romRead: lut count mismatch");
    addr_t A;
    address_prepare(c, addr, vrom, &A);
    uint32_t* layer = malloc(4 * cw * nluts);
    memcpy(layer, luts, 4 * cw * nluts);
    uint32_t* tmp = malloc(4 * cw);
    size_t size = nluts;
    for (uint32_t d = 0; d < highBits; d++) {
        const size_t half = size / 2;
        for (size_t k = 0; k < half; k++) {
            cmux32(c, SELRAW(&A, lowBits + d), SELFD(&A, lowBits + d),
                   layer + (2 * k + 1) * cw, layer + 2 * k * cw, tmp);
            memcpy(layer + k * cw, tmp, 4 * cw);
        }
        size = half;
    }
    uint32_t* acc = malloc(4 * cw);
    uint32_t* rot = malloc(4 * cw);
    memcpy(acc, layer, 4 * cw);
    for (uint32_t d = 0; d < lowBits; d++) {
        const uint32_t shift = 32u << d;
        poly_rotate32(rot, acc, N, 2 * N - shift);
        poly_rotate32(rot + N, acc + N, N, 2 * N - shift);
        cmux32(c, SELRAW(&A, d), SELFD(&A, d), rot, acc, tmp);
        memcpy(acc, tmp, 4 * cw);
    }
    uint32_t* se = malloc(4 * (N + 1));
    for (uint32_t k = 0; k < 32; k++) {
        sample_extract32(acc, N, k, se);
        iks(c, se, out + (size_t)k * (n + 1));
    }
    free(se);
    free(acc);
    free(rot);
    free(tmp);
    free(layer);
    address_free(&A);
    return 0;
}

static int image_bit(const uint8_t* image, size_t bit) { return (image[bit / 8] >> (bit % 8)) & 1; }

/* encryptBitPoly (mem.cpp:184-194) */
static void encrypt_bit_poly(orc_ctx* c, const uint32_t* bits, int trivial, uint32_t* out)
{
    const uint32_t N = c->p.N1;
    if (!trivial) {
        orc_trlwe_encrypt(c, bits, c->p.alpha1, out);
        return;
    }
    memset(out, 0, 4 * N);
    for (uint32_t i = 0; i < N; i++)
        out[N + i] = bits[i] ? kMu32 : 0u - kMu32;
}

int orc_encrypt_ram(orc_ctx* c, const uint8_t* image, uint32_t v, uint32_t w, int trivial,
                    uint32_t* out) /* mem.cpp:202-222 */
{
    const uint32_t N = c->p.N1, words = 1u << v;
    uint32_t* mv = calloc(N, 4);
    size_t pos = 0;
    for (uint32_t j = 0; j < w; j++)
        for (uint32_t A = 0; A < words; A++) {
            mv[0] = (uint32_t)image_bit(image, (size_t)A * w + j);
            encrypt_bit_poly(c, mv, trivial, out + pos);
            pos += 2 * (size_t)N;
        }
    free(mv);
    return 0;
}

int orc_decrypt_ram(const orc_ctx* c, const uint32_t* ram, uint32_t v, uint32_t w,
                    uint8_t* image) /* mem.cpp:224-234 */
{
    const uint32_t N = c->p.N1, words = 1u << v;
    memset(image, 0, ((size_t)w << v) / 8);
    for (uint32_t j = 0; j < w; j++)
        for (uint32_t A = 0; A < words; A++) {
            const uint32_t* cell = ram + ((size_t)j * words + A) * 2 * N;
            if ((int32_t)orc_trlwe_phase_at(c, cell, 0) >= 0) {
                const size_t bit = (size_t)A * w + j;
                image[bit / 8] |= (uint8_t)(1u << (bit % 8));
            }
        }
    return 0;
}

int orc_encrypt_rom(orc_ctx* c, const uint8_t* image, uint32_t depth_bytes, int trivial,
                    uint32_t* out) /* mem.cpp:236-263 */
{
    const uint32_t N = c->p.N1;
    const size_t totalBits = (size_t)depth_bytes * 8;
    const uint32_t numLuts = orc_rom_luts(c, depth_bytes);
    uint32_t* bits = malloc(4 * N);
    for (uint32_t t = 0; t < numLuts; t++) {
        for (uint32_t k = 0; k < N; k++) {
            const size_t bit = (size_t)t * N + k;
            bits[k] = bit < totalBits && image_bit(image, bit) ? 1 : 0;
        }
        encrypt_bit_poly(c, bits, trivial, out + (size_t)t * 2 * N);
    }
    free(bits);
    return 0;
}
