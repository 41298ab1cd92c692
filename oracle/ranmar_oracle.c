/* TEST INFRASTRUCTURE ONLY (oracle/) — see ranmar_oracle.h. Plain-C
 * restatement of /root/reference/proj/include/ranmar; each function cites
 * the reference lines it follows. Deliberately scalar and literal: it is the
 * checker, not a fast path. Compiled with -ffp-contract=off so the float
 * recurrence and the gaussian are evaluated exactly as written. */
#include "ranmar_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- core --- */

/* init.hpp:18-51 (checked; throws above max_seed, init.hpp:19-20). */
int or_init(uint32_t seed, or_state* out) {
    if (seed > OR_MAX_SEED) return 1;
    or_init_unchecked(seed, out);
    return 0;
}

/* init.hpp:22-49: signed seed split with C truncating division (seed 0 gives
 * ij = 0, kl = -1), then 97 lanes x 24 bits of the Marsaglia bit mixer
 * ((ii*jj)%179)*kk%179 — the code's Remainder, not the paper's Quotient
 * — accumulated at weight 2^31, 2^30, ... and >> 8. */
void or_init_unchecked(uint32_t seed, or_state* out) {
    const int ij = ((int)seed - 1) / 30082;
    const int kl = ((int)seed - 1) - 30082 * ij;
    int ii = (ij / 177) % 177 + 2;
    int jj = ij % 177 + 2;
    int kk = (kl / 169) % 178 + 1;
    int ll = kl % 169;
    memset(out, 0, sizeof *out);
    for (int lane = 0; lane < OR_LONG_LAG; ++lane) {
        uint32_t acc = 0, t = 1u << 31;
        for (int bit = 0; bit < 24; ++bit) {
            const int mm = ((ii * jj) % 179) * kk % 179;
            ii = jj;
            jj = kk;
            kk = mm;
            ll = (53 * ll + 1) % 169;
            if ((ll * mm) % 64 >= 32) acc += t;
            t >>= 1;
        }
        out->lane[lane] = acc >> 8;
    }
    out->i = OR_LONG_LAG - 1;
    out->j = OR_SHORT_LAG - 1;
    out->v = OR_ARITH_START;
}

/* core.hpp:54-66 */
uint32_t or_step(or_state* s) {
    const uint32_t u = (s->lane[s->i] - s->lane[s->j]) & OR_MASK;
    s->lane[s->i] = u;
    s->i = s->i == 0 ? OR_LONG_LAG - 1 : s->i - 1;
    s->j = s->j == 0 ? OR_LONG_LAG - 1 : s->j - 1;
    uint32_t v = s->v + (OR_ARITH_MOD - OR_ARITH_DELTA);
    if (v >= OR_ARITH_MOD) v -= OR_ARITH_MOD;
    s->v = v;
    return (u - v) & OR_MASK;
}

void or_step_n(or_state* s, uint64_t n, uint32_t* out) {
    for (uint64_t k = 0; k < n; ++k) {
        const uint32_t u = or_step(s);
        if (out) out[k] = u;
    }
}

/* core.hpp:75-79 */
int or_value_of(uint32_t u24, double* out) {
    if (u24 > OR_MASK) return 1;
    *out = (double)u24 * 0x1p-24;
    return 0;
}

/* ---------------------------------------------------------- float path --- */

/* reference/float_ranmar.hpp:50-80 */
int or_init_float(uint32_t seed, or_float_state* f) {
    if (seed > OR_MAX_SEED) return 1;
    const int ij = ((int)seed - 1) / 30082;
    const int kl = ((int)seed - 1) - 30082 * ij;
    int ii = (ij / 177) % 177 + 2;
    int jj = ij % 177 + 2;
    int kk = (kl / 169) % 178 + 1;
    int ll = kl % 169;
    for (int lane = 0; lane < OR_LONG_LAG; ++lane) {
        double s = 0.0, t = 0.5;
        for (int bit = 0; bit < 24; ++bit) {
            const int mm = ((ii * jj) % 179) * kk % 179;
            ii = jj;
            jj = kk;
            kk = mm;
            ll = (53 * ll + 1) % 169;
            if ((ll * mm) % 64 >= 32) s += t;
            t *= 0.5;
        }
        f->x[lane] = s;
    }
    f->c = 362436.0 / 16777216.0;
    f->i = OR_LONG_LAG - 1;
    f->j = OR_SHORT_LAG - 1;
    return 0;
}

/* reference/float_ranmar.hpp:33-46 (Algorithm 1, five branches, binary64). */
double or_step_float(or_float_state* s) {
    double y = s->x[s->i] - s->x[s->j];
    if (y < 0.0) y += 1.0;
    s->x[s->i] = y;
    s->i = s->i == 0 ? OR_LONG_LAG - 1 : s->i - 1;
    s->j = s->j == 0 ? OR_LONG_LAG - 1 : s->j - 1;
    s->c -= 7654321.0 / 16777216.0;
    if (s->c < 0.0) s->c += 16777213.0 / 16777216.0;
    y -= s->c;
    if (y < 0.0) y += 1.0;
    return y;
}

void or_step_float_n(or_float_state* s, uint64_t n, double* out) {
    for (uint64_t k = 0; k < n; ++k) out[k] = or_step_float(s);
}

/* ----------------------------------------------------------- poly ring --- */

/* polyring.hpp:60-80: fold degree <= 192 down with t^97 = 1 - t^64,
 * descending, 32-bit wraparound, final mask. */
void or_reduce_trinomial(const uint32_t* raw, int n, uint32_t* out97) {
    uint32_t c[193];
    memset(c, 0, sizeof c);
    for (int k = 0; k < n && k < 193; ++k) c[k] = raw[k];
    for (int k = 192; k >= 97; --k) {
        const uint32_t hi = c[k];
        c[k - 97] += hi;
        c[k - 33] -= hi;
        c[k] = 0;
    }
    for (int k = 0; k < 97; ++k) out97[k] = c[k] & OR_MASK;
}

/* polyring.hpp:85-98: schoolbook with 64-bit accumulation, then fold. */
void or_mul_mod(const uint32_t* a, const uint32_t* b, uint32_t* out97) {
    uint64_t acc[193];
    uint32_t raw[193];
    memset(acc, 0, sizeof acc);
    for (int i = 0; i < 97; ++i) {
        const uint64_t ai = a[i];
        if (ai == 0) continue;
        for (int j = 0; j < 97; ++j) acc[i + j] += ai * b[j];
    }
    for (int k = 0; k < 193; ++k) raw[k] = (uint32_t)acc[k] & OR_MASK;
    or_reduce_trinomial(raw, 193, out97);
}

/* polyring.hpp:101-109 */
void or_mul_by_t(const uint32_t* p, uint32_t* out97) {
    uint32_t q[97];
    const uint32_t top = p[96];
    for (int k = 96; k >= 1; --k) q[k] = p[k - 1];
    q[0] = top;
    q[64] = (q[64] - top) & OR_MASK;
    memcpy(out97, q, sizeof q);
}

/* polyring.hpp:113-124: left-to-right square-and-multiply over J's bits. */
void or_pow_t_mod(const or_j256* j, uint32_t* out97) {
    uint32_t acc[97];
    memset(acc, 0, sizeof acc);
    acc[0] = 1;
    for (int k = or_j256_msb(j); k >= 0; --k) {
        or_mul_mod(acc, acc, acc);
        if ((j->limb[k / 64] >> (k % 64)) & 1u) or_mul_by_t(acc, acc);
    }
    memcpy(out97, acc, sizeof acc);
}

/* ---------------------------------------------------------------- jump --- */

/* jump.hpp:32-37 */
void or_canonicalize(const or_state* s, uint32_t* u97) {
    for (int k = 0; k < 97; ++k) u97[k] = s->lane[(s->i + 97 - k) % 97];
}

/* jump.hpp:42-48 */
void or_decanonicalize(const uint32_t* u97, or_state* out) {
    out->i = OR_LONG_LAG - 1;
    out->j = OR_SHORT_LAG - 1;
    for (int k = 0; k < 97; ++k) out->lane[96 - k] = u97[k];
}

/* jump.hpp:52-57 */
void or_apply_companion(const uint32_t* u, uint32_t* out97) {
    uint32_t o[97];
    for (int k = 0; k + 1 < 97; ++k) o[k] = u[k + 1];
    o[96] = (u[0] - u[64]) & OR_MASK;
    memcpy(out97, o, sizeof o);
}

/* jump.hpp:60-76: pow_t_mod, then Horner acc = b96 u; acc = A(acc) + b_k u. */
void or_jump_fib(const uint32_t* u, const or_j256* j, uint32_t* out97) {
    uint32_t p[97], acc[97];
    or_pow_t_mod(j, p);
    const uint64_t top = p[96];
    for (int k = 0; k < 97; ++k) acc[k] = (uint32_t)(top * u[k]) & OR_MASK;
    for (int deg = 95; deg >= 0; --deg) {
        or_apply_companion(acc, acc);
        const uint64_t b = p[deg];
        if (b == 0) continue;
        for (int k = 0; k < 97; ++k) acc[k] = (uint32_t)(acc[k] + b * u[k]) & OR_MASK;
    }
    memcpy(out97, acc, sizeof acc);
}

/* jump.hpp:79-86: v' = (v + m - ((J mod m) * d mod m)) mod m. */
uint32_t or_jump_arith(uint32_t v, const or_j256* j) {
    const uint64_t jm = or_j256_mod_u32(j, OR_ARITH_MOD);
    const uint64_t dec = (jm * OR_ARITH_DELTA) % OR_ARITH_MOD;
    return (uint32_t)(((uint64_t)v + (OR_ARITH_MOD - dec)) % OR_ARITH_MOD);
}

/* jump.hpp:90-95 */
void or_jump_state(const or_state* in, const or_j256* j, or_state* out) {
    uint32_t u[97], w[97];
    or_canonicalize(in, u);
    or_jump_fib(u, j, w);
    const uint32_t v = or_jump_arith(in->v, j);
    or_decanonicalize(w, out);
    out->v = v;
}

/* jump.hpp:108-124, streams [first, first+n): stream `first` by the
 * independent jump (first * J, :121), the rest incrementally (:119). */
int or_make_streams(const or_state* base, const or_j256* j, uint64_t first, uint64_t n,
                    or_state* out) {
    if (n == 0) return 1;                 /* jump.hpp:111 */
    if (or_j256_is_zero(j)) return 1;     /* jump.hpp:112: block_length < 1 */
    or_state s;
    if (first == 0) {
        s = *base;
    } else {
        or_j256 kj;
        or_j256_mul_u64(j, first, &kj);
        or_jump_state(base, &kj, &s);
    }
    out[0] = s;
    for (uint64_t k = 1; k < n; ++k) or_jump_state(&out[k - 1], j, &out[k]);
    return 0;
}

/* ------------------------------------------------------------ J helpers --- */

void or_j256_from_u64(uint64_t x, or_j256* out) {
    memset(out, 0, sizeof *out);
    out->limb[0] = x;
}

int or_j256_is_zero(const or_j256* a) {
    return (a->limb[0] | a->limb[1] | a->limb[2] | a->limb[3]) == 0;
}

int or_j256_msb(const or_j256* a) {
    for (int k = 3; k >= 0; --k)
        if (a->limb[k]) return 64 * k + 63 - __builtin_clzll(a->limb[k]);
    return -1;
}

uint32_t or_j256_mod_u32(const or_j256* a, uint32_t m) {
    unsigned __int128 r = 0;
    for (int k = 3; k >= 0; --k) r = ((r << 64) | a->limb[k]) % m;
    return (uint32_t)r;
}

void or_j256_mul_u64(const or_j256* a, uint64_t k, or_j256* out) {
    unsigned __int128 carry = 0;
    or_j256 r;
    for (int w = 0; w < 4; ++w) {
        const unsigned __int128 p = (unsigned __int128)a->limb[w] * k + carry;
        r.limb[w] = (uint64_t)p;
        carry = p >> 64;
    }
    *out = r;
}

void or_j256_add(const or_j256* a, const or_j256* b, or_j256* out) {
    unsigned __int128 carry = 0;
    or_j256 r;
    for (int w = 0; w < 4; ++w) {
        const unsigned __int128 s = (unsigned __int128)a->limb[w] + b->limb[w] + carry;
        r.limb[w] = (uint64_t)s;
        carry = s >> 64;
    }
    *out = r;
}

/* jumpcount.hpp:16-47: decimal, "2^k", "2^k-1", "2^k+1" (k <= 10^6 there;
 * here the value must also fit 256 bits, else error 2). */
int or_j256_parse(const char* text, or_j256* out) {
    memset(out, 0, sizeof *out);
    if (!text || !*text) return 1;
    if (text[0] == '2' && text[1] == '^') {
        const char* p = text + 2;
        unsigned long k = 0;
        int n = 0;
        while (*p >= '0' && *p <= '9') {
            k = k * 10 + (unsigned long)(*p - '0');
            if (k > 1000000) return 1;
            ++p;
            ++n;
        }
        if (n == 0) return 1;
        int delta = 0;
        if (strcmp(p, "-1") == 0) delta = -1;
        else if (strcmp(p, "+1") == 0) delta = 1;
        else if (*p) return 1;
        if (k > 256 || (k == 256 && delta >= 0)) return 2;
        if (k < 256) out->limb[k / 64] = 1ull << (k % 64);
        if (delta == 1) {
            or_j256 one;
            or_j256_from_u64(1, &one);
            or_j256_add(out, &one, out);
        } else if (delta == -1) { /* subtract one with borrow */
            for (int w = 0; w < 4; ++w) {
                if (out->limb[w]-- != 0) break;
            }
        }
        return 0;
    }
    for (const char* p = text; *p; ++p)
        if (*p < '0' || *p > '9') return 1;
    for (const char* p = text; *p; ++p) {
        or_j256 t;
        or_j256_mul_u64(out, 10, &t);
        /* overflow check: t / 10 must give back out */
        if (or_j256_msb(out) >= 252) return 2;
        or_j256 d;
        or_j256_from_u64((uint64_t)(*p - '0'), &d);
        or_j256_add(&t, &d, out);
    }
    return 0;
}

/* ------------------------------------------------------------ workloads --- */

void or_generate_u32(or_state* states, uint64_t n_streams, uint64_t per_stream, uint32_t* out) {
    for (uint64_t k = 0; k < n_streams; ++k)
        or_step_n(&states[k], per_stream, out + k * per_stream);
}

/* next_f64 (core.hpp:70-72) narrowed to binary32: exact for 24-bit outputs. */
void or_generate_f32(or_state* states, uint64_t n_streams, uint64_t per_stream, float* out) {
    for (uint64_t k = 0; k < n_streams; ++k)
        for (uint64_t t = 0; t < per_stream; ++t)
            out[k * per_stream + t] = (float)((double)or_step(&states[k]) * 0x1p-24);
}

void or_consume(or_state* states, uint64_t n_streams, uint64_t per_stream, uint64_t* sums,
                uint32_t* hist) {
    for (uint64_t k = 0; k < n_streams; ++k) {
        uint64_t sum = 0;
        uint32_t* h = hist + k * 256;
        memset(h, 0, 256 * sizeof *h);
        for (uint64_t t = 0; t < per_stream; ++t) {
            const uint32_t u = or_step(&states[k]);
            sum += u;
            ++h[u >> 16];
        }
        sums[k] = sum;
    }
}

/* The gaussian convention's log(): CORRECTLY ROUNDED binary64 log, so the
 * repo's gaussian() equals LAMMPS' RanMars::gaussian() form
 * fac = sqrt(-2.0*log(rsq)/rsq) with any correctly rounded libm log (glibc's
 * log is correctly rounded except in rare cases, where it is 1 ulp off). The
 * method restates the published two-phase scheme of CRlibm / CORE-MATH
 * (Ziv's strategy): a fast double-double evaluation with a rigorous error
 * bound and a rounding test, and an accurate path (~2^-103) for the rare
 * inputs whose log lies too close to a rounding boundary. The constants come
 * from tools/gen_crlog.py (crlog_table.inc, the same file as the device's);
 * every operation below is one IEEE binary64 operation (-ffp-contract=off;
 * fma() is the correctly rounded fused multiply-add), so the device
 * (csrc/gauss_math.cuh crlog) reproduces each step bit for bit.
 *
 *   x = 2^e m, m in [1,2), i = top 7 bits of m, h = (i >= CRLOG_SPLIT)
 *   z = m r_i - 1                        exact (|z| < 2^-7, r_i = R_i/256)
 *   log x = (e+h) ln2 + T_i + log1p(z)   T_i = -log(r_i 2^h) (table)
 *
 * Fast-path error (absolute, derived in DESIGN.md §5.2):
 *   |log x - (yh + yl)| <= 2^-49 |z^3| + 2^-88 |yh|;
 * the test accepts yh when yh + (yl +- bound) round to the same double.
 * x must be a positive normal double: gaussian()'s rsq is in [2^-46, 1). */
#define CRLOG_TABLE_QUAL static const
#include "crlog_table.inc"

static void or_two_sum(double a, double b, double* s, double* e) {
    const double t = a + b;
    const double bb = t - a;
    *e = (a - (t - bb)) + (b - bb);
    *s = t;
}

/* the argument reduction shared by both phases */
static void or_crlog_reduce(double x, int* i, double* ed, double* z) {
    uint64_t b;
    memcpy(&b, &x, 8);
    *i = (int)((b >> 45) & 127);
    *ed = (double)((int)(b >> 52) - 1023 + (*i >= CRLOG_SPLIT));
    const uint64_t mb = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    double m;
    memcpy(&m, &mb, 8);
    *z = fma(m, crlog_r[*i], -1.0);
}

/* Accurate phase: log1p(z) by its Taylor series to z^15 (truncation
 * < 2^-109 relative), terms 8..15 in double, 7..1 in double-double Horner;
 * (e+h) ln2 as an exact head, an exact double-double middle and a tail;
 * T_i as three doubles; everything summed in double-double. *ok = 0 when the
 * rounding test at 2^-98 fails too (never on the gaussian domain: the GPU
 * sweep ranmar_crlog_sweep_dev checks all 2^46 inputs, and the few it finds
 * undecided are tabulated with their correctly rounded logs, crlog_hard). */
double or_crlog_accurate(double x, int* ok) {
    int i;
    double ed, z;
    or_crlog_reduce(x, &i, &ed, &z);
    double p = CRLOG_A15;
    p = fma(p, z, CRLOG_A14);
    p = fma(p, z, CRLOG_A13);
    p = fma(p, z, CRLOG_A12);
    p = fma(p, z, CRLOG_A11);
    p = fma(p, z, CRLOG_A10);
    p = fma(p, z, CRLOG_A9);
    p = fma(p, z, CRLOG_A8);
    static const double ch[8] = {0, 1.0, -0.5, CRLOG_A3H, CRLOG_A4H, CRLOG_A5H, CRLOG_A6H, CRLOG_A7H};
    static const double cl[8] = {0, 0.0, 0.0, CRLOG_A3L, CRLOG_A4L, CRLOG_A5L, CRLOG_A6L, CRLOG_A7L};
    double ph = p, pl = 0.0;
    for (int k = 7; k >= 1; --k) {
        /* (ph, pl) = (ph, pl) * z + c_k */
        const double th = ph * z;
        const double tl = fma(pl, z, fma(ph, z, -th));
        double s, e;
        or_two_sum(th, ch[k], &s, &e);
        e = e + (tl + cl[k]);
        ph = s + e;
        pl = e - (ph - s);
    }
    {   /* log1p(z) = (ph, pl) * z */
        const double th = ph * z;
        const double tl = fma(pl, z, fma(ph, z, -th));
        ph = th + tl;
        pl = tl - (ph - th);
    }
    /* K + T: head e ln2_hi + t1 (Fast2Sum: |e ln2_hi| >= |t1| or e = 0) */
    const double k1 = ed * CRLOG_LN2_HI;
    const double t1 = crlog_t12[2 * i], t2 = crlog_t12[2 * i + 1], t3 = crlog_t3[i];
    double hi = k1 + t1;
    double lo = t1 - (hi - k1);
    const double k2h = ed * CRLOG_LN2_MID;
    const double k2l = fma(ed, CRLOG_LN2_MID, -k2h);
    const double small = (k2l + t3) + ed * CRLOG_LN2_LO;
    double s, e;
    /* + k2h */
    or_two_sum(hi, k2h, &s, &e);
    e = e + lo;
    hi = s + e;
    lo = e - (hi - s);
    /* + t2 */
    or_two_sum(hi, t2, &s, &e);
    e = e + lo;
    hi = s + e;
    lo = e - (hi - s);
    /* + log1p(z) */
    or_two_sum(hi, ph, &s, &e);
    e = e + ((lo + pl) + small);
    hi = s + e;
    lo = e - (hi - s);
    const double d = fabs(hi) * 0x1p-98;
    *ok = (hi + (lo + d)) == (hi + (lo - d));
    if (!*ok) /* the few domain inputs that even this cannot decide are tabulated */
        for (int k = 0; k < CRLOG_NHARD; ++k)
            if (x == crlog_hard[2 * k]) {
                *ok = 1;
                return crlog_hard[2 * k + 1];
            }
    return hi;
}

/* Fast phase; *fast = 1 when its rounding test decided the result. */
double or_crlog_ex(double x, int* fast) {
    int i;
    double ed, z;
    or_crlog_reduce(x, &i, &ed, &z);
    /* log1p(z) = z - z^2/2 + z^3 q(z), q = 1/3 - z/4 + ... - z^7/10 */
    const double zh = z * z;
    const double zl = fma(z, z, -zh);
    double q = CRLOG_C10;
    q = fma(q, z, CRLOG_C9);
    q = fma(q, z, CRLOG_C8);
    q = fma(q, z, CRLOG_C7);
    q = fma(q, z, CRLOG_C6);
    q = fma(q, z, CRLOG_C5);
    q = fma(q, z, CRLOG_C4);
    q = fma(q, z, CRLOG_C3);
    const double z3 = z * zh;
    const double hh = -0.5 * zh;            /* exact */
    const double s1 = z + hh;               /* Fast2Sum: |z| >= |hh| */
    const double e1 = hh - (s1 - z);
    const double lo1 = fma(z3, q, e1 + (-0.5 * zl));
    /* K + T_i: Fast2Sum (|e ln2_hi| >= |t1| unless e = 0) */
    const double k1 = ed * CRLOG_LN2_HI;    /* exact: 42-bit head */
    const double t1 = crlog_t12[2 * i], t2 = crlog_t12[2 * i + 1];
    const double ah = k1 + t1;
    const double al = t1 - (ah - k1);
    /* + log1p head: Fast2Sum, exact because |ah| >= |s1| whenever ah != 0
     * (|s1| < 2^-7; a nonzero ah is at least |T_i| >= 2^-6.4 or |e ln2| - 0.35) */
    const double bh = ah + s1;
    const double bl = s1 - (bh - ah);
    double lo = fma(ed, CRLOG_LN2_MID, t2) + al;
    lo = lo + bl;
    lo = lo + lo1;
    const double yh = bh + lo;               /* Fast2Sum: |bh| >= |lo| */
    const double yl = lo - (yh - bh);
    const double d = fma(fabs(z3), 0x1p-49, fabs(yh) * 0x1p-88);
    if ((yh + (yl + d)) == (yh + (yl - d))) {
        *fast = 1;
        return yh;
    }
    *fast = 0;
    int ok;
    return or_crlog_accurate(x, &ok);
}

double or_crlog(double x) {
    int fast;
    return or_crlog_ex(x, &fast);
}

/* Diagnostics for tests: over rsq = s / 2^46, s = s0 .. s0 + n - 1, the s
 * whose fast phase fails (up to cap of them, returns the total count). */
uint64_t or_crlog_scan(uint64_t s0, uint64_t n, uint64_t* fails, uint64_t cap) {
    uint64_t c = 0;
    for (uint64_t k = 0; k < n; ++k) {
        const double x = (double)(s0 + k) * 0x1p-46;
        int fast;
        (void)or_crlog_ex(x, &fast);
        if (!fast) {
            if (c < cap) fails[c] = s0 + k;
            ++c;
        }
    }
    return c;
}

int or_gauss_use_libm_log = 0; /* diagnostic: 1 = glibc log() instead of or_crlog */
/* set by or_gaussian for each NEW pair: glibc's log(rsq) != or_crlog(rsq) */
int or_gauss_last_log_differs = 0;

/* Repo-defined gaussian(): Marsaglia polar method on uniform() = next_f64
 * (core.hpp:70-72). Pair convention as in Numerical Recipes' gasdev: draw
 * v1 then v2 (each 2u-1), reject while rsq >= 1 or rsq == 0, return v2*fac
 * and cache v1*fac for the next call (LAMMPS RanMars::gaussian's form); log
 * is the correctly rounded or_crlog above, every other operation a single
 * IEEE binary64 operation. */
double or_gaussian(or_gauss_state* g) {
    if (g->has_saved) {
        g->has_saved = 0;
        return g->saved;
    }
    double v1, v2, rsq;
    do {
        v1 = 2.0 * ((double)or_step(&g->s) * 0x1p-24) - 1.0;
        v2 = 2.0 * ((double)or_step(&g->s) * 0x1p-24) - 1.0;
        rsq = v1 * v1 + v2 * v2;
    } while (rsq >= 1.0 || rsq == 0.0);
    const double lg = or_gauss_use_libm_log ? log(rsq) : or_crlog(rsq);
    or_gauss_last_log_differs = or_gauss_use_libm_log && lg != or_crlog(rsq);
    const double fac = sqrt(-2.0 * lg / rsq);
    g->saved = v1 * fac;
    g->has_saved = 1;
    return v2 * fac;
}

void or_gaussian_fill(or_gauss_state* g, uint64_t n_atoms, uint64_t per_step, uint64_t steps,
                      double* out) {
    or_gaussian_fill_flags(g, n_atoms, per_step, steps, out, NULL);
}

/* The same, and (libm mode) flags[idx] = 1 when deviate idx comes from a pair
 * whose rsq has glibc log(rsq) != correctly rounded log(rsq). A deviate
 * cached before the call counts as unflagged. */
void or_gaussian_fill_flags(or_gauss_state* g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* out, uint8_t* flags) {
    for (uint64_t a = 0; a < n_atoms; ++a) {
        int pending = 0;
        for (uint64_t st = 0; st < steps; ++st)
            for (uint64_t c = 0; c < per_step; ++c) {
                const uint64_t idx = (st * n_atoms + a) * per_step + c;
                const int cached = g[a].has_saved != 0;
                out[idx] = or_gaussian(&g[a]);
                if (flags) {
                    flags[idx] = (uint8_t)(cached ? pending : or_gauss_last_log_differs);
                    if (!cached) pending = or_gauss_last_log_differs;
                }
            }
    }
}

/* Repo-defined fix-langevin-style consumer (no
 * reference counterpart, LAMMPS is not in the container). One stream per atom;
 * atoms outside the group draw nothing. Every operation rounds separately
 * (-ffp-contract=off); the device kernel langevin_kernel performs the same
 * sequence. noise 0: r = uniform() - 0.5; noise 1: r = gaussian(). */
int or_langevin(or_gauss_state* g, uint64_t n_atoms, const double* v, double* f,
                const int32_t* type, const int32_t* mask, int32_t groupbit,
                const double* gfactor1, const double* gfactor2, int32_t n_types, double tsqrt,
                int noise) {
    int bad_type = 0;
    for (uint64_t a = 0; a < n_atoms; ++a) {
        if (mask && !(mask[a] & groupbit)) continue;
        const int32_t t = type[a];
        if (t < 0 || t > n_types) {
            bad_type = 1;
            continue;
        }
        const double g1 = gfactor1[t];
        const double g2 = gfactor2[t] * tsqrt;
        for (int d = 0; d < 3; ++d) {
            const double r = noise ? or_gaussian(&g[a])
                                   : (double)or_step(&g[a].s) * 0x1p-24 - 0.5;
            const double fd = g1 * v[3 * a + d] + g2 * r;
            f[3 * a + d] = f[3 * a + d] + fd;
        }
    }
    return bad_type;
}

/* ---------------------------------------------------------- text state --- */

/* serialize.hpp:21-40: "ranmar24 v1", 1-based cursors, v, 97 lanes. */
long or_to_text(const or_state* s, char* buf, long cap) {
    long n = snprintf(buf, (size_t)cap, "ranmar24 v1\ni %d j %d\nv %u\n", s->i + 1, s->j + 1,
                      s->v);
    if (n < 0 || n >= cap) return -1;
    for (int k = 0; k < 97; ++k) {
        const int w = snprintf(buf + n, (size_t)(cap - n), "u %d %u\n", k + 1, s->lane[k]);
        if (w < 0 || w >= cap - n) return -1;
        n += w;
    }
    return n;
}

/* serialize.hpp:81-136 (strict parser); returns 0 or 1 (invalid_argument). */
static const char* or_line(const char** text, int* len) {
    const char* t = *text;
    if (!*t) return NULL;
    const char* nl = strchr(t, '\n');
    const int n = nl ? (int)(nl - t) : (int)strlen(t);
    *text = nl ? nl + 1 : t + n;
    *len = (n > 0 && t[n - 1] == '\r') ? n - 1 : n;
    return t;
}

static int or_take_uint(const char** p, const char* end, uint64_t* v) {
    uint64_t x = 0;
    int n = 0;
    while (*p < end && **p >= '0' && **p <= '9') {
        x = x * 10 + (uint64_t)(**p - '0');
        if (x > 0xFFFFFFFFull) return 1;
        ++*p;
        ++n;
    }
    if (n == 0) return 1;
    *v = x;
    return 0;
}

static int or_take_lit(const char** p, const char* end, const char* lit) {
    const size_t n = strlen(lit);
    if ((size_t)(end - *p) < n || strncmp(*p, lit, n) != 0) return 1;
    *p += n;
    return 0;
}

int or_from_text(const char* text, or_state* out) {
    int len;
    const char* l = or_line(&text, &len);
    if (!l || len != 11 || strncmp(l, "ranmar24 v1", 11) != 0) return 1;
    memset(out, 0, sizeof *out);
    uint64_t i, j, v;
    if (!(l = or_line(&text, &len))) return 1;
    const char* p = l;
    const char* e = l + len;
    if (or_take_lit(&p, e, "i ") || or_take_uint(&p, e, &i) || or_take_lit(&p, e, " j ") ||
        or_take_uint(&p, e, &j) || p != e)
        return 1;
    if (i < 1 || i > 97 || j < 1 || j > 97) return 1;
    if ((i + 97 - j) % 97 != 64) return 1;
    out->i = (int32_t)i - 1;
    out->j = (int32_t)j - 1;
    if (!(l = or_line(&text, &len))) return 1;
    p = l;
    e = l + len;
    if (or_take_lit(&p, e, "v ") || or_take_uint(&p, e, &v) || p != e) return 1;
    if (v >= OR_ARITH_MOD) return 1;
    out->v = (uint32_t)v;
    for (int k = 0; k < 97; ++k) {
        uint64_t idx, lane;
        if (!(l = or_line(&text, &len))) return 1;
        p = l;
        e = l + len;
        if (or_take_lit(&p, e, "u ") || or_take_uint(&p, e, &idx) || or_take_lit(&p, e, " ") ||
            or_take_uint(&p, e, &lane) || p != e)
            return 1;
        if (idx != (uint64_t)k + 1) return 1;
        if (lane > OR_MASK) return 1;
        out->lane[k] = (uint32_t)lane;
    }
    for (; *text; ++text)
        if (*text != '\n' && *text != '\r' && *text != ' ' && *text != '\t') return 1;
    return 0;
}
