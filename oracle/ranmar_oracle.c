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

/* The gaussian convention's log(): a fixed sequence of IEEE operations
 * (binary64 +, -, *, / and fused multiply-add, each correctly rounded) so the
 * device can reproduce it bit for bit. x = 2^k m with m in (sqrt2/2, sqrt2],
 * f = m - 1 (exact), s = f / (2 + f), log1p(f) = 2 atanh(s) with the Taylor
 * series of atanh to s^21 (|s| <= 0.1716, truncation < 2^-60 relative), and
 * k ln2 added as a 42-bit head (exact k * head) plus a tail. Accuracy ~1 ulp
 * (the rounding of s dominates); x must be a positive normal double, which
 * rsq in (0, 1) of the polar method always is (rsq >= 2^-46). */
double or_glog(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    int k = (int)((b >> 52) & 0x7FF) - 1023;
    const uint64_t mb = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    double m;
    memcpy(&m, &mb, 8);
    if (m > 0x1.6a09e667f3bcdp+0) { /* sqrt(2) */
        m *= 0.5;
        k += 1;
    }
    const double f = m - 1.0;
    const double s = f / (2.0 + f);
    const double z = s * s;
    double p = 0x1.8618618618618p-5;     /* 1/21 */
    p = fma(p, z, 0x1.af286bca1af28p-5); /* 1/19 */
    p = fma(p, z, 0x1.e1e1e1e1e1e1ep-5); /* 1/17 */
    p = fma(p, z, 0x1.1111111111111p-4); /* 1/15 */
    p = fma(p, z, 0x1.3b13b13b13b14p-4); /* 1/13 */
    p = fma(p, z, 0x1.745d1745d1746p-4); /* 1/11 */
    p = fma(p, z, 0x1.c71c71c71c71cp-4); /* 1/9 */
    p = fma(p, z, 0x1.2492492492492p-3); /* 1/7 */
    p = fma(p, z, 0x1.999999999999ap-3); /* 1/5 */
    p = fma(p, z, 0x1.5555555555555p-2); /* 1/3 */
    const double t = s * z;
    const double l1p = 2.0 * fma(t, p, s); /* 2 atanh(s) */
    const double kd = (double)k;
    return fma(kd, 0x1.62e42fefa3800p-1, fma(kd, 0x1.ef35793c76730p-45, l1p));
}

int or_gauss_use_libm_log = 0; /* diagnostic: 1 = glibc log() instead of or_glog */

/* Repo-defined gaussian(): Marsaglia polar method on uniform() = next_f64
 * (core.hpp:70-72). Pair convention as in Numerical Recipes' gasdev: draw
 * v1 then v2 (each 2u-1), reject while rsq >= 1 or rsq == 0, return v2*fac
 * and cache v1*fac for the next call; log is or_glog above, every other
 * operation a single IEEE binary64 operation. NOT pinned to LAMMPS (absent). */
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
    const double lg = or_gauss_use_libm_log ? log(rsq) : or_glog(rsq);
    const double fac = sqrt(-2.0 * lg / rsq);
    g->saved = v1 * fac;
    g->has_saved = 1;
    return v2 * fac;
}

void or_gaussian_fill(or_gauss_state* g, uint64_t n_atoms, uint64_t per_step, uint64_t steps,
                      double* out) {
    for (uint64_t a = 0; a < n_atoms; ++a)
        for (uint64_t st = 0; st < steps; ++st)
            for (uint64_t c = 0; c < per_step; ++c)
                out[(st * n_atoms + a) * per_step + c] = or_gaussian(&g[a]);
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
