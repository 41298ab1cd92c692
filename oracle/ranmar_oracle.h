/* TEST INFRASTRUCTURE ONLY (oracle/). The product never includes, links or
 * calls this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it, and only as the checker.
 *
 * Plain-C restatement of the reference's CPU algorithm for the hot path
 * (arXiv 2512.00093, /root/reference/proj/include/ranmar). Every function
 * cites the reference file:line it restates. Pinned against the reference's
 * frozen known answers (tests/golden/known_answers.json) and against the
 * reference itself compiled in place (oracle/_ref/libranmar_ref.so, fixtures
 * in tests/golden/ref_vectors.json made by oracle/gen_golden.py).
 *
 * The one function with no reference counterpart is or_gaussian_*: the
 * reference has no gaussian(). Its convention
 * (Marsaglia polar, Numerical-Recipes "gasdev" pairing) is defined HERE and
 * is therefore "parity unpinned" against LAMMPS.
 */
#ifndef RANMAR_ORACLE_H
#define RANMAR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* core.hpp:17-24 */
#define OR_LONG_LAG 97
#define OR_SHORT_LAG 33
#define OR_MASK 0x00FFFFFFu
#define OR_ARITH_MOD 16777213u
#define OR_ARITH_DELTA 7654321u
#define OR_ARITH_START 362436u
#define OR_MAX_SEED 900000000u

/* core.hpp:29-49 — byte-identical to ranmar::RanmarState (400 B). */
typedef struct or_state {
    uint32_t lane[97];
    int32_t i, j;
    uint32_t v;
} or_state;

/* Jump count J: 256-bit little-endian limbs (jumpcount.hpp:13 uses an
 * unbounded cpp_int; the generator period is ~2^144). */
typedef struct or_j256 {
    uint64_t limb[4];
} or_j256;

/* Returns 0, or 1 where the reference throws std::invalid_argument. */
int or_init(uint32_t seed, or_state* out);
/* Same arithmetic without the seed range check (for BASELINE config 3). */
void or_init_unchecked(uint32_t seed, or_state* out);
uint32_t or_step(or_state* s);
void or_step_n(or_state* s, uint64_t n, uint32_t* out);
int or_value_of(uint32_t u24, double* out);

/* Float recurrence (reference/float_ranmar.hpp:33-80). */
typedef struct or_float_state {
    double x[97];
    double c;
    int32_t i, j;
} or_float_state;
int or_init_float(uint32_t seed, or_float_state* out);
double or_step_float(or_float_state* s);
void or_step_float_n(or_float_state* s, uint64_t n, double* out);

/* Polynomial ring Z/2^24[t]/(t^97 + t^64 - 1) (polyring.hpp:60-124). */
void or_reduce_trinomial(const uint32_t* raw, int n, uint32_t* out97);
void or_mul_mod(const uint32_t* a, const uint32_t* b, uint32_t* out97);
void or_mul_by_t(const uint32_t* p, uint32_t* out97);
void or_pow_t_mod(const or_j256* j, uint32_t* out97);

/* Jump (jump.hpp:32-124). */
void or_canonicalize(const or_state* s, uint32_t* u97);
void or_decanonicalize(const uint32_t* u97, or_state* out /* lanes, i, j only */);
void or_apply_companion(const uint32_t* u97, uint32_t* out97);
void or_jump_fib(const uint32_t* u97, const or_j256* j, uint32_t* out97);
uint32_t or_jump_arith(uint32_t v, const or_j256* j);
void or_jump_state(const or_state* in, const or_j256* j, or_state* out);
/* Streams [first, first + n) of make_streams(base, J); both StreamModes agree. */
int or_make_streams(const or_state* base, const or_j256* j, uint64_t first, uint64_t n,
                    or_state* out);

/* Jump-count helpers. */
void or_j256_from_u64(uint64_t x, or_j256* out);
int or_j256_parse(const char* text, or_j256* out); /* jumpcount.hpp:16-47 */
void or_j256_mul_u64(const or_j256* a, uint64_t k, or_j256* out);
void or_j256_add(const or_j256* a, const or_j256* b, or_j256* out);
int or_j256_is_zero(const or_j256* a);
int or_j256_msb(const or_j256* a); /* -1 for zero */
uint32_t or_j256_mod_u32(const or_j256* a, uint32_t m);

/* Workloads (BASELINE configs), stream-major outputs. */
void or_generate_u32(or_state* states, uint64_t n_streams, uint64_t per_stream, uint32_t* out);
void or_generate_f32(or_state* states, uint64_t n_streams, uint64_t per_stream, float* out);
void or_consume(or_state* states, uint64_t n_streams, uint64_t per_stream, uint64_t* sums,
                uint32_t* hist /* n_streams x 256, bin = u >> 16 */);

/* Repo-defined gaussian() (no reference counterpart). */
typedef struct or_gauss_state {
    or_state s;
    double saved;
    uint32_t has_saved;
    uint32_t pad;
} or_gauss_state;
double or_crlog(double x);                    /* correctly rounded log, x > 0 normal */
double or_crlog_ex(double x, int* fast);      /* *fast: the fast phase decided */
double or_crlog_accurate(double x, int* ok);  /* accurate phase alone */
uint64_t or_crlog_scan(uint64_t s0, uint64_t n, uint64_t* fails, uint64_t cap);
extern int or_gauss_use_libm_log;
double or_gaussian(or_gauss_state* g);
/* Repo-defined fix-langevin-style consumer; returns 1 if an atom type was out
 * of [0, n_types] (that atom is skipped). */
int or_langevin(or_gauss_state* g, uint64_t n_atoms, const double* v, double* f,
                const int32_t* type, const int32_t* mask, int32_t groupbit,
                const double* gfactor1, const double* gfactor2, int32_t n_types, double tsqrt,
                int noise);
void or_gaussian_fill(or_gauss_state* g, uint64_t n_atoms, uint64_t per_step, uint64_t steps,
                      double* out /* [step][atom][per_step] */);
void or_gaussian_fill_flags(or_gauss_state* g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* out, uint8_t* flags);

/* Text state (serialize.hpp:21-136). */
long or_to_text(const or_state* s, char* buf, long cap);
int or_from_text(const char* text, or_state* out);

#ifdef __cplusplus
}
#endif
#endif
