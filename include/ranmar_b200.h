/* ranmar_b200.h — C ABI of the B200-native RANMAR generator + exact jump-ahead.
 *
 * Drop-in boundary for the reference library ranmar24
 * (/root/reference/proj/include/ranmar, header-only C++20, arXiv 2512.00093).
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj). Plain C types only: no torch, no C++.
 *
 * Conventions
 *  - Return value: RANMAR_OK (0) or a RANMAR_E* code; ranmar_last_error()
 *    gives a thread-local message. RANMAR_EINVAL is returned exactly where
 *    the reference throws std::invalid_argument (SURVEY §8b "Errors").
 *  - "_dev" functions take device pointers and a cudaStream_t passed as
 *    void*; they run on the CURRENT device (cudaSetDevice), are asynchronous
 *    and stream-ordered, never allocate, never synchronise and never read
 *    device memory back to the host, so a sequence of them can be captured
 *    in a CUDA graph. They need the device's one-time resources from
 *    ranmar_device_setup(device, stream) (else RANMAR_ESTATE). There is no
 *    CPU fallback: without a usable CUDA device they return RANMAR_ECUDA.
 *  - "ranmar_ctx_*" functions take HOST buffers and do the host<->device
 *    copies themselves (pinned/pageable both accepted), synchronously.
 *  - Stream-major output layout: out[k * per_stream + n] is output n (0-based)
 *    of stream k.
 */
#ifndef RANMAR_B200_H
#define RANMAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RANMAR_ABI_VERSION 2

enum {
    RANMAR_OK = 0,
    RANMAR_EINVAL = 1, /* the reference throws std::invalid_argument here */
    RANMAR_ERANGE = 2, /* jump count or size outside what the ABI represents */
    RANMAR_ECUDA = 3,  /* CUDA runtime/launch failure or no device */
    RANMAR_ESTATE = 4, /* a device state violated the invariants (see ranmar_device_status) */
    RANMAR_ENOMEM = 5  /* workspace too small / allocation failed */
};

/* ranmar::RanmarState (core.hpp:29-49), byte-identical: 97 lanes < 2^24 in a
 * ring, 0-based cursors i, j with (i - j) mod 97 == 64, arithmetic residue
 * v < 2^24 - 3. sizeof == 400. */
typedef struct ranmar_state {
    uint32_t lane[97];
    int32_t i;
    int32_t j;
    uint32_t v;
} ranmar_state;

/* ranmar::JumpCount (jumpcount.hpp:13, an unbounded cpp_int) as 256-bit
 * little-endian limbs; the generator's period is ~2^144. */
typedef struct ranmar_jump_count {
    uint64_t limb[4];
} ranmar_jump_count;

/* State + the cached second polar deviate of gaussian() (416 B). */
typedef struct ranmar_gauss_state {
    ranmar_state s;
    double saved;
    uint32_t has_saved;
    uint32_t pad;
} ranmar_gauss_state;

/* ranmar::reference::FloatState (reference/float_ranmar.hpp:22-29): the
 * classic floating-point generator, 97 doubles + c + cursors (792 B). */
typedef struct ranmar_float_state {
    double x[97];
    double c;
    int32_t i;
    int32_t j;
} ranmar_float_state;

typedef struct ranmar_ctx ranmar_ctx;

/* ------------------------------------------------------------ host, no GPU */
int ranmar_abi_version(void);
const char* ranmar_last_error(void);

/* ranmar::init(seed)             init.hpp:18-51 (EINVAL if seed > 900000000, :19-20) */
int ranmar_init(uint32_t seed, ranmar_state* out);
/* Same seed expansion without the range check (BASELINE config 3 uses seed
 * 987654321, which ranmar::init rejects; documented deviation). */
int ranmar_init_unchecked(uint32_t seed, ranmar_state* out);
/* ranmar::reference::init_float(seed) float_ranmar.hpp:50-80 (EINVAL above
 * 900000000): x[k] = lane/2^24, c = 362436/2^24, the float image of init. */
int ranmar_init_float(uint32_t seed, ranmar_float_state* out);
/* ranmar::value_of(u24)          core.hpp:75-79 (EINVAL if u24 > 2^24-1) */
int ranmar_value_of(uint32_t u24, double* out);
/* ranmar::parse_jump_count(text) jumpcount.hpp:16-47 (EINVAL on bad text;
 * ERANGE if the value does not fit 256 bits) */
int ranmar_parse_jump_count(const char* text, ranmar_jump_count* out);
/* ranmar::jump_arith(a, J).v     jump.hpp:79-86 (closed form, host) */
int ranmar_jump_arith(uint32_t v, const ranmar_jump_count* j, uint32_t* out);
/* ranmar::to_text / from_text    serialize.hpp:21-40 / :81-136. to_text
 * returns the length written (cap must hold it + NUL) or -1. */
long ranmar_to_text(const ranmar_state* s, char* buf, long cap);
int ranmar_from_text(const char* text, ranmar_state* out);

/* -------------------------------------------------- device ops (async) --- */

/* One-time, per-device setup for the _dev entry points (allocates and
 * synchronises; idempotent, thread-safe): the sticky status word and the
 * table of t^(2^k) mod the characteristic polynomial that every jump uses
 * (the squarings of polyring.hpp:113-124, ~0.3 ms). `stream` belongs to
 * `device`; the caller's current device is restored. ranmar_ctx_create calls it. */
int ranmar_device_setup(int device, void* stream);

/* Workspace bytes needed by ranmar_make_streams_dev / ranmar_jump_dev for n
 * streams. */
size_t ranmar_make_streams_workspace(uint64_t n);

/* Streams [first, first + n) of ranmar::make_streams(base, J, ·)
 * (jump.hpp:108-124): stream k starts at s_{kJ} of `base` (a HOST state).
 * Stream 0 is `base` itself, like make_streams' streams.front(); every other
 * stream is in jump_state's normalised layout (jump.hpp:42-48). Both
 * StreamModes give these states (test_jump.cpp:191-196). EINVAL if n == 0 or
 * J == 0 (jump.hpp:111-112). first + n must be < 2^63. */
int ranmar_make_streams_dev(const ranmar_state* base, const ranmar_jump_count* j, uint64_t first,
                            uint64_t n, ranmar_state* d_out, void* d_workspace,
                            size_t workspace_bytes, void* stream);

/* The same with the base state in DEVICE memory (d_base). An invalid base
 * raises the status bit (ranmar_device_status) instead of RANMAR_ESTATE. */
int ranmar_make_streams_from_dev(const ranmar_state* d_base, const ranmar_jump_count* j,
                                 uint64_t first, uint64_t n, ranmar_state* d_out,
                                 void* d_workspace, size_t workspace_bytes, void* stream);

/* d_out[k] = ranmar::jump_state(d_in[k], J) for k < n (jump.hpp:90-95).
 * d_in == d_out is allowed. A state violating the invariants raises the
 * status bit (its output is unspecified; nothing is read outside it). */
int ranmar_jump_dev(const ranmar_state* d_in, ranmar_state* d_out, uint64_t n,
                    const ranmar_jump_count* j, void* d_workspace, size_t workspace_bytes,
                    void* stream);

/* ranmar::poly::pow_t_mod<24>(J) (polyring.hpp:113-124) into d_coeff[97]. */
int ranmar_pow_t_mod_dev(const ranmar_jump_count* j, uint32_t* d_coeff, void* stream);

/* per_stream calls of ranmar::step (core.hpp:54-66) on each of n_streams
 * device states, advancing them in place exactly as step() would (ring
 * contents and cursors included). Outputs: u24 in u32, next_f64 narrowed to
 * f32 (exact), or next_f64 (core.hpp:70-72). */
int ranmar_generate_u32_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            uint32_t* d_out, void* stream);
int ranmar_generate_f32_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            float* d_out, void* stream);
int ranmar_generate_f64_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                            double* d_out, void* stream);

/* per_stream calls of reference::step_float (float_ranmar.hpp:33-46, the
 * classic Algorithm 1 in binary64) on each device float state; bit-identical
 * to the integer path's outputs / 2^24. States advance in place. */
int ranmar_generate_float_dev(ranmar_float_state* d_states, uint64_t n_streams,
                              uint64_t per_stream, double* d_out, void* stream);

/* ONE stream, `count` outputs at full GPU width: the stream is split into
 * substreams of 8,192 outputs starting at s_{k 8192} (make_streams), so the
 * outputs land in order in d_out[0 .. count), and *d_state (device) ends
 * exactly as `count` calls of step() leave it (same ring layout). d_ws:
 * ranmar_generate_single_workspace(count) bytes (0 for count <= 8192). The
 * state stays on the device (an invalid one raises the status bit). */
size_t ranmar_generate_single_workspace(uint64_t count);
int ranmar_generate_single_u32_dev(ranmar_state* d_state, uint64_t count, uint32_t* d_out,
                                   void* d_ws, size_t ws_bytes, void* stream);
int ranmar_generate_single_f32_dev(ranmar_state* d_state, uint64_t count, float* d_out,
                                   void* d_ws, size_t ws_bytes, void* stream);

/* Consume-in-kernel (no uniform is stored): per stream, the u64 sum of its
 * per_stream 24-bit outputs and a 256-bin histogram of (u >> 16);
 * d_hist is n_streams x 256 u32. States advance in place. */
int ranmar_consume_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                       uint64_t* d_sums, uint32_t* d_hist, void* stream);

/* gaussian() (no reference counterpart; Marsaglia polar, NR gasdev pairing):
 * for each atom, steps x per_step calls; d_out[(step * n_atoms + atom) *
 * per_step + c] (per_step < 2^32). States (and the cached deviate) advance in
 * place. */
int ranmar_gaussian_f64_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t per_step,
                            uint64_t steps, double* d_out, void* stream);

/* gaussian() consumed in-kernel (no reference counterpart):
 * for each atom, count gaussian() calls (the cached deviate first, as
 * ranmar_gaussian_f64_dev with per_step = count, steps = 1) summed in call
 * order, d_out[2 atom] = s1, d_out[2 atom + 1] = s2 with s1 = RN(s1 + x),
 * s2 = RN(s2 + RN(x * x)); nothing else is stored. States and caches advance
 * exactly as that ranmar_gaussian_f64_dev call would leave them. */
int ranmar_gaussian_moments_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, uint64_t count, double* d_out,
                                void* stream);

/* Fix-langevin-style per-atom consumer (no reference counterpart; SURVEY
 * §8f rows 3-4): one stream per atom, uniforms/gaussians consumed in-kernel.
 * For each atom a with d_mask == NULL or (d_mask[a] & groupbit) != 0, with
 * t = d_type[a] in [0, n_types], g1 = d_gfactor1[t], g2 = d_gfactor2[t] * tsqrt:
 *   for d = 0..2:  r = uniform() - 0.5      (RANMAR_NOISE_UNIFORM)
 *                  r = gaussian()           (RANMAR_NOISE_GAUSSIAN)
 *                  d_f[3a+d] = d_f[3a+d] + (g1 * d_v[3a+d] + g2 * r)
 * every operation rounded separately. d_v, d_f are n_atoms x 3 doubles
 * (LAMMPS v[i][d], f[i][d]); d_gfactor* hold n_types + 1 doubles. States
 * advance in place; a type outside [0, n_types] sets status bit 2. */
#define RANMAR_NOISE_UNIFORM 0
#define RANMAR_NOISE_GAUSSIAN 1
int ranmar_langevin_dev(ranmar_gauss_state* d_g, uint64_t n_atoms, const double* d_v,
                        double* d_f, const int32_t* d_type, const int32_t* d_mask,
                        int32_t groupbit, const double* d_gfactor1, const double* d_gfactor2,
                        int32_t n_types, double tsqrt, int noise, void* stream);

/* The same force update with gaussian noise drawn beforehand: d_noise holds
 * this step's 3 deviates per atom (n_atoms x 3 f64, e.g. the slice
 * out + step * 3 n_atoms of one ranmar_gaussian_f64_dev launch with
 * per_step = 3 over many steps). Equal to ranmar_langevin_dev with
 * RANMAR_NOISE_GAUSSIAN, step by step, when every atom is in the group at every
 * step (replaces: the fix-langevin loop of PAPER.md:46-47, repo convention). */
int ranmar_langevin_noise_dev(uint64_t n_atoms, const double* d_noise, const double* d_v,
                              double* d_f, const int32_t* d_type, const int32_t* d_mask,
                              int32_t groupbit, const double* d_gfactor1, const double* d_gfactor2,
                              int32_t n_types, double tsqrt, void* stream);

/* Stream bank: n streams transposed slot-major (99 u32 words per stream:
 * 97 ring slots, v, the initial cursor) for consumers that draw the same
 * number of outputs from every stream per launch, so every access of a launch
 * is coalesced. t = outputs drawn from each stream since from_states; the
 * round trip to_states(from_states(S), t) is byte-identical to t calls of
 * step() on each state. ranmar_langevin_bank_dev is ranmar_langevin_dev with
 * RANMAR_NOISE_UNIFORM, no mask, on a bank (every stream draws 3 outputs; an
 * atom with a bad type keeps its force, is flagged, and still draws); it
 * returns with the bank at t + 3. */
uint64_t ranmar_bank_words(uint64_t n);
int ranmar_bank_from_states_dev(const ranmar_state* d_states, uint64_t n, uint32_t* d_bank,
                                void* stream);
int ranmar_bank_to_states_dev(const uint32_t* d_bank, uint64_t n, uint64_t t,
                              ranmar_state* d_states, void* stream);
int ranmar_langevin_bank_dev(uint32_t* d_bank, uint64_t n_atoms, uint64_t t, const double* d_v,
                             double* d_f, const int32_t* d_type, const double* d_gfactor1,
                             const double* d_gfactor2, int32_t n_types, double tsqrt,
                             void* stream);

/* Diagnostic: compares gaussian()'s branch-free fp64 divide / sqrt with the
 * CUDA library's correctly rounded ones on n operand sets drawn from seed
 * (rsq = s / 2^46); adds the number of bitwise mismatches to *d_mismatches. */
int ranmar_fp64_selfcheck_dev(uint64_t n, uint64_t seed, unsigned long long* d_mismatches,
                              void* stream);

/* Diagnostic: exhaustive check of gaussian()'s correctly rounded log on
 * rsq = s / 2^46, s in [s0, s0 + n) (the whole domain is s in [1, 2^46)).
 * Adds to d_counts[0..3]: inputs the fast phase could not decide, inputs the
 * accurate phase could not decide either, (mode 1) fast/accurate disagreements,
 * and the number of inputs recorded in d_fails[0 .. cap) (no particular order):
 * the fast-phase failures (modes 0, 1) or the accurate-phase failures (mode 2). */
int ranmar_crlog_sweep_dev(uint64_t s0, uint64_t n, int32_t mode, unsigned long long* d_counts,
                           uint64_t* d_fails, uint64_t cap, void* stream);

/* The same gaussian() calls for FEW streams with MANY calls each: one warp per
 * stream (serves the scalar RanMars-style facade). d_out[s * count + q] is
 * call q of stream s. States and cached deviates advance in place. */
int ranmar_gaussian_stream_f64_dev(ranmar_gauss_state* d_g, uint64_t n_streams, uint64_t count,
                                   double* d_out, void* stream);

/* Device-side persistence (bulk serialize.hpp:21-136). to_text: d_text gets
 * the concatenated "ranmar24 v1" texts of n device states, d_offsets[0..n]
 * their start offsets (d_offsets[n] = total bytes); text_cap must be at least
 * ranmar_to_text_bound(n). A state violating the invariants (cursors, v,
 * 24-bit lanes) gets an empty text and raises the status bit. from_text: parses texts [d_offsets[k],
 * d_offsets[k+1]) with the reference's strict rules; d_err[k] = 0 or the
 * 1-based line of the first error (where from_text throws invalid_argument),
 * d_states[k] written only on success. */
uint64_t ranmar_to_text_bound(uint64_t n);
size_t ranmar_text_workspace(uint64_t n);
int ranmar_to_text_dev(const ranmar_state* d_states, uint64_t n, char* d_text, uint64_t text_cap,
                       uint64_t* d_offsets, void* d_workspace, size_t workspace_bytes,
                       void* stream);
int ranmar_from_text_dev(const char* d_text, const uint64_t* d_offsets, uint64_t n,
                         ranmar_state* d_states, int32_t* d_err, void* stream);

/* Sticky status bits of the current device (bit 0: a kernel met a state with
 * bad cursors / v >= m; bit 2: ranmar_langevin_dev met an atom type outside
 * [0, n_types]). Synchronises the device. clear != 0 resets them. */
int ranmar_device_status(uint32_t* flags, int clear);

/* Number of kernels this library has launched in this process (all devices);
 * diagnostic evidence for benchmarks ("gpu_launches"). */
uint64_t ranmar_kernel_launches(void);

/* The state isomorphism of float_ranmar.hpp:3-8 on the device: d_out[k] =
 * the float state of d_states[k] (x = lane / 2^24, c = v / 2^24, same
 * cursors), so float streams can start from integer jumps. */
int ranmar_float_from_states_dev(const ranmar_state* d_states, uint64_t n, ranmar_float_state* d_out,
                                 void* stream);

/* Per-step trace for the scalar step()/next_f64() of the C++ facade: for
 * step n of stream k, at index k * per_stream + n: d_u = the output
 * (core.hpp:65), d_x = the word step() writes into lane[i] (core.hpp:56-57),
 * d_v = the residue after the step (core.hpp:61-63). States advance in place. */
int ranmar_generate_trace_dev(ranmar_state* d_states, uint64_t n_streams, uint64_t per_stream,
                              uint32_t* d_u, uint32_t* d_x, uint32_t* d_v, void* stream);
/* The same for reference::step_float (float_ranmar.hpp:33-46): outputs, the
 * values written into x[i] and the new c. */
int ranmar_generate_float_trace_dev(ranmar_float_state* d_states, uint64_t n_streams,
                                    uint64_t per_stream, double* d_out, double* d_y, double* d_c,
                                    void* stream);
/* ranmar::poly on the device: d_out[q] = d_a[q] * d_b[q] mod phi (mul_mod,
 * polyring.hpp:85-98) for q < n (97 words each), and d_out[q] = d_raw[q] mod
 * phi (reduce_trinomial, polyring.hpp:60-80; 193 raw words each). */
int ranmar_poly_mul_mod_dev(const uint32_t* d_a, const uint32_t* d_b, uint32_t* d_out, uint64_t n,
                            void* stream);
int ranmar_poly_reduce_dev(const uint32_t* d_raw, uint32_t* d_out, uint64_t n, void* stream);

/* The calling thread's current CUDA device (cudaGetDevice), for callers that
 * do not include the CUDA runtime headers. */
int ranmar_current_device(int* device);

/* ------------------------------------------- host-buffer ops (sync, e2e) --- */
int ranmar_ctx_create(int device, ranmar_ctx** out);
void ranmar_ctx_destroy(ranmar_ctx* ctx);
/* ranmar::make_streams(seed, J, n) (jump.hpp:108-124) -> h_out[n]. */
int ranmar_ctx_make_streams(ranmar_ctx* ctx, uint32_t seed, const ranmar_jump_count* j,
                            uint64_t first, uint64_t n, ranmar_state* h_out);
/* ranmar::jump_state on host arrays. */
int ranmar_ctx_jump(ranmar_ctx* ctx, const ranmar_state* h_in, ranmar_state* h_out, uint64_t n,
                    const ranmar_jump_count* j);
/* Generation into host memory, pipelined in chunks (copy-out overlapped with
 * generation). h_states advance in place. */
int ranmar_ctx_generate_u32(ranmar_ctx* ctx, ranmar_state* h_states, uint64_t n_streams,
                            uint64_t per_stream, uint32_t* h_out);
int ranmar_ctx_generate_f32(ranmar_ctx* ctx, ranmar_state* h_states, uint64_t n_streams,
                            uint64_t per_stream, float* h_out);
int ranmar_ctx_consume(ranmar_ctx* ctx, ranmar_state* h_states, uint64_t n_streams,
                       uint64_t per_stream, uint64_t* h_sums, uint32_t* h_hist);
/* count gaussian() calls on each of n HOST gauss states (advanced in place),
 * h_out[s * count + q]; one warp per stream on the device. */
int ranmar_ctx_gaussian_stream(ranmar_ctx* ctx, ranmar_gauss_state* h_g, uint64_t n_streams,
                               uint64_t count, double* h_out);
/* Bytes moved host->device and device->host by the last ctx call. */
int ranmar_ctx_last_traffic(ranmar_ctx* ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* Host-buffer forms of the trace, pow_t_mod and poly primitives (the C++
 * facade's step(), reference::step_float(), poly::pow_t_mod / mul_mod /
 * reduce_trinomial). */
int ranmar_ctx_generate_trace(ranmar_ctx* ctx, ranmar_state* h_states, uint64_t n,
                              uint64_t per_stream, uint32_t* h_u, uint32_t* h_x, uint32_t* h_v);
int ranmar_ctx_float_trace(ranmar_ctx* ctx, ranmar_float_state* h_states, uint64_t n,
                           uint64_t per_stream, double* h_out, double* h_y, double* h_c);
int ranmar_ctx_pow_t_mod(ranmar_ctx* ctx, const ranmar_jump_count* j, uint32_t* h_coeff);
int ranmar_ctx_poly_mul_mod(ranmar_ctx* ctx, const uint32_t* h_a, const uint32_t* h_b,
                            uint32_t* h_out, uint64_t n);
int ranmar_ctx_poly_reduce(ranmar_ctx* ctx, const uint32_t* h_raw, uint32_t* h_out, uint64_t n);

/* Host-buffer forms of the trace, pow_t_mod and poly primitives (the C++
 * facade's step(), reference::step_float(), poly::pow_t_mod / mul_mod /
 * reduce_trinomial). */
int ranmar_ctx_generate_trace(ranmar_ctx* ctx, ranmar_state* h_states, uint64_t n,
                              uint64_t per_stream, uint32_t* h_u, uint32_t* h_x, uint32_t* h_v);
int ranmar_ctx_float_trace(ranmar_ctx* ctx, ranmar_float_state* h_states, uint64_t n,
                           uint64_t per_stream, double* h_out, double* h_y, double* h_c);
int ranmar_ctx_pow_t_mod(ranmar_ctx* ctx, const ranmar_jump_count* j, uint32_t* h_coeff);
int ranmar_ctx_poly_mul_mod(ranmar_ctx* ctx, const uint32_t* h_a, const uint32_t* h_b,
                            uint32_t* h_out, uint64_t n);
int ranmar_ctx_poly_reduce(ranmar_ctx* ctx, const uint32_t* h_raw, uint32_t* h_out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* RANMAR_B200_H */
