/* The C ABI used from plain C: make_streams + generate on
 * the device, checked against the reference's frozen answers (test_core.cpp:
 * 121-123: the first outputs of seed 12345 are stream 0's). Run by
 * tests/test_facade.py on a GPU; exit code 0 = all checks passed. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "ranmar_b200.h"

#define CHECK(x)                                                                   \
    do {                                                                           \
        if (!(x)) {                                                                \
            printf("[FAIL] %s:%d: %s (%s)\n", __FILE__, __LINE__, #x, ranmar_last_error()); \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(void) {
    const uint32_t first10[10] = {1905444, 14595391, 174918,   4925251,  346329,
                                  1286474, 5077740,  10808695, 10092480, 6540075};
    ranmar_state base;
    CHECK(ranmar_init(12345, &base) == RANMAR_OK);
    CHECK(ranmar_init(900000001, &base) == RANMAR_EINVAL); /* init.hpp:19-20 */
    CHECK(ranmar_init(12345, &base) == RANMAR_OK);
    ranmar_jump_count J;
    CHECK(ranmar_parse_jump_count("2^40", &J) == RANMAR_OK);

    const uint64_t n = 300, per = 64;
    ranmar_state* d_states = NULL;
    uint32_t* d_out = NULL;
    void* d_ws = NULL;
    const size_t ws = ranmar_make_streams_workspace(n);
    CHECK(cudaMalloc((void**)&d_states, n * sizeof(ranmar_state)) == cudaSuccess);
    CHECK(cudaMalloc((void**)&d_out, n * per * sizeof(uint32_t)) == cudaSuccess);
    CHECK(cudaMalloc(&d_ws, ws) == cudaSuccess);
    /* the _dev entry points never allocate: the device's one-time resources
     * come from ranmar_device_setup (RANMAR_ESTATE until then) */
    CHECK(ranmar_make_streams_dev(&base, &J, 0, n, d_states, d_ws, ws, NULL) == RANMAR_ESTATE);
    CHECK(ranmar_device_setup(0, NULL) == RANMAR_OK);
    CHECK(ranmar_make_streams_dev(&base, &J, 0, n, d_states, d_ws, ws, NULL) == RANMAR_OK);
    CHECK(ranmar_generate_u32_dev(d_states, n, per, d_out, NULL) == RANMAR_OK);
    uint32_t* h = (uint32_t*)malloc(n * per * sizeof(uint32_t));
    CHECK(cudaMemcpy(h, d_out, n * per * sizeof(uint32_t), cudaMemcpyDeviceToHost) == cudaSuccess);
    for (int k = 0; k < 10; ++k) CHECK(h[k] == first10[k]);
    /* stream 1 starts 2^40 outputs later: its first output equals jumping the
     * base by 2^40 on the host-buffer path */
    ranmar_ctx* ctx = NULL;
    CHECK(ranmar_ctx_create(0, &ctx) == RANMAR_OK);
    ranmar_state s1;
    CHECK(ranmar_ctx_jump(ctx, &base, &s1, 1, &J) == RANMAR_OK);
    uint32_t one = 0;
    CHECK(ranmar_ctx_generate_u32(ctx, &s1, 1, 1, &one) == RANMAR_OK);
    CHECK(one == h[per]);
    uint32_t flags = 1;
    CHECK(ranmar_device_status(&flags, 1) == RANMAR_OK && flags == 0);
    ranmar_ctx_destroy(ctx);
    free(h);
    cudaFree(d_states);
    cudaFree(d_out);
    cudaFree(d_ws);
    printf("abi_example: all checks passed\n");
    return 0;
}
