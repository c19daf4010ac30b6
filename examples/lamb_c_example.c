/*
 * lamb_c_example.c — the C ABI used from plain C (no Python, no torch): one rank, the toy
 * table of BASELINE configs[0] (t0 [64,48] decay, t1 [48] no decay, t2 [128,64] decay), master
 * weights and gradients from the synthetic generator, two LAMB steps on the default stream,
 * then the per-tensor trust ratios and the first master weights read back.
 *
 *   gcc -std=c11 -O2 -I include examples/lamb_c_example.c -o /tmp/lamb_c_example \
 *       -L paper_2402_15627_b200 -llamb -Wl,-rpath,$PWD/paper_2402_15627_b200 -lm
 *   /tmp/lamb_c_example            (needs a B200)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "lamb.h"
#include "lamb_synth.h"

#define CHECK(h, call)                                                                  \
    do {                                                                                \
        lamb_status st_ = (call);                                                       \
        if (st_ != LAMB_OK) {                                                           \
            fprintf(stderr, "%s -> %d: %s\n", #call, (int)st_, lamb_last_error(h));    \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(void) {
    const lamb_tensor tensors[3] = {{64 * 48, 0, 0}, {48, 1, 0}, {128 * 64, 0, 0}};
    /* lr 2^-10, beta1 0.9, beta2 0.999, eps 1e-6; weight decay 0.01 on matrices, 0 on vectors */
    const lamb_group groups[2] = {{0.0009765625f, 0.9f, 0.999f, 1e-6f, 0.01f, 1, 1},
                                  {0.0009765625f, 0.9f, 0.999f, 1e-6f, 0.0f, 1, 1}};
    const lamb_synth_tensor spec[3] = {{LAMB_INIT_UNIFORM, -10}, {LAMB_INIT_ZERO, -8}, {LAMB_INIT_UNIFORM, -10}};
    lamb_config cfg = {1, 0, 0, LAMB_COMM_FUSED, 0, 0.0f, 0};   /* D = 1 on device 0 */
    lamb_t h = NULL;
    CHECK(NULL, lamb_create(tensors, 3, groups, 2, &cfg, NULL, &h));
    lamb_plan_view plan;
    CHECK(h, lamb_query_plan(h, &plan));
    printf("plan: %lld tensors, %lld bucket(s), flat size %lld\n", (long long)plan.n_tensors,
           (long long)plan.n_buckets, (long long)plan.flat_size);
    const uint64_t seed = 0x4D454741ull;   /* BASE_SEED + config index 0 */
    CHECK(h, lamb_synth_init(h, spec, seed, NULL));
    for (int t = 1; t <= 2; ++t) {
        CHECK(h, lamb_synth_grads(h, spec, seed, 1, (uint32_t)t, NULL));   /* PER_RANK, rank 0 */
        CHECK(h, lamb_step(h, NULL, t, NULL));
    }
    double w2[3], u2[3];
    float ratio[3];
    CHECK(h, lamb_get_tensor_stats(h, w2, u2, ratio));
    for (int i = 0; i < 3; ++i)
        printf("tensor %d: ||w|| = %.6f  ||u|| = %.6f  trust ratio = %.6f\n", i, sqrt(w2[i]), sqrt(u2[i]), ratio[i]);
    float* w = (float*)malloc(sizeof(float) * (size_t)plan.shard_size);
    CHECK(h, lamb_get_state(h, LAMB_BUF_W, w, 0, NULL));
    printf("w[0..3] = %.8f %.8f %.8f %.8f\n", w[0], w[1], w[2], w[3]);
    free(w);
    printf("kernels launched: %lld\n", (long long)lamb_launch_count(h));
    lamb_destroy(h);
    return 0;
}
