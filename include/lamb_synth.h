/*
 * lamb_synth.h — seeded synthetic inputs for tests and the bench (NOT part of the method).
 *
 * Fills a handle's buffers on the device with the input recipe of DESIGN.md §4 (SURVEY.md
 * §8(d)): Philox4x32-10 (Salmon et al. SC'11, Random123 definition) keyed by
 *   key = (seed & 0xFFFFFFFF, (seed >> 32) ^ (stream << 24) ^ rank_term)
 *   ctr = (q & 0xFFFFFFFF, q >> 32, tensor_id, step),  q = e / 4, word e % 4,
 * where e is the element index inside its tensor (independent of layout and world size).
 * The CPU oracle implements the same generator separately (oracle/lamb_oracle.c); the two
 * are pinned independently by Random123 known-answer vectors.
 */
#ifndef LAMB_SYNTH_H_
#define LAMB_SYNTH_H_

#include <stdint.h>
#include "lamb.h"

#ifdef __cplusplus
extern "C" {
#endif

#define LAMB_INIT_UNIFORM 0   /* w = (int(x >> 8) - 2^23) * 2^-28, uniform on [-1/32, 1/32) */
#define LAMB_INIT_ONE 1       /* w = 1 */
#define LAMB_INIT_ZERO 2      /* w = 0 */

typedef struct {
    int32_t init;   /* LAMB_INIT_* */
    int32_t gexp;   /* gradient exponent base E: value = +-(1 + mant/128) * 2^(E - ((x>>5)&3)),
                       0 when (x & 0xF) == 0 */
} lamb_synth_tensor;

/* Initialises the master weights from the generator (stream 1, step 0, rank_term 0): this
 * rank's w slices, m = v = 0, the whole bf16 param buffer.  spec[n_tensors] is host memory.
 * Marks the master as set (like lamb_set_master).  Synchronises `stream`. */
lamb_status lamb_synth_init(lamb_t h, const lamb_synth_tensor* spec, uint64_t seed, void* stream);

/* Writes the generator's bf16 gradients (stream 2) for `step` and `rank_term` (0 for
 * REPLICATED inputs, rank + 1 for PER_RANK) into the library grad buffer; padding = 0.
 * Asynchronous on `stream`. */
lamb_status lamb_synth_grads(lamb_t h, const lamb_synth_tensor* spec, uint64_t seed,
                             uint32_t rank_term, uint32_t step, void* stream);

/* Philox4x32-10 of one (ctr, key) on the DEVICE (known-answer test of the GPU generator).
 * ctr[4], key[2], out[4] are host arrays.  Synchronous. */
lamb_status lamb_synth_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* LAMB_SYNTH_H_ */
