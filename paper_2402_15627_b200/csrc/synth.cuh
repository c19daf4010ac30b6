// synth.cuh — device tables for the synthetic-input generator (internal).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lamb {

struct SynthTables {
    const int64_t* tensor_off;   // [T] flat offsets
    const int64_t* numel;        // [T]
    const int32_t* init;         // [T]
    const int32_t* gexp;         // [T]
    int64_t n_tensors;
    const int64_t* shard_base;   // [B]
    const int64_t* bucket_base;  // [B]
    const int64_t* bucket_slice; // [B]  S_b / D
    int64_t n_buckets;
    int32_t rank;
};

cudaError_t synth_grads(const SynthTables& t, uint64_t seed, uint32_t rank_term, uint32_t step,
                        uint16_t* grad, int64_t flat, cudaStream_t s);
cudaError_t synth_init(const SynthTables& t, uint64_t seed, __nv_bfloat16* params, int64_t flat,
                       float* w, int64_t shard, cudaStream_t s);
cudaError_t synth_philox(const uint32_t* in6_dev, uint32_t* out4_dev);

}  // namespace lamb
