// synth.cu — seeded synthetic inputs on the device (include/lamb_synth.h).  Not part of the
// method: it writes the grads/weights the bench and the GPU tests feed to lamb_step.
// Philox4x32-10 per Salmon et al. (SC'11); keying per DESIGN.md §4.  Implemented here
// independently of the oracle's generator; both are pinned by Random123 KAT vectors.
#include <cuda_runtime.h>

#include <cstdint>

#include "synth.cuh"

namespace lamb {

__host__ __device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t a = 0xD2511F53ull * c[0];
        const uint64_t b = 0xCD9E8D57ull * c[2];
        const uint32_t x0 = (uint32_t)(b >> 32) ^ c[1] ^ k0;
        const uint32_t x1 = (uint32_t)b;
        const uint32_t x2 = (uint32_t)(a >> 32) ^ c[3] ^ k1;
        const uint32_t x3 = (uint32_t)a;
        c[0] = x0; c[1] = x1; c[2] = x2; c[3] = x3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// 4 words for elements e = 4q .. 4q+3 of `tensor` (e is the index inside the tensor)
__device__ __forceinline__ void gen4(uint64_t seed, uint32_t stream, uint32_t rank_term,
                                     uint32_t tensor, uint32_t step, uint64_t q, uint32_t out[4]) {
    out[0] = (uint32_t)q;
    out[1] = (uint32_t)(q >> 32);
    out[2] = tensor;
    out[3] = step;
    philox10(out, (uint32_t)seed, (uint32_t)(seed >> 32) ^ (stream << 24) ^ rank_term);
}

__device__ __forceinline__ int find_tensor(const int64_t* off, int64_t T, int64_t f) {
    int64_t lo = 0, hi = T - 1;   // last tensor with off <= f
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= f) lo = mid; else hi = mid - 1;
    }
    return (int)lo;
}

__device__ __forceinline__ uint16_t grad_bits(uint32_t x, int gexp) {
    if ((x & 0xFu) == 0u) return 0;
    const uint32_t sign = (x >> 4) & 1u;
    const int ex = gexp - (int)((x >> 5) & 3u);
    const uint32_t mant = (x >> 7) & 0x7Fu;
    return (uint16_t)((sign << 15) | ((uint32_t)(ex + 127) << 7) | mant);
}

__device__ __forceinline__ float weight_val(uint32_t x, int init) {
    if (init == 1) return 1.0f;
    if (init == 2) return 0.0f;
    const int k = (int)(x >> 8) - 8388608;
    return (float)k * 3.7252902984619140625e-09f;   // 2^-28, exact
}

// flat bf16 grads: one thread per 4 flat elements (tensor starts are 8-aligned so the 4
// elements share one Philox call)
__global__ void synth_grads_kernel(SynthTables t, uint64_t seed, uint32_t rank_term, uint32_t step,
                                   uint16_t* __restrict__ grad, int64_t flat) {
    for (int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; f < flat;
         f += (int64_t)gridDim.x * blockDim.x * 4) {
        const int i = find_tensor(t.tensor_off, t.n_tensors, f);
        const int64_t e = f - t.tensor_off[i];
        uint16_t o[4] = {0, 0, 0, 0};
        if (e < t.numel[i]) {
            uint32_t x[4];
            gen4(seed, 2u, rank_term, (uint32_t)i, step, (uint64_t)e >> 2, x);
            for (int k = 0; k < 4; ++k)
                if (e + k < t.numel[i]) o[k] = grad_bits(x[k], t.gexp[i]);
        }
        *reinterpret_cast<uint2*>(grad + f) =
            make_uint2((uint32_t)o[0] | ((uint32_t)o[1] << 16), (uint32_t)o[2] | ((uint32_t)o[3] << 16));
    }
}

// fp32 weight for flat element range [f, f+4) -> out[4] (0 in padding)
__device__ __forceinline__ void weights4(const SynthTables& t, uint64_t seed, int64_t f, float out[4]) {
    const int i = find_tensor(t.tensor_off, t.n_tensors, f);
    const int64_t e = f - t.tensor_off[i];
    out[0] = out[1] = out[2] = out[3] = 0.0f;
    if (e < t.numel[i]) {
        uint32_t x[4];
        gen4(seed, 1u, 0u, (uint32_t)i, 0u, (uint64_t)e >> 2, x);
        for (int k = 0; k < 4; ++k)
            if (e + k < t.numel[i]) out[k] = weight_val(x[k], t.init[i]);
    }
}

// whole flat bf16 param buffer
__global__ void synth_params_kernel(SynthTables t, uint64_t seed, __nv_bfloat16* __restrict__ p,
                                    int64_t flat) {
    for (int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; f < flat;
         f += (int64_t)gridDim.x * blockDim.x * 4) {
        float w[4];
        weights4(t, seed, f, w);
        for (int k = 0; k < 4; ++k) p[f + k] = __float2bfloat16_rn(w[k]);
    }
}

// this rank's fp32 w shard: shard index s -> bucket (shard_base) -> flat
__global__ void synth_shard_kernel(SynthTables t, uint64_t seed, float* __restrict__ w, int64_t shard) {
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; s < shard;
         s += (int64_t)gridDim.x * blockDim.x * 4) {
        const int b = find_tensor(t.shard_base, t.n_buckets, s);
        const int64_t f = t.bucket_base[b] + (int64_t)t.rank * t.bucket_slice[b] + (s - t.shard_base[b]);
        float v[4];
        weights4(t, seed, f, v);
        *reinterpret_cast<float4*>(w + s) = make_float4(v[0], v[1], v[2], v[3]);
    }
}

__global__ void philox_kat_kernel(const uint32_t* in, uint32_t* out) {
    uint32_t c[4] = {in[0], in[1], in[2], in[3]};
    philox10(c, in[4], in[5]);
    for (int k = 0; k < 4; ++k) out[k] = c[k];
}

cudaError_t synth_grads(const SynthTables& t, uint64_t seed, uint32_t rank_term, uint32_t step,
                        uint16_t* grad, int64_t flat, cudaStream_t s) {
    synth_grads_kernel<<<148 * 16, 256, 0, s>>>(t, seed, rank_term, step, grad, flat);
    return cudaGetLastError();
}

cudaError_t synth_init(const SynthTables& t, uint64_t seed, __nv_bfloat16* params, int64_t flat,
                       float* w, int64_t shard, cudaStream_t s) {
    synth_params_kernel<<<148 * 16, 256, 0, s>>>(t, seed, params, flat);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    synth_shard_kernel<<<148 * 16, 256, 0, s>>>(t, seed, w, shard);
    return cudaGetLastError();
}

cudaError_t synth_philox(const uint32_t* in6_dev, uint32_t* out4_dev) {
    philox_kat_kernel<<<1, 1>>>(in6_dev, out4_dev);
    return cudaGetLastError();
}

}  // namespace lamb
