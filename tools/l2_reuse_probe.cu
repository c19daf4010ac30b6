// l2_reuse_probe.cu — does pass B's re-read of m, v, w hit L2 when it runs right after pass A
// on the same (small enough) tensor?  Streams a pass-A-shaped kernel (read g bf16, m, v, w;
// write m, v) over S elements, then a pass-B-shaped kernel (read m, v, w; write w, p bf16) over
// the same S elements, forward or reverse order, and compares pass B's time with pass B after
// an L2 flush.  Store policy of pass A: streaming (.cs, evict-first) or default.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_reuse_probe tools/l2_reuse_probe.cu
//   tools/l2_reuse_probe            -> one JSON line per (S, A-store policy, B order)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

template <bool CS>
__global__ void passA(const uint2* g, float4* m, float4* v, const float4* w, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const uint2 gg = __ldcs(g + i);
        float4 a = m[i], b = v[i];
        const float4 c = w[i];
        const float gf = __uint_as_float(gg.x << 16) + __uint_as_float(gg.y & 0xffff0000u);
        a.x = 0.9f * a.x + 0.1f * gf + 1e-9f * c.x;
        b.x = 0.999f * b.x + 0.001f * gf * gf + 1e-9f * c.y;
        if (CS) {
            __stcs(m + i, a);
            __stcs(v + i, b);
        } else {
            m[i] = a;
            v[i] = b;
        }
    }
}

template <bool REV>
__global__ void passB(const float4* m, const float4* v, float4* w, uint2* p, int64_t n4) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
        // REV: blocks walk the array from its end (the most recently written lines first)
        const int64_t i = REV ? n4 - 1 - k : k;
        const float4 a = __ldcs(m + i), b = __ldcs(v + i);
        float4 c = __ldcs(w + i);
        c.x -= 1e-3f * a.x / (sqrtf(b.x) + 1e-6f);
        __stcs(w + i, c);
        __stcs(p + i, make_uint2(__float_as_uint(c.x), __float_as_uint(c.y)));
    }
}

__global__ void flush(float4* buf, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_float4(0.f, 1.f, 2.f, 3.f);
}

int main() {
    const int64_t maxS = 64ll << 20;   // elements
    uint2 *g, *p;
    float4 *m, *v, *w, *fl;
    CK(cudaMalloc(&g, maxS * 2));
    CK(cudaMalloc(&p, maxS * 2));
    CK(cudaMalloc(&m, maxS * 4));
    CK(cudaMalloc(&v, maxS * 4));
    CK(cudaMalloc(&w, maxS * 4));
    const int64_t fl4 = (512ll << 20) / 16;   // 512 MB flush buffer
    CK(cudaMalloc(&fl, fl4 * 16));
    CK(cudaMemset(g, 0, maxS * 2));
    CK(cudaMemset(m, 0, maxS * 4));
    CK(cudaMemset(v, 0, maxS * 4));
    CK(cudaMemset(w, 0, maxS * 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = sms * 8, tpb = 256;
    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    for (int64_t S : {1ll << 20, 2ll << 20, 4ll << 20, 6ll << 20, 8ll << 20, 12ll << 20, 16ll << 20, 32ll << 20,
                      64ll << 20}) {
        const int64_t n4 = S / 4;
        for (int cs = 0; cs < 2; ++cs) {
            for (int rev = 0; rev < 3; ++rev) {   // rev 2 = cold pass B (flush between A and B)
                float bestA = 1e30f, bestB = 1e30f;
                for (int rep = 0; rep < 5; ++rep) {
                    flush<<<grid, tpb>>>(fl, fl4);
                    CK(cudaEventRecord(e0));
                    if (cs) passA<true><<<grid, tpb>>>(g, m, v, w, n4);
                    else passA<false><<<grid, tpb>>>(g, m, v, w, n4);
                    CK(cudaEventRecord(e1));
                    if (rev == 2) flush<<<grid, tpb>>>(fl, fl4);
                    cudaEvent_t eb;
                    CK(cudaEventCreate(&eb));
                    CK(cudaEventRecord(eb));
                    if (rev == 1) passB<true><<<grid, tpb>>>(m, v, w, p, n4);
                    else passB<false><<<grid, tpb>>>(m, v, w, p, n4);
                    CK(cudaEventRecord(e2));
                    CK(cudaEventSynchronize(e2));
                    float a, b;
                    CK(cudaEventElapsedTime(&a, e0, e1));
                    CK(cudaEventElapsedTime(&b, eb, e2));
                    CK(cudaEventDestroy(eb));
                    bestA = a < bestA ? a : bestA;
                    bestB = b < bestB ? b : bestB;
                }
                const double bytesB = (double)S * 18.0;
                printf("{\"S_M\": %.0f, \"a_store\": \"%s\", \"b\": \"%s\", \"a_ms\": %.4f, \"b_ms\": %.4f, "
                       "\"b_GBps_algo\": %.0f}\n",
                       S / 1048576.0, cs ? "cs" : "default", rev == 2 ? "cold" : rev ? "reverse" : "forward",
                       bestA, bestB, bytesB / (bestB * 1e-3) / 1e9);
                fflush(stdout);
            }
        }
    }
    return 0;
}
