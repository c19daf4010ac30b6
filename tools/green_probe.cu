// green_probe.cu — can a kernel launched into a green-context stream (a real SM partition,
// CUDA 12.4+ driver API) use memory from the primary context, and does it stay on its SMs?
// Probe for NEXT #2 (overlap): prints JSON.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/green_probe tools/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

#define CU(x)                                                                  \
    do {                                                                       \
        CUresult r = (x);                                                      \
        if (r != CUDA_SUCCESS) {                                               \
            const char* s = nullptr;                                           \
            cuGetErrorString(r, &s);                                           \
            printf("{\"error\": \"%s: %s\"}\n", #x, s ? s : "?");              \
            return 0;                                                          \
        }                                                                      \
    } while (0)

__global__ void probe(int* smids, float* buf, int n) {
    int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) smids[blockIdx.x] = smid;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = 2.f * buf[i] + 1.f;
}

int main() {
    CU(cuInit(0));
    CUdevice dev;
    CU(cuDeviceGet(&dev, 0));
    cudaSetDevice(0);
    cudaFree(0);
    const int n = 1 << 24, blocks = 1024;
    float* buf;
    int* smids;
    cudaMalloc(&buf, n * 4);
    cudaMalloc(&smids, blocks * 4);
    std::vector<float> h(n, 1.f);
    cudaMemcpy(buf, h.data(), n * 4, cudaMemcpyHostToDevice);
    CUdevResource res;
    CU(cuDeviceGetDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM));
    unsigned int ngroups = 1;
    CUdevResource part, rest;
    CU(cuDevSmResourceSplitByCount(&part, &ngroups, &res, &rest, 0, 32));
    CUdevResourceDesc desc;
    CU(cuDevResourceGenerateDesc(&desc, &part, 1));
    CUgreenCtx g;
    CU(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s;
    CU(cuGreenCtxStreamCreate(&s, g, CU_STREAM_NON_BLOCKING, 0));
    probe<<<blocks, 256, 0, (cudaStream_t)s>>>(smids, buf, n);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)s);
    std::vector<int> sm(blocks);
    cudaMemcpy(sm.data(), smids, blocks * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h.data(), buf, n * 4, cudaMemcpyDeviceToHost);
    std::set<int> used(sm.begin(), sm.end());
    bool ok = true;
    for (int i = 0; i < n; ++i) ok = ok && h[i] == 3.f;
    printf("{\"green_sms\": %u, \"rest_sms\": %u, \"launch\": \"%s\", \"distinct_smids\": %zu, \"data_ok\": %d}\n",
           part.sm.smCount, rest.sm.smCount, cudaGetErrorString(e), used.size(), (int)ok);
    return 0;
}
