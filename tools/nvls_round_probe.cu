// nvls_round_probe.cu — what does the NVSwitch return for multimem.ld_reduce...acc::f32.bf16x2?
// (NVLS mode, reading Z23.)  Single process, D GPUs, one multicast object over D buffers: GPU g's
// buffer holds N bf16 inputs (host-generated, seeded), GPU 0 issues the ld_reduce over all N
// positions, and inputs + results are written to a binary file for offline analysis against
// candidate rounding rules (tools/nvls_round_fit.py).  No part of the library or the oracle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_round_probe tools/nvls_round_probe.cu -lcuda
//   /tmp/nvls_round_probe <D> <out.bin>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                                            \
    do {                                                                                                 \
        cudaError_t e = (x);                                                                             \
        if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } \
    } while (0)
#define CU(x)                                                                                            \
    do {                                                                                                 \
        CUresult r = (x);                                                                                \
        if (r != CUDA_SUCCESS) { fprintf(stderr, "%s:%d CUresult %d\n", __FILE__, __LINE__, (int)r); exit(1); } \
    } while (0)

__global__ void reduce_kernel(const uint16_t* mc, uint16_t* out, size_t n, int acc32) {
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i >= n) return;
    uint4 r;
    if (acc32)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc + i) : "memory");
    else
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc + i) : "memory");
    *reinterpret_cast<uint4*>(out + i) = r;
}

static uint16_t bf16_of(float f) {   // inputs are generated exactly representable
    uint32_t b;
    memcpy(&b, &f, 4);
    return (uint16_t)(b >> 16);
}

int main(int argc, char** argv) {
    const int D = argc > 1 ? atoi(argv[1]) : 2;
    const char* path = argc > 2 ? argv[2] : "nvls_round.bin";
    const size_t N = 1 << 20;
    CU(cuInit(0));
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    if (ng < D) { printf("{\"error\": \"need %d GPUs\"}\n", D); return 0; }
    std::vector<CUdevice> dev(D);
    for (int g = 0; g < D; ++g) {
        CU(cuDeviceGet(&dev[g], g));
        CK(cudaSetDevice(g));
        CK(cudaFree(0));
    }
    // inputs: half "generator-like" (±(1+m/128) 2^e, e in [-13,-8], 1/16 zeros), half wide
    // (random sign, exponent in [-30, 0], any mantissa), seeded
    std::mt19937_64 rng(12345);
    std::vector<std::vector<uint16_t>> in(D, std::vector<uint16_t>(N));
    for (int g = 0; g < D; ++g)
        for (size_t i = 0; i < N; ++i) {
            const uint64_t x = rng();
            float v;
            if (i < N / 2) {
                if ((x & 15) == 0) v = 0.f;
                else v = ((x >> 4) & 1 ? -1.f : 1.f) * (1.f + (float)((x >> 7) & 127) / 128.f) *
                         ldexpf(1.f, -8 - (int)((x >> 5) & 3) - (int)((x >> 14) & 1) * 2);
            } else {
                v = ((x >> 4) & 1 ? -1.f : 1.f) * (1.f + (float)((x >> 7) & 127) / 128.f) *
                    ldexpf(1.f, -(int)((x >> 20) % 31));
            }
            in[g][i] = bf16_of(v);
        }
    CUmulticastObjectProp mp = {};
    mp.numDevices = D;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = N * 2;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t total = (N * 2 + gran - 1) / gran * gran;
    mp.size = total;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int g = 0; g < D; ++g) CU(cuMulticastAddDevice(mc, dev[g]));
    std::vector<CUmemAccessDesc> acc(D);
    for (int g = 0; g < D; ++g) {
        acc[g].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[g].location.id = g;
        acc[g].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    for (int g = 0; g < D; ++g) {
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = g;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CUmemGenericAllocationHandle mem;
        CU(cuMemCreate(&mem, total, &ap, 0));
        CUdeviceptr p;
        CU(cuMemAddressReserve(&p, total, gran, 0, 0));
        CU(cuMemMap(p, total, 0, mem, 0));
        CU(cuMemSetAccess(p, total, acc.data(), D));
        CU(cuMulticastBindMem(mc, 0, mem, 0, total, 0));
        CK(cudaSetDevice(g));
        CK(cudaMemcpy(reinterpret_cast<void*>(p), in[g].data(), N * 2, cudaMemcpyHostToDevice));
    }
    CUdeviceptr mva;
    CU(cuMemAddressReserve(&mva, total, gran, 0, 0));
    CU(cuMemMap(mva, total, 0, mc, 0));
    CU(cuMemSetAccess(mva, total, acc.data(), D));
    for (int g = 0; g < D; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
    FILE* f = fopen(path, "wb");
    const int32_t hdr[2] = {D, (int32_t)N};
    fwrite(hdr, 4, 2, f);
    for (int g = 0; g < D; ++g) fwrite(in[g].data(), 2, N, f);
    for (int acc32 = 1; acc32 >= 0; --acc32) {
        for (int g = 0; g < D; ++g) {   // every GPU issues the reduction (does the issuer matter?)
            CK(cudaSetDevice(g));
            uint16_t* out;
            CK(cudaMalloc(&out, N * 2));
            reduce_kernel<<<(unsigned)(N / 8 / 256), 256>>>(reinterpret_cast<const uint16_t*>(mva), out, N, acc32);
            CK(cudaDeviceSynchronize());
            std::vector<uint16_t> res(N);
            CK(cudaMemcpy(res.data(), out, N * 2, cudaMemcpyDeviceToHost));
            fwrite(res.data(), 2, N, f);
            CK(cudaFree(out));
        }
    }
    fclose(f);
    printf("{\"D\": %d, \"N\": %zu, \"file\": \"%s\"}\n", D, N, path);
    return 0;
}
