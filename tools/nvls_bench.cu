// nvls_bench.cu — NVLink SHARP (NVLS, multicast) vs unicast peer access for the two
// collectives of the LAMB step, single process driving D GPUs.
//   AG  : every GPU publishes its slice of a bf16 buffer to all GPUs
//         mc = one multimem.st per 16 B to the multicast address; uc = D-1 peer stores
//   RS  : every GPU reduces its slice over all GPUs
//         mc_bf16 = multimem.ld_reduce.add.acc::f32.v4.bf16x2 (result rounded to bf16)
//         mc_f32  = multimem.ld_reduce.add.v4.f32 on fp32 inputs (2x the bytes)
//         uc_bf16 = D peer loads of bf16, fp32 sum (what the fused pass A does)
// Reports, per variant, the slowest GPU's time and the per-GPU in-bound GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_bench tools/nvls_bench.cu -lcuda
//   tools/nvls_bench <D> <MiB of the full bf16 buffer>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)
#define CU(x)                                                                              \
    do {                                                                                   \
        CUresult r = (x);                                                                  \
        if (r != CUDA_SUCCESS) {                                                           \
            const char* s = nullptr;                                                       \
            cuGetErrorString(r, &s);                                                       \
            printf("{\"error\": \"%s: %s\"}\n", #x, s ? s : "?");                          \
            exit(0);                                                                       \
        }                                                                                  \
    } while (0)

struct Peers {
    char* p[8];
};

__global__ void ag_mc(char* mc, const char* mine, size_t off, size_t bytes) {
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(mine + off + i);
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + off + i),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
}

__global__ void ag_uc(Peers P, int D, int me, size_t off, size_t bytes) {
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(P.p[me] + off + i);
        for (int j = 0; j < D; ++j)
            if (j != me) *reinterpret_cast<uint4*>(P.p[j] + off + i) = v;
    }
}

__global__ void rs_mc_bf16(const char* mc, float* out, size_t off, size_t bytes) {
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16) {
        uint32_t a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + off + i) : "memory");
        float* o = out + i / 2;
        o[0] = __uint_as_float(a << 16); o[1] = __uint_as_float(a & 0xffff0000u);
        o[2] = __uint_as_float(b << 16); o[3] = __uint_as_float(b & 0xffff0000u);
        o[4] = __uint_as_float(c << 16); o[5] = __uint_as_float(c & 0xffff0000u);
        o[6] = __uint_as_float(d << 16); o[7] = __uint_as_float(d & 0xffff0000u);
    }
}

__global__ void rs_mc_f32(const char* mc, float* out, size_t off, size_t bytes) {
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + off + i) : "memory");
        *reinterpret_cast<float4*>(out + i / 4) = make_float4(a, b, c, d);
    }
}

__global__ void rs_uc_bf16(Peers P, int D, float* out, size_t off, size_t bytes) {
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)gridDim.x * blockDim.x * 16) {
        float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = 0; j < D; ++j) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(P.p[j] + off + i));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            for (int k = 0; k < 4; ++k) {
                s[2 * k] += __uint_as_float(w[k] << 16);
                s[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
            }
        }
        for (int k = 0; k < 8; ++k) out[i / 2 + k] = s[k];
    }
}

// Pipelined pair: half the blocks reduce-scatter region A while the other half all-gather
// region B (RS of bucket b+1 || AG of bucket b).  mc: multimem ld_reduce + multimem.st;
// uc: peer loads + peer stores (the fused passes' patterns).
__global__ void pipe_mc(char* mc, const char* mine, float* out, size_t offA, size_t offB, size_t bytes) {
    const unsigned half = gridDim.x / 2;
    const bool rs = blockIdx.x < half;
    const size_t b0 = (size_t)(rs ? blockIdx.x : blockIdx.x - half);
    for (size_t i = (b0 * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)half * blockDim.x * 16) {
        if (rs) {
            uint32_t a, b, c, d;
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + offA + i) : "memory");
            *reinterpret_cast<uint4*>(reinterpret_cast<char*>(out) + i) = make_uint4(a, b, c, d);
        } else {
            const uint4 v = *reinterpret_cast<const uint4*>(mine + offB + i);
            asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + offB + i),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
    }
}

__global__ void pipe_uc(Peers P, int D, int me, float* out, size_t offA, size_t offB, size_t bytes) {
    const unsigned half = gridDim.x / 2;
    const bool rs = blockIdx.x < half;
    const size_t b0 = (size_t)(rs ? blockIdx.x : blockIdx.x - half);
    for (size_t i = (b0 * blockDim.x + threadIdx.x) * 16; i < bytes; i += (size_t)half * blockDim.x * 16) {
        if (rs) {
            float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int j = 0; j < D; ++j) {
                const uint4 v = __ldcs(reinterpret_cast<const uint4*>(P.p[j] + offA + i));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                for (int k = 0; k < 4; ++k) {
                    s[2 * k] += __uint_as_float(w[k] << 16);
                    s[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
                }
            }
            for (int k = 0; k < 8; ++k) out[i / 2 + k] = s[k];
        } else {
            const uint4 v = *reinterpret_cast<const uint4*>(P.p[me] + offB + i);
            for (int j = 0; j < D; ++j)
                if (j != me) *reinterpret_cast<uint4*>(P.p[j] + offB + i) = v;
        }
    }
}

int main(int argc, char** argv) {
    const int D = argc > 1 ? atoi(argv[1]) : 2;
    const size_t mib = argc > 2 ? (size_t)atoll(argv[2]) : 1024;
    CU(cuInit(0));
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < D) { printf("{\"error\": \"need %d GPUs\"}\n", D); return 0; }
    std::vector<CUdevice> dev(D);
    int mcs = 1;
    for (int g = 0; g < D; ++g) {
        CU(cuDeviceGet(&dev[g], g));
        int s = 0;
        CU(cuDeviceGetAttribute(&s, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[g]));
        mcs &= s;
        CK(cudaSetDevice(g));
        CK(cudaFree(0));   // primary context
    }
    if (!mcs) { printf("{\"D\": %d, \"multicast_supported\": 0}\n", D); return 0; }
    // one buffer of `bytes` per GPU (bf16 data; the f32 RS uses a second, 2x buffer)
    size_t bytes = mib << 20;
    CUmulticastObjectProp mp = {};
    mp.numDevices = D;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = 2 * bytes;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    size_t total = (3 * bytes + gran - 1) / gran * gran;   // [0,bytes) bf16, [bytes, 3 bytes) f32
    mp.size = total;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int g = 0; g < D; ++g) CU(cuMulticastAddDevice(mc, dev[g]));
    std::vector<CUmemGenericAllocationHandle> mem(D);
    std::vector<char*> uva(D);
    std::vector<CUmemAccessDesc> acc(D);
    for (int g = 0; g < D; ++g) {
        acc[g].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[g].location.id = g;
        acc[g].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    size_t ugran = 0;
    for (int g = 0; g < D; ++g) {
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = g;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CU(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        CU(cuMemCreate(&mem[g], total, &ap, 0));
        CUdeviceptr p;
        CU(cuMemAddressReserve(&p, total, gran > ugran ? gran : ugran, 0, 0));
        CU(cuMemMap(p, total, 0, mem[g], 0));
        CU(cuMemSetAccess(p, total, acc.data(), D));   // every GPU can reach every buffer
        uva[g] = reinterpret_cast<char*>(p);
        CU(cuMulticastBindMem(mc, 0, mem[g], 0, total, 0));
    }
    CUdeviceptr mva;
    CU(cuMemAddressReserve(&mva, total, gran, 0, 0));
    CU(cuMemMap(mva, total, 0, mc, 0));
    CU(cuMemSetAccess(mva, total, acc.data(), D));
    char* mcp = reinterpret_cast<char*>(mva);
    std::vector<float*> out(D);
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMalloc(&out[g], 2 * bytes));
        CK(cudaMemset(uva[g], 0x3c, total));   // bf16 ~1.0-ish patterns; f32 region too
    }
    Peers P;
    for (int g = 0; g < D; ++g) P.p[g] = uva[g];
    const size_t slice = bytes / D;   // per-GPU slice of the bf16 buffer
    auto timeit = [&](auto launch) {
        float best = 1e30f;
        std::vector<cudaEvent_t> e0(D), e1(D);
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventCreate(&e0[g]));
            CK(cudaEventCreate(&e1[g]));
        }
        for (int rep = 0; rep < 6; ++rep) {
            for (int g = 0; g < D; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
            for (int g = 0; g < D; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventRecord(e0[g]));
                launch(g);
                CK(cudaEventRecord(e1[g]));
            }
            float worst = 0;
            for (int g = 0; g < D; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventSynchronize(e1[g]));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
                worst = ms > worst ? ms : worst;
            }
            if (rep > 0) best = worst < best ? worst : best;
        }
        return best;
    };
    const int grid = 148 * 4, blk = 256;
    const double in_bf16 = (double)slice * (D - 1);   // bytes each GPU must receive (AG / RS-pull)
    float t_ag_mc = timeit([&](int g) { ag_mc<<<grid, blk>>>(mcp, uva[g], g * slice, slice); });
    float t_ag_uc = timeit([&](int g) { ag_uc<<<grid, blk>>>(P, D, g, g * slice, slice); });
    float t_rs_mcb = timeit([&](int g) { rs_mc_bf16<<<grid, blk>>>(mcp, out[g], g * slice, slice); });
    float t_rs_mcf = timeit([&](int g) { rs_mc_f32<<<grid, blk>>>(mcp + bytes, out[g], 2 * g * slice, 2 * slice); });
    float t_rs_uc = timeit([&](int g) { rs_uc_bf16<<<grid, blk>>>(P, D, out[g], g * slice, slice); });
    // pipelined RS(A) || AG(B): regions A = [0, bytes/2), B = [bytes/2, bytes) of the bf16 buffer
    const size_t hs = bytes / 2 / D;   // per-GPU slice of each region
    float t_pipe_mc = timeit([&](int g) { pipe_mc<<<grid, blk>>>(mcp, uva[g], out[g], g * hs, bytes / 2 + g * hs, hs); });
    float t_pipe_uc = timeit([&](int g) { pipe_uc<<<grid, blk>>>(P, D, g, out[g], g * hs, bytes / 2 + g * hs, hs); });
    float t_seq_uc = timeit([&](int g) {
        rs_uc_bf16<<<grid, blk>>>(P, D, out[g], g * hs, hs);
        ag_uc<<<grid, blk>>>(P, D, g, bytes / 2 + g * hs, hs);
    });
    CK(cudaGetLastError());
    printf("{\"D\": %d, \"pipelined_half_buffers\": 1, \"rs_then_ag_uc_ms\": %.3f, \"rs_par_ag_uc_ms\": %.3f, "
           "\"rs_par_ag_mc_ms\": %.3f}\n", D, t_seq_uc, t_pipe_uc, t_pipe_mc);
    auto gbs = [&](double b, float ms) { return b / (ms * 1e-3) / 1e9; };
    printf("{\"D\": %d, \"MiB\": %zu, \"multicast_supported\": 1, \"slice_MiB\": %.1f, "
           "\"ag_mc_ms\": %.3f, \"ag_uc_ms\": %.3f, \"rs_mc_bf16_ms\": %.3f, \"rs_mc_f32_ms\": %.3f, \"rs_uc_bf16_ms\": %.3f, "
           "\"ag_mc_in_GBps\": %.1f, \"ag_uc_in_GBps\": %.1f, \"rs_uc_in_GBps\": %.1f}\n",
           D, mib, slice / 1048576.0, t_ag_mc, t_ag_uc, t_rs_mcb, t_rs_mcf, t_rs_uc, gbs(in_bf16, t_ag_mc),
           gbs(in_bf16, t_ag_uc), gbs(in_bf16, t_rs_uc));
    return 0;
}
