// p2p_bench.cu — single-process NVLink microbenchmark for the fused passes' access patterns.
// Every GPU g pulls (loads) or pushes (stores) `bytes` from/to each of the other D-1 GPUs at
// the same time (the all-to-all shape of pass A's reduce-scatter / pass B's all-gather),
// with 8 B or 16 B per lane.  Reports the per-GPU in-bound GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_bench tools/p2p_bench.cu
//   tools/p2p_bench <D> <MiB per peer>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

struct Ptrs {
    const char* src[8];
    char* dst[8];
};

template <typename V, bool PUSH>
__global__ void a2a(Ptrs P, int D, int me, size_t bytes_per_peer, char* local) {
    // peers round-robin over the grid's blocks: block b serves peer (me + 1 + b % (D-1)) % D
    const size_t nv = bytes_per_peer / sizeof(V);
    const int np = D - 1;
    const int j = (me + 1 + (int)(blockIdx.x % np)) % D;
    const size_t nb = gridDim.x / np;
    const size_t b = blockIdx.x / np;
    for (size_t k = b * blockDim.x + threadIdx.x; k < nv; k += nb * blockDim.x) {
        if (PUSH) {
            reinterpret_cast<V*>(P.dst[j] + (size_t)me * bytes_per_peer)[k] =
                reinterpret_cast<const V*>(local + (size_t)j * bytes_per_peer)[k];
        } else {
            reinterpret_cast<V*>(local + (size_t)j * bytes_per_peer)[k] =
                __ldcs(reinterpret_cast<const V*>(P.src[j] + (size_t)me * bytes_per_peer) + k);
        }
    }
}

template <typename V, bool PUSH>
__global__ void a2a_s(Ptrs P, int D, int me, size_t bytes_per_peer, size_t nbytes, char* local) {
    const size_t nv = nbytes / sizeof(V);
    const int np = D - 1;
    const int j = (me + 1 + (int)(blockIdx.x % np)) % D;
    const size_t nb = gridDim.x / np;
    const size_t b = blockIdx.x / np;
    for (size_t k = b * blockDim.x + threadIdx.x; k < nv; k += nb * blockDim.x) {
        if (PUSH) {
            reinterpret_cast<V*>(P.dst[j] + (size_t)me * bytes_per_peer)[k] =
                reinterpret_cast<const V*>(local + (size_t)j * bytes_per_peer)[k];
        } else {
            reinterpret_cast<V*>(local + (size_t)j * bytes_per_peer)[k] =
                __ldcs(reinterpret_cast<const V*>(P.src[j] + (size_t)me * bytes_per_peer) + k);
        }
    }
}

template <typename V, bool PUSH>
float run(int D, size_t bpp, std::vector<char*>& remote, std::vector<char*>& local, int grid) {
    std::vector<cudaEvent_t> e0(D), e1(D);
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
    }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            Ptrs P;
            for (int j = 0; j < D; ++j) {
                P.src[j] = remote[j];
                P.dst[j] = remote[j];
            }
            CK(cudaEventRecord(e0[g]));
            a2a<V, PUSH><<<grid, 256>>>(P, D, g, bpp, local[g]);
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
        best = worst < best ? worst : best;
    }
    return (float)(bpp * (D - 1)) / (best * 1e-3f) / 1e9f;
}

// Copy-engine all-to-all: every GPU issues one cudaMemcpyPeerAsync per peer, each on its own
// stream (PUSH: from the GPU's local buffer into the peer; pull: from the peer into local).
float run_ce(int D, size_t bpp, std::vector<char*>& remote, std::vector<char*>& local, bool push, int split) {
    std::vector<cudaEvent_t> e0(D), e1(D);
    std::vector<std::vector<cudaStream_t>> st(D);
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
        st[g].resize((D - 1) * split);
        for (auto& x : st[g]) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventRecord(e0[g], 0));
            int k = 0;
            for (int j = 0; j < D; ++j) {
                if (j == g) continue;
                for (int q = 0; q < split; ++q, ++k) {
                    const size_t lo = bpp * q / split, n = bpp * (q + 1) / split - lo;
                    CK(cudaStreamWaitEvent(st[g][k], e0[g], 0));
                    if (push)
                        CK(cudaMemcpyPeerAsync(remote[j] + (size_t)g * bpp + lo, j, local[g] + (size_t)j * bpp + lo,
                                               g, n, st[g][k]));
                    else
                        CK(cudaMemcpyPeerAsync(local[g] + (size_t)j * bpp + lo, g, remote[j] + (size_t)g * bpp + lo,
                                               j, n, st[g][k]));
                }
            }
            for (auto& x : st[g]) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, x));
                CK(cudaStreamWaitEvent(0, ev, 0));
                CK(cudaEventDestroy(ev));
            }
            CK(cudaEventRecord(e1[g], 0));
        }
        float worst = 0;
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventSynchronize(e1[g]));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
            worst = ms > worst ? ms : worst;
        }
        best = worst < best ? worst : best;
    }
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        for (auto& x : st[g]) CK(cudaStreamDestroy(x));
    }
    return (float)(bpp * (D - 1)) / (best * 1e-3f) / 1e9f;
}

// SM pushes/pulls on the first (1 - ce_frac) of every peer's bytes while the copy engines move
// the rest, all at once: does the fabric give more than either path alone?
float run_mixed(int D, size_t bpp, std::vector<char*>& remote, std::vector<char*>& local, int grid, double ce_frac,
                bool push) {
    const size_t ce_b = (size_t)(bpp * ce_frac) / 4096 * 4096, sm_b = bpp - ce_b;
    std::vector<cudaEvent_t> e0(D), e1(D);
    std::vector<std::vector<cudaStream_t>> st(D);
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
        st[g].resize(D);
        for (auto& x : st[g]) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventRecord(e0[g], 0));
            Ptrs P;
            for (int j = 0; j < D; ++j) {
                P.src[j] = remote[j];
                P.dst[j] = remote[j];
            }
            // SM part: the same a2a kernel over the first sm_b bytes of each peer block (stride bpp)
            if (sm_b) {
                CK(cudaStreamWaitEvent(st[g][0], e0[g], 0));
                if (push) a2a_s<uint4, true><<<grid, 256, 0, st[g][0]>>>(P, D, g, bpp, sm_b, local[g]);
                else a2a_s<uint4, false><<<grid, 256, 0, st[g][0]>>>(P, D, g, bpp, sm_b, local[g]);
            }
            int k = 1;
            for (int j = 0; j < D && ce_b; ++j) {
                if (j == g) continue;
                CK(cudaStreamWaitEvent(st[g][k], e0[g], 0));
                if (push)
                    CK(cudaMemcpyPeerAsync(remote[j] + (size_t)g * bpp + sm_b, j, local[g] + (size_t)j * bpp + sm_b, g,
                                           ce_b, st[g][k]));
                else
                    CK(cudaMemcpyPeerAsync(local[g] + (size_t)j * bpp + sm_b, g, remote[j] + (size_t)g * bpp + sm_b, j,
                                           ce_b, st[g][k]));
                ++k;
            }
            for (auto& x : st[g]) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, x));
                CK(cudaStreamWaitEvent(0, ev, 0));
                CK(cudaEventDestroy(ev));
            }
            CK(cudaEventRecord(e1[g], 0));
        }
        float worst = 0;
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventSynchronize(e1[g]));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
            worst = ms > worst ? ms : worst;
        }
        best = worst < best ? worst : best;
    }
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        for (auto& x : st[g]) CK(cudaStreamDestroy(x));
    }
    return (float)(bpp * (D - 1)) / (best * 1e-3f) / 1e9f;
}

// TMA bulk pulls (what pass A's producer does): one CTA per SM, one elected thread streams
// `chunk`-byte pieces of the peers' blocks into an S-stage shared-memory ring with
// cp.async.bulk (mbarrier complete_tx); one consumer warp only releases the stages (no compute,
// no HBM write): the ceiling of the pull pattern itself.  Items go round robin over the peers.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void a2a_tma(Ptrs P, int D, int me, size_t bytes_per_peer, int chunk, int S) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)chunk * S);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) {
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(full + k)), "r"(1));
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(empty + k)), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int np = D - 1;
    const size_t per_peer = bytes_per_peer / chunk, total = per_peer * np;
    if (threadIdx.x == 0) {
        int k = 0;
        uint32_t ph = 0;
        for (size_t it = blockIdx.x; it < total; it += gridDim.x) {
            asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                         ::"r"(su32(empty + k)), "r"(ph ^ 1) : "memory");
            const int j = (me + 1 + (int)(it % np)) % D;
            const char* src = P.src[j] + (size_t)me * bytes_per_peer + (it / np) * chunk;
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(full + k)), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm + (size_t)k * chunk)), "l"(src), "r"(chunk), "r"(su32(full + k)) : "memory");
            if (++k == S) { k = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int k = 0;
        uint32_t ph = 0;
        for (size_t it = blockIdx.x; it < total; it += gridDim.x) {
            asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                         ::"r"(su32(full + k)), "r"(ph) : "memory");
            asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(empty + k)) : "memory");
            if (++k == S) { k = 0; ph ^= 1; }
        }
    }
}

float run_tma(int D, size_t bpp, std::vector<char*>& remote, int sms, int chunk, int S) {
    const size_t smem = (size_t)chunk * S + 16 * S;
    std::vector<cudaEvent_t> e0(D), e1(D);
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaFuncSetAttribute(a2a_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
    }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        for (int g = 0; g < D; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        for (int g = 0; g < D; ++g) {
            CK(cudaSetDevice(g));
            Ptrs P;
            for (int j = 0; j < D; ++j) P.src[j] = P.dst[j] = remote[j];
            CK(cudaEventRecord(e0[g]));
            a2a_tma<<<sms, 64, smem>>>(P, D, g, bpp, chunk, S);
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
        best = worst < best ? worst : best;
    }
    return (float)(bpp * (D - 1)) / (best * 1e-3f) / 1e9f;
}

int main(int argc, char** argv) {
    const int D = argc > 1 ? atoi(argv[1]) : 2;
    const size_t mib = argc > 2 ? (size_t)atoll(argv[2]) : 512;
    const size_t bpp = mib << 20;
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < D) {
        fprintf(stderr, "need %d GPUs, have %d\n", D, n);
        return 1;
    }
    std::vector<char*> remote(D), local(D);
    int sms = 0;
    for (int g = 0; g < D; ++g) {
        CK(cudaSetDevice(g));
        for (int j = 0; j < D; ++j)
            if (j != g) CK(cudaDeviceEnablePeerAccess(j, 0));
        CK(cudaMalloc(&remote[g], bpp * D));
        CK(cudaMalloc(&local[g], bpp * D));
        CK(cudaMemset(remote[g], 1, bpp * D));
        CK(cudaMemset(local[g], 2, bpp * D));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g));
    }
    printf("{\"D\": %d, \"MiB_per_peer\": %zu", D, mib);
    if (argc > 3 && atoi(argv[3]) == 1) {   // TMA pull sweep only
        for (int chunk : {8192, 16384, 32768})
            for (int S : {4, 8, 16, 24})
                if ((size_t)chunk * S <= 200 * 1024)
                    printf(", \"tma_pull_c%d_s%d\": %.1f", chunk, S, run_tma(D, bpp, remote, sms, chunk, S));
        printf("}\n");
        return 0;
    }
    for (int mult : {3, 6, 12}) {   // multiples of 3 so every peer gets the same block count
        const int grid = sms * mult;
        printf(", \"pull8_x%d\": %.1f", mult, run<uint2, false>(D, bpp, remote, local, grid));
        printf(", \"pull16_x%d\": %.1f", mult, run<uint4, false>(D, bpp, remote, local, grid));
        printf(", \"push8_x%d\": %.1f", mult, run<uint2, true>(D, bpp, remote, local, grid));
        printf(", \"push16_x%d\": %.1f", mult, run<uint4, true>(D, bpp, remote, local, grid));
    }
    for (int split : {1, 4}) {
        printf(", \"ce_push_s%d\": %.1f", split, run_ce(D, bpp, remote, local, true, split));
        printf(", \"ce_pull_s%d\": %.1f", split, run_ce(D, bpp, remote, local, false, split));
    }
    for (double f : {0.1, 0.2, 0.3, 0.4}) {
        printf(", \"mixed_push_ce%.1f\": %.1f", f, run_mixed(D, bpp, remote, local, sms * 6, f, true));
        printf(", \"mixed_pull_ce%.1f\": %.1f", f, run_mixed(D, bpp, remote, local, sms * 6, f, false));
    }
    printf("}\n");
    return 0;
}
