// lamb_kernels.cu — the hot path of the sharded LAMB step on sm_100a.
//
// Pass A  (rows a1+a2): g = grad_scale * sum_j f32(G_j)     [fused reduce-scatter: G_j are
//          the ranks' bf16 grad buffers read over NVLink, fp32 sum in fixed order j=0..D-1]
//          m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2       [Adam moments, You et al. Alg. 2]
//          u = (m c1) / (sqrt(v c2) + eps) + wd w            [bias correction Z5, eps Z4, Z7]
//          per item: sum w^2, sum u^2 in fp64                 [segmented norms, row a3]
// Finalize (a3+a4): per segment fixed-order sum of item partials; straddlers exchanged over
//          NVLink and summed in rank order; ratio = ||w||/||u|| (1 on a zero norm, Z9).
// Pass B  (a5+a6): recompute u bit-identically, w -= (lr ratio) u, p = bf16_rne(w) stored to
//          every rank's param buffer [fused all-gather over NVLink].
// PAPER.md cites: LAMB §3.1; ZeRO-2 RS/AG §2, §3.2 P:312-328.
//
// All three are HBM/NVLink streaming kernels (~1 flop/B): no tensor cores.  Design for B200:
// 128-bit coalesced loads with L1::no_allocate, several independent chunks per lane in
// flight, a persistent grid of (148 x resident CTAs) warps walking the item table.
#include "lamb_kernels.cuh"

namespace lamb {

// ------------------------------------------------------------ memory helpers
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_ro_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_ro_u2(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_f4(float* p, float4 v) {
    asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void st_u2(void* p, uint2 v) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
}
// bf16 -> f32 is exact: the bf16 bits are the high half of the f32.
__device__ __forceinline__ float bf_lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf_hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // cvt.rn.bf16x2.f32 (RNE, Z15)
    return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------ the LAMB element math
// Both passes call exactly these functions with explicit-rounding intrinsics (no FMA
// contraction, no fast-math), so pass B recomputes the same u bits pass A normed.
__device__ __forceinline__ void adam_moments(float g, float& m, float& v, const GroupConst& G) {
    m = __fmaf_rn(G.b1, m, __fmul_rn(G.omb1, g));
    v = __fmaf_rn(G.b2, v, __fmul_rn(G.omb2, __fmul_rn(g, g)));
}
__device__ __forceinline__ float lamb_update(float m, float v, float w, const GroupConst& G) {
    const float mh = __fmul_rn(m, G.c1);
    const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(v, G.c2)), G.eps);
    return __fmaf_rn(G.wd, w, __fdiv_rn(mh, den));
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// ------------------------------------------------------------ pass A
// NS > 0: NS bf16 sources (fused reduce-scatter, NS = D); NS == 0: fp32 reduced shard (g32).
template <int NS, int U>
__global__ void __launch_bounds__(kThreads) pass_a_kernel(const __grid_constant__ StepParams P) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    for (int64_t it = P.item_begin + gw; it < P.item_end; it += nw) {
        const Item I = P.items[it];
        const GroupConst& G = P.groups[I.group];
        float* const wp = P.w + I.shard_off;
        float* const mp = P.m + I.shard_off;
        float* const vp = P.v + I.shard_off;
        double sw = 0.0, su = 0.0;
        for (int c0 = 0; c0 < I.n_chunk; c0 += 32 * U) {
            float4 g[U], m[U], v[U], w[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int c = c0 + k * 32 + lane;
                if (c < I.n_chunk) {
                    const int64_t e = 4 * (int64_t)c;
                    m[k] = ld_stream_f4(mp + e);
                    v[k] = ld_stream_f4(vp + e);
                    w[k] = ld_ro_f4(wp + e);
                    if constexpr (NS == 0) {
                        g[k] = ld_ro_f4(P.g32 + I.shard_off + e);
                    } else {
                        uint2 raw[NS];
#pragma unroll
                        for (int j = 0; j < NS; ++j) raw[j] = ld_ro_u2(P.gsrc[j] + I.flat_off + e);
                        // fp32 accumulation in fixed rank order j = 0..D-1 (reading Z11)
                        float4 s = make_float4(bf_lo(raw[0].x), bf_hi(raw[0].x),
                                               bf_lo(raw[0].y), bf_hi(raw[0].y));
#pragma unroll
                        for (int j = 1; j < NS; ++j) {
                            s.x = __fadd_rn(s.x, bf_lo(raw[j].x));
                            s.y = __fadd_rn(s.y, bf_hi(raw[j].x));
                            s.z = __fadd_rn(s.z, bf_lo(raw[j].y));
                            s.w = __fadd_rn(s.w, bf_hi(raw[j].y));
                        }
                        g[k] = s;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int c = c0 + k * 32 + lane;
                if (c < I.n_chunk) {
                    const int64_t e = 4 * (int64_t)c;
                    float gs[4] = {g[k].x, g[k].y, g[k].z, g[k].w};
                    float ms[4] = {m[k].x, m[k].y, m[k].z, m[k].w};
                    float vs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
                    const float ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        adam_moments(__fmul_rn(gs[q], P.grad_scale), ms[q], vs[q], G);
                        const float u = lamb_update(ms[q], vs[q], ws[q], G);
                        sw = fma((double)ws[q], (double)ws[q], sw);
                        su = fma((double)u, (double)u, su);
                    }
                    st_f4(mp + e, make_float4(ms[0], ms[1], ms[2], ms[3]));
                    st_f4(vp + e, make_float4(vs[0], vs[1], vs[2], vs[3]));
                }
            }
        }
        sw = warp_sum(sw);
        su = warp_sum(su);
        if (lane == 0) P.partials[it] = make_double2(sw, su);
    }
}

// ------------------------------------------------------------ pass B
template <int ND, int U>
__global__ void __launch_bounds__(kThreads) pass_b_kernel(const __grid_constant__ StepParams P) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    for (int64_t it = P.item_begin + gw; it < P.item_end; it += nw) {
        const Item I = P.items[it];
        const GroupConst& G = P.groups[I.group];
        const float scale = P.scale[I.tensor];
        float* const wp = P.w + I.shard_off;
        const float* const mp = P.m + I.shard_off;
        const float* const vp = P.v + I.shard_off;
        for (int c0 = 0; c0 < I.n_chunk; c0 += 32 * U) {
            float4 m[U], v[U], w[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int c = c0 + k * 32 + lane;
                if (c < I.n_chunk) {
                    const int64_t e = 4 * (int64_t)c;
                    m[k] = ld_ro_f4(mp + e);
                    v[k] = ld_ro_f4(vp + e);
                    w[k] = ld_stream_f4(wp + e);
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int c = c0 + k * 32 + lane;
                if (c < I.n_chunk) {
                    const int64_t e = 4 * (int64_t)c;
                    const float ms[4] = {m[k].x, m[k].y, m[k].z, m[k].w};
                    const float vs[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
                    float ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        ws[q] = __fmaf_rn(-scale, lamb_update(ms[q], vs[q], ws[q], G), ws[q]);
                    st_f4(wp + e, make_float4(ws[0], ws[1], ws[2], ws[3]));
                    const uint2 pb = make_uint2(pack_bf16x2(ws[0], ws[1]), pack_bf16x2(ws[2], ws[3]));
#pragma unroll
                    for (int j = 0; j < ND; ++j) st_u2(P.pdst[j] + I.flat_off + e, pb);
                }
            }
        }
    }
    if constexpr (ND > 1) __threadfence_system();   // peer stores visible before the barrier
}

// ------------------------------------------------------------ finalize
__device__ __forceinline__ void trust_ratio(double w2, double u2, const GroupConst& G, int tensor,
                                            const FinalizeParams& P) {
    const double wn = sqrt(w2), un = sqrt(u2);
    const double ratio = G.adapt ? ((wn > 0.0 && un > 0.0) ? wn / un : 1.0) : 1.0;
    P.scale[tensor] = (float)((double)G.lr * ratio);
    P.w_sq[tensor] = w2;
    P.u_sq[tensor] = u2;
    P.ratio[tensor] = (float)ratio;
}

// One warp per segment: fixed-order sum of its item partials (lane-strided, then xor tree).
__global__ void __launch_bounds__(256) finalize_segments_kernel(const __grid_constant__ FinalizeParams P) {
    const int lane = threadIdx.x & 31;
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (s >= P.n_segs) return;
    const SegDesc S = P.segs[s];
    double w2 = 0.0, u2 = 0.0;
    for (int64_t i = S.item_begin + lane; i < S.item_end; i += 32) {
        const double2 q = P.partials[i];
        w2 += q.x;
        u2 += q.y;
    }
    w2 = warp_sum(w2);
    u2 = warp_sum(u2);
    if (lane == 0) {
        if (S.strad_slot < 0) {
            trust_ratio(w2, u2, P.groups[S.group], S.tensor, P);
        } else {
            const double2 val = make_double2(w2, u2);
            for (int j = 0; j < P.world; ++j)
                P.xrow[j][(int64_t)P.rank * P.n_strad + S.strad_slot] = val;
        }
    }
    if (P.world > 1) __threadfence_system();
}

// One thread per straddler this rank touches: sum the D rows in rank order.
__global__ void finalize_straddlers_kernel(const __grid_constant__ FinalizeParams P) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P.n_local_strad) return;
    const int slot = P.strad_slots[k];
    double w2 = 0.0, u2 = 0.0;
    for (int j = 0; j < P.world; ++j) {
        const double2 q = P.xbuf[(int64_t)j * P.n_strad + slot];
        w2 += q.x;
        u2 += q.y;
    }
    trust_ratio(w2, u2, P.groups[P.strad_group[k]], P.strad_tensor[k], P);
}

// ------------------------------------------------------------ cross-GPU barrier
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A.flags[j] -> rank j's flag array (uint64[LAMB_MAX_RANKS]); slot i of rank j's array holds
// the last epoch rank i announced to j.  Every rank runs the same sequence of barriers, so the
// epoch counters agree.  A peer that does not arrive within 30 s sets *err (host-mapped) and
// the kernel exits instead of hanging the GPU.
struct BarrierArgs {
    uint64_t* flags[LAMB_MAX_RANKS];
};
__global__ void barrier_kernel_v(const __grid_constant__ BarrierArgs A, uint64_t* epoch, int rank,
                                 int world, int* err) {
    __shared__ uint64_t e;
    if (threadIdx.x == 0) {
        e = *epoch + 1;
        *epoch = e;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < world) {
        __threadfence_system();
        st_release_sys(A.flags[j] + rank, e);
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(A.flags[rank] + j) < e) {
            if (globaltimer() - t0 > 30ull * 1000000000ull) {
                atomicExch(err, 1);
                break;
            }
            __nanosleep(64);
        }
    }
}

// ------------------------------------------------------------ casts
__global__ void upcast_bf16_kernel(const __nv_bfloat16* __restrict__ src, float* __restrict__ dst,
                                   int64_t n) {
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
        const uint2 r = ld_ro_u2(src + i);   // n is a multiple of 128 (bucket sizes)
        st_f4(dst + i, make_float4(bf_lo(r.x), bf_hi(r.x), bf_lo(r.y), bf_hi(r.y)));
    }
}
__global__ void cast_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                 int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

// ------------------------------------------------------------ host launchers
template <int NS>
static constexpr int unroll_a() { return NS <= 1 ? 4 : 2; }

template <int NS>
static cudaError_t pass_a_ns(const StepParams& p, int grid, cudaStream_t s) {
    pass_a_kernel<NS, unroll_a<NS>()><<<grid, kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_pass_a(const StepParams& p, int nsrc, bool g32, int grid, cudaStream_t s) {
    if (p.item_end <= p.item_begin) return cudaSuccess;
    if (g32) return pass_a_ns<0>(p, grid, s);
    switch (nsrc) {
        case 1: return pass_a_ns<1>(p, grid, s);
        case 2: return pass_a_ns<2>(p, grid, s);
        case 3: return pass_a_ns<3>(p, grid, s);
        case 4: return pass_a_ns<4>(p, grid, s);
        case 5: return pass_a_ns<5>(p, grid, s);
        case 6: return pass_a_ns<6>(p, grid, s);
        case 7: return pass_a_ns<7>(p, grid, s);
        case 8: return pass_a_ns<8>(p, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int ND>
static cudaError_t pass_b_nd(const StepParams& p, int grid, cudaStream_t s) {
    pass_b_kernel<ND, 4><<<grid, kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_pass_b(const StepParams& p, int ndst, int grid, cudaStream_t s) {
    if (p.item_end <= p.item_begin) return cudaSuccess;
    switch (ndst) {
        case 1: return pass_b_nd<1>(p, grid, s);
        case 2: return pass_b_nd<2>(p, grid, s);
        case 3: return pass_b_nd<3>(p, grid, s);
        case 4: return pass_b_nd<4>(p, grid, s);
        case 5: return pass_b_nd<5>(p, grid, s);
        case 6: return pass_b_nd<6>(p, grid, s);
        case 7: return pass_b_nd<7>(p, grid, s);
        case 8: return pass_b_nd<8>(p, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <typename K>
static int occupancy_grid(int device, K kernel) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    return sms * per_sm;
}

int pass_grid(int device, int nsrc, bool g32, bool pass_b, int ndst) {
    // All variants share the launch shape; size by the heaviest register user of each pass.
    if (pass_b) return occupancy_grid(device, pass_b_kernel<8, 4>);
    (void)nsrc;
    (void)g32;
    (void)ndst;
    return occupancy_grid(device, pass_a_kernel<8, unroll_a<8>()>);
}

cudaError_t launch_finalize_segments(const FinalizeParams& p, cudaStream_t s) {
    if (p.n_segs <= 0) return cudaSuccess;
    const int64_t warps_per_block = 8;
    const int64_t blocks = (p.n_segs + warps_per_block - 1) / warps_per_block;
    finalize_segments_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finalize_straddlers(const FinalizeParams& p, cudaStream_t s) {
    if (p.n_local_strad <= 0) return cudaSuccess;
    finalize_straddlers_kernel<<<(p.n_local_strad + 127) / 128, 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_barrier(uint64_t* const* flags, uint64_t* epoch, int rank, int world,
                           int* err_flag, cudaStream_t s) {
    BarrierArgs a;
    for (int j = 0; j < LAMB_MAX_RANKS; ++j) a.flags[j] = j < world ? flags[j] : nullptr;
    barrier_kernel_v<<<1, 32, 0, s>>>(a, epoch, rank, world, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_upcast_bf16(const __nv_bfloat16* src, float* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    upcast_bf16_kernel<<<148 * 8, 256, 0, s>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_cast_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    cast_bf16_kernel<<<148 * 8, 256, 0, s>>>(src, dst, n);
    return cudaGetLastError();
}

}  // namespace lamb
