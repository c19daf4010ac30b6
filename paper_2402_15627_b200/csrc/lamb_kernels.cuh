// lamb_kernels.cuh — device-side data structures of the LAMB step (internal, not ABI).
//
// HBM layout: flat bf16 grad and param buffers in plan order (bucket after
// bucket, 8-aligned tensors, zero padding); this rank's fp32 w, m, v shards in shard-local
// order (its slice of bucket 0, then bucket 1, ...).  Work is cut into ITEMS: contiguous
// pieces of ONE segment (tensor ∩ slice), <= kItemElems elements, 8-aligned starts.  One warp
// owns one item at a time, so every per-item norm partial is an unsegmented, fixed-order
// reduction (deterministic, no float atomics) — the "tensor-boundary table" of the north star
// is the item -> segment -> tensor mapping.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/lamb.h"

namespace lamb {

// LAMB_DEBUG build (liblamb_debug.so, paper_2402_15627_b200/build.py): device-side checks in
// place of compute-sanitizer, which is closed on this GPU pool — item bounds and alignment
// against the buffers' extents, a tag per ring stage (the item the producer filled must be the
// one the consumers expect: a ring-phase or early-overwrite error shows up as a mismatch),
// bounded mbarrier waits (deadlock -> message + trap), segment / straddler / barrier-epoch
// bounds.  A failed check prints "LAMB_DEBUG ..." and traps.  The release build compiles none of it.
#ifdef LAMB_DEBUG
#define LAMB_DCHECK(cond, fmt, ...)                                                            \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("LAMB_DEBUG %s:%d block %d thread %d: check (%s) failed: " fmt "\n", __FILE__,     \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x, #cond, ##__VA_ARGS__);             \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define LAMB_DCHECK(cond, fmt, ...) \
    do {                            \
    } while (0)
#endif

constexpr int kThreads = 256;          // threads per CTA of the streaming passes
constexpr int kChunk = 4;              // elements per lane access (16 B fp32, 8 B bf16)
constexpr int64_t kItemElems = 4096;   // max elements per work item (multiple of 8)

struct __align__(32) Item {
    int64_t shard_off;   // first element in the fp32 shard (multiple of 8)
    int64_t flat_off;    // same element in the flat bf16 buffers
    int32_t n_chunk;     // ceil(len / 4) (len rounded up to 8: the tail is zero padding)
    int32_t tensor;
    int32_t group;
    int32_t seg;
};

struct __align__(16) SegDesc {
    int64_t item_begin, item_end;   // items of this segment (contiguous)
    int32_t tensor, group;
    int32_t strad_slot;             // index in the global straddler list, -1 if none
    int32_t pad;
};

// Per-step constants of one group (host computes c1 = 1/(1-b1^t), c2 = 1/(1-b2^t) in double).
struct GroupConst {
    float lr, b1, omb1, b2, omb2, eps, wd, c1, c2;
    int32_t adapt;
};

// Pre-step state, written on the device by clip_combine_kernel:
// gs = grad_scale * inv_loss_scale * clip (fp32, what pass A multiplies the reduced sum by),
// skip = 1 when the global gradient norm is not finite (the whole step is a no-op).
struct ClipState {
    double grad_norm;
    float gs;
    float clip;
    int32_t skip;
    int32_t pad;
};

struct ClipParams {
    const double2* partials;        // [n_items] .x = sum of squares of the item's reduced grads
    int64_t n_items;
    double* rows[LAMB_MAX_RANKS];   // rank j's clip row buffer (double[D]); this rank writes slot `rank`
    const double* my_rows;          // this rank's row buffer
    int32_t world, rank;
    float grad_scale, inv_loss_scale, max_grad_norm;
    ClipState* out;
    double* block_sums;             // [kClipBlocks] scratch of the two-level sum
};
constexpr int kClipBlocksMax = 296;

struct StepParams {
    const Item* items;
    int64_t item_begin, item_end;
    // pass A gradient sources: flat bf16 grad buffers of ranks 0..nsrc-1 (peer-mapped), or
    // g32 = this rank's fp32 reduced-gradient shard (NCCL mode)
    const __nv_bfloat16* gsrc[LAMB_MAX_RANKS];
    const float* g32;
    float grad_scale;
    float* w;
    float* m;
    float* v;
    double2* partials;        // [n_items] (sum w^2, sum u^2)
    const float* scale;       // [T] lr * ratio (pass B)
    const ClipState* clip;    // non-null: pre-step enabled (gs from device, skip flag)
    float* g32_out;           // grad_stats: materialise the fp32 reduced sums here (FUSED + clip)
    __nv_bfloat16* pdst[LAMB_MAX_RANKS];   // param buffers pass B stores into
    const GroupConst* groups;  // device table [n_groups], refreshed each step by the prologue
    int32_t self_src;          // index of this rank's own (local) source in gsrc
    int32_t staged;            // 1: sources j != self_src are shard-ordered staging buffers
                               // (copy-engine schedule): addressed by shard_off, not flat_off
    // copy-engine schedule, pass A: walk the items in reverse (buckets arrive in backward order)
    // and wait per bucket until gflags[b * world + j] >= gflag_target for every j != self_src
    int32_t reverse, world;
    const int32_t* item_bucket;
    const uint64_t* gflags;
    uint64_t gflag_target;
    int* err;
    uint64_t timeout_ns;
    // NVLS mode (LAMB_COMM_NVLS): multicast addresses of the flat grad and
    // param buffers (one address reaches the same offset on every rank through the NVSwitch)
    const __nv_bfloat16* gmc;   // pass A: multimem.ld_reduce (switch-side fp32 sum, bf16 result)
    __nv_bfloat16* pmc;         // pass B: multimem.st (one store lands in every rank's buffer)
    // extents, checked by the LAMB_DEBUG build only (bounds of every item it touches)
    int64_t shard_elems, flat_elems, n_items;
    int32_t n_tensors;
};

struct FinalizeParams {
    const SegDesc* segs;
    int64_t n_segs;
    const double2* partials;
    float* scale;             // [T]
    double* w_sq;             // [T] stats
    double* u_sq;
    float* ratio;
    // straddler exchange: xrow[j] points at rank j's exchange buffer ([D][n_strad] double2);
    // this rank writes its row (index `rank`) into every rank's buffer.
    double2* xrow[LAMB_MAX_RANKS];
    int32_t world, rank;
    int32_t n_strad;
    // straddler finalize: local slots this rank touches
    const int32_t* strad_slots;     // [n_local_strad] slot index
    const int32_t* strad_tensor;    // [n_local_strad]
    const int32_t* strad_group;     // [n_local_strad]
    int32_t n_local_strad;
    const double2* xbuf;            // this rank's exchange buffer
    const ClipState* clip;          // skip flag (pre-step)
    const GroupConst* groups;       // device table [n_groups]
    int64_t n_items;                // extents, checked by the LAMB_DEBUG build only
    int32_t n_tensors;
};

// Per-step constants of every group, written to device memory by one tiny kernel launched on
// the step's stream before the step (so a captured CUDA graph of the step replays correctly).
struct GroupTable {
    GroupConst g[LAMB_MAX_GROUPS];
};

// Host launchers (lamb_kernels.cu).  The streaming passes size their own persistent grids
// (TMA kernels: one CTA per SM; LDG kernels: SMs x resident CTAs); `budget` > 0 caps the CTA
// count (lamb_set_max_ctas), 0 = a full wave.
cudaError_t launch_self_check(const Item* items, int64_t n_items, const float* w, const float* m, const float* v,
                              const __nv_bfloat16* grad, const __nv_bfloat16* param, const int64_t* shard_pad,
                              int64_t n_shard_pad, const int64_t* flat_pad, int64_t n_flat_pad,
                              const uint64_t* const* peer_flags, int world, unsigned long long* out,
                              cudaStream_t s);
cudaError_t launch_prologue(const GroupTable& t, int n_groups, GroupConst* dst, cudaStream_t s);
cudaError_t launch_pass_a(const StepParams& p, int nsrc, bool g32, int budget, cudaStream_t s);
cudaError_t launch_pass_b(const StepParams& p, int ndst, int budget, cudaStream_t s);
// NVLS mode: pass A reduces the gradients through the switch (p.gmc), pass B stores the params
// through it (p.pmc)
cudaError_t launch_pass_a_nvls(const StepParams& p, int budget, cudaStream_t s);
cudaError_t launch_pass_b_nvls(const StepParams& p, int budget, cudaStream_t s);
cudaError_t launch_grad_stats(const StepParams& p, int nsrc, bool materialise, int budget, cudaStream_t s);
cudaError_t launch_clip_finalize(const ClipParams& p, cudaStream_t s);
cudaError_t launch_clip_combine(const ClipParams& p, cudaStream_t s);
cudaError_t launch_finalize_segments(const FinalizeParams& p, cudaStream_t s);
cudaError_t launch_finalize_straddlers(const FinalizeParams& p, cudaStream_t s);
cudaError_t launch_barrier(uint64_t* const* flags, uint64_t* epoch, int rank, int world,
                           int* err_flag, cudaStream_t s, uint64_t timeout_ns);
cudaError_t launch_gather(const __nv_bfloat16* const* peers, __nv_bfloat16* dst, int64_t base, int64_t slice,
                          int world, int rank, cudaStream_t s);
// copy-engine schedule: raise flags (system-scope release stores, e.g. in peers' sync buffers)
// and wait for flags[(b * world + j)] >= v for b in [b0, b1), j != rank (bounded; err on timeout)
cudaError_t launch_flag_store(uint64_t* const* ptrs, int n, uint64_t v, cudaStream_t s);
cudaError_t launch_flag_wait(const uint64_t* flags, int64_t b0, int64_t b1, int world, int rank, uint64_t v,
                             int* err_flag, uint64_t timeout_ns, cudaStream_t s);
cudaError_t launch_upcast_bf16(const __nv_bfloat16* src, float* dst, int64_t n, cudaStream_t s);
cudaError_t launch_cast_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t s);

}  // namespace lamb
