// ctx.hpp — the handle behind lamb_t (internal, not ABI).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lamb.h"
#include "lamb_kernels.cuh"
#include "planner.hpp"

using lamb::GroupConst;
using lamb::Item;
using lamb::Plan;
using lamb::SegDesc;

struct CheckpointJob;   // checkpoint.cu
struct NvlsState;       // nvls.cu

struct lamb_plan_ctx {
    Plan plan;
};

struct lamb_ctx {
    Plan plan;
    lamb_config cfg{};
    std::vector<lamb_group> groups;
    std::string err;
    int device = 0;
    bool master_set = false;
    int64_t launches = 0;
    // device buffers (own)
    __nv_bfloat16* grad = nullptr;     // flat
    __nv_bfloat16* param = nullptr;    // flat
    float *w = nullptr, *m = nullptr, *v = nullptr;   // shard
    Item* items = nullptr;
    int64_t n_items = 0;
    // FUSED whole-table pass B order: [0, n_items_b_plain) non-straddler items, then straddler
    // items (null when this rank touches no straddler)
    Item* items_b = nullptr;
    int64_t n_items_b_plain = 0;
    cudaStream_t x_stream = nullptr;   // FUSED: straddler exchange concurrent with pass B
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool no_strad_hide = false;        // LAMB_NO_STRAD_HIDE (A/B timing)
    std::vector<int64_t> bucket_item_begin;   // [B+1] items of bucket b: [b], [b+1)
    std::vector<int64_t> bucket_seg_begin;    // [B+1] this rank's segments of bucket b
    std::vector<int64_t> bucket_strad_begin;  // [B+1] this rank's local straddler slots of bucket b
    std::vector<uint8_t> bucket_has_strad;    // [B] bucket holds a straddler (same on all ranks)
    double2* partials = nullptr;
    SegDesc* segs = nullptr;
    float* scale = nullptr;
    double *w_sq = nullptr, *u_sq = nullptr;
    float* ratio = nullptr;
    int32_t *strad_slots = nullptr, *strad_tensor = nullptr, *strad_group = nullptr;
    int32_t n_local_strad = 0;
    // sync buffer: [flags uint64 x 8][epoch uint64][pad][xbuf double2 x D x n_strad]
    char* sync = nullptr;
    size_t sync_bytes = 0;
    int* err_flag_host = nullptr;   // host-mapped
    int* err_flag_dev = nullptr;
    // peers (FUSED): index j = rank j (own entry = own pointer)
    __nv_bfloat16* peer_grad[LAMB_MAX_RANKS] = {};
    __nv_bfloat16* peer_param[LAMB_MAX_RANKS] = {};
    char* peer_sync[LAMB_MAX_RANKS] = {};
    uint32_t peer_ipc[LAMB_MAX_RANKS] = {};   // bit k: mapping k (grad, param, sync, stage) is CUDA-IPC-opened
    // NVLS mode (LAMB_COMM_NVLS): grad / param are VMM allocations bound to multicast objects;
    // peer_grad / peer_param are fd-imported mappings of the peers' allocations (not CUDA IPC)
    NvlsState* nvls = nullptr;
    __nv_bfloat16* mc_grad = nullptr;    // multicast address of the flat grad buffer
    __nv_bfloat16* mc_param = nullptr;   // multicast address of the flat param buffer
    // D > 1 with every peer's buffers mapped (FUSED or NVLS): barriers, straddler rows and the
    // deferred gather go through peer memory
    bool peer_mode() const {
        return cfg.world_size > 1 && (cfg.comm_mode == LAMB_COMM_FUSED || cfg.comm_mode == LAMB_COMM_NVLS);
    }
    bool nvls_mode() const { return cfg.world_size > 1 && cfg.comm_mode == LAMB_COMM_NVLS; }
    // NCCL (null in FUSED mode created by lamb_create_with_allgather: the step needs no NCCL)
    ncclComm_t comm = nullptr;
    lamb_allgather_fn host_ag = nullptr;   // bootstrap all-gather, set only inside lamb_create_*
    void* host_ag_user = nullptr;
    cudaStream_t comm_stream = nullptr;
    float* g32 = nullptr;          // NCCL mode: reduced fp32 grad shard
    float* up32[2] = {nullptr, nullptr};   // NCCL mode: upcast staging, 2 buckets
    int64_t max_bucket = 0;
    std::vector<cudaEvent_t> ev_rs, ev_b;   // NCCL mode: per-bucket RS done / pass B done
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;
    cudaEvent_t ev_grad_free = nullptr;                  // grad buffer may be overwritten
    // lamb_step_host: copy streams and events (created on first use)
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr, work_stream = nullptr;
    cudaEvent_t ev_h2d = nullptr, ev_params = nullptr, ev_d2h = nullptr, ev_call = nullptr;
    cudaEvent_t pre_b_event = nullptr;   // step_impl waits on it before pass B (lamb_step_host)
    // lamb_step_host per-bucket pipeline: grads of b landed / consumed, params of b ready /
    // downloaded (one event each per bucket)
    std::vector<cudaEvent_t> ev_hb, ev_gf, ev_pb, ev_db;
    cudaEvent_t gf_override = nullptr;   // step_impl records "grads consumed" here if set
    bool host_whole = false;             // LAMB_HOST_WHOLE: whole-step pipeline (A/B timing)
    cudaEvent_t grad_free_event() const { return gf_override ? gf_override : ev_grad_free; }
    int max_ctas = 0;   // SM budget of the streaming passes (0 = one full wave)
    lamb::GroupConst* d_groups = nullptr;   // per-step group constants (prologue kernel)
    // lamb_self_check: padding ranges and counters (built on first use)
    bool pad_built = false;
    int64_t *d_shard_pad = nullptr, *d_flat_pad = nullptr;
    int64_t n_shard_pad = 0, n_flat_pad = 0;
    unsigned long long* d_check = nullptr;
    // LAMB_FLAG_GRAPH
    cudaGraphExec_t graph_exec = nullptr;
    cudaStream_t cap_stream = nullptr;
    // what the captured graph froze: pre-step on/off and SM budget (launch sequence) and the
    // pre-step scalars passed to its kernels by value (max_grad_norm, inv_loss_scale bits)
    std::array<int64_t, 3> graph_key{{-1, -1, -1}};
    int64_t graph_launches = 0;
    uint64_t barrier_timeout_ns = 30000000000ull;   // LAMB_BARRIER_TIMEOUT_MS at create
    // synth tables (device)
    int64_t *d_tensor_off = nullptr, *d_numel = nullptr, *d_shard_base = nullptr,
            *d_bucket_base = nullptr, *d_bucket_slice = nullptr;
    // timing
    std::vector<cudaEvent_t> tev;   // [max_steps][LAMB_N_PHASES + 1]
    int32_t t_max = 0, t_n = 0;

    // pre-step (NEXT #3): global grad-norm clipping, loss-scale unscale, non-finite skip
    float max_grad_norm = 0.f, inv_loss_scale = 1.f;
    lamb::ClipState* d_clip = nullptr;
    double* d_clip_blocks = nullptr;
    bool prestep() const { return max_grad_norm > 0.f || inv_loss_scale != 1.f; }
    // checkpoint (two-stage save: pinned staging + background writer thread)
    float* ck_stage = nullptr;          // pinned host, 3 x shard_size
    uint64_t session = 0;               // random at create, rank 0's value on every rank
    uint64_t ck_seq = 0;                // saves so far (same on every rank: collective calls)
    std::thread ck_thread;
    lamb_status ck_status = LAMB_OK;
    std::string ck_error;

    // copy-engine schedule (LAMB_FLAG_CE, FUSED D > 1): shard-ordered staging of the D-1 peers'
    // gradient slices (peers push into it), per-(bucket, source) arrival flags in the sync buffer
    __nv_bfloat16* stage = nullptr;                    // [(D-1) x shard_size], IPC-shared
    __nv_bfloat16* peer_stage[LAMB_MAX_RANKS] = {};
    size_t ce_off = 0;                                 // byte offset of the CE flags in sync
    cudaStream_t ce_stream = nullptr;
    cudaEvent_t ev_ce_in = nullptr, ev_ce_pushed = nullptr, ev_ce_params = nullptr;
    bool ce() const { return stage != nullptr; }
    int32_t* d_item_bucket = nullptr;   // [n_items] bucket of each item (staged pass A waits)
    // Flag values are an internal per-handle epoch (identical on every rank: all ranks make the
    // same sequence of collective calls), never the caller's step: a rollback or a repeated step
    // number cannot make a stale flag satisfy a new wait.  Round k's gradient pushes raise
    // gflags to k + 1 (= ce_epoch + 1), lamb_step_staged of round k + 1 waits for that, then
    // sets ce_epoch = k + 1 and its param pushes raise pflags to it.
    uint64_t ce_epoch = 0;
    int64_t ce_staged_step = 0;      // `step` of the last lamb_step_staged (wait_params checks it)
    int64_t ce_pushes_pending = 0;   // gradient pushes since the last staged step
    bool staged_now = false;   // inside lamb_step_staged (step_impl: flag wait + staged sources)
    // gflag[b * D + j]: rank j's gradient slice of bucket b landed in this rank's staging;
    // pflag[b * D + j]: rank j's param slice of bucket b landed in this param buffer (values:
    // ce_epoch above)
    uint64_t* gflag(int j) const { return reinterpret_cast<uint64_t*>((j < 0 ? sync : peer_sync[j]) + ce_off); }
    uint64_t* pflag(int j) const { return gflag(j) + (size_t)plan.n_buckets() * cfg.world_size; }

    uint64_t* flags(int j) const { return reinterpret_cast<uint64_t*>(peer_sync[j]); }
    uint64_t* epoch() const { return reinterpret_cast<uint64_t*>(sync + 8 * LAMB_MAX_RANKS); }
    // sync buffer layout: [0,64) barrier flags, [64,72) epoch, [128,192) clip rows (double[8]),
    // [256, ...) straddler exchange rows (double2[D][n_strad])
    double* clip_rows(int j) const { return reinterpret_cast<double*>((j < 0 ? sync : peer_sync[j]) + 128); }
    double2* xbuf(int j) const {
        return reinterpret_cast<double2*>((j < 0 ? sync : peer_sync[j]) + 256);
    }
};


// Every entry point runs on its handle's device and restores the caller's current device on
// return (a process may hold handles on several GPUs; torch's "cuda" means the current one).
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// error plumbing shared by the implementation files
lamb_status lamb_fail(lamb_ctx* h, lamb_status st, const std::string& msg);
// bootstrap all-gather of lamb_create (NCCL or the caller's host all-gather), lamb_api.cu
lamb_status lamb_bootstrap_allgather(lamb_ctx* h, const void* mine, void* all, size_t bytes);
// NVLS mode buffers (nvls.cu): allocate + bind + map (COLLECTIVE, inside lamb_create), release
lamb_status lamb_nvls_setup(lamb_ctx* h);
void lamb_nvls_free(lamb_ctx* h);
#define CUDA_TRY(h, call)                                                                     \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return lamb_fail(h, e_ == cudaErrorMemoryAllocation ? LAMB_ENOMEM : LAMB_ECUDA,   \
                             std::string(#call) + ": " + cudaGetErrorString(e_));             \
    } while (0)
#define NCCL_TRY(h, call)                                                                     \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return lamb_fail(h, LAMB_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)
