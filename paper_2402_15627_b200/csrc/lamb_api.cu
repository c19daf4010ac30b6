// lamb_api.cu — implementation of include/lamb.h and include/lamb_synth.h.
//
// lamb_create: planner (row a0) -> work items -> device buffers -> NCCL communicator ->
// (FUSED) CUDA-IPC mapping of every peer's grad / param / sync buffers over NVLink.
// lamb_step (rows a1-a7), FUSED mode, all on the caller's stream:
//     barrier("grads ready") -> pass A (peer bf16 loads, fp32 sum = fused reduce-scatter)
//     -> finalize segments (+ straddler rows stored into every peer) -> barrier
//     -> finalize straddlers -> pass B (bf16 params stored into every peer = fused
//     all-gather) -> barrier("params complete").
// NCCL mode (baseline): per bucket upcast + ncclReduceScatter(fp32) on a comm stream,
// overlapped with pass A of earlier buckets; ncclAllGather(fp64) of straddler rows;
// per-bucket ncclAllGather(bf16) of params overlapped with pass B of later buckets.
// D = 1: pass A -> finalize -> pass B.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <unistd.h>

#include <chrono>
#include <cmath>
#include <random>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lamb.h"
#include "../../include/lamb_synth.h"
#ifdef LAMB_DEBUG
#include "../../include/lamb_debug.h"
#endif
#include "lamb_kernels.cuh"
#include "planner.hpp"
#include "synth.cuh"
#include "ctx.hpp"

using namespace lamb;


// ------------------------------------------------------------------ error plumbing
static thread_local std::string g_last_error_storage;

lamb_status lamb_fail(lamb_ctx* h, lamb_status st, const std::string& msg) {
    g_last_error_storage = msg;
    if (h) h->err = msg;
    return st;
}
static inline lamb_status fail(lamb_ctx* h, lamb_status st, const std::string& msg) { return lamb_fail(h, st, msg); }
#define g_last_error g_last_error_storage

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
    *p = nullptr;
    if (n == 0) n = 1;
    return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

template <typename T>
static cudaError_t upload(T** p, const std::vector<T>& v) {
    cudaError_t e = dalloc(p, v.size());
    if (e != cudaSuccess) return e;
    if (v.empty()) return cudaSuccess;
    return cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// ------------------------------------------------------------------ planner ABI
extern "C" lamb_status lamb_plan_create(const lamb_tensor* tensors, int64_t n_tensors,
                                        int32_t world_size, int32_t rank, int64_t cap,
                                        lamb_plan_t* out) {
    if (!out || !tensors || n_tensors < 1) return fail(nullptr, LAMB_EINVAL, "bad arguments");
    std::vector<int64_t> numel(n_tensors);
    std::vector<int32_t> grp(n_tensors);
    for (int64_t i = 0; i < n_tensors; ++i) {
        numel[i] = tensors[i].numel;
        grp[i] = tensors[i].group;
    }
    auto* p = new lamb_plan_ctx();
    std::string why = build_plan(numel.data(), grp.data(), n_tensors, world_size, rank, cap, &p->plan);
    if (!why.empty()) {
        delete p;
        return fail(nullptr, LAMB_EINVAL, why);
    }
    *out = p;
    return LAMB_OK;
}

static void fill_view(const Plan& p, lamb_plan_view* v) {
    v->n_tensors = p.n_tensors();
    v->n_buckets = p.n_buckets();
    v->n_segments = p.n_segments();
    v->n_straddlers = (int64_t)p.straddlers.size();
    v->flat_size = p.flat_size;
    v->shard_size = p.shard_size;
    v->world_size = p.world;
    v->rank = p.rank;
    v->tensor_off = p.tensor_off.data();
    v->tensor_bucket = p.tensor_bucket.data();
    v->buckets = p.buckets.data();
    v->segments = p.segments.data();
    v->straddlers = p.straddlers.data();
}

extern "C" lamb_status lamb_plan_get(lamb_plan_t plan, lamb_plan_view* out) {
    if (!plan || !out) return fail(nullptr, LAMB_EINVAL, "null argument");
    fill_view(plan->plan, out);
    return LAMB_OK;
}

extern "C" void lamb_plan_destroy(lamb_plan_t plan) { delete plan; }

// ------------------------------------------------------------------ lifecycle
extern "C" lamb_status lamb_get_unique_id(uint8_t id[LAMB_UNIQUE_ID_BYTES]) {
    if (!id) return fail(nullptr, LAMB_EINVAL, "null id");
    static_assert(sizeof(ncclUniqueId) == LAMB_UNIQUE_ID_BYTES, "nccl id size");
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return fail(nullptr, LAMB_ENCCL, ncclGetErrorString(r));
    memcpy(id, &u, sizeof(u));
    return LAMB_OK;
}

static std::string check_group(const lamb_group& g) {
    if (!(g.lr >= 0.f)) return "lr must be >= 0";
    if (!(g.beta1 >= 0.f && g.beta1 < 1.f)) return "beta1 must be in [0,1)";
    if (!(g.beta2 >= 0.f && g.beta2 < 1.f)) return "beta2 must be in [0,1)";
    if (!(g.eps >= 0.f)) return "eps must be >= 0";
    if (!(g.weight_decay >= 0.f)) return "weight_decay must be >= 0";
    if (g.adapt != 0 && g.adapt != 1) return "adapt must be 0 or 1";
    if (g.bias_correction != 0 && g.bias_correction != 1) return "bias_correction must be 0 or 1";
    return std::string();
}

static void free_ctx(lamb_ctx* h) {
    if (!h) return;
    if (h->ck_thread.joinable()) h->ck_thread.join();
    DeviceGuard device_guard_(h->device);
    if (h->ck_stage) cudaFreeHost(h->ck_stage);
    cudaDeviceSynchronize();
    lamb_nvls_free(h);   // NVLS: VMM grad/param + peer views + multicast (nulls the pointers)
    for (int j = 0; j < h->cfg.world_size && j < LAMB_MAX_RANKS; ++j) {
        // only IPC-opened peer mappings (peers in other processes); other entries alias this
        // rank's buffers or a same-process peer's own allocation
        if (h->peer_ipc[j] & 1u) cudaIpcCloseMemHandle(h->peer_grad[j]);
        if (h->peer_ipc[j] & 2u) cudaIpcCloseMemHandle(h->peer_param[j]);
        if (h->peer_ipc[j] & 4u) cudaIpcCloseMemHandle(h->peer_sync[j]);
        if (h->peer_ipc[j] & 8u) cudaIpcCloseMemHandle(h->peer_stage[j]);
    }
    void* ptrs[] = {h->grad, h->param, h->w, h->m, h->v, h->items, h->items_b, h->stage, h->d_item_bucket, h->partials, h->segs, h->scale,
                    h->w_sq, h->u_sq, h->ratio, h->strad_slots, h->strad_tensor, h->strad_group,
                    h->sync, h->g32, h->up32[0], h->up32[1], h->d_clip, h->d_clip_blocks, h->d_groups, h->d_shard_pad, h->d_flat_pad, h->d_check, h->d_tensor_off, h->d_numel,
                    h->d_shard_base, h->d_bucket_base, h->d_bucket_slice};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->err_flag_host) cudaFreeHost(h->err_flag_host);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    for (auto* vec : {&h->ev_rs, &h->ev_b, &h->tev, &h->ev_hb, &h->ev_gf, &h->ev_pb, &h->ev_db})
        for (cudaEvent_t e : *vec) cudaEventDestroy(e);
    for (cudaEvent_t e : {h->ev_start, h->ev_done, h->ev_grad_free, h->ev_h2d, h->ev_params, h->ev_d2h,
                          h->ev_call, h->ev_fork, h->ev_join, h->ev_ce_in, h->ev_ce_pushed, h->ev_ce_params})
        if (e) cudaEventDestroy(e);
    for (cudaStream_t st : {h->comm_stream, h->h2d_stream, h->d2h_stream, h->work_stream, h->cap_stream,
                            h->x_stream, h->ce_stream})
        if (st) cudaStreamDestroy(st);
    if (h->comm) ncclCommDestroy(h->comm);
    delete h;
}

static lamb_status build_tables(lamb_ctx* h) {
    const Plan& p = h->plan;
    const int64_t nseg = p.n_segments();
    std::vector<Item> items;
    std::vector<SegDesc> segs(nseg);
    std::vector<int64_t> strad_slot_of(p.n_tensors(), -1);
    for (size_t k = 0; k < p.straddlers.size(); ++k) strad_slot_of[p.straddlers[k]] = (int64_t)k;
    std::vector<int32_t> ls_slot, ls_tensor, ls_group;
    const int64_t B = p.n_buckets();
    h->bucket_item_begin.assign(B + 1, 0);
    h->bucket_seg_begin.assign(B + 1, 0);
    h->bucket_strad_begin.assign(B + 1, 0);
    h->bucket_has_strad.assign(B, 0);
    for (int64_t t : p.straddlers) h->bucket_has_strad[p.tensor_bucket[t]] = 1;
    int64_t b = 0;
    for (int64_t s = 0; s < nseg; ++s) {
        const int64_t t = p.segments[4 * s], soff = p.segments[4 * s + 1];
        const int64_t len = p.segments[4 * s + 3];
        const int64_t tb = p.tensor_bucket[t];
        while (b < tb) {
            ++b;
            h->bucket_item_begin[b] = (int64_t)items.size();
            h->bucket_seg_begin[b] = s;
            h->bucket_strad_begin[b] = (int64_t)ls_slot.size();
        }
        const int64_t slice = p.buckets[4 * tb + 1] / p.world;
        const int64_t flat0 = p.buckets[4 * tb] + (int64_t)p.rank * slice + (soff - p.shard_base[tb]);
        // the segment rounded up to 8 stays inside zero padding (P2: next start is 8-aligned,
        // P6: slice ends are 128-aligned)
        const int64_t len8 = (len + 7) / 8 * 8;
        segs[s].item_begin = (int64_t)items.size();
        for (int64_t o = 0; o < len8; o += kItemElems) {
            const int64_t n = std::min<int64_t>(kItemElems, len8 - o);
            Item it;
            it.shard_off = soff + o;
            it.flat_off = flat0 + o;
            it.n_chunk = (int32_t)(n / kChunk);
            it.tensor = (int32_t)t;
            it.group = p.group[t];
            it.seg = (int32_t)s;
            items.push_back(it);
        }
        segs[s].item_end = (int64_t)items.size();
        segs[s].tensor = (int32_t)t;
        segs[s].group = p.group[t];
        segs[s].strad_slot = (int32_t)strad_slot_of[t];
        segs[s].pad = 0;
        if (strad_slot_of[t] >= 0) {
            ls_slot.push_back((int32_t)strad_slot_of[t]);
            ls_tensor.push_back((int32_t)t);
            ls_group.push_back(p.group[t]);
        }
    }
    while (b < B) {
        ++b;
        h->bucket_item_begin[b] = (int64_t)items.size();
        h->bucket_seg_begin[b] = nseg;
        h->bucket_strad_begin[b] = (int64_t)ls_slot.size();
    }
    h->n_items = (int64_t)items.size();
    h->n_local_strad = (int32_t)ls_slot.size();
    CUDA_TRY(h, upload(&h->items, items));
    {
        std::vector<int32_t> ib(items.size());
        for (int64_t k = 0; k < B; ++k)
            for (int64_t i = h->bucket_item_begin[k]; i < h->bucket_item_begin[k + 1]; ++i) ib[i] = (int32_t)k;
        CUDA_TRY(h, upload(&h->d_item_bucket, ib));
    }
    if (p.world > 1 && h->n_local_strad > 0) {
        // pass B order for the whole-table FUSED step: items of non-straddler tensors first (their
        // trust ratios are final after the local finalize), straddler items last (they wait for the
        // cross-rank exchange, which runs on a side stream meanwhile)
        std::vector<Item> ib;
        ib.reserve(items.size());
        for (const Item& it : items)
            if (strad_slot_of[it.tensor] < 0) ib.push_back(it);
        h->n_items_b_plain = (int64_t)ib.size();
        for (const Item& it : items)
            if (strad_slot_of[it.tensor] >= 0) ib.push_back(it);
        CUDA_TRY(h, upload(&h->items_b, ib));
    }
    CUDA_TRY(h, upload(&h->segs, segs));
    CUDA_TRY(h, upload(&h->strad_slots, ls_slot));
    CUDA_TRY(h, upload(&h->strad_tensor, ls_tensor));
    CUDA_TRY(h, upload(&h->strad_group, ls_group));
    CUDA_TRY(h, dalloc(&h->partials, (size_t)h->n_items));
    const size_t T = (size_t)p.n_tensors();
    CUDA_TRY(h, dalloc(&h->scale, T));
    CUDA_TRY(h, dalloc(&h->w_sq, T));
    CUDA_TRY(h, dalloc(&h->u_sq, T));
    CUDA_TRY(h, dalloc(&h->ratio, T));
    CUDA_TRY(h, cudaMemset(h->w_sq, 0xFF, T * sizeof(double)));   // NaN = not touched
    CUDA_TRY(h, cudaMemset(h->u_sq, 0xFF, T * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->ratio, 0xFF, T * sizeof(float)));
    // synth tables
    std::vector<int64_t> bb(B), bs(B);
    for (int64_t k = 0; k < B; ++k) {
        bb[k] = p.buckets[4 * k];
        bs[k] = p.buckets[4 * k + 1] / p.world;
        h->max_bucket = std::max(h->max_bucket, p.buckets[4 * k + 1]);
    }
    CUDA_TRY(h, upload(&h->d_tensor_off, p.tensor_off));
    CUDA_TRY(h, upload(&h->d_numel, p.numel));
    CUDA_TRY(h, upload(&h->d_shard_base, p.shard_base));
    CUDA_TRY(h, upload(&h->d_bucket_base, bb));
    CUDA_TRY(h, upload(&h->d_bucket_slice, bs));
    return LAMB_OK;
}

// Bootstrap exchange: every rank contributes `bytes` bytes, `all` receives D * bytes in rank
// order.  Through NCCL (device staging) when the handle has a communicator, else through the
// caller's host all-gather (lamb_create_with_allgather).
lamb_status lamb_bootstrap_allgather(lamb_ctx* h, const void* mine, void* all, size_t bytes) {
    const int D = h->cfg.world_size;
    if (h->host_ag) {
        if (h->host_ag(mine, all, bytes, h->host_ag_user) != 0)
            return fail(h, LAMB_EINVAL, "lamb_create: the caller's all-gather failed");
        return LAMB_OK;
    }
    char* dbuf = nullptr;
    CUDA_TRY(h, cudaMalloc(&dbuf, bytes * (D + 1)));
    // freed on every return path, the error returns of the TRY macros included
    std::unique_ptr<char, cudaError_t (*)(void*)> guard(dbuf, cudaFree);
    CUDA_TRY(h, cudaMemcpy(dbuf + bytes * D, mine, bytes, cudaMemcpyHostToDevice));
    NCCL_TRY(h, ncclAllGather(dbuf + bytes * D, dbuf, bytes, ncclChar, h->comm, 0));
    CUDA_TRY(h, cudaMemcpy(all, dbuf, bytes * D, cudaMemcpyDeviceToHost));
    return LAMB_OK;
}

static lamb_status setup_comm(lamb_ctx* h, const uint8_t* id) {
    const int D = h->cfg.world_size, r = h->cfg.rank;
    if (!h->host_ag) {
        ncclUniqueId u;
        memcpy(&u, id, sizeof(u));
        NCCL_TRY(h, ncclCommInitRank(&h->comm, D, u, r));
    }
    {
        // collective-misuse check: every rank must pass the same tables and config (except
        // rank/device) — a 64-bit FNV-1a hash of them is all-gathered and compared
        uint64_t hv = 1469598103934665603ull;
        auto mix = [&](const void* data, size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(data);
            for (size_t i = 0; i < n; ++i) hv = (hv ^ b[i]) * 1099511628211ull;
        };
        mix(h->plan.numel.data(), h->plan.numel.size() * 8);
        mix(h->plan.group.data(), h->plan.group.size() * 4);
        mix(h->groups.data(), h->groups.size() * sizeof(lamb_group));
        const int64_t cfgv[4] = {h->cfg.world_size, h->cfg.comm_mode, h->plan.cap, (int64_t)h->cfg.flags};
        mix(cfgv, sizeof(cfgv));
        mix(&h->cfg.grad_scale, sizeof(float));
        // with it travels each rank's random session id; rank 0's becomes everyone's (it tags
        // the per-rank commit records of checkpoints, checkpoint.cu)
        const uint64_t mine[2] = {hv, h->session};
        std::vector<uint64_t> all(2 * (size_t)D);
        lamb_status st = lamb_bootstrap_allgather(h, mine, all.data(), sizeof(mine));
        if (st != LAMB_OK) return st;
        for (int j = 0; j < D; ++j)
            if (all[2 * j] != hv)
                return fail(h, LAMB_EINVAL, "lamb_create: rank " + std::to_string(j) +
                                                " passed a different tensor/group table or config");
        h->session = all[1];
    }
    for (int j = 0; j < D; ++j) {
        h->peer_grad[j] = h->grad;
        h->peer_param[j] = h->param;
        h->peer_sync[j] = h->sync;
    }
    if (!h->peer_mode()) return LAMB_OK;
    if (h->nvls_mode()) {
        // NVLS: grad / param are multicast-bound VMM allocations, peers mapped by fd (nvls.cu)
        lamb_status st = lamb_nvls_setup(h);
        if (st != LAMB_OK) return st;
    }
    // exchange IPC handles of grad / param / sync (+ the CE staging) in one all-gather (NVLS:
    // only the sync buffer travels as a CUDA-IPC handle).  With them travel the process id, the
    // device and the raw pointers: a peer in THIS process (several ranks driven by one process,
    // one thread per GPU) is mapped by peer access, not by IPC, which cannot open a handle of
    // its own process.
    struct PeerRec {
        cudaIpcMemHandle_t ipc[4];
        void* raw[4];
        uint64_t process;   // process identity: random per process (pids repeat across containers)
        int32_t device, pad;
    };
    PeerRec mine;
    memset(&mine, 0, sizeof(mine));
    const bool nv = h->nvls_mode();
    const int nh = nv ? 1 : (h->ce() ? 4 : 3);
    void* bufs[4] = {nv ? (void*)h->sync : (void*)h->grad, (void*)h->param, (void*)h->sync, (void*)h->stage};
    for (int k = 0; k < nh; ++k) {
        CUDA_TRY(h, cudaIpcGetMemHandle(&mine.ipc[k], bufs[k]));
        mine.raw[k] = bufs[k];
    }
    static const uint64_t process_token = [] {
        std::random_device rd;
        return ((uint64_t)rd() << 32) ^ (uint64_t)rd() ^ ((uint64_t)getpid() << 20) ^
               (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
    }();
    mine.process = process_token;
    mine.device = h->device;
    std::vector<PeerRec> all((size_t)D);
    {
        lamb_status st = lamb_bootstrap_allgather(h, &mine, all.data(), sizeof(PeerRec));
        if (st != LAMB_OK) return st;
    }
    for (int j = 0; j < D; ++j) {
        if (j == r) continue;
        const bool local = all[j].process == mine.process;
        if (local && all[j].device != h->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(all[j].device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else CUDA_TRY(h, e);
        }
        void* q[4] = {nullptr, nullptr, nullptr, nullptr};
        for (int k = 0; k < nh; ++k) {
            if (local) {
                q[k] = all[j].raw[k];
            } else {
                CUDA_TRY(h, cudaIpcOpenMemHandle(&q[k], all[j].ipc[k], cudaIpcMemLazyEnablePeerAccess));
                h->peer_ipc[j] |= 1u << (nv ? 2 : k);   // which mappings free_ctx must close
            }
        }
        if (nv) {
            h->peer_sync[j] = static_cast<char*>(q[0]);
            continue;
        }
        h->peer_grad[j] = static_cast<__nv_bfloat16*>(q[0]);
        h->peer_param[j] = static_cast<__nv_bfloat16*>(q[1]);
        h->peer_sync[j] = static_cast<char*>(q[2]);
        if (h->ce()) h->peer_stage[j] = static_cast<__nv_bfloat16*>(q[3]);
    }
    // make sure every rank has mapped everything before the first step
    CUDA_TRY(h, cudaDeviceSynchronize());
    {
        const uint8_t ok = 1;
        std::vector<uint8_t> oks(D);
        lamb_status st = lamb_bootstrap_allgather(h, &ok, oks.data(), 1);
        if (st != LAMB_OK) return st;
    }
    return LAMB_OK;
}

static lamb_status create_impl(const lamb_tensor* tensors, int64_t n_tensors, const lamb_group* groups,
                               int32_t n_groups, const lamb_config* cfg, const uint8_t* id,
                               lamb_allgather_fn host_ag, void* host_ag_user, lamb_t* out) {
    if (!out || !tensors || !groups || !cfg) return fail(nullptr, LAMB_EINVAL, "null argument");
    *out = nullptr;
    if (n_groups < 1 || n_groups > LAMB_MAX_GROUPS)
        return fail(nullptr, LAMB_EINVAL, "n_groups must be in [1, 64]");
    for (int32_t k = 0; k < n_groups; ++k) {
        std::string why = check_group(groups[k]);
        if (!why.empty()) return fail(nullptr, LAMB_EINVAL, "group " + std::to_string(k) + ": " + why);
    }
    if (n_tensors < 1) return fail(nullptr, LAMB_EINVAL, "n_tensors must be >= 1");
    for (int64_t i = 0; i < n_tensors; ++i) {
        if (tensors[i].group < 0 || tensors[i].group >= n_groups)
            return fail(nullptr, LAMB_EINVAL, "tensor " + std::to_string(i) + ": group out of range");
        if (tensors[i].reserved != 0) return fail(nullptr, LAMB_EINVAL, "reserved must be 0");
    }
    if (cfg->world_size > 1 && !id && !host_ag) return fail(nullptr, LAMB_EINVAL, "unique id required for D > 1");
    if (cfg->world_size > 1 && host_ag && cfg->comm_mode == LAMB_COMM_NCCL)
        return fail(nullptr, LAMB_EINVAL, "the host all-gather bootstrap needs LAMB_COMM_FUSED or NVLS (no NCCL communicator)");
    if (cfg->world_size > 1 && cfg->comm_mode != LAMB_COMM_NCCL && cfg->comm_mode != LAMB_COMM_FUSED &&
        cfg->comm_mode != LAMB_COMM_NVLS)
        return fail(nullptr, LAMB_EUNSUPPORTED, "unknown comm_mode");
    if (cfg->world_size > 1 && cfg->comm_mode == LAMB_COMM_NVLS && (cfg->flags & LAMB_FLAG_CE))
        return fail(nullptr, LAMB_EUNSUPPORTED, "LAMB_FLAG_CE is a FUSED-mode schedule (not NVLS)");
    if (!(cfg->grad_scale >= 0.f)) return fail(nullptr, LAMB_EINVAL, "grad_scale must be >= 0");

    auto* h = new lamb_ctx();
    h->cfg = *cfg;
    h->host_ag = host_ag;
    h->host_ag_user = host_ag_user;
    {
        // failure detection: bound on every cross-GPU wait (a missing peer must not hang the GPU)
        const char* e = getenv("LAMB_BARRIER_TIMEOUT_MS");
        const long ms = e ? atol(e) : 30000;
        h->barrier_timeout_ns = (uint64_t)(ms > 0 ? ms : 30000) * 1000000ull;
    }
    h->device = cfg->device;
    {
        std::random_device rd;
        h->session = ((uint64_t)rd() << 32) ^ (uint64_t)rd() ^
                     (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count() ^ ((uint64_t)getpid() << 17);
    }
    h->groups.assign(groups, groups + n_groups);
    if (h->cfg.grad_scale == 0.f) h->cfg.grad_scale = 1.0f / (float)cfg->world_size;
    std::vector<int64_t> numel(n_tensors);
    std::vector<int32_t> grp(n_tensors);
    for (int64_t i = 0; i < n_tensors; ++i) {
        numel[i] = tensors[i].numel;
        grp[i] = tensors[i].group;
    }
    std::string why = build_plan(numel.data(), grp.data(), n_tensors, cfg->world_size, cfg->rank,
                                 cfg->bucket_cap_elems, &h->plan);
    if (!why.empty()) {
        fail(nullptr, LAMB_EINVAL, why);
        delete h;
        return LAMB_EINVAL;
    }
    lamb_status st = LAMB_OK;
    auto bail = [&](lamb_status s) {
        g_last_error = h->err;
        free_ctx(h);
        return s;
    };
    DeviceGuard device_guard_(cfg->device);
    if (!device_guard_.ok) {
        fail(h, LAMB_ECUDA, "cudaSetDevice(" + std::to_string(cfg->device) + ") failed");
        return bail(LAMB_ECUDA);
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10 || prop.minor != 0) {
        fail(h, LAMB_EUNSUPPORTED, "device is not sm_100 (B200); no fallback path exists");
        return bail(LAMB_EUNSUPPORTED);
    }
#define STEP(x)                      \
    do {                             \
        st = (x);                    \
        if (st != LAMB_OK) return bail(st); \
    } while (0)
#define CUDA_STEP(x)                                                                         \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            st = fail(h, e_ == cudaErrorMemoryAllocation ? LAMB_ENOMEM : LAMB_ECUDA,         \
                      std::string(#x) + ": " + cudaGetErrorString(e_));                      \
            return bail(st);                                                                 \
        }                                                                                    \
    } while (0)
    const Plan& p = h->plan;
    const int D = cfg->world_size;
    if (!(D > 1 && cfg->comm_mode == LAMB_COMM_NVLS)) {   // NVLS: multicast-bound VMM, setup_comm
        CUDA_STEP(dalloc(&h->grad, (size_t)p.flat_size));
        CUDA_STEP(dalloc(&h->param, (size_t)p.flat_size));
        CUDA_STEP(cudaMemset(h->grad, 0, (size_t)p.flat_size * 2));
        CUDA_STEP(cudaMemset(h->param, 0, (size_t)p.flat_size * 2));
    }
    CUDA_STEP(dalloc(&h->w, (size_t)p.shard_size));
    CUDA_STEP(dalloc(&h->m, (size_t)p.shard_size));
    CUDA_STEP(dalloc(&h->v, (size_t)p.shard_size));
    CUDA_STEP(cudaMemset(h->w, 0, (size_t)p.shard_size * 4));
    CUDA_STEP(cudaMemset(h->m, 0, (size_t)p.shard_size * 4));
    CUDA_STEP(cudaMemset(h->v, 0, (size_t)p.shard_size * 4));
    STEP(build_tables(h));
    h->sync_bytes = 256 + sizeof(double2) * (size_t)D * std::max<size_t>(1, p.straddlers.size());
    const bool want_ce = D > 1 && cfg->comm_mode == LAMB_COMM_FUSED && (cfg->flags & LAMB_FLAG_CE);
    if (want_ce) {
        // copy-engine schedule: arrival flags after the straddler rows; the staging buffer
        h->ce_off = (h->sync_bytes + 63) & ~(size_t)63;
        h->sync_bytes = h->ce_off + 2 * sizeof(uint64_t) * (size_t)p.n_buckets() * D;
        CUDA_STEP(dalloc(&h->stage, (size_t)(D - 1) * (size_t)p.shard_size));
        CUDA_STEP(cudaMemset(h->stage, 0, (size_t)(D - 1) * (size_t)p.shard_size * 2));
    }
    CUDA_STEP(dalloc(&h->sync, h->sync_bytes));
    CUDA_STEP(cudaMemset(h->sync, 0, h->sync_bytes));
    CUDA_STEP(dalloc(&h->d_clip, 1));
    CUDA_STEP(dalloc(&h->d_groups, LAMB_MAX_GROUPS));
    CUDA_STEP(dalloc(&h->d_clip_blocks, lamb::kClipBlocksMax));
    CUDA_STEP(cudaMemset(h->d_clip, 0, sizeof(lamb::ClipState)));
    CUDA_STEP(cudaHostAlloc(&h->err_flag_host, sizeof(int), cudaHostAllocMapped));
    *h->err_flag_host = 0;
    CUDA_STEP(cudaHostGetDevicePointer(&h->err_flag_dev, h->err_flag_host, 0));
    CUDA_STEP(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
    CUDA_STEP(cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming));
    CUDA_STEP(cudaEventCreateWithFlags(&h->ev_grad_free, cudaEventDisableTiming));
    for (int j = 0; j < LAMB_MAX_RANKS; ++j) {
        h->peer_grad[j] = h->grad;
        h->peer_param[j] = h->param;
        h->peer_sync[j] = h->sync;
    }
    if (D > 1) {
        STEP(setup_comm(h, id));
        if (h->peer_mode()) {
            CUDA_STEP(cudaStreamCreateWithFlags(&h->x_stream, cudaStreamNonBlocking));
            CUDA_STEP(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
            CUDA_STEP(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
            const char* e = getenv("LAMB_NO_STRAD_HIDE");
            h->no_strad_hide = e && *e && *e != '0';
            if (h->ce()) {
                CUDA_STEP(cudaStreamCreateWithFlags(&h->ce_stream, cudaStreamNonBlocking));
                for (cudaEvent_t* e2 : {&h->ev_ce_in, &h->ev_ce_pushed, &h->ev_ce_params})
                    CUDA_STEP(cudaEventCreateWithFlags(e2, cudaEventDisableTiming));
            }
        }
        if (cfg->comm_mode == LAMB_COMM_NCCL) {
            CUDA_STEP(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
            CUDA_STEP(dalloc(&h->g32, (size_t)p.shard_size));
            CUDA_STEP(cudaMemset(h->g32, 0, (size_t)p.shard_size * 4));
            CUDA_STEP(dalloc(&h->up32[0], (size_t)h->max_bucket));
            CUDA_STEP(dalloc(&h->up32[1], (size_t)h->max_bucket));
            const int64_t B = p.n_buckets();
            for (auto* vec : {&h->ev_rs, &h->ev_b}) {
                vec->resize(B);
                for (auto& e : *vec) CUDA_STEP(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
        }
    }
    CUDA_STEP(cudaDeviceSynchronize());
    *out = h;
    return LAMB_OK;
#undef STEP
#undef CUDA_STEP
}

extern "C" lamb_status lamb_create(const lamb_tensor* tensors, int64_t n_tensors, const lamb_group* groups,
                                   int32_t n_groups, const lamb_config* cfg, const uint8_t* id, lamb_t* out) {
    return create_impl(tensors, n_tensors, groups, n_groups, cfg, id, nullptr, nullptr, out);
}

extern "C" lamb_status lamb_create_with_allgather(const lamb_tensor* tensors, int64_t n_tensors,
                                                  const lamb_group* groups, int32_t n_groups,
                                                  const lamb_config* cfg, lamb_allgather_fn allgather,
                                                  void* user, lamb_t* out) {
    if (!allgather) return fail(nullptr, LAMB_EINVAL, "null all-gather callback");
    lamb_status st = create_impl(tensors, n_tensors, groups, n_groups, cfg, nullptr, allgather, user, out);
    if (st == LAMB_OK) {
        (*out)->host_ag = nullptr;   // only valid during the call
        (*out)->host_ag_user = nullptr;
    }
    return st;
}

extern "C" void lamb_destroy(lamb_t h) { free_ctx(h); }

// ------------------------------------------------------------------ the step
static void group_consts(const lamb_ctx* h, int64_t t, GroupConst* out) {
    for (size_t k = 0; k < h->groups.size(); ++k) {
        const lamb_group& g = h->groups[k];
        GroupConst& c = out[k];
        c.lr = g.lr;
        c.b1 = g.beta1;
        c.b2 = g.beta2;
        c.omb1 = (float)(1.0 - (double)g.beta1);   // exact for fp32 betas in [0.5, 1)
        c.omb2 = (float)(1.0 - (double)g.beta2);
        c.eps = g.eps;
        c.wd = g.weight_decay;
        // bias correction in double on the host (reading Z14), passed as fp32
        c.c1 = g.bias_correction ? (float)(1.0 / (1.0 - std::pow((double)g.beta1, (double)t))) : 1.0f;
        c.c2 = g.bias_correction ? (float)(1.0 / (1.0 - std::pow((double)g.beta2, (double)t))) : 1.0f;
        c.adapt = g.adapt;
    }
}

static inline void mark(lamb_ctx* h, int phase, cudaStream_t s) {
    if (h->t_n < h->t_max) cudaEventRecord(h->tev[(size_t)h->t_n * (LAMB_N_PHASES + 1) + phase], s);
}

#define LAUNCH(h, call)                                                                       \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail(h, LAMB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
        ++(h)->launches;                                                                      \
    } while (0)

// One LAMB step over the buckets [b0, b1) (the whole table for lamb_step, one bucket for
// lamb_step_bucket).  Every tensor lives in exactly one bucket, so a bucket range is a
// self-contained LAMB update; only the pre-step's global norm needs the whole table.
// defer_ag: pass B writes only this rank's slices; the all-gather is lamb_gather_bucket.
static lamb_status step_impl(lamb_ctx* h, const void* grads, int64_t t, cudaStream_t s, int64_t b0,
                             int64_t b1, bool defer_ag) {
    const Plan& p = h->plan;
    // SM budget (lamb_set_max_ctas): fewer persistent CTAs leave SMs to concurrent compute;
    // 0 = every pass sizes a full persistent wave itself
    const int grid_a = h->max_ctas, grid_b = h->max_ctas;
    const int D = h->cfg.world_size, r = h->cfg.rank;
    const bool fused = h->peer_mode();   // FUSED or NVLS: barriers and exchanges through peer memory
    const bool nvls = h->nvls_mode();
    const bool nccl = D > 1 && h->cfg.comm_mode == LAMB_COMM_NCCL;
    const bool whole = b0 == 0 && b1 == p.n_buckets();
    bool strad = false;   // a bucket in range holds a straddler (identical on every rank)
    for (int64_t b = b0; b < b1; ++b) strad = strad || h->bucket_has_strad[b];

    StepParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.items = h->items;
    sp.item_begin = h->bucket_item_begin[b0];
    sp.item_end = h->bucket_item_begin[b1];
    sp.grad_scale = h->cfg.grad_scale;
    sp.self_src = h->cfg.world_size > 1 ? h->cfg.rank : 0;
    sp.w = h->w;
    sp.m = h->m;
    sp.v = h->v;
    sp.partials = h->partials;
    sp.scale = h->scale;
    sp.groups = h->d_groups;
    sp.shard_elems = p.shard_size;   // extents for the LAMB_DEBUG build's bounds checks
    sp.flat_elems = p.flat_size;
    sp.n_items = h->n_items;
    sp.n_tensors = (int32_t)p.n_tensors();
    FinalizeParams fp;
    memset(&fp, 0, sizeof(fp));
    fp.n_items = h->n_items;
    fp.n_tensors = (int32_t)p.n_tensors();
    fp.segs = h->segs + h->bucket_seg_begin[b0];
    fp.n_segs = h->bucket_seg_begin[b1] - h->bucket_seg_begin[b0];
    fp.partials = h->partials;
    fp.scale = h->scale;
    fp.w_sq = h->w_sq;
    fp.u_sq = h->u_sq;
    fp.ratio = h->ratio;
    fp.world = D;
    fp.rank = r;
    fp.n_strad = (int32_t)p.straddlers.size();
    fp.strad_slots = h->strad_slots + h->bucket_strad_begin[b0];
    fp.strad_tensor = h->strad_tensor + h->bucket_strad_begin[b0];
    fp.strad_group = h->strad_group + h->bucket_strad_begin[b0];
    fp.n_local_strad = (int32_t)(h->bucket_strad_begin[b1] - h->bucket_strad_begin[b0]);
    fp.xbuf = h->xbuf(-1);
    fp.groups = h->d_groups;
    const bool pre = h->prestep();
    lamb::ClipParams cp;
    memset(&cp, 0, sizeof(cp));
    if (pre) {
        if (!whole) return fail(h, LAMB_EUNSUPPORTED, "the pre-step (clip / loss scale) needs the whole table: use lamb_step");
        if (nvls) return fail(h, LAMB_EUNSUPPORTED, "the pre-step is not available in NVLS mode");
        if (!h->g32 && D > 1) {   // FUSED + pre-step: the fp32 reduced shard lives here
            CUDA_TRY(h, dalloc(&h->g32, (size_t)p.shard_size));
        }
        sp.clip = h->d_clip;
        fp.clip = h->d_clip;
        cp.partials = h->partials;
        cp.n_items = h->n_items;
        for (int j = 0; j < D; ++j) cp.rows[j] = h->clip_rows(fused ? j : -1);
        cp.my_rows = h->clip_rows(-1);
        cp.world = D;
        cp.rank = r;
        cp.grad_scale = h->cfg.grad_scale;
        cp.inv_loss_scale = h->inv_loss_scale;
        cp.max_grad_norm = h->max_grad_norm;
        cp.out = h->d_clip;
        cp.block_sums = h->d_clip_blocks;
    }

    mark(h, 0, s);
    if (!nccl) {
        // ---------------- D = 1 or FUSED
        uint64_t* flags[LAMB_MAX_RANKS];
        for (int j = 0; j < D; ++j) flags[j] = h->flags(j);
        if (h->staged_now) {
            // copy-engine schedule: pass A waits per bucket for the peers' slices (in-kernel,
            // walking the buckets in the order the backward pushed them)
        } else if (fused) {
            LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
        }
        mark(h, 1, s);
        for (int j = 0; j < D; ++j)
            sp.gsrc[j] = fused ? h->peer_grad[j] : (grads ? (const __nv_bfloat16*)grads : h->grad);
        if (h->staged_now) {
            for (int j = 0; j < D; ++j)
                sp.gsrc[j] = j == r ? h->grad : h->stage + (size_t)(j - (j > r)) * (size_t)p.shard_size;
            sp.staged = 1;
            sp.reverse = 1;
            sp.world = D;
            sp.item_bucket = h->d_item_bucket;
            sp.gflags = h->gflag(-1);
            sp.gflag_target = h->ce_epoch + 1;   // this round's pushes (internal epoch, not t)
            sp.err = h->err_flag_dev;
            sp.timeout_ns = h->barrier_timeout_ns;
        }
        if (pre) {
            // pre-step: global ||g||^2 (FUSED: the reduce-scatter happens here, into g32)
            sp.g32_out = h->g32;
            LAUNCH(h, launch_grad_stats(sp, D, fused, grid_a, s));
            LAUNCH(h, launch_clip_finalize(cp, s));
            if (fused) {
                LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
                LAUNCH(h, launch_clip_combine(cp, s));
                sp.g32 = h->g32;
                LAUNCH(h, launch_pass_a(sp, 0, true, grid_a, s));
            } else {
                LAUNCH(h, launch_pass_a(sp, D, false, grid_a, s));
            }
        } else if (nvls) {
            sp.gmc = h->mc_grad;   // reduce-scatter through the switch (reading Z23)
            LAUNCH(h, launch_pass_a_nvls(sp, grid_a, s));
        } else {
            LAUNCH(h, launch_pass_a(sp, D, false, grid_a, s));
        }
        if (!fused) CUDA_TRY(h, cudaEventRecord(h->grad_free_event(), s));   // D = 1: grads consumed
        mark(h, 2, s);
        for (int j = 0; j < D; ++j) fp.xrow[j] = h->xbuf(fused ? j : -1);
        LAUNCH(h, launch_finalize_segments(fp, s));
        mark(h, 3, s);
        const bool push = fused && !defer_ag;
        for (int j = 0; j < D; ++j) sp.pdst[j] = push ? h->peer_param[j] : h->param;
        sp.pmc = h->mc_param;
        // pass B: FUSED pushes to the D param buffers, NVLS stores once through the switch
        auto pass_b = [&](const StepParams& q, cudaStream_t st) -> cudaError_t {
            return (push && nvls) ? launch_pass_b_nvls(q, grid_b, st) : launch_pass_b(q, push ? D : 1, grid_b, st);
        };
        // Straddler exchange hidden behind pass B (whole-table FUSED step): pass B streams the
        // non-straddler items while a side stream runs barrier + straddler finalize; the
        // straddler items follow once their ratios are final.  Every barrier stays in one
        // global order on every rank (the pre-B barrier precedes the fork).
        const bool hide = fused && strad && whole && !defer_ag && h->items_b && !h->no_strad_hide;
        if (hide) {
            if (h->pre_b_event) {
                CUDA_TRY(h, cudaStreamWaitEvent(s, h->pre_b_event, 0));
                LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
            }
            CUDA_TRY(h, cudaEventRecord(h->ev_fork, s));
            CUDA_TRY(h, cudaStreamWaitEvent(h->x_stream, h->ev_fork, 0));
            LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, h->x_stream, h->barrier_timeout_ns));
            if (fp.n_local_strad > 0) LAUNCH(h, launch_finalize_straddlers(fp, h->x_stream));
            CUDA_TRY(h, cudaEventRecord(h->ev_join, h->x_stream));
            mark(h, 4, s);
            StepParams sb = sp;
            sb.items = h->items_b;
            sb.item_begin = 0;
            sb.item_end = h->n_items_b_plain;
            LAUNCH(h, pass_b(sb, s));
            CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_join, 0));
            sb.item_begin = h->n_items_b_plain;
            sb.item_end = h->n_items;
            LAUNCH(h, pass_b(sb, s));
        } else {
            if (fused && strad) {
                // straddler rows travel through peer memory: barrier, then sum in rank order
                LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
                if (fp.n_local_strad > 0) LAUNCH(h, launch_finalize_straddlers(fp, s));
            }
            mark(h, 4, s);
            if (h->pre_b_event) {
                // lamb_step_host: the previous step's download of the param buffer(s) must finish
                // before pass B rewrites them — on every rank, since pass B stores into peers
                CUDA_TRY(h, cudaStreamWaitEvent(s, h->pre_b_event, 0));
                if (fused) LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
            }
            LAUNCH(h, pass_b(sp, s));
        }
        mark(h, 5, s);
        if (fused) {
            // params complete everywhere, and every rank finished reading this rank's grads
            LAUNCH(h, launch_barrier(flags, h->epoch(), r, D, h->err_flag_dev, s, h->barrier_timeout_ns));
            CUDA_TRY(h, cudaEventRecord(h->grad_free_event(), s));
        }
        mark(h, 6, s);
        return LAMB_OK;
    }

    // ---------------- NCCL baseline, per-bucket pipeline on (s, comm_stream)
    const __nv_bfloat16* gsrc = grads ? (const __nv_bfloat16*)grads : h->grad;
    CUDA_TRY(h, cudaEventRecord(h->ev_start, s));
    CUDA_TRY(h, cudaStreamWaitEvent(h->comm_stream, h->ev_start, 0));
    mark(h, 1, s);
    sp.g32 = h->g32;
    for (int64_t b = b0; b < b1; ++b) {
        const int64_t base = p.buckets[4 * b], S = p.buckets[4 * b + 1];
        float* up = h->up32[b & 1];
        // the staging buffer is reused every other bucket; comm_stream order guarantees the
        // reduce-scatter that read it has finished before the next upcast overwrites it
        LAUNCH(h, launch_upcast_bf16(gsrc + base, up, S, h->comm_stream));
        NCCL_TRY(h, ncclReduceScatter(up, h->g32 + p.shard_base[b], (size_t)(S / D), ncclFloat,
                                      ncclSum, h->comm, h->comm_stream));
        CUDA_TRY(h, cudaEventRecord(h->ev_rs[b], h->comm_stream));
    }
    if (pre) {
        // the global norm needs every bucket's reduced gradient: wait for all RS first
        for (int64_t b = b0; b < b1; ++b) CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_rs[b], 0));
        LAUNCH(h, launch_grad_stats(sp, 0, false, grid_a, s));
        LAUNCH(h, launch_clip_finalize(cp, s));
        double* rows = h->clip_rows(-1);
        NCCL_TRY(h, ncclAllGather(rows + r, rows, 1, ncclDouble, h->comm, s));
        LAUNCH(h, launch_clip_combine(cp, s));
        LAUNCH(h, launch_pass_a(sp, 0, true, grid_a, s));
    } else {
        for (int64_t b = b0; b < b1; ++b) {
            CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_rs[b], 0));
            sp.item_begin = h->bucket_item_begin[b];
            sp.item_end = h->bucket_item_begin[b + 1];
            LAUNCH(h, launch_pass_a(sp, 0, true, grid_a, s));
        }
    }
    mark(h, 2, s);
    for (int j = 0; j < D; ++j) fp.xrow[j] = h->xbuf(-1);
    LAUNCH(h, launch_finalize_segments(fp, s));
    mark(h, 3, s);
    if (strad) {
        const size_t n = p.straddlers.size() * 2;
        double* xb = reinterpret_cast<double*>(h->xbuf(-1));
        NCCL_TRY(h, ncclAllGather(xb + (size_t)r * n, xb, n, ncclDouble, h->comm, s));
        if (fp.n_local_strad > 0) LAUNCH(h, launch_finalize_straddlers(fp, s));
    }
    mark(h, 4, s);
    if (h->pre_b_event) CUDA_TRY(h, cudaStreamWaitEvent(s, h->pre_b_event, 0));   // see above
    sp.pdst[0] = h->param;
    for (int64_t b = b0; b < b1; ++b) {
        sp.item_begin = h->bucket_item_begin[b];
        sp.item_end = h->bucket_item_begin[b + 1];
        LAUNCH(h, launch_pass_b(sp, 1, grid_b, s));
        if (defer_ag) continue;
        CUDA_TRY(h, cudaEventRecord(h->ev_b[b], s));
        CUDA_TRY(h, cudaStreamWaitEvent(h->comm_stream, h->ev_b[b], 0));
        const int64_t base = p.buckets[4 * b], sl = p.buckets[4 * b + 1] / D;
        NCCL_TRY(h, ncclAllGather(h->param + base + (int64_t)r * sl, h->param + base, (size_t)sl,
                                  ncclBfloat16, h->comm, h->comm_stream));
    }
    CUDA_TRY(h, cudaEventRecord(h->ev_done, h->comm_stream));
    CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_done, 0));
    CUDA_TRY(h, cudaEventRecord(h->grad_free_event(), s));
    mark(h, 5, s);
    mark(h, 6, s);
    return LAMB_OK;
}

static lamb_status check_async(lamb_ctx* h) {
    if (h->err_flag_host && *(volatile int*)h->err_flag_host)
        return fail(h, LAMB_ECUDA, "cross-GPU barrier timed out in an earlier step (peer missing)");
    // an asynchronous fault of this handle's earlier work (sticky context errors surface here);
    // the thread's last-error slot is not consulted: it may hold another library's error
    const cudaError_t e = cudaEventQuery(h->ev_grad_free);
    if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(h, LAMB_ECUDA, std::string("CUDA error from earlier work: ") + cudaGetErrorString(e));
    if (h->comm) {
        ncclResult_t ae;
        if (ncclCommGetAsyncError(h->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
            return fail(h, LAMB_ENCCL, std::string("NCCL async error: ") + ncclGetErrorString(ae));
    }
    return LAMB_OK;
}

// Per-step group constants (bias corrections for this t, current lr) -> device table.
static lamb_status prologue(lamb_ctx* h, int64_t t, cudaStream_t s) {
    lamb::GroupTable T;
    memset(&T, 0, sizeof(T));
    group_consts(h, t, T.g);
    LAUNCH(h, lamb::launch_prologue(T, (int)h->groups.size(), h->d_groups, s));
    return LAMB_OK;
}

// LAMB_FLAG_GRAPH: the whole step (everything after the prologue) captured once into a CUDA
// graph and replayed; re-captured when a setting changes that the graph froze: the launch
// sequence (pre-step on/off, SM budget) or a value passed to its kernels (the pre-step's
// max_grad_norm / inv_loss_scale).
static lamb_status graph_step(lamb_ctx* h, cudaStream_t s) {
    uint32_t clip_bits, scale_bits;
    memcpy(&clip_bits, &h->max_grad_norm, 4);
    memcpy(&scale_bits, &h->inv_loss_scale, 4);
    const std::array<int64_t, 3> key{{(h->prestep() ? 1 : 0) | ((int64_t)h->max_ctas << 1), (int64_t)clip_bits,
                                      (int64_t)scale_bits}};
    if (!h->graph_exec || key != h->graph_key) {
        if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = nullptr;
        if (!h->cap_stream) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
        if (h->prestep() && h->cfg.world_size > 1 && !h->g32)   // no allocation inside a capture
            CUDA_TRY(h, dalloc(&h->g32, (size_t)h->plan.shard_size));
        const int32_t t_max = h->t_max;
        h->t_max = 0;   // no per-phase events inside the graph
        const int64_t l0 = h->launches;
        CUDA_TRY(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
        lamb_status st = step_impl(h, nullptr, 1, h->cap_stream, 0, h->plan.n_buckets(), false);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(h->cap_stream, &g);
        h->t_max = t_max;
        if (st != LAMB_OK) return st;
        if (ce != cudaSuccess) return fail(h, LAMB_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        h->graph_launches = h->launches - l0;
        h->launches = l0;
        ce = cudaGraphInstantiate(&h->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return fail(h, LAMB_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
        h->graph_key = key;
    }
    CUDA_TRY(h, cudaGraphLaunch(h->graph_exec, s));
    h->launches += h->graph_launches;
    // the graph's own record of ev_grad_free was captured, not executed on a stream; record it
    // eagerly after the replay so check_async / lamb_step_host can query and wait on it
    CUDA_TRY(h, cudaEventRecord(h->ev_grad_free, s));
    return LAMB_OK;
}

extern "C" lamb_status lamb_step(lamb_t h, const void* grads, int64_t step, void* stream) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (step < 1) return fail(h, LAMB_EINVAL, "step must be >= 1");
    if (grads && h->peer_mode())
        return fail(h, LAMB_EINVAL, "external grads are not allowed in FUSED / NVLS mode with D > 1");
    if (!h->master_set) return fail(h, LAMB_ESTATE, "lamb_step before lamb_set_master / lamb_synth_init");
    lamb_status st = check_async(h);
    if (st != LAMB_OK) return st;
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    st = prologue(h, step, s);
    if (st != LAMB_OK) return st;
    const bool graph = (h->cfg.flags & LAMB_FLAG_GRAPH) && !grads && !h->pre_b_event &&
                       !(h->cfg.world_size > 1 && h->cfg.comm_mode == LAMB_COMM_NCCL);
    if (graph) return graph_step(h, s);
    st = step_impl(h, grads, step, s, 0, h->plan.n_buckets(), false);
    if (h->t_n < h->t_max) ++h->t_n;
    return st;
}

extern "C" lamb_status lamb_step_bucket(lamb_t h, int64_t bucket, int64_t step, int32_t flags, void* stream) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (bucket < 0 || bucket >= h->plan.n_buckets()) return fail(h, LAMB_EINVAL, "bucket out of range");
    if (step < 1) return fail(h, LAMB_EINVAL, "step must be >= 1");
    if (flags & ~LAMB_BUCKET_DEFER_AG) return fail(h, LAMB_EINVAL, "unknown flags");
    if (!h->master_set) return fail(h, LAMB_ESTATE, "lamb_step_bucket before lamb_set_master / lamb_synth_init");
    lamb_status st = check_async(h);
    if (st != LAMB_OK) return st;
    DeviceGuard device_guard_(h->device);
    const int32_t t_max = h->t_max;
    h->t_max = 0;   // per-bucket calls are not phase-timed
    st = prologue(h, step, static_cast<cudaStream_t>(stream));
    if (st == LAMB_OK)
        st = step_impl(h, nullptr, step, static_cast<cudaStream_t>(stream), bucket, bucket + 1,
                       (flags & LAMB_BUCKET_DEFER_AG) != 0);
    h->t_max = t_max;
    return st;
}

extern "C" lamb_status lamb_gather_bucket(lamb_t h, int64_t bucket, void* stream) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (bucket < 0 || bucket >= h->plan.n_buckets()) return fail(h, LAMB_EINVAL, "bucket out of range");
    const Plan& p = h->plan;
    const int D = p.world, r = p.rank;
    if (D == 1) return LAMB_OK;
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t base = p.buckets[4 * bucket], sl = p.buckets[4 * bucket + 1] / D;
    if (h->peer_mode()) {
        // pull the peers' slices over NVLink; they were completed before the barrier that
        // ended their lamb_step_bucket, and are not rewritten before this rank's next
        // barrier of this bucket
        LAUNCH(h, lamb::launch_gather(const_cast<const __nv_bfloat16* const*>(h->peer_param), h->param,
                                      base, sl, D, r, s));
        return LAMB_OK;
    }
    NCCL_TRY(h, ncclAllGather(h->param + base + (int64_t)r * sl, h->param + base, (size_t)sl,
                              ncclBfloat16, h->comm, s));
    return LAMB_OK;
}

// ------------------------------------------------------------------ copy-engine schedule
static lamb_status ce_check(lamb_ctx* h, int64_t bucket, int64_t step) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (!h->ce()) return fail(h, LAMB_EUNSUPPORTED, "handle created without LAMB_FLAG_CE (FUSED, D > 1)");
    if (bucket < -1 || bucket >= h->plan.n_buckets()) return fail(h, LAMB_EINVAL, "bucket out of range");
    if (step < 1) return fail(h, LAMB_EINVAL, "step must be >= 1");
    if (h->prestep()) return fail(h, LAMB_EUNSUPPORTED, "the pre-step needs lamb_step (global norm before pass A)");
    return check_async(h);
}

extern "C" lamb_status lamb_push_grads_bucket(lamb_t h, int64_t bucket, int64_t step, void* stream) {
    lamb_status st = ce_check(h, bucket, step);
    if (st != LAMB_OK) return st;
    if (bucket < 0) return fail(h, LAMB_EINVAL, "bucket out of range");
    DeviceGuard device_guard_(h->device);
    const Plan& p = h->plan;
    const int D = p.world, r = p.rank;
    const int64_t base = p.buckets[4 * bucket], sl = p.buckets[4 * bucket + 1] / D, sb = p.shard_base[bucket];
    CUDA_TRY(h, cudaEventRecord(h->ev_ce_in, static_cast<cudaStream_t>(stream)));
    CUDA_TRY(h, cudaStreamWaitEvent(h->ce_stream, h->ev_ce_in, 0));
    uint64_t* fl[LAMB_MAX_RANKS];
    int nf = 0;
    for (int j = 0; j < D; ++j) {
        if (j == r) continue;
        // peer j's staging slot for source r, at j's (= every rank's) shard offset of bucket b
        __nv_bfloat16* dst = h->peer_stage[j] + (size_t)(r - (r > j)) * (size_t)p.shard_size + sb;
        CUDA_TRY(h, cudaMemcpyAsync(dst, h->grad + base + (int64_t)j * sl, (size_t)sl * 2, cudaMemcpyDefault,
                                    h->ce_stream));
        fl[nf++] = h->gflag(j) + bucket * D + r;
    }
    LAUNCH(h, lamb::launch_flag_store(fl, nf, h->ce_epoch + 1, h->ce_stream));
    CUDA_TRY(h, cudaEventRecord(h->ev_ce_pushed, h->ce_stream));
    ++h->ce_pushes_pending;
    return LAMB_OK;
}

extern "C" lamb_status lamb_step_staged(lamb_t h, int64_t step, void* stream) {
    lamb_status st = ce_check(h, -1, step);
    if (st != LAMB_OK) return st;
    if (!h->master_set) return fail(h, LAMB_ESTATE, "lamb_step_staged before lamb_set_master / lamb_synth_init");
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Plan& p = h->plan;
    const int D = p.world, r = p.rank;
    st = prologue(h, step, s);
    if (st != LAMB_OK) return st;
    h->staged_now = true;
    st = step_impl(h, nullptr, step, s, 0, p.n_buckets(), /*defer_ag=*/true);
    h->staged_now = false;
    if (h->t_n < h->t_max) ++h->t_n;
    if (st != LAMB_OK) return st;
    ++h->ce_epoch;
    h->ce_staged_step = step;
    h->ce_pushes_pending = 0;
    // the grad buffer is rewritten by the next backward: this rank's pushes must have read it
    // (joined here, after the update, so the last bucket's push overlaps pass A)
    CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_ce_pushed, 0));
    // the all-gather on the copy engines, bucket order (the next forward's order)
    CUDA_TRY(h, cudaEventRecord(h->ev_ce_params, s));
    CUDA_TRY(h, cudaStreamWaitEvent(h->ce_stream, h->ev_ce_params, 0));
    for (int64_t b = 0; b < p.n_buckets(); ++b) {
        const int64_t base = p.buckets[4 * b], sl = p.buckets[4 * b + 1] / D;
        const int64_t off = base + (int64_t)r * sl;
        uint64_t* fl[LAMB_MAX_RANKS];
        int nf = 0;
        for (int j = 0; j < D; ++j) {
            if (j == r) continue;
            CUDA_TRY(h, cudaMemcpyAsync(h->peer_param[j] + off, h->param + off, (size_t)sl * 2, cudaMemcpyDefault,
                                        h->ce_stream));
            fl[nf++] = h->pflag(j) + b * D + r;
        }
        LAUNCH(h, lamb::launch_flag_store(fl, nf, h->ce_epoch, h->ce_stream));
    }
    return LAMB_OK;
}

extern "C" lamb_status lamb_wait_params_bucket(lamb_t h, int64_t bucket, int64_t step, void* stream) {
    lamb_status st = ce_check(h, bucket, step);
    if (st != LAMB_OK) return st;
    if (bucket < 0) return fail(h, LAMB_EINVAL, "bucket out of range");
    if (h->ce_epoch == 0) return fail(h, LAMB_ESTATE, "no lamb_step_staged yet: no params to wait for");
    if (step != h->ce_staged_step)
        return fail(h, LAMB_EINVAL, "params of step " + std::to_string(step) + " requested, the last staged step is " +
                                        std::to_string(h->ce_staged_step));
    DeviceGuard device_guard_(h->device);
    LAUNCH(h, lamb::launch_flag_wait(h->pflag(-1), bucket, bucket + 1, h->plan.world, h->plan.rank, h->ce_epoch,
                                     h->err_flag_dev, h->barrier_timeout_ns, static_cast<cudaStream_t>(stream)));
    return LAMB_OK;
}

extern "C" lamb_status lamb_step_host(lamb_t h, const uint16_t* host_grads, uint16_t* host_params,
                                      int64_t step, void* stream) {
    // Pipeline on internal streams, per bucket and across consecutive calls (§3.2
    // overlap "on a model chunk basis"; here the chunks hide the LAMB work and the
    // two copy directions behind each other on the host link):
    //   copy-in  (h2d)  : grads of bucket b, as soon as the previous step's pass A of bucket b
    //                     released that part of the grad buffer;
    //   work            : the LAMB update of bucket b (lamb_step_bucket: pass A, norms, ratios,
    //                     pass B) once its grads landed; pass B also waits for the previous
    //                     step's download of bucket b (it rewrites those params);
    //   copy-out (d2h)  : params of bucket b as soon as its pass B finished.
    // Every tensor lives in one bucket, so the per-bucket update is the exact LAMB step
    // (bit-identical to lamb_step: tests).  With the pre-step (global clip / loss scale) the
    // whole table is one unit: whole-step pipeline.  `stream` gets a dependency on the last
    // download; the first call also orders the pipeline after the work already on `stream`.
    if (!h || !host_grads || !host_params) return fail(h, LAMB_EINVAL, "null argument");
    if (step < 1) return fail(h, LAMB_EINVAL, "step must be >= 1");
    if (!h->master_set) return fail(h, LAMB_ESTATE, "lamb_step_host before lamb_set_master / lamb_synth_init");
    lamb_status st = check_async(h);
    if (st != LAMB_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceGuard device_guard_(h->device);
    const Plan& p = h->plan;
    const int64_t B = p.n_buckets();
    if (!h->h2d_stream) {
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking));
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->work_stream, cudaStreamNonBlocking));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_h2d, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_params, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_d2h, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_call, cudaEventDisableTiming));
        for (auto* vec : {&h->ev_hb, &h->ev_gf, &h->ev_pb, &h->ev_db}) {
            vec->resize(B);
            for (auto& e : *vec) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        h->host_whole = getenv("LAMB_HOST_WHOLE") && *getenv("LAMB_HOST_WHOLE") && *getenv("LAMB_HOST_WHOLE") != '0';
        CUDA_TRY(h, cudaEventRecord(h->ev_call, s));
        CUDA_TRY(h, cudaStreamWaitEvent(h->work_stream, h->ev_call, 0));
        CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_call, 0));
    }
    // an earlier lamb_step may still read the grad buffer
    CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_grad_free, 0));
    if (h->host_whole || h->prestep()) {
        const size_t bytes = (size_t)p.flat_size * 2;
        // the per-bucket pipeline of the previous call may still use the buffers
        for (int64_t b = 0; b < B; ++b) CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_gf[b], 0));
        CUDA_TRY(h, cudaMemcpyAsync(h->grad, host_grads, bytes, cudaMemcpyHostToDevice, h->h2d_stream));
        CUDA_TRY(h, cudaEventRecord(h->ev_h2d, h->h2d_stream));
        CUDA_TRY(h, cudaStreamWaitEvent(h->work_stream, h->ev_h2d, 0));
        for (int64_t b = 0; b < B; ++b) CUDA_TRY(h, cudaStreamWaitEvent(h->work_stream, h->ev_db[b], 0));
        h->pre_b_event = h->ev_d2h;   // previous download (a never-recorded event is a no-op)
        st = lamb_step(h, nullptr, step, h->work_stream);
        h->pre_b_event = nullptr;
        if (st != LAMB_OK) return st;
        CUDA_TRY(h, cudaEventRecord(h->ev_params, h->work_stream));
        CUDA_TRY(h, cudaStreamWaitEvent(h->d2h_stream, h->ev_params, 0));
        CUDA_TRY(h, cudaMemcpyAsync(host_params, h->param, bytes, cudaMemcpyDeviceToHost, h->d2h_stream));
        CUDA_TRY(h, cudaEventRecord(h->ev_d2h, h->d2h_stream));
        CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_d2h, 0));
        return LAMB_OK;
    }
    // a whole-step call before may still download / own the param buffer
    CUDA_TRY(h, cudaStreamWaitEvent(h->work_stream, h->ev_d2h, 0));
    for (int64_t b = 0; b < B; ++b) {
        const int64_t base = p.buckets[4 * b], S = p.buckets[4 * b + 1];
        CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_gf[b], 0));
        CUDA_TRY(h, cudaMemcpyAsync(h->grad + base, host_grads + base, (size_t)S * 2, cudaMemcpyHostToDevice,
                                    h->h2d_stream));
        CUDA_TRY(h, cudaEventRecord(h->ev_hb[b], h->h2d_stream));
    }
    const int32_t t_max = h->t_max;
    h->t_max = 0;   // per-bucket calls are not phase-timed
    st = prologue(h, step, h->work_stream);
    for (int64_t b = 0; b < B && st == LAMB_OK; ++b) {
        const int64_t base = p.buckets[4 * b], S = p.buckets[4 * b + 1];
        cudaError_t ce = cudaStreamWaitEvent(h->work_stream, h->ev_hb[b], 0);
        if (ce != cudaSuccess) {
            st = fail(h, LAMB_ECUDA, std::string("cudaStreamWaitEvent: ") + cudaGetErrorString(ce));
            break;
        }
        h->pre_b_event = h->ev_db[b];   // previous download of this bucket
        h->gf_override = h->ev_gf[b];   // this bucket's grads consumed
        st = step_impl(h, nullptr, step, h->work_stream, b, b + 1, false);
        h->pre_b_event = nullptr;
        h->gf_override = nullptr;
        if (st != LAMB_OK) break;
        ce = cudaEventRecord(h->ev_pb[b], h->work_stream);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(h->d2h_stream, h->ev_pb[b], 0);
        if (ce == cudaSuccess)
            ce = cudaMemcpyAsync(host_params + base, h->param + base, (size_t)S * 2, cudaMemcpyDeviceToHost,
                                 h->d2h_stream);
        if (ce == cudaSuccess) ce = cudaEventRecord(h->ev_db[b], h->d2h_stream);
        if (ce != cudaSuccess) st = fail(h, LAMB_ECUDA, std::string("bucket pipeline: ") + cudaGetErrorString(ce));
    }
    h->t_max = t_max;
    if (st != LAMB_OK) return st;
    CUDA_TRY(h, cudaEventRecord(h->ev_d2h, h->d2h_stream));
    CUDA_TRY(h, cudaStreamWaitEvent(s, h->ev_d2h, 0));
    return LAMB_OK;
}

// ------------------------------------------------------------------ queries / state
extern "C" lamb_status lamb_query_plan(lamb_t h, lamb_plan_view* out) {
    if (!h || !out) return fail(h, LAMB_EINVAL, "null argument");
    fill_view(h->plan, out);
    return LAMB_OK;
}

extern "C" lamb_status lamb_buffer(lamb_t h, int32_t which, void** dev_ptr, int64_t* n) {
    if (!h || !dev_ptr || !n) return fail(h, LAMB_EINVAL, "null argument");
    switch (which) {
        case LAMB_BUF_GRAD: *dev_ptr = h->grad; *n = h->plan.flat_size; return LAMB_OK;
        case LAMB_BUF_PARAM: *dev_ptr = h->param; *n = h->plan.flat_size; return LAMB_OK;
        case LAMB_BUF_W: *dev_ptr = h->w; *n = h->plan.shard_size; return LAMB_OK;
        case LAMB_BUF_M: *dev_ptr = h->m; *n = h->plan.shard_size; return LAMB_OK;
        case LAMB_BUF_V: *dev_ptr = h->v; *n = h->plan.shard_size; return LAMB_OK;
        case LAMB_BUF_GSUM:
            if (!h->g32) return fail(h, LAMB_ESTATE, "no materialised reduced gradient on this path");
            *dev_ptr = h->g32;
            *n = h->plan.shard_size;
            return LAMB_OK;
    }
    return fail(h, LAMB_EINVAL, "unknown buffer");
}

extern "C" lamb_status lamb_set_master(lamb_t h, const float* full, int32_t on_device, void* stream) {
    if (!h || !full) return fail(h, LAMB_EINVAL, "null argument");
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Plan& p = h->plan;
    // Host source: staged bucket by bucket through ONE device buffer of the largest bucket
    // (4 * max S_b bytes; 160 MB at the default cap), so the call works at configs whose state
    // fills the GPU (a flat_size fp32 temporary would be 87 GB for the 175B slice).  Each
    // bucket: H2D into the buffer, own slice -> w (D2D), whole bucket -> bf16 params.
    float* tmp = nullptr;
    // freed on every return path; an error return synchronises first so that no queued copy
    // still uses it (the success path synchronises below)
    auto release = [s](float* q) {
        cudaStreamSynchronize(s);
        cudaFree(q);
    };
    std::unique_ptr<float, decltype(release)> guard(nullptr, release);
    if (!on_device) {
        CUDA_TRY(h, dalloc(&tmp, (size_t)h->max_bucket));
        guard.reset(tmp);
    }
    for (int64_t b = 0; b < p.n_buckets(); ++b) {
        const int64_t base = p.buckets[4 * b], S = p.buckets[4 * b + 1], sl = S / p.world;
        const float* src = full + base;
        if (!on_device) {
            CUDA_TRY(h, cudaMemcpyAsync(tmp, full + base, (size_t)S * 4, cudaMemcpyHostToDevice, s));
            src = tmp;
        }
        CUDA_TRY(h, cudaMemcpyAsync(h->w + p.shard_base[b], src + (int64_t)p.rank * sl, (size_t)sl * 4,
                                    cudaMemcpyDeviceToDevice, s));
        LAUNCH(h, launch_cast_to_bf16(src, h->param + base, S, s));
    }
    CUDA_TRY(h, cudaMemsetAsync(h->m, 0, (size_t)p.shard_size * 4, s));
    CUDA_TRY(h, cudaMemsetAsync(h->v, 0, (size_t)p.shard_size * 4, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    h->master_set = true;
    return LAMB_OK;
}

extern "C" lamb_status lamb_get_state(lamb_t h, int32_t which, float* dst, int32_t on_device, void* stream) {
    if (!h || !dst) return fail(h, LAMB_EINVAL, "null argument");
    const float* src = which == LAMB_BUF_W ? h->w : which == LAMB_BUF_M ? h->m : which == LAMB_BUF_V ? h->v : nullptr;
    if (!src) return fail(h, LAMB_EINVAL, "which must be LAMB_BUF_W/M/V");
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(h, cudaMemcpyAsync(dst, src, (size_t)h->plan.shard_size * 4,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    return LAMB_OK;
}

extern "C" lamb_status lamb_get_tensor_stats(lamb_t h, double* w_sq, double* u_sq, float* ratio) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    DeviceGuard device_guard_(h->device);
    CUDA_TRY(h, cudaDeviceSynchronize());
    const size_t T = (size_t)h->plan.n_tensors();
    if (w_sq) CUDA_TRY(h, cudaMemcpy(w_sq, h->w_sq, T * 8, cudaMemcpyDeviceToHost));
    if (u_sq) CUDA_TRY(h, cudaMemcpy(u_sq, h->u_sq, T * 8, cudaMemcpyDeviceToHost));
    if (ratio) CUDA_TRY(h, cudaMemcpy(ratio, h->ratio, T * 4, cudaMemcpyDeviceToHost));
    return LAMB_OK;
}

extern "C" lamb_status lamb_set_lr(lamb_t h, int32_t group, float lr) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (group < 0 || group >= (int32_t)h->groups.size()) return fail(h, LAMB_EINVAL, "group out of range");
    if (!(lr >= 0.f)) return fail(h, LAMB_EINVAL, "lr must be >= 0");
    h->groups[group].lr = lr;
    return LAMB_OK;
}

// ------------------------------------------------------------------ SM partition (NEXT #2)
// Green contexts (CUDA 12.4+ driver API), resolved through cudaGetDriverEntryPoint so the
// library carries no link-time dependency on libcuda (it still loads on a driverless host).
template <typename F>
static bool driver_fn(const char* name, F* out) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    *out = reinterpret_cast<F>(fn);
    return true;
}

extern "C" lamb_status lamb_sm_partition(int32_t device, int32_t lamb_sms, void** lamb_stream,
                                         void** compute_stream, int32_t* got_sms) {
    if (!lamb_stream || !compute_stream || lamb_sms < 1) return fail(nullptr, LAMB_EINVAL, "bad arguments");
    CUresult (*getDev)(CUdevice*, int) = nullptr;
    CUresult (*getRes)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*split)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                      unsigned int) = nullptr;
    CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
    CUresult (*gcCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
    CUresult (*gcStream)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
    DeviceGuard device_guard_(device);
    if (!device_guard_.ok || cudaFree(nullptr) != cudaSuccess)
        return fail(nullptr, LAMB_ECUDA, "cannot initialise the device");
    if (!driver_fn("cuDeviceGet", &getDev) || !driver_fn("cuDeviceGetDevResource", &getRes) ||
        !driver_fn("cuDevSmResourceSplitByCount", &split) || !driver_fn("cuDevResourceGenerateDesc", &genDesc) ||
        !driver_fn("cuGreenCtxCreate", &gcCreate) || !driver_fn("cuGreenCtxStreamCreate", &gcStream))
        return fail(nullptr, LAMB_EUNSUPPORTED, "green contexts are not available from this driver");
    CUdevice dev;
    CUdevResource all, part, rest;
    unsigned int ng = 1;
    if (getDev(&dev, device) != CUDA_SUCCESS || getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
        split(&part, &ng, &all, &rest, 0, (unsigned)lamb_sms) != CUDA_SUCCESS || ng != 1)
        return fail(nullptr, LAMB_EUNSUPPORTED, "cannot split the SMs");
    CUdevResourceDesc d1, d2;
    CUgreenCtx g1, g2;
    CUstream s1, s2;
    if (genDesc(&d1, &part, 1) != CUDA_SUCCESS || genDesc(&d2, &rest, 1) != CUDA_SUCCESS ||
        gcCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        gcCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        gcStream(&s1, g1, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
        gcStream(&s2, g2, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
        return fail(nullptr, LAMB_EUNSUPPORTED, "cannot create the green contexts");
    *lamb_stream = s1;
    *compute_stream = s2;
    if (got_sms) *got_sms = (int32_t)part.sm.smCount;
    return LAMB_OK;
}

// ------------------------------------------------------------------ self-check (§4.3)
// Padding ranges: shard positions not covered by a segment rounded up to 8 (w/m/v must stay 0)
// and flat positions not covered by any tensor (grad/param must stay 0).  Built on first use.
static lamb_status build_padding(lamb_ctx* h) {
    if (h->pad_built) return LAMB_OK;
    const Plan& p = h->plan;
    std::vector<int64_t> sh, fl;
    int64_t pos = 0;
    for (int64_t k = 0; k < p.n_segments(); ++k) {
        const int64_t soff = p.segments[4 * k + 1], len = p.segments[4 * k + 3];
        if (soff > pos) sh.insert(sh.end(), {pos, soff});
        pos = soff + len;   // [len, len8) is padding too: checked below as part of the gap
    }
    if (p.shard_size > pos) sh.insert(sh.end(), {pos, p.shard_size});
    pos = 0;
    for (int64_t i = 0; i < p.n_tensors(); ++i) {
        if (p.tensor_off[i] > pos) fl.insert(fl.end(), {pos, p.tensor_off[i]});
        pos = p.tensor_off[i] + p.numel[i];
    }
    if (p.flat_size > pos) fl.insert(fl.end(), {pos, p.flat_size});
    CUDA_TRY(h, upload(&h->d_shard_pad, sh));
    CUDA_TRY(h, upload(&h->d_flat_pad, fl));
    h->n_shard_pad = (int64_t)sh.size() / 2;
    h->n_flat_pad = (int64_t)fl.size() / 2;
    CUDA_TRY(h, dalloc(&h->d_check, 5));
    h->pad_built = true;
    return LAMB_OK;
}

extern "C" lamb_status lamb_self_check(lamb_t h, int64_t counts[5], void* stream) {
    if (!h || !counts) return fail(h, LAMB_EINVAL, "null argument");
    if (!h->master_set) return fail(h, LAMB_ESTATE, "nothing to check: master not set");
    DeviceGuard device_guard_(h->device);
    lamb_status st = build_padding(h);
    if (st != LAMB_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t* flags[LAMB_MAX_RANKS];
    for (int j = 0; j < h->cfg.world_size; ++j) flags[j] = h->flags(j);
    LAUNCH(h, lamb::launch_self_check(h->items, h->n_items, h->w, h->m, h->v, h->grad, h->param, h->d_shard_pad,
                                      h->n_shard_pad, h->d_flat_pad, h->n_flat_pad, flags, h->cfg.world_size,
                                      h->d_check, s));
    unsigned long long c[5];
    CUDA_TRY(h, cudaMemcpyAsync(c, h->d_check, sizeof(c), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    for (int k = 0; k < 5; ++k) counts[k] = (int64_t)c[k];
    return LAMB_OK;
}

#ifdef LAMB_DEBUG
extern "C" lamb_status lamb_debug_corrupt_item(lamb_t h, int64_t item, int64_t flat_off) {
    if (!h || item < 0 || item >= h->n_items) return fail(h, LAMB_EINVAL, "item out of range");
    DeviceGuard device_guard_(h->device);
    CUDA_TRY(h, cudaDeviceSynchronize());
    for (Item* tab : {h->items, h->items_b}) {
        if (!tab) continue;
        Item it;
        CUDA_TRY(h, cudaMemcpy(&it, tab + item, sizeof(Item), cudaMemcpyDeviceToHost));
        it.flat_off = flat_off;
        CUDA_TRY(h, cudaMemcpy(tab + item, &it, sizeof(Item), cudaMemcpyHostToDevice));
    }
    return LAMB_OK;
}
#endif

extern "C" lamb_status lamb_set_max_ctas(lamb_t h, int32_t max_ctas) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (max_ctas < 0) return fail(h, LAMB_EINVAL, "max_ctas must be >= 0");
    h->max_ctas = max_ctas;
    return LAMB_OK;
}

extern "C" lamb_status lamb_set_grad_clip(lamb_t h, float max_grad_norm) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (!(max_grad_norm >= 0.f)) return fail(h, LAMB_EINVAL, "max_grad_norm must be >= 0");
    h->max_grad_norm = max_grad_norm;
    return LAMB_OK;
}

extern "C" lamb_status lamb_set_loss_scale(lamb_t h, float inv_loss_scale) {
    if (!h) return fail(nullptr, LAMB_EINVAL, "null handle");
    if (!(inv_loss_scale > 0.f) || !std::isfinite(inv_loss_scale))
        return fail(h, LAMB_EINVAL, "inv_loss_scale must be finite and > 0");
    h->inv_loss_scale = inv_loss_scale;
    return LAMB_OK;
}

extern "C" lamb_status lamb_get_step_info(lamb_t h, lamb_step_info* out) {
    if (!h || !out) return fail(h, LAMB_EINVAL, "null argument");
    DeviceGuard device_guard_(h->device);
    CUDA_TRY(h, cudaDeviceSynchronize());
    lamb::ClipState cs;
    CUDA_TRY(h, cudaMemcpy(&cs, h->d_clip, sizeof(cs), cudaMemcpyDeviceToHost));
    if (!h->prestep()) {
        out->grad_norm = NAN;
        out->clip = 1.f;
        out->skipped = 0;
        return LAMB_OK;
    }
    out->grad_norm = cs.grad_norm;
    out->clip = cs.clip;
    out->skipped = cs.skip;
    return LAMB_OK;
}

extern "C" lamb_status lamb_timing_begin(lamb_t h, int32_t max_steps) {
    if (!h || max_steps < 0) return fail(h, LAMB_EINVAL, "bad argument");
    if (!(h->cfg.flags & LAMB_FLAG_TIMING)) return fail(h, LAMB_ESTATE, "handle created without LAMB_FLAG_TIMING");
    DeviceGuard device_guard_(h->device);
    CUDA_TRY(h, cudaDeviceSynchronize());
    for (cudaEvent_t e : h->tev) cudaEventDestroy(e);
    h->tev.assign((size_t)max_steps * (LAMB_N_PHASES + 1), nullptr);
    for (auto& e : h->tev) CUDA_TRY(h, cudaEventCreate(&e));
    h->t_max = max_steps;
    h->t_n = 0;
    return LAMB_OK;
}

extern "C" lamb_status lamb_timing_read(lamb_t h, float* ms, int32_t* n_steps) {
    if (!h || !n_steps) return fail(h, LAMB_EINVAL, "null argument");
    DeviceGuard device_guard_(h->device);
    *n_steps = h->t_n;
    for (int32_t k = 0; k < h->t_n; ++k) {
        CUDA_TRY(h, cudaEventSynchronize(h->tev[(size_t)k * (LAMB_N_PHASES + 1) + LAMB_N_PHASES]));
        for (int ph = 0; ph < LAMB_N_PHASES; ++ph) {
            float x = 0.f;
            CUDA_TRY(h, cudaEventElapsedTime(&x, h->tev[(size_t)k * (LAMB_N_PHASES + 1) + ph],
                                             h->tev[(size_t)k * (LAMB_N_PHASES + 1) + ph + 1]));
            if (ms) ms[(size_t)k * LAMB_N_PHASES + ph] = x;
        }
    }
    return LAMB_OK;
}

extern "C" int64_t lamb_launch_count(lamb_t h) { return h ? h->launches : -1; }

extern "C" const char* lamb_last_error(lamb_t h) {
    return h ? h->err.c_str() : g_last_error.c_str();
}

// ------------------------------------------------------------------ synth ABI
static lamb_status synth_tables(lamb_ctx* h, const lamb_synth_tensor* spec, SynthTables* t,
                                int32_t** d_init, int32_t** d_gexp) {
    const int64_t T = h->plan.n_tensors();
    std::vector<int32_t> init(T), gexp(T);
    for (int64_t i = 0; i < T; ++i) {
        if (spec[i].init < 0 || spec[i].init > 2) return fail(h, LAMB_EINVAL, "bad init kind");
        init[i] = spec[i].init;
        gexp[i] = spec[i].gexp;
    }
    CUDA_TRY(h, upload(d_init, init));
    CUDA_TRY(h, upload(d_gexp, gexp));
    t->tensor_off = h->d_tensor_off;
    t->numel = h->d_numel;
    t->init = *d_init;
    t->gexp = *d_gexp;
    t->n_tensors = T;
    t->shard_base = h->d_shard_base;
    t->bucket_base = h->d_bucket_base;
    t->bucket_slice = h->d_bucket_slice;
    t->n_buckets = h->plan.n_buckets();
    t->rank = h->plan.rank;
    return LAMB_OK;
}

extern "C" lamb_status lamb_synth_init(lamb_t h, const lamb_synth_tensor* spec, uint64_t seed, void* stream) {
    if (!h || !spec) return fail(h, LAMB_EINVAL, "null argument");
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    SynthTables t;
    int32_t *di = nullptr, *dg = nullptr;
    lamb_status st = synth_tables(h, spec, &t, &di, &dg);
    if (st == LAMB_OK) {
        cudaError_t e = synth_init(t, seed, h->param, h->plan.flat_size, h->w, h->plan.shard_size, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(h->m, 0, (size_t)h->plan.shard_size * 4, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(h->v, 0, (size_t)h->plan.shard_size * 4, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(h, LAMB_ECUDA, std::string("synth_init: ") + cudaGetErrorString(e));
    }
    if (di) cudaFree(di);
    if (dg) cudaFree(dg);
    if (st == LAMB_OK) h->master_set = true;
    return st;
}

extern "C" lamb_status lamb_synth_grads(lamb_t h, const lamb_synth_tensor* spec, uint64_t seed,
                                        uint32_t rank_term, uint32_t step, void* stream) {
    if (!h || !spec) return fail(h, LAMB_EINVAL, "null argument");
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    SynthTables t;
    int32_t *di = nullptr, *dg = nullptr;
    lamb_status st = synth_tables(h, spec, &t, &di, &dg);
    if (st == LAMB_OK) {
        cudaError_t e = synth_grads(t, seed, rank_term, step, reinterpret_cast<uint16_t*>(h->grad),
                                    h->plan.flat_size, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(h, LAMB_ECUDA, std::string("synth_grads: ") + cudaGetErrorString(e));
    }
    if (di) cudaFree(di);
    if (dg) cudaFree(dg);
    return st;
}

extern "C" lamb_status lamb_synth_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    if (!ctr || !key || !out) return fail(nullptr, LAMB_EINVAL, "null argument");
    uint32_t in[6] = {ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]};
    uint32_t* d = nullptr;
    CUDA_TRY(nullptr, cudaMalloc(&d, 10 * sizeof(uint32_t)));
    std::unique_ptr<uint32_t, cudaError_t (*)(void*)> guard(d, cudaFree);   // freed on every path
    CUDA_TRY(nullptr, cudaMemcpy(d, in, sizeof(in), cudaMemcpyHostToDevice));
    CUDA_TRY(nullptr, synth_philox(d, d + 6));
    CUDA_TRY(nullptr, cudaMemcpy(out, d + 6, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    return LAMB_OK;
}
