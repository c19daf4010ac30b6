/*
 * lamb.h — C ABI of the B200-native sharded LAMB step (ABI v1).
 *
 * What this library computes is the data-parallel hot path of MegaScale (arXiv 2402.15627):
 *   - the LAMB optimizer the paper adopts to grow the batch 4x (§3.1 P:288-293,
 *     citing You et al. 2020 `You2020Large`; update rule = that paper's Algorithm 2,
 *     readings Z1-Z9 in DESIGN.md §3),
 *   - on ZeRO-2 data parallelism: gradients reduce-scattered, optimizer state sharded,
 *     parameters all-gathered (§2, Fig. fig:dp-zero; §3.2).
 * One lamb_step = (a1) reduce-scatter of bf16 gradients with fp32 accumulation, (a2) Adam
 * moments + update vector on the local shard, (a3) segmented per-tensor ||w||^2, ||u||^2 and
 * their cross-shard combine, (a4) trust ratio, (a5) w <- w - lr*ratio*u and the bf16 cast,
 * (a6) all-gather of the bf16 parameters.
 *
 * Conventions (all functions):
 *   - Return LAMB_OK or an error code; lamb_last_error(h) (h may be NULL) holds a message.
 *   - Pointers are plain host or device pointers as stated per argument.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Collective calls (marked COLLECTIVE) must be made by all world_size ranks with
 *     identical tensor/group tables, config (except rank/device) and step.
 *   - One handle is not thread-safe; several handles per process are allowed, on the same or
 *     on different devices (tests/test_gpu_parity.py::test_two_devices_in_one_process).
 *   - There is no CPU fallback: a device that is not sm_100 gives LAMB_EUNSUPPORTED.
 */
#ifndef LAMB_H_
#define LAMB_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAMB_ABI_VERSION 1
#define LAMB_MAX_GROUPS 64      /* hyper-parameter groups per handle */
#define LAMB_MAX_RANKS 8        /* ranks of one NVSwitch node */
#define LAMB_UNIQUE_ID_BYTES 128

typedef struct lamb_ctx* lamb_t;          /* one per (rank, device, parameter set) */
typedef struct lamb_plan_ctx* lamb_plan_t;

typedef enum {
    LAMB_OK = 0,
    LAMB_EINVAL = 1,        /* bad argument (see each function) */
    LAMB_ENOMEM = 2,        /* device or host allocation failed */
    LAMB_ECUDA = 3,         /* CUDA runtime error (incl. asynchronous faults, barrier timeout) */
    LAMB_ENCCL = 4,         /* NCCL error */
    LAMB_ESTATE = 5,        /* call out of order (e.g. lamb_step before the master is set) */
    LAMB_EUNSUPPORTED = 6   /* not an sm_100 device, unsupported mode or feature */
} lamb_status;

/* Parameter-tensor table row ("layer" = one tensor, reading Z2).  numel >= 1. */
typedef struct {
    int64_t numel;
    int32_t group;          /* index into the group table */
    int32_t reserved;       /* must be 0 */
} lamb_tensor;

/* Hyper-parameter group.  The fp32 values ARE the contract (reading Z6).
 * beta1, beta2 in [0,1); eps >= 0; lr >= 0; weight_decay >= 0.
 * adapt = 1: LAMB trust ratio ||w||/||u|| (fallback 1 on a zero norm, Z9);
 * adapt = 0: ratio 1 (exactly AdamW, Z8).  bias_correction = 1: Adam bias correction (Z5). */
typedef struct {
    float lr, beta1, beta2, eps, weight_decay;
    int32_t adapt, bias_correction;
} lamb_group;

/* comm_mode */
#define LAMB_COMM_NCCL 0     /* baseline: NCCL reduce-scatter(fp32)/all-gather(fp64)/all-gather(bf16) */
#define LAMB_COMM_FUSED 1    /* default: reduce-scatter fused into pass A (NVLink peer loads,
                                fp32 sum), all-gather fused into pass B (NVLink peer stores) */
#define LAMB_COMM_NVLS 2     /* opt-in (§2): both
                                collectives THROUGH the NVSwitch.  Pass A reduce-scatters with
                                multimem.ld_reduce (the switch adds the D bf16 gradients in fp32
                                and returns the sum rounded ONCE to bf16: g = grad_scale *
                                bf16_rne(sum_j G_j), reading Z23 — a documented variant, not the
                                exact fp32 sum of the other modes), pass B all-gathers with one
                                multimem.st per chunk.  The flat grad / param buffers are VMM
                                allocations bound to two multicast objects (file descriptors
                                exchanged over Unix-domain sockets during lamb_create).  Needs D
                                distinct multicast-capable GPUs (EUNSUPPORTED otherwise, on every
                                rank); no pre-step (lamb_step: EUNSUPPORTED), no LAMB_FLAG_CE */
/* flags */
#define LAMB_FLAG_TIMING 1   /* record CUDA events around every phase (lamb_timing_*) */
#define LAMB_FLAG_GRAPH 2    /* lamb_step replays one captured CUDA graph of the whole step
                                (D = 1 and FUSED, library grad buffer; no per-phase timing) */
#define LAMB_FLAG_CE 4       /* FUSED, D > 1: also set up the copy-engine schedule
                                (lamb_push_grads_bucket / lamb_step_staged /
                                lamb_wait_params_bucket): a (D-1) x shard bf16 staging buffer */

typedef struct {
    int32_t world_size;        /* D >= 1, <= LAMB_MAX_RANKS; D = 1 needs no unique id */
    int32_t rank;              /* [0, D) */
    int32_t device;            /* CUDA device ordinal of this rank */
    int32_t comm_mode;         /* LAMB_COMM_*; ignored at D = 1 */
    int64_t bucket_cap_elems;  /* bucket cap (rule P3); 0 -> 40,000,000 */
    float grad_scale;          /* reduced gradient = grad_scale * sum_j G_j; 0 -> 1/D (Z10) */
    int32_t flags;             /* LAMB_FLAG_* */
} lamb_config;

/* Read-only views of the shard/bucket plan (row a0, rules P1-P7 in DESIGN.md §2).
 * All tables are int64, host memory owned by the handle, valid until destroy. */
typedef struct {
    int64_t n_tensors, n_buckets, n_segments, n_straddlers;
    int64_t flat_size;          /* elements of the flat bf16 grad / param buffers */
    int64_t shard_size;         /* elements of this rank's fp32 w/m/v shard = flat_size / D */
    int32_t world_size, rank;
    const int64_t* tensor_off;      /* [n_tensors] flat offset of each tensor (8-aligned, P2) */
    const int64_t* tensor_bucket;   /* [n_tensors] */
    const int64_t* buckets;         /* [n_buckets][4] = {base, S_b, t_begin, t_end} (P3-P5) */
    const int64_t* segments;        /* [n_segments][4] = {tensor, shard_off, tensor_off, len}
                                       of THIS rank, shard order (P6-P7) */
    const int64_t* straddlers;      /* [n_straddlers] tensors with >= 2 segments, ascending */
} lamb_plan_view;

/* ---------------- host-only planner (row a0; no device needed) ---------------- */
/* Builds the plan of `rank` for a world of `world_size`.  cap = 0 -> 40,000,000.
 * EINVAL: n_tensors < 1, numel < 1, world_size not in [1, LAMB_MAX_RANKS], rank out of range,
 * cap < 0. */
lamb_status lamb_plan_create(const lamb_tensor* tensors, int64_t n_tensors, int32_t world_size,
                             int32_t rank, int64_t cap, lamb_plan_t* out);
lamb_status lamb_plan_get(lamb_plan_t plan, lamb_plan_view* out);
void lamb_plan_destroy(lamb_plan_t plan);

/* ---------------- lifecycle ---------------- */
/* Rank 0 creates the NCCL unique id; the caller broadcasts the 128 bytes (torch.distributed). */
lamb_status lamb_get_unique_id(uint8_t id[LAMB_UNIQUE_ID_BYTES]);

/* COLLECTIVE.  Plans, allocates (library-owned: flat bf16 grad and param buffers, zeroed;
 * fp32 w/m/v shards), creates the NCCL communicator and, in LAMB_COMM_FUSED, maps every
 * peer's grad/param/exchange buffers over NVLink (CUDA IPC; peer access for ranks of the same
 * process); in LAMB_COMM_NVLS the grad/param buffers are multicast-bound VMM allocations
 * (csrc/nvls.cu).  `id` may be NULL when D = 1.
 * EINVAL: see lamb_plan_create, n_groups not in [1, LAMB_MAX_GROUPS], group out of range,
 * bad hyper-parameters, reserved != 0, or (D > 1) another rank passed a different table /
 * config (a hash is all-gathered and compared; every rank fails).  ENOMEM, ECUDA, ENCCL,
 * EUNSUPPORTED (device not sm_100, peers not NVLink-reachable in FUSED mode, an unknown
 * comm_mode, LAMB_FLAG_CE with NVLS, or in NVLS mode: no multicast support or ranks sharing a
 * GPU — then on every rank).
 * Failure detection: every cross-GPU wait is bounded by LAMB_BARRIER_TIMEOUT_MS (environment,
 * default 30000); a peer that does not arrive makes the next call return LAMB_ECUDA, after
 * which the handle must be destroyed. */
lamb_status lamb_create(const lamb_tensor* tensors, int64_t n_tensors, const lamb_group* groups,
                        int32_t n_groups, const lamb_config* cfg,
                        const uint8_t id[LAMB_UNIQUE_ID_BYTES], lamb_t* out);

/* Host all-gather supplied by the caller (e.g. over its torch.distributed process group):
 * every rank passes `bytes` bytes in `send`; on return `recv` holds rank j's bytes at offset
 * j * bytes for every j in [0, D).  Returns 0 on success.  Called only during
 * lamb_create_with_allgather, on the calling thread, the same number of times on every rank. */
typedef int (*lamb_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);

/* COLLECTIVE.  lamb_create for LAMB_COMM_FUSED (or NVLS) without an NCCL communicator: the table/config
 * hash and the CUDA-IPC handles of every rank's grad/param/sync buffers are exchanged through
 * `allgather` (§3.2 P:312-317 needs only the RS/AG data paths, which FUSED runs in the
 * pass kernels over peer memory; NCCL there serves only as bootstrap).  Ranks may share a
 * device: D processes on fewer GPUs time-slice it, which exercises the D-rank kernels and
 * protocol on any box (tests; not a performance configuration).  Ranks may also live in one
 * process (one thread per GPU calling this concurrently): peers in the same process are mapped
 * by peer access instead of CUDA IPC (tools/nvlink_bytes_1proc.py).  Everything else as
 * lamb_create.  EINVAL: allgather NULL, D > 1 with comm_mode not FUSED or NVLS, the callback
 * returned non-zero, or the lamb_create conditions. */
lamb_status lamb_create_with_allgather(const lamb_tensor* tensors, int64_t n_tensors,
                                       const lamb_group* groups, int32_t n_groups,
                                       const lamb_config* cfg, lamb_allgather_fn allgather, void* user,
                                       lamb_t* out);

/* COLLECTIVE, asynchronous, stream-ordered on `stream`.  Gradients are read from the
 * library grad buffer (lamb_buffer(LAMB_BUF_GRAD)) — every rank holds its full flat bf16
 * gradient there, padding elements zero — or, when `grads` != NULL (D = 1 or NCCL mode),
 * from a caller-owned device buffer with the same layout.  When `stream` reaches the end of
 * the step: every rank's param buffer holds bf16_rne(w) of the updated params, each shard
 * holds the updated fp32 w, m, v.  No host synchronisation.  step >= 1 is LAMB's t.
 * EINVAL: step < 1, grads != NULL in FUSED mode with D > 1.  ESTATE: master not set.
 * ECUDA/ENCCL: launch failures or an asynchronous fault/timeout of an earlier step. */
lamb_status lamb_step(lamb_t h, const void* grads, int64_t step, void* stream);

/* COLLECTIVE.  End-to-end variant with HOST buffers: copies `host_grads` (flat bf16,
 * flat_size elements, pinned for full speed) into the grad buffer, runs the step, and copies
 * the full updated bf16 param buffer back into `host_params` (flat_size elements).
 * The copies and the update run as a per-bucket pipeline on internal streams (§3.2
 * P:318-319, overlap per model chunk): bucket b's upload starts once the previous step's pass A
 * of b released it, b's update (pass A, norms, ratios, pass B — exact per bucket, every tensor
 * lives in one bucket) once its grads landed and the previous download of b finished, b's
 * download once its pass B finished; consecutive calls overlap the same way.  With the pre-step
 * enabled (lamb_set_grad_clip / lamb_set_loss_scale) the whole table is one unit.  The first
 * call is ordered after the work on `stream`; later calls are ordered among themselves (do not
 * interleave with lamb_step without synchronising).  `host_grads` must hold the gradients when
 * the call is made and stay unchanged until `stream` completes; `stream` completes once
 * host_params holds the params.  EINVAL: null buffers, step < 1.  ESTATE: master not set. */
lamb_status lamb_step_host(lamb_t h, const uint16_t* host_grads, uint16_t* host_params,
                           int64_t step, void* stream);

/* ---------------- per-bucket stepping: overlap with backward/forward --------
 * PAPER.md §3.2: the reduce-scatter of a model chunk starts right after its
 * backward, the all-gather right before its forward (prefetched for the first chunk).  Every
 * tensor lives in exactly one bucket, so the complete LAMB update of a bucket (RS, moments,
 * segmented norms incl. straddlers, trust ratio, apply, cast) can run as soon as that bucket's
 * gradients are final, overlapped with the backward of the remaining buckets. */
#define LAMB_BUCKET_DEFER_AG 1   /* pass B writes only this rank's slices; gather later */
/* COLLECTIVE (all ranks, same bucket order), asynchronous on `stream`: the LAMB step of
 * bucket `bucket` (0 <= bucket < n_buckets).  Without LAMB_BUCKET_DEFER_AG the bucket's params
 * are all-gathered at the end (as lamb_step); with it, call lamb_gather_bucket before the
 * bucket's next forward.  Calling it for every bucket once equals one lamb_step.
 * EINVAL: bucket out of range, step < 1, unknown flags.  ESTATE: master not set.
 * EUNSUPPORTED: the pre-step is enabled (its global norm needs the whole table). */
lamb_status lamb_step_bucket(lamb_t h, int64_t bucket, int64_t step, int32_t flags, void* stream);
/* SM budget: caps the persistent grid of the streaming passes at max_ctas CTAs (256 threads;
 * 0 = one full wave, the default) so that a concurrently running compute stream keeps the
 * remaining SMs.  Applies to subsequent lamb_step / lamb_step_bucket calls.  EINVAL: < 0. */
lamb_status lamb_set_max_ctas(lamb_t h, int32_t max_ctas);
/* Splits `device`'s SMs into two green contexts (CUDA 12.4+ driver API): lamb_sms SMs (rounded
 * up to the hardware's SM-group granularity; the count is returned in *got_sms) and the rest,
 * and returns one non-blocking stream in each.  Kernels launched into a stream run only on its
 * SMs — the hard partition that overlapping lamb_step_bucket with compute needs (a cuBLAS
 * SM-count target is only a heuristic).  Streams live until process exit.
 * EINVAL: bad arguments.  EUNSUPPORTED: driver without green contexts. */
lamb_status lamb_sm_partition(int32_t device, int32_t lamb_sms, void** lamb_stream, void** compute_stream,
                              int32_t* got_sms);
/* Deferred all-gather of one bucket's bf16 params (FUSED: NVLink pull of the D-1 peer slices;
 * NCCL: ncclAllGather, COLLECTIVE).  No-op at D = 1. */
lamb_status lamb_gather_bucket(lamb_t h, int64_t bucket, void* stream);

/* ---------------- copy-engine schedule (§3.2, on B200) ----------------
 * The paper overlaps the DP reduce-scatter with the backward and the all-gather with the next
 * forward.  Here the transfers ride the copy engines (DMA over NVLink, no SMs), so the compute
 * keeps every SM; the LAMB math then runs after the backward on local HBM only.  Needs
 * LAMB_FLAG_CE at create (FUSED, D > 1).  Results are bit-identical to lamb_step (same sums in
 * the same rank order).  EUNSUPPORTED: handle without LAMB_FLAG_CE, or the pre-step enabled.
 *
 * Arrival flags carry an internal per-handle round number, not `step`, so a rollback
 * (lamb_checkpoint_load) or a repeated step number can never let a stale flag release a wait.
 *
 * lamb_push_grads_bucket — COLLECTIVE per bucket, called as soon as the backward has written
 *   bucket b's gradients into the library grad buffer (ordered after the work on `stream`):
 *   copies this rank's gradients of every peer's slice of b into that peer's staging buffer
 *   (one cudaMemcpyAsync per peer on an internal copy stream) and raises the peer's arrival
 *   flag for this round.  Buckets may be pushed in any order (backward order is the natural);
 *   a bucket's gradients must be final (gradient accumulation: push after the last
 *   micro-batch only).
 * lamb_step_staged — COLLECTIVE, after every bucket was pushed: pass A (own slice + D-1 staged
 *   slices, local HBM) walks the buckets in reverse (the order the backward pushed them) and
 *   waits in-kernel, per bucket and bounded by LAMB_BARRIER_TIMEOUT_MS, until all peers' slices
 *   of step `step` landed — so the last bucket's transfer overlaps pass A of the others; then
 *   segmented norms with the straddler exchange, pass B into this rank's own param slices;
 *   then the copy stream pushes the own
 *   param slices of every bucket (bucket order) into every peer's param buffer — the
 *   all-gather, deferred into the next forward.
 * lamb_wait_params_bucket — before bucket b's forward: `stream` waits until every peer's
 *   param slice of b from lamb_step_staged(step) landed in this rank's param buffer.  `step`
 *   must be the step of the last lamb_step_staged (EINVAL otherwise; ESTATE before the first). */
lamb_status lamb_push_grads_bucket(lamb_t h, int64_t bucket, int64_t step, void* stream);
lamb_status lamb_step_staged(lamb_t h, int64_t step, void* stream);
lamb_status lamb_wait_params_bucket(lamb_t h, int64_t bucket, int64_t step, void* stream);


/* COLLECTIVE (barrier-free teardown of this rank's peer mappings and communicator). */
void lamb_destroy(lamb_t h);

/* ---------------- queries, state, hooks ---------------- */
lamb_status lamb_query_plan(lamb_t h, lamb_plan_view* out);

#define LAMB_BUF_GRAD 0    /* bf16 [flat_size], caller writes gradients here */
#define LAMB_BUF_PARAM 1   /* bf16 [flat_size], updated params after each step */
#define LAMB_BUF_W 2       /* fp32 [shard_size] master weights, shard-local order */
#define LAMB_BUF_M 3       /* fp32 [shard_size] first moment (stored uncorrected, Z5) */
#define LAMB_BUF_V 4       /* fp32 [shard_size] second moment */
#define LAMB_BUF_GSUM 5    /* fp32 [shard_size] reduced gradient sum_j G_j of the last step
                              (before grad_scale), shard order; exists only where the path
                              materialises it: NCCL mode, or FUSED with the pre-step enabled
                              (else LAMB_ESTATE) — for exactness checks (pin H10) */
/* Device pointer + element count of a library buffer; valid until lamb_destroy. */
lamb_status lamb_buffer(lamb_t h, int32_t which, void** dev_ptr, int64_t* n_elems);

/* Sets the fp32 master from a FULL flat fp32 array (flat_size elements, plan layout,
 * padding 0; host memory if on_device = 0): copies this rank's slices into w, zeroes m and
 * v, writes bf16_rne into the whole param buffer.  A host source is staged bucket by bucket
 * through one temporary device buffer of the largest bucket (4 * max S_b bytes), whatever
 * flat_size is.  Synchronous w.r.t. `stream`.  ENOMEM: that buffer. */
lamb_status lamb_set_master(lamb_t h, const float* full_flat, int32_t on_device, void* stream);

/* Copies this rank's shard of W/M/V (LAMB_BUF_W/M/V; shard_size floats, shard order) to
 * dst (host if on_device = 0).  Synchronises `stream`. */
lamb_status lamb_get_state(lamb_t h, int32_t which, float* dst, int32_t on_device, void* stream);

/* Per tensor, from the last completed step (synchronises the device): ||w||^2 and ||u||^2
 * (fp64, full tensor after the cross-shard combine) and the trust ratio.  Arrays have
 * n_tensors entries; only tensors with a segment on this rank are written (others NaN).
 * Any pointer may be NULL. */
lamb_status lamb_get_tensor_stats(lamb_t h, double* w_sq, double* u_sq, float* ratio);

/* Changes a group's learning rate for subsequent steps (schedules live outside, Z13). */
lamb_status lamb_set_lr(lamb_t h, int32_t group, float lr);

/* ---------------- pre-step: clipping, loss scale, non-finite skip ----
 * Enabled while max_grad_norm > 0 or inv_loss_scale != 1.  Each step then computes the GLOBAL
 * norm gn = ||grad_scale * inv_loss_scale * sum_j G_j|| over all tensors and ranks
 * (deterministic: fixed-order partials, rank-order combine), skips the whole step on the
 * device if gn is not finite (w, m, v, params, stats untouched), and otherwise multiplies the
 * reduced gradient by inv_loss_scale * min(1, max_grad_norm / (gn + 1e-6)) (the
 * torch.nn.utils.clip_grad_norm_ rule) before the LAMB update.  Costs one extra read of the
 * local bf16 grads at D = 1; at D > 1 (FUSED) the reduce-scatter moves into the extra pass,
 * which writes the fp32 reduced shard that pass A then reads (4 * shard_size bytes allocated on
 * first use).  Values are host settings used by subsequent steps. */
typedef struct {
    double grad_norm;   /* global norm of the unclipped, unscaled-by-clip gradient; NaN if disabled */
    float clip;         /* applied clip coefficient (1 = none) */
    int32_t skipped;    /* 1 if the step was skipped (non-finite gradient) */
} lamb_step_info;
/* EINVAL: max_grad_norm < 0 or NaN (0 disables clipping). */
lamb_status lamb_set_grad_clip(lamb_t h, float max_grad_norm);
/* EINVAL: inv_loss_scale not finite or <= 0 (1 disables unscaling). */
lamb_status lamb_set_loss_scale(lamb_t h, float inv_loss_scale);
/* Synchronises the device; reports the last step's pre-step outcome. */
lamb_status lamb_get_step_info(lamb_t h, lamb_step_info* out);

/* ---------------- checkpoint / resume with reshard (§4.4) ----------------
 * File format (little endian; one file per checkpoint, written by all ranks at disjoint
 * offsets): header {char magic[8] = "LAMBCKPT"; u32 version = 2; u32 world size that saved;
 * i64 n_tensors, step, n_params, data_off; u64 session, save_seq} + i64 numel[n_tensors] +
 * u64 commit[8] (one word per saving rank, written after its data is durable), zero-padded to
 * data_off (multiple of 4096); then fp32 arrays W, M, V of n_params elements each in table
 * order, no padding.  Independent of D, bucket cap and alignment: load at any world size. */
/* COLLECTIVE.  Stage 1 (blocking): copies this rank's w/m/v shard into pinned host staging
 * (allocated on first use: 12 * shard_size bytes) after the work already on `stream`.
 * Stage 2 (background host thread): writes this rank's segments into `path`.tmp.<n> (rank 0
 * writes the header and sizes the file), makes them durable, writes its commit word; the rank
 * that finds every rank's commit word in place renames the file to `path` (atomic: a crash or
 * an I/O error on any rank leaves the previous checkpoint at `path` intact).  Returns after
 * stage 1; training may continue.  A second save first waits for the previous one.
 * EINVAL: null path.  ESTATE: master not set.  ENOMEM: staging allocation. */
lamb_status lamb_checkpoint_save(lamb_t h, const char* path, int64_t step, void* stream);
/* Waits for this rank's background write of the last save; EINVAL with the I/O error if it
 * failed (reported once: the next save or load starts clean).  `path` is complete once every
 * rank's wait returned LAMB_OK (the last rank to commit renames it). */
lamb_status lamb_checkpoint_wait(lamb_t h);
/* COLLECTIVE.  Reads only this rank's segments of W, M, V from `path` (saved at any world
 * size), uploads them, rebuilds the bf16 param buffer (own slices cast, then all-gathered),
 * marks the master set and returns the saved step in *step (may be NULL).  Synchronous.
 * EINVAL: unreadable file, wrong magic/version, a different parameter table, or a commit word
 * missing (a partition never completed).  ESTATE: copy-engine gradient pushes of a step that
 * was not taken are pending. */
lamb_status lamb_checkpoint_load(lamb_t h, const char* path, int64_t* step, void* stream);

/* ---------------- self-check (§4.3 P:163-193 diagnostic tests) ----------------
 * Device-side audit of this rank's state, e.g. before resuming on a replacement machine.
 * counts[0]: shard entries with a non-finite w, m or v, or v < 0;
 * counts[1]: own-slice params that differ from bf16_rne(w);
 * counts[2]: nonzero w/m/v in the shard's padding;  counts[3]: nonzero grad/param padding
 *            (a caller wrote outside a tensor view);
 * counts[4]: peer mappings that read back as poisoned (FUSED).  All zero = healthy.
 * Synchronises `stream`.  ESTATE: master not set. */
lamb_status lamb_self_check(lamb_t h, int64_t counts[5], void* stream);

/* ---------------- measurement (CUDA events, §5.1 P:21-35 style) ---------------- */
#define LAMB_PH_BARRIER_IN 0   /* cross-GPU "grads ready" barrier (FUSED, D > 1) */
#define LAMB_PH_PASS_A 1       /* a1+a2: (fused RS) + moments + update + partial norms */
#define LAMB_PH_FINALIZE 2     /* a3+a4: segment sums, local trust ratios */
#define LAMB_PH_EXCHANGE 3     /* a3 cross-shard combine of straddlers + their ratios */
#define LAMB_PH_PASS_B 4       /* a5+a6: apply + bf16 cast (+ fused AG stores) */
#define LAMB_PH_BARRIER_OUT 5  /* cross-GPU "params complete" barrier */
#define LAMB_N_PHASES 6
/* Needs LAMB_FLAG_TIMING.  Starts recording the next `max_steps` steps. */
lamb_status lamb_timing_begin(lamb_t h, int32_t max_steps);
/* Synchronises and writes ms[n][LAMB_N_PHASES] for the n recorded steps; *n_steps = n. */
lamb_status lamb_timing_read(lamb_t h, float* ms, int32_t* n_steps);
/* Number of kernels this handle has launched (all steps so far). */
int64_t lamb_launch_count(lamb_t h);

const char* lamb_last_error(lamb_t h);

#ifdef __cplusplus
}
#endif
#endif /* LAMB_H_ */
