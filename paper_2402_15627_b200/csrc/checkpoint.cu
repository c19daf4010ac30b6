// checkpoint.cu — sharded LAMB state checkpoint / resume with reshard.
//
// PAPER.md §4.4: two-stage checkpointing — stage 1, every GPU worker copies its
// on-chip state into pinned host memory (blocking, "several seconds" thanks to PCIe);
// stage 2, a background process writes host memory to storage while training continues.
// Recovery: workers that share a state partition should not all read it; here no
// rank ever reads more than its own ZeRO-2 partition, and the replicated bf16 params are
// rebuilt by an all-gather instead of being read D times.
//
// File format v2 (little endian, one file per checkpoint, written by all ranks at disjoint
// offsets): header {magic "LAMBCKPT", u32 version = 2, u32 world size that saved,
// i64 n_tensors, i64 step, i64 n_params, i64 data_off, u64 session, u64 save_seq} +
// i64 numel[n_tensors] + u64 commit[8], zero-padded to data_off (multiple of 4096); then three
// fp32 arrays W, M, V of n_params elements each, in table order without padding (tensor i
// occupies [cum_i, cum_i + numel_i)).  The layout does not depend on D, the bucket cap or
// alignment, so a checkpoint saved at any world size loads at any other (reshard).
//
// Atomic commit: ranks write `path.tmp.<save_seq>`; after its data is durable each rank
// stores its commit word commit[r] = tag(session, save_seq, step, r) and re-reads all of them;
// the rank that sees all world_saved words valid renames the file to `path` (atomic; the
// previous checkpoint at `path` stays intact until then).  A crashed or failed rank therefore
// leaves `path` untouched, and load verifies every commit word, so a partial file is refused
// instead of loading zeros or stale data.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <string>

#include "ctx.hpp"

namespace {

constexpr char kMagic[8] = {'L', 'A', 'M', 'B', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 2;

struct Header {
    char magic[8];
    uint32_t version;
    uint32_t world_saved;
    int64_t n_tensors, step, n_params, data_off;
    uint64_t session, save_seq;
};

int64_t commit_offset(int64_t T) { return (int64_t)(sizeof(Header) + 8 * T); }
int64_t data_offset(int64_t T) { return (commit_offset(T) + 8 * LAMB_MAX_RANKS + 4095) / 4096 * 4096; }

// splitmix64 finaliser over the fields; never 0 (0 = not committed)
uint64_t commit_tag(uint64_t session, uint64_t seq, int64_t step, int rank) {
    uint64_t x = session ^ (seq * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)step << 8) ^ (uint64_t)(rank + 1);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x ? x : 1;
}

bool pwrite_all(int fd, const void* buf, size_t n, off_t off) {
    const char* p = static_cast<const char*>(buf);
    while (n > 0) {
        ssize_t k = pwrite(fd, p, n, off);
        if (k <= 0) return false;
        p += k;
        n -= (size_t)k;
        off += k;
    }
    return true;
}

bool pread_all(int fd, void* buf, size_t n, off_t off) {
    char* p = static_cast<char*>(buf);
    while (n > 0) {
        ssize_t k = pread(fd, p, n, off);
        if (k <= 0) return false;
        p += k;
        n -= (size_t)k;
        off += k;
    }
    return true;
}

// File I/O of one rank's segments: split into <= 64 MiB pieces, served by a pool of host
// threads (pread/pwrite at disjoint offsets are thread-safe).
struct IoTask {
    float* host;
    off_t off;
    size_t bytes;
};

std::vector<IoTask> segment_tasks(const Plan& p, float* stage, const std::vector<int64_t>& cum, int64_t doff) {
    const int64_t N = cum.back();
    const size_t sh = (size_t)p.shard_size;
    const size_t piece = 64u << 20;
    std::vector<IoTask> tasks;
    for (int64_t k = 0; k < p.n_segments(); ++k) {
        const int64_t t = p.segments[4 * k], soff = p.segments[4 * k + 1];
        const int64_t toff = p.segments[4 * k + 2], len = p.segments[4 * k + 3];
        for (int x = 0; x < 3; ++x) {
            float* h = stage + x * sh + soff;
            off_t off = doff + ((int64_t)x * N + cum[t] + toff) * 4;
            size_t left = (size_t)len * 4;
            while (left > 0) {
                const size_t n = left < piece ? left : piece;
                tasks.push_back({h, off, n});
                h += n / 4;
                off += (off_t)n;
                left -= n;
            }
        }
    }
    return tasks;
}

bool run_io(int fd, const std::vector<IoTask>& tasks, bool write) {
    const int nthreads = (int)std::min<size_t>(8, std::max<size_t>(1, tasks.size()));
    std::atomic<size_t> next{0};
    std::atomic<bool> ok{true};
    auto worker = [&]() {
        for (size_t i = next++; i < tasks.size() && ok; i = next++) {
            const IoTask& T = tasks[i];
            const bool r = write ? pwrite_all(fd, T.host, T.bytes, T.off) : pread_all(fd, T.host, T.bytes, T.off);
            if (!r) ok = false;
        }
    };
    std::vector<std::thread> pool;
    for (int i = 1; i < nthreads; ++i) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    return ok;
}

std::vector<int64_t> prefix(const Plan& p) {
    std::vector<int64_t> cum(p.n_tensors() + 1, 0);
    for (int64_t i = 0; i < p.n_tensors(); ++i) cum[i + 1] = cum[i] + p.numel[i];
    return cum;
}

lamb_status ensure_stage(lamb_ctx* h) {
    if (!h->ck_stage) {
        CUDA_TRY(h, cudaHostAlloc(reinterpret_cast<void**>(&h->ck_stage),
                                  3 * (size_t)h->plan.shard_size * sizeof(float), cudaHostAllocDefault));
    }
    return LAMB_OK;
}

}  // namespace

extern "C" lamb_status lamb_checkpoint_wait(lamb_t h) {
    if (!h) return lamb_fail(nullptr, LAMB_EINVAL, "null handle");
    if (h->ck_thread.joinable()) h->ck_thread.join();
    if (h->ck_status != LAMB_OK) {
        // reported once: a failed save must not block every later save or load
        const lamb_status st = h->ck_status;
        h->ck_status = LAMB_OK;
        return lamb_fail(h, st, h->ck_error);
    }
    return LAMB_OK;
}

extern "C" lamb_status lamb_checkpoint_save(lamb_t h, const char* path, int64_t step, void* stream) {
    if (!h || !path) return lamb_fail(h, LAMB_EINVAL, "null argument");
    if (!h->master_set) return lamb_fail(h, LAMB_ESTATE, "nothing to save: master not set");
    lamb_status st = lamb_checkpoint_wait(h);   // one save in flight at a time
    if (st != LAMB_OK) return st;
    st = ensure_stage(h);
    if (st != LAMB_OK) return st;
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = (size_t)h->plan.shard_size;
    // stage 1 (blocking): device shards -> pinned host
    CUDA_TRY(h, cudaMemcpyAsync(h->ck_stage, h->w, n * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->ck_stage + n, h->m, n * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->ck_stage + 2 * n, h->v, n * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    // stage 2 (background): this rank's segments -> path.tmp.<seq>, commit word, rename
    h->ck_status = LAMB_OK;
    h->ck_error.clear();
    const uint64_t seq = h->ck_seq++;
    const std::string file(path), tmp = file + ".tmp." + std::to_string(seq);
    const uint64_t session = h->session;
    h->ck_thread = std::thread([h, file, tmp, step, seq, session]() {
        const Plan& p = h->plan;
        const std::vector<int64_t> cum = prefix(p);
        const int64_t T = p.n_tensors(), N = cum[T], doff = data_offset(T);
        auto fail_io = [&](const char* what, const std::string& f) {
            h->ck_status = LAMB_EINVAL;
            h->ck_error = std::string("checkpoint save: ") + what + " " + f + ": " + strerror(errno);
        };
        int fd = open(tmp.c_str(), O_RDWR | O_CREAT, 0644);
        if (fd < 0) return fail_io("open", tmp);
        auto bail = [&](const char* what) {
            fail_io(what, tmp);   // before close(), which may overwrite errno
            close(fd);
        };
        if (p.rank == 0) {
            // the header without the commit words (each rank writes its own)
            std::vector<char> hdr((size_t)commit_offset(T), 0);
            Header H;
            memset(&H, 0, sizeof(H));
            memcpy(H.magic, kMagic, 8);
            H.version = kVersion;
            H.world_saved = (uint32_t)p.world;
            H.n_tensors = T;
            H.step = step;
            H.n_params = N;
            H.data_off = doff;
            H.session = session;
            H.save_seq = seq;
            memcpy(hdr.data(), &H, sizeof(H));
            memcpy(hdr.data() + sizeof(H), p.numel.data(), 8 * (size_t)T);
            // never truncate below data written by other ranks: size the file exactly
            if (ftruncate(fd, doff + 3 * N * 4) != 0 || !pwrite_all(fd, hdr.data(), hdr.size(), 0))
                return bail("header");
        }
        if (!run_io(fd, segment_tasks(p, h->ck_stage, cum, doff), true)) return bail("write");
        if (fdatasync(fd) != 0) return bail("fdatasync");
        // this rank's data (and rank 0's header) is durable: commit it
        const uint64_t mine = commit_tag(session, seq, step, p.rank);
        if (!pwrite_all(fd, &mine, 8, commit_offset(T) + 8 * p.rank) || fdatasync(fd) != 0) return bail("commit");
        uint64_t words[LAMB_MAX_RANKS] = {};
        if (!pread_all(fd, words, 8 * (size_t)p.world, commit_offset(T))) return bail("commit read");
        close(fd);
        for (int r = 0; r < p.world; ++r)
            if (words[r] != commit_tag(session, seq, step, r)) return;   // a later rank renames
        // every rank committed: publish atomically.  Two ranks may both see the last word; the
        // second rename finds the temporary gone, which is success.
        if (rename(tmp.c_str(), file.c_str()) != 0 && !(errno == ENOENT && access(file.c_str(), F_OK) == 0))
            fail_io("rename", tmp);
    });
    return LAMB_OK;
}

extern "C" lamb_status lamb_checkpoint_load(lamb_t h, const char* path, int64_t* step, void* stream) {
    if (!h || !path) return lamb_fail(h, LAMB_EINVAL, "null argument");
    if (h->ce_pushes_pending > 0)
        return lamb_fail(h, LAMB_ESTATE, "checkpoint load: gradients of an untaken step were pushed (copy-engine "
                                         "schedule); run lamb_step_staged first");
    lamb_status st = lamb_checkpoint_wait(h);
    if (st != LAMB_OK) return st;
    const Plan& p = h->plan;
    const std::vector<int64_t> cum = prefix(p);
    const int64_t T = p.n_tensors(), N = cum[T];
    int fd = open(path, O_RDONLY);
    if (fd < 0) return lamb_fail(h, LAMB_EINVAL, std::string("checkpoint load: open ") + path + ": " + strerror(errno));
    Header H;
    std::vector<int64_t> numel(T);
    bool ok = pread_all(fd, &H, sizeof(H), 0) && memcmp(H.magic, kMagic, 8) == 0 && H.version == kVersion &&
              H.n_tensors == T && H.n_params == N && H.data_off == data_offset(T) &&
              H.world_saved >= 1 && H.world_saved <= LAMB_MAX_RANKS &&
              pread_all(fd, numel.data(), 8 * (size_t)T, sizeof(H)) && numel == p.numel;
    if (!ok) {
        close(fd);
        return lamb_fail(h, LAMB_EINVAL, std::string("checkpoint load: ") + path +
                                             " is not a checkpoint of this parameter table");
    }
    {
        // every saving rank's commit word: a partially written checkpoint is refused
        uint64_t words[LAMB_MAX_RANKS] = {};
        if (!pread_all(fd, words, 8 * (size_t)H.world_saved, commit_offset(T))) words[0] = 0;
        for (uint32_t r = 0; r < H.world_saved; ++r)
            if (words[r] != commit_tag(H.session, H.save_seq, H.step, (int)r)) {
                close(fd);
                return lamb_fail(h, LAMB_EINVAL, std::string("checkpoint load: ") + path + " is incomplete (rank " +
                                                     std::to_string(r) + " of " + std::to_string(H.world_saved) +
                                                     " never committed its partition)");
            }
    }
    st = ensure_stage(h);
    if (st != LAMB_OK) {
        close(fd);
        return st;
    }
    const size_t sh = (size_t)p.shard_size;
    memset(h->ck_stage, 0, 3 * sh * sizeof(float));   // padding stays exactly zero
    ok = run_io(fd, segment_tasks(p, h->ck_stage, cum, H.data_off), false);
    close(fd);
    if (!ok) return lamb_fail(h, LAMB_EINVAL, std::string("checkpoint load: short read of ") + path);
    DeviceGuard device_guard_(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(h, cudaMemcpyAsync(h->w, h->ck_stage, sh * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->m, h->ck_stage + sh, sh * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->v, h->ck_stage + 2 * sh, sh * 4, cudaMemcpyHostToDevice, s));
    // params: cast own slices, then all-gather them (ranks never read other partitions)
    for (int64_t b = 0; b < p.n_buckets(); ++b) {
        const int64_t base = p.buckets[4 * b], sl = p.buckets[4 * b + 1] / p.world;
        CUDA_TRY(h, lamb::launch_cast_to_bf16(h->w + p.shard_base[b], h->param + base + (int64_t)p.rank * sl, sl, s));
        ++h->launches;
    }
    if (h->peer_mode()) {   // FUSED or NVLS: peers' param buffers are mapped
        // FUSED: every rank's own slices are cast -> barrier -> pull the peers' slices over
        // NVLink -> barrier (no rank rewrites its slices while a peer may still read them)
        uint64_t* flags[LAMB_MAX_RANKS];
        for (int j = 0; j < p.world; ++j) flags[j] = h->flags(j);
        CUDA_TRY(h, lamb::launch_barrier(flags, h->epoch(), p.rank, p.world, h->err_flag_dev, s, h->barrier_timeout_ns));
        for (int64_t b = 0; b < p.n_buckets(); ++b) {
            const int64_t base = p.buckets[4 * b], sl = p.buckets[4 * b + 1] / p.world;
            CUDA_TRY(h, lamb::launch_gather(const_cast<const __nv_bfloat16* const*>(h->peer_param), h->param, base,
                                            sl, p.world, p.rank, s));
            ++h->launches;
        }
        CUDA_TRY(h, lamb::launch_barrier(flags, h->epoch(), p.rank, p.world, h->err_flag_dev, s, h->barrier_timeout_ns));
        h->launches += 2;
    } else if (p.world > 1) {
        NCCL_TRY(h, ncclGroupStart());
        for (int64_t b = 0; b < p.n_buckets(); ++b) {
            const int64_t base = p.buckets[4 * b], sl = p.buckets[4 * b + 1] / p.world;
            NCCL_TRY(h, ncclAllGather(h->param + base + (int64_t)p.rank * sl, h->param + base, (size_t)sl,
                                      ncclBfloat16, h->comm, s));
        }
        NCCL_TRY(h, ncclGroupEnd());
    }
    CUDA_TRY(h, cudaStreamSynchronize(s));
    h->master_set = true;
    if (step) *step = H.step;
    return LAMB_OK;
}
