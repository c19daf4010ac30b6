// nvls.cu — buffers of the NVLS mode (LAMB_COMM_NVLS).
//
// PAPER.md §2 P:695-697 splits the DP all-reduce into a reduce-scatter and an all-gather; on one
// NVSwitch node both can run THROUGH the switch: a multimem.ld_reduce on a multicast address
// makes the switch read the same offset from every rank's buffer and add the values (pass A's
// reduce-scatter), and one multimem.st lands in every rank's buffer (pass B's all-gather).  That
// needs the flat grad and param buffers to be physical allocations bound to two multicast
// objects that span the D GPUs — VMM memory (cuMemCreate), not cudaMalloc:
//
//   1. each rank creates its grad and param allocations (POSIX-fd shareable) and maps them;
//   2. rank 0 creates the two multicast objects (numDevices = D);
//   3. the file descriptors travel over Unix-domain sockets (SCM_RIGHTS): every rank sends its
//      two allocation fds to every peer (the peers map them — the unicast peer views that the
//      deferred gather, the checkpoint reload and the self-check use), rank 0 also sends the
//      two multicast fds;
//   4. every rank adds its device to both multicast objects -> barrier -> binds its own
//      allocations -> barrier -> maps the multicast objects (the addresses pass A / pass B use).
//
// The barriers are the handle's bootstrap all-gather (NCCL or the caller's host all-gather);
// every phase ends with an all-gathered status byte, so a failure on one rank fails lamb_create on
// all of them instead of leaving peers waiting.  Driver API entry points are resolved through
// cudaGetDriverEntryPoint (no link-time libcuda dependency: the library still loads on a
// driverless host, tests/test_abi.py).
#include <cuda.h>
#include <cuda_runtime.h>

#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.hpp"

namespace {

struct Drv {
    CUresult (*deviceGet)(CUdevice*, int) = nullptr;
    CUresult (*deviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    CUresult (*addressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*allocGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char* name, F* out) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !fn)
        return false;
    *out = reinterpret_cast<F>(fn);
    return true;
}

const Drv& drv() {
    static const Drv d = [] {
        Drv x;
        x.ok = entry("cuDeviceGet", &x.deviceGet) && entry("cuDeviceGetAttribute", &x.deviceGetAttribute) &&
               entry("cuMemCreate", &x.memCreate) && entry("cuMemRelease", &x.memRelease) &&
               entry("cuMemExportToShareableHandle", &x.memExport) &&
               entry("cuMemImportFromShareableHandle", &x.memImport) &&
               entry("cuMemAddressReserve", &x.addressReserve) && entry("cuMemAddressFree", &x.addressFree) &&
               entry("cuMemMap", &x.memMap) && entry("cuMemUnmap", &x.memUnmap) &&
               entry("cuMemSetAccess", &x.memSetAccess) &&
               entry("cuMemGetAllocationGranularity", &x.allocGranularity) &&
               entry("cuMulticastCreate", &x.mcCreate) && entry("cuMulticastAddDevice", &x.mcAddDevice) &&
               entry("cuMulticastBindMem", &x.mcBindMem) && entry("cuMulticastUnbind", &x.mcUnbind) &&
               entry("cuMulticastGetGranularity", &x.mcGranularity);
        return x;
    }();
    return d;
}

std::string cu_err(const char* what, CUresult r) { return std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")"; }

// ---------------------------------------------------------------- fd passing (SCM_RIGHTS)
struct FdMsg {
    int32_t rank;
    int32_t nfd;
};

sockaddr_un sock_addr(uint64_t session, int rank, socklen_t* len) {
    sockaddr_un a;
    memset(&a, 0, sizeof(a));
    a.sun_family = AF_UNIX;
    // abstract namespace (leading NUL): no file, gone when the last descriptor closes
    const int n = snprintf(a.sun_path + 1, sizeof(a.sun_path) - 1, "lamb-nvls-%016llx-%d",
                           (unsigned long long)session, rank);
    *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
    return a;
}

bool send_fds(uint64_t session, int to, int me, const std::vector<int>& fds, std::string* why) {
    const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) return *why = "socket()", false;
    socklen_t len;
    sockaddr_un a = sock_addr(session, to, &len);
    bool ok = false;
    for (int attempt = 0; attempt < 3000 && !ok; ++attempt) {   // the peer listens before the barrier
        ok = connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0;
        if (!ok) usleep(1000);
    }
    if (!ok) {
        close(s);
        return *why = "connect() to rank " + std::to_string(to), false;
    }
    FdMsg m{me, (int32_t)fds.size()};
    iovec io{&m, sizeof(m)};
    std::vector<char> ctl(CMSG_SPACE(sizeof(int) * fds.size()));
    msghdr h;
    memset(&h, 0, sizeof(h));
    h.msg_iov = &io;
    h.msg_iovlen = 1;
    h.msg_control = ctl.data();
    h.msg_controllen = ctl.size();
    cmsghdr* c = CMSG_FIRSTHDR(&h);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int) * fds.size());
    memcpy(CMSG_DATA(c), fds.data(), sizeof(int) * fds.size());
    ok = sendmsg(s, &h, 0) == (ssize_t)sizeof(m);
    close(s);
    if (!ok) *why = "sendmsg() to rank " + std::to_string(to);
    return ok;
}

bool recv_fds(int listener, int timeout_ms, int* from, std::vector<int>* fds, std::string* why) {
    pollfd p{listener, POLLIN, 0};
    if (poll(&p, 1, timeout_ms) != 1) return *why = "timed out waiting for a peer's descriptors", false;
    const int c = accept4(listener, nullptr, nullptr, SOCK_CLOEXEC);
    if (c < 0) return *why = "accept()", false;
    ucred cred;
    socklen_t clen = sizeof(cred);
    if (getsockopt(c, SOL_SOCKET, SO_PEERCRED, &cred, &clen) != 0 || cred.uid != getuid()) {
        close(c);   // only processes of this user may hand us memory
        return *why = "descriptor message from another user", false;
    }
    FdMsg m{-1, 0};
    iovec io{&m, sizeof(m)};
    std::vector<char> ctl(CMSG_SPACE(sizeof(int) * 8));
    msghdr h;
    memset(&h, 0, sizeof(h));
    h.msg_iov = &io;
    h.msg_iovlen = 1;
    h.msg_control = ctl.data();
    h.msg_controllen = ctl.size();
    const ssize_t n = recvmsg(c, &h, MSG_CMSG_CLOEXEC);
    close(c);
    cmsghdr* cm = CMSG_FIRSTHDR(&h);
    if (n != (ssize_t)sizeof(m) || !cm || cm->cmsg_type != SCM_RIGHTS || m.nfd < 1 || m.nfd > 8)
        return *why = "malformed descriptor message", false;
    fds->resize(m.nfd);
    memcpy(fds->data(), CMSG_DATA(cm), sizeof(int) * m.nfd);
    *from = m.rank;
    return true;
}

}  // namespace

struct NvlsState {
    CUdevice dev = 0;
    size_t bytes = 0;                                  // per buffer (rounded to the granularity)
    CUmemGenericAllocationHandle mem[2] = {0, 0};      // own grad, param
    CUdeviceptr va[2] = {0, 0};
    CUmemGenericAllocationHandle peer_mem[LAMB_MAX_RANKS][2] = {};
    CUdeviceptr peer_va[LAMB_MAX_RANKS][2] = {};
    CUmemGenericAllocationHandle mc[2] = {0, 0};       // multicast objects
    bool bound[2] = {false, false};
    CUdeviceptr mc_va[2] = {0, 0};
};

// all-gathered status byte: LAMB_OK only if every rank's `st` is LAMB_OK
static lamb_status agree(lamb_ctx* h, lamb_status st) {
    const uint8_t mine = st == LAMB_OK ? 1 : 0;
    std::vector<uint8_t> all(h->cfg.world_size);
    lamb_status s2 = lamb_bootstrap_allgather(h, &mine, all.data(), 1);
    if (s2 != LAMB_OK) return s2;
    if (st != LAMB_OK) return st;
    for (int j = 0; j < h->cfg.world_size; ++j)
        if (!all[j]) return lamb_fail(h, LAMB_EUNSUPPORTED, "NVLS setup failed on rank " + std::to_string(j));
    return LAMB_OK;
}

static lamb_status map_local(lamb_ctx* h, NvlsState* S, CUmemGenericAllocationHandle mem, CUdeviceptr* va) {
    const Drv& d = drv();
    CUresult r = d.addressReserve(va, S->bytes, S->bytes >= (1ull << 21) ? (1ull << 21) : 0, 0, 0);
    if (r != CUDA_SUCCESS) return lamb_fail(h, LAMB_ENOMEM, cu_err("cuMemAddressReserve", r));
    r = d.memMap(*va, S->bytes, 0, mem, 0);
    if (r != CUDA_SUCCESS) return lamb_fail(h, LAMB_ECUDA, cu_err("cuMemMap", r));
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = h->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = d.memSetAccess(*va, S->bytes, &acc, 1);
    if (r != CUDA_SUCCESS) return lamb_fail(h, LAMB_ECUDA, cu_err("cuMemSetAccess", r));
    return LAMB_OK;
}

lamb_status lamb_nvls_setup(lamb_ctx* h) {
    const int D = h->cfg.world_size, r = h->cfg.rank;
    auto* S = new NvlsState();
    h->nvls = S;
    const Drv& d = drv();
    lamb_status st = LAMB_OK;

    // ---- phase 0: capability and distinct devices (NVLS needs one GPU per rank)
    if (!d.ok) st = lamb_fail(h, LAMB_EUNSUPPORTED, "NVLS: driver without the VMM / multicast entry points");
    int mc_ok = 0;
    if (st == LAMB_OK && (d.deviceGet(&S->dev, h->device) != CUDA_SUCCESS ||
                          d.deviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, S->dev) != CUDA_SUCCESS ||
                          !mc_ok))
        st = lamb_fail(h, LAMB_EUNSUPPORTED, "NVLS: device does not support multicast objects");
    cudaDeviceProp prop;
    char uuid[16] = {0};
    if (st == LAMB_OK && cudaGetDeviceProperties(&prop, h->device) == cudaSuccess) memcpy(uuid, prop.uuid.bytes, 16);
    {
        std::vector<char> all((size_t)D * 16);
        lamb_status s2 = lamb_bootstrap_allgather(h, uuid, all.data(), 16);
        if (s2 != LAMB_OK) return s2;
        for (int j = 0; j < D && st == LAMB_OK; ++j)
            for (int k = 0; k < j; ++k)
                if (!memcmp(&all[16 * j], &all[16 * k], 16))
                    st = lamb_fail(h, LAMB_EUNSUPPORTED, "NVLS: ranks " + std::to_string(k) + " and " + std::to_string(j) +
                                                             " share a GPU (multicast needs one GPU per rank)");
    }
    if ((st = agree(h, st)) != LAMB_OK) return st;

    // ---- phase 1: own allocations, multicast objects (rank 0), the listening socket
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)D;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = (size_t)h->plan.flat_size * 2;
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = h->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g_mc = 0, g_mem = 0;
    CUresult cr = d.mcGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (cr == CUDA_SUCCESS) cr = d.allocGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (cr != CUDA_SUCCESS) st = lamb_fail(h, LAMB_EUNSUPPORTED, cu_err("NVLS granularity query", cr));
    const size_t gran = std::max<size_t>(std::max(g_mc, g_mem), 1);
    S->bytes = (mp.size + gran - 1) / gran * gran;
    mp.size = S->bytes;
    for (int b = 0; b < 2 && st == LAMB_OK; ++b) {
        cr = d.memCreate(&S->mem[b], S->bytes, &ap, 0);
        if (cr != CUDA_SUCCESS) st = lamb_fail(h, LAMB_ENOMEM, cu_err("cuMemCreate", cr));
        else st = map_local(h, S, S->mem[b], &S->va[b]);
    }
    if (st == LAMB_OK && r == 0)
        for (int b = 0; b < 2 && st == LAMB_OK; ++b)
            if ((cr = d.mcCreate(&S->mc[b], &mp)) != CUDA_SUCCESS) st = lamb_fail(h, LAMB_EUNSUPPORTED, cu_err("cuMulticastCreate", cr));
    std::vector<int> my_fds;
    for (int b = 0; b < 2 && st == LAMB_OK; ++b) {
        int fd = -1;
        if ((cr = d.memExport(&fd, S->mem[b], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS)
            st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMemExportToShareableHandle", cr));
        else my_fds.push_back(fd);
    }
    for (int b = 0; b < 2 && st == LAMB_OK && r == 0; ++b) {
        int fd = -1;
        if ((cr = d.memExport(&fd, S->mc[b], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS)
            st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMemExportToShareableHandle(multicast)", cr));
        else my_fds.push_back(fd);
    }
    int listener = -1;
    if (st == LAMB_OK) {
        listener = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
        socklen_t len;
        sockaddr_un a = sock_addr(h->session, r, &len);
        if (listener < 0 || bind(listener, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(listener, LAMB_MAX_RANKS) != 0)
            st = lamb_fail(h, LAMB_ECUDA, "NVLS: cannot open the descriptor socket");
    }
    auto close_all = [&]() {
        for (int fd : my_fds) close(fd);
        my_fds.clear();
        if (listener >= 0) close(listener);
        listener = -1;
    };
    if ((st = agree(h, st)) != LAMB_OK) {
        close_all();
        return st;
    }

    // ---- phase 2: descriptors to every peer (connections queue in the backlog: no ordering)
    std::string why;
    for (int j = 0; j < D && st == LAMB_OK; ++j)
        if (j != r && !send_fds(h->session, j, r, my_fds, &why)) st = lamb_fail(h, LAMB_ECUDA, "NVLS: " + why);
    std::vector<std::vector<int>> got(D);
    for (int k = 0; k < D - 1 && st == LAMB_OK; ++k) {
        int from = -1;
        std::vector<int> fds;
        const int timeout_ms = (int)std::min<uint64_t>(h->barrier_timeout_ns / 1000000ull, 600000ull);
        if (!recv_fds(listener, timeout_ms, &from, &fds, &why)) st = lamb_fail(h, LAMB_ECUDA, "NVLS: " + why);
        else if (from < 0 || from >= D || from == r || !got[from].empty() || (int)fds.size() != (from == 0 ? 4 : 2)) {
            for (int fd : fds) close(fd);
            st = lamb_fail(h, LAMB_ECUDA, "NVLS: unexpected descriptor message");
        } else {
            got[from] = fds;
        }
    }
    close_all();
    // ---- phase 3: map the peers' allocations (unicast views), import the multicast objects
    for (int j = 0; j < D && st == LAMB_OK; ++j) {
        if (j == r) continue;
        for (int b = 0; b < 2 && st == LAMB_OK; ++b) {
            cr = d.memImport(&S->peer_mem[j][b], (void*)(intptr_t)got[j][b], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
            if (cr != CUDA_SUCCESS) st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMemImportFromShareableHandle", cr));
            else st = map_local(h, S, S->peer_mem[j][b], &S->peer_va[j][b]);
        }
        if (st == LAMB_OK && j == 0 && r != 0)
            for (int b = 0; b < 2 && st == LAMB_OK; ++b)
                if ((cr = d.memImport(&S->mc[b], (void*)(intptr_t)got[0][2 + b], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)) !=
                    CUDA_SUCCESS)
                    st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMemImportFromShareableHandle(multicast)", cr));
    }
    for (auto& v : got)
        for (int fd : v) close(fd);
    for (int b = 0; b < 2 && st == LAMB_OK; ++b)
        if ((cr = d.mcAddDevice(S->mc[b], S->dev)) != CUDA_SUCCESS) st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMulticastAddDevice", cr));
    if ((st = agree(h, st)) != LAMB_OK) return st;

    // ---- phase 4: every device added -> bind own memory; then map the multicast objects
    for (int b = 0; b < 2 && st == LAMB_OK; ++b) {
        if ((cr = d.mcBindMem(S->mc[b], 0, S->mem[b], 0, S->bytes, 0)) != CUDA_SUCCESS)
            st = lamb_fail(h, LAMB_ECUDA, cu_err("cuMulticastBindMem", cr));
        else S->bound[b] = true;
    }
    if ((st = agree(h, st)) != LAMB_OK) return st;
    for (int b = 0; b < 2 && st == LAMB_OK; ++b) st = map_local(h, S, S->mc[b], &S->mc_va[b]);
    if (st == LAMB_OK) {
        h->grad = reinterpret_cast<__nv_bfloat16*>(S->va[0]);
        h->param = reinterpret_cast<__nv_bfloat16*>(S->va[1]);
        h->mc_grad = reinterpret_cast<__nv_bfloat16*>(S->mc_va[0]);
        h->mc_param = reinterpret_cast<__nv_bfloat16*>(S->mc_va[1]);
        for (int j = 0; j < D; ++j) {
            h->peer_grad[j] = j == r ? h->grad : reinterpret_cast<__nv_bfloat16*>(S->peer_va[j][0]);
            h->peer_param[j] = j == r ? h->param : reinterpret_cast<__nv_bfloat16*>(S->peer_va[j][1]);
        }
        if (cudaMemset(h->grad, 0, S->bytes) != cudaSuccess || cudaMemset(h->param, 0, S->bytes) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess)
            st = lamb_fail(h, LAMB_ECUDA, "NVLS: zeroing the buffers failed");
    }
    return agree(h, st);
}

void lamb_nvls_free(lamb_ctx* h) {
    NvlsState* S = h->nvls;
    if (!S) return;
    const Drv& d = drv();
    if (d.ok) {
        for (int b = 0; b < 2; ++b) {
            if (S->mc_va[b]) {
                d.memUnmap(S->mc_va[b], S->bytes);
                d.addressFree(S->mc_va[b], S->bytes);
            }
            if (S->bound[b]) d.mcUnbind(S->mc[b], S->dev, 0, S->bytes);
            if (S->mc[b]) d.memRelease(S->mc[b]);
            for (int j = 0; j < LAMB_MAX_RANKS; ++j) {
                if (S->peer_va[j][b]) {
                    d.memUnmap(S->peer_va[j][b], S->bytes);
                    d.addressFree(S->peer_va[j][b], S->bytes);
                }
                if (S->peer_mem[j][b]) d.memRelease(S->peer_mem[j][b]);
            }
            if (S->va[b]) {
                d.memUnmap(S->va[b], S->bytes);
                d.addressFree(S->va[b], S->bytes);
            }
            if (S->mem[b]) d.memRelease(S->mem[b]);
        }
    }
    delete S;
    h->nvls = nullptr;
    h->grad = h->param = nullptr;
    h->mc_grad = h->mc_param = nullptr;
    for (int j = 0; j < LAMB_MAX_RANKS; ++j) h->peer_grad[j] = h->peer_param[j] = nullptr;
}
