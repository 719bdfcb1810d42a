// Multi-GPU data path of the head-sharded decode step.
//
// KV heads split over ranks (GQA: a rank's query heads read only its own KV
// heads), so a layer step has exactly one exchange: every rank's attention
// outputs [batch][heads_local][G][d] are gathered into the full
// [batch][kv_heads][G][d] on every rank.  NCCL is loaded at run time
// (libnccl.so.2; the process's NCCL when one is already loaded) so the
// library has no link-time dependency on it:
//   tier 1: ncclAllGather into a staging buffer + one permute kernel;
//   tier 2: the same call on ncclMemAlloc buffers registered as symmetric
//           windows (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC, NCCL >=
//           2.27): NCCL's low-latency symmetric kernels over NVLink/NVSwitch.
// The decode step writes its outputs straight into the (registered) send
// buffer (saap_comm_send_buffer), so no copy precedes the collective.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "api.cuh"
#include "args.cuh"

namespace saap_b200 {

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    // optional (NCCL >= 2.27): symmetric windows
    ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*MemFree)(void*) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) {
        if (!n.h) fail(SAAP_ERR_UNSUPPORTED, "comm: libnccl.so.2 could not be loaded");
        return n;
    }
    tried = true;
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) fail(SAAP_ERR_UNSUPPORTED, std::string("comm: libnccl.so.2 could not be loaded: ") + dlerror());
    auto sym = [&](const char* name) { return dlsym(n.h, name); };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    n.GetVersion = (decltype(n.GetVersion))sym("ncclGetVersion");
    n.MemAlloc = (decltype(n.MemAlloc))sym("ncclMemAlloc");
    n.MemFree = (decltype(n.MemFree))sym("ncclMemFree");
    n.WindowRegister = (decltype(n.WindowRegister))sym("ncclCommWindowRegister");
    n.WindowDeregister = (decltype(n.WindowDeregister))sym("ncclCommWindowDeregister");
    if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllGather || !n.GetErrorString) {
        n.h = nullptr;
        fail(SAAP_ERR_UNSUPPORTED, "comm: libnccl.so.2 lacks the core API");
    }
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SAAP_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

// recv [nranks][batch][hl][G*d] -> out [batch][nranks][hl][G*d] (float4 moves)
__global__ void permute_heads_kernel(const float4* __restrict__ recv, float4* __restrict__ out,
                                     uint32_t nranks, uint32_t batch, uint32_t hl, uint32_t row4) {
    const size_t total = (size_t)nranks * batch * hl * row4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t e = i % row4, t = i / row4;
        const uint32_t h = (uint32_t)(t % hl), b = (uint32_t)((t / hl) % batch),
                       r = (uint32_t)(t / ((size_t)hl * batch));
        out[(((size_t)b * nranks + r) * hl + h) * row4 + e] = recv[i];
    }
}

}  // namespace
}  // namespace saap_b200

using namespace saap_b200;

struct saap_comm {
    saap_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0;
    bool symmetric = false;  // tier 2 buffers registered
    void* send = nullptr;
    void* recv = nullptr;
    size_t cap = 0;  // bytes per rank block (send), recv = nranks * cap
    ncclWindow_t wsend = nullptr, wrecv = nullptr;
};

// fused output exchange over peer memory (CUDA IPC mappings)
struct saap_p2p {
    saap_ctx* ctx = nullptr;
    int nranks = 0, rank = 0;
    uint64_t bytes = 0;          // full output bytes (the counter sits after them)
    char* base = nullptr;        // this rank's allocation: [full outputs | counter | expected]
    std::vector<char*> peer;     // mapped bases, rank order (own = base)
    float** d_out = nullptr;     // device [nranks] full-buffer pointers
    uint32_t** d_flag = nullptr; // device [nranks] counter pointers
    bool opened = false;
};

namespace saap_b200 {
namespace {
constexpr uint64_t kP2pTail = 256;  // counter + expected-arrivals word after the outputs
__global__ void p2p_wait_kernel(volatile uint32_t* flag, uint32_t* expect, uint32_t arrivals) {
    const uint32_t target = *expect + arrivals;
    uint32_t v;
    do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    } while ((int32_t)(v - target) < 0);
    *expect = target;
}
}  // namespace

void p2p_fill(saap_ctx* c, CombineArgs& ca) {
    saap_p2p* p = c->p2p;
    ca.p2p_out = p->d_out;
    ca.p2p_flag = p->d_flag;
    ca.p2p_n = (uint32_t)p->nranks;
    ca.p2p_hl = c->p2p_hl;
    ca.p2p_h0 = c->p2p_h0;
    ca.p2p_kvh = c->p2p_kvh;
}
}  // namespace saap_b200

namespace {

void release_buffers(saap_comm* m) {
    Nccl& n = nccl();
    if (m->wsend) n.WindowDeregister(m->comm, m->wsend);
    if (m->wrecv) n.WindowDeregister(m->comm, m->wrecv);
    m->wsend = m->wrecv = nullptr;
    if (m->symmetric) {
        if (m->send) n.MemFree(m->send);
        if (m->recv) n.MemFree(m->recv);
    } else {
        if (m->send) cudaFree(m->send);
        if (m->recv) cudaFree(m->recv);
    }
    m->send = m->recv = nullptr;
    m->cap = 0;
}

// (Collective: every rank grows with the same size.)  Symmetric windows when
// the NCCL in the process has them, plain device buffers otherwise.
void ensure_buffers(saap_comm* m, size_t bytes) {
    if (bytes <= m->cap) return;
    Nccl& n = nccl();
    SAAP_CUDA(cudaStreamSynchronize(m->ctx->stream));
    release_buffers(m);
    const size_t cap = (bytes + 4095) & ~size_t(4095);
    bool sym = n.MemAlloc && n.MemFree && n.WindowRegister && n.WindowDeregister && m->nranks > 1;
    if (sym) {
        sym = n.MemAlloc(&m->send, cap) == ncclSuccess &&
              n.MemAlloc(&m->recv, cap * m->nranks) == ncclSuccess &&
              n.WindowRegister(m->comm, m->send, cap, &m->wsend, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess &&
              n.WindowRegister(m->comm, m->recv, cap * m->nranks, &m->wrecv,
                               NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
        m->symmetric = true;  // (release path for MemAlloc'd buffers)
        if (!sym) release_buffers(m);
    }
    m->symmetric = sym;
    if (!sym) {
        SAAP_CUDA(cudaMalloc(&m->send, cap));
        SAAP_CUDA(cudaMalloc(&m->recv, cap * m->nranks));
    }
    m->cap = cap;
}

}  // namespace

extern "C" {

int saap_comm_unique_id(uint8_t* id) {
    return guard([&] {
        need(id, "comm: id");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int saap_comm_init(saap_ctx* c, int nranks, int rank, const uint8_t* id, saap_comm** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(id, "comm: id");
        need(out, "comm: out");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            invalid("comm: rank " + std::to_string(rank) + " of " + std::to_string(nranks));
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        auto* m = new saap_comm;
        m->ctx = c;
        m->nranks = nranks;
        m->rank = rank;
        const ncclResult_t r = nccl().CommInitRank(&m->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete m;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = m;
    });
}

int saap_comm_destroy(saap_comm* m) {
    return guard([&] {
        if (!m) return;
        DeviceGuard dg(m->ctx);
        cudaStreamSynchronize(m->ctx->stream);
        release_buffers(m);
        nccl().CommDestroy(m->comm);
        delete m;
    });
}

int saap_comm_info(const saap_comm* m, int* nranks, int* rank, int* symmetric, int* nccl_version) {
    return guard([&] {
        need(m, "comm");
        if (nranks) *nranks = m->nranks;
        if (rank) *rank = m->rank;
        if (symmetric) *symmetric = m->symmetric ? 1 : 0;
        if (nccl_version) {
            *nccl_version = 0;
            if (nccl().GetVersion) nccl().GetVersion(nccl_version);
        }
    });
}

int saap_comm_send_buffer(saap_comm* m, uint64_t bytes, void** out) {
    return guard([&] {
        need(m, "comm");
        need(out, "comm: out");
        DeviceGuard dg(m->ctx);
        ensure_buffers(m, bytes);
        *out = m->send;
    });
}

int saap_shard_heads(uint64_t kv_heads, int nranks, int rank, uint64_t* head0, uint64_t* heads_local) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            invalid("shard: rank " + std::to_string(rank) + " of " + std::to_string(nranks));
        if (kv_heads % (uint64_t)nranks)
            invalid("shard: " + std::to_string(kv_heads) + " KV heads do not split over " +
                    std::to_string(nranks) + " ranks");
        const uint64_t hl = kv_heads / (uint64_t)nranks;
        if (head0) *head0 = (uint64_t)rank * hl;
        if (heads_local) *heads_local = hl;
    });
}

int saap_allgather_heads(saap_ctx* c, saap_comm* m, const float* out_local, uint64_t batch,
                         uint64_t heads_local, uint64_t G, uint64_t d, float* out_full) {
    return guard([&] {
        DeviceGuard dg(c);
        need(m, "comm");
        need(out_local, "allgather: local outputs");
        need(out_full, "allgather: full outputs");
        if (m->ctx != c) invalid("allgather: the communicator belongs to another context");
        const uint64_t row = G * d;
        if (row % 4) unsupported("allgather: G*d must be a multiple of 4");
        const uint64_t elems = batch * heads_local * row;
        if (elems == 0) return;
        ensure_buffers(m, elems * 4);
        const cudaStream_t st = c->stream;
        if (out_local != m->send)
            SAAP_CUDA(cudaMemcpyAsync(m->send, out_local, elems * 4, cudaMemcpyDeviceToDevice, st));
        nccl_check(nccl().AllGather(m->send, m->recv, elems, ncclFloat32, m->comm, st), "ncclAllGather");
        const uint64_t total4 = (uint64_t)m->nranks * elems / 4;
        const uint32_t threads = 256;
        const uint32_t blocks = (uint32_t)std::min<uint64_t>((total4 + threads - 1) / threads, 4 * 148);
        permute_heads_kernel<<<blocks, threads, 0, st>>>((const float4*)m->recv, (float4*)out_full,
                                                        (uint32_t)m->nranks, (uint32_t)batch,
                                                        (uint32_t)heads_local, (uint32_t)(row / 4));
        SAAP_CUDA(cudaGetLastError());
        c->launches++;
    });
}

int saap_p2p_create(saap_ctx* c, int nranks, int rank, uint64_t full_bytes, saap_p2p** out) {
    return guard([&] {
        DeviceGuard dg(c);
        need(out, "p2p: out");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            invalid("p2p: rank " + std::to_string(rank) + " of " + std::to_string(nranks));
        if (full_bytes == 0 || full_bytes % 16) invalid("p2p: full buffer bytes must be a positive multiple of 16");
        auto* p = new saap_p2p;
        p->ctx = c;
        p->nranks = nranks;
        p->rank = rank;
        p->bytes = full_bytes;
        if (cudaMalloc(&p->base, full_bytes + kP2pTail) != cudaSuccess) {
            delete p;
            fail(SAAP_ERR_CUDA, "p2p: cudaMalloc");
        }
        SAAP_CUDA(cudaMemset(p->base, 0, full_bytes + kP2pTail));
        *out = p;
    });
}

int saap_p2p_handle(saap_p2p* p, uint8_t* handle64) {
    return guard([&] {
        need(p, "p2p");
        need(handle64, "p2p: handle");
        DeviceGuard dg(p->ctx);
        cudaIpcMemHandle_t h;
        SAAP_CUDA(cudaIpcGetMemHandle(&h, p->base));
        static_assert(sizeof(h) == 64, "IPC handle size");
        std::memcpy(handle64, &h, 64);
    });
}

int saap_p2p_open(saap_p2p* p, const uint8_t* all) {
    return guard([&] {
        need(p, "p2p");
        need(all, "p2p: handles");
        DeviceGuard dg(p->ctx);
        if (p->opened) invalid("p2p: already open");
        p->peer.assign(p->nranks, nullptr);
        for (int r = 0; r < p->nranks; ++r) {
            if (r == p->rank) {
                p->peer[r] = p->base;
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, all + 64 * (size_t)r, 64);
            void* q = nullptr;
            SAAP_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
            p->peer[r] = (char*)q;
        }
        std::vector<float*> outs(p->nranks);
        std::vector<uint32_t*> flags(p->nranks);
        for (int r = 0; r < p->nranks; ++r) {
            outs[r] = (float*)p->peer[r];
            flags[r] = (uint32_t*)(p->peer[r] + p->bytes);
        }
        SAAP_CUDA(cudaMalloc(&p->d_out, p->nranks * sizeof(float*)));
        SAAP_CUDA(cudaMalloc(&p->d_flag, p->nranks * sizeof(uint32_t*)));
        SAAP_CUDA(cudaMemcpy(p->d_out, outs.data(), p->nranks * sizeof(float*), cudaMemcpyHostToDevice));
        SAAP_CUDA(cudaMemcpy(p->d_flag, flags.data(), p->nranks * sizeof(uint32_t*), cudaMemcpyHostToDevice));
        p->opened = true;
    });
}

int saap_p2p_buffer(saap_p2p* p, void** full_out) {
    return guard([&] {
        need(p, "p2p");
        need(full_out, "p2p: out");
        *full_out = p->base;
    });
}

int saap_p2p_attach(saap_ctx* c, saap_p2p* p, uint64_t heads_local, uint64_t head0, uint64_t kv_heads) {
    return guard([&] {
        need(c, "context");
        if (c->capturing) invalid("saap_p2p_attach during graph capture");
        if (p && !p->opened) invalid("p2p: attach before open");
        if (p && (heads_local == 0 || head0 + heads_local > kv_heads))
            invalid("p2p: heads " + std::to_string(head0) + "+" + std::to_string(heads_local) + " of " +
                    std::to_string(kv_heads));
        c->p2p = p;
        c->p2p_hl = (uint32_t)heads_local;
        c->p2p_h0 = (uint32_t)head0;
        c->p2p_kvh = (uint32_t)kv_heads;
        // saved host-API step graphs hold the old combine arguments
        for (auto& g : c->host_graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        c->host_graphs.clear();
    });
}

int saap_p2p_wait(saap_ctx* c, saap_p2p* p, uint64_t arrivals) {
    return guard([&] {
        DeviceGuard dg(c);
        need(p, "p2p");
        if (!p->opened) invalid("p2p: wait before open");
        uint32_t* flag = (uint32_t*)(p->base + p->bytes);
        p2p_wait_kernel<<<1, 1, 0, c->stream>>>(flag, flag + 1, (uint32_t)arrivals);
        SAAP_CUDA(cudaGetLastError());
        c->launches++;
    });
}

int saap_p2p_read(saap_p2p* p, void* host, uint64_t bytes) {
    return guard([&] {
        need(p, "p2p");
        need(host, "p2p: host");
        DeviceGuard dg(p->ctx);
        if (bytes > p->bytes) invalid("p2p: read past the full buffer");
        SAAP_CUDA(cudaStreamSynchronize(p->ctx->stream));
        SAAP_CUDA(cudaMemcpy(host, p->base, bytes, cudaMemcpyDeviceToHost));
    });
}

int saap_p2p_destroy(saap_p2p* p) {
    return guard([&] {
        if (!p) return;
        DeviceGuard dg(p->ctx);
        cudaStreamSynchronize(p->ctx->stream);
        if (p->ctx->p2p == p) p->ctx->p2p = nullptr;
        for (int r = 0; r < (int)p->peer.size(); ++r)
            if (r != p->rank && p->peer[r]) cudaIpcCloseMemHandle(p->peer[r]);
        if (p->d_out) cudaFree(p->d_out);
        if (p->d_flag) cudaFree(p->d_flag);
        if (p->base) cudaFree(p->base);
        delete p;
    });
}

}  // extern "C"
