// comm.cu -- rank-to-rank exchange of the distributed matvec.
//
// Two transports behind one interface:
//   * NCCL (one process per GPU): grouped ncclSend / ncclRecv for the two all-to-all
//     transposes of each matvec and ncclAllReduce for the Krylov dot products, all on the
//     context stream.  libnccl is loaded with dlopen at vc_init_distributed time, so the library
//     itself has no link-time NCCL dependency.
//   * in-process thread group (any number of contexts in one process, possibly on one GPU,
//     each driven by its own host thread): host barriers plus stream-ordered peer copies and
//     events.  No kernel ever waits on another rank, so ranks may share a GPU; this is how the
//     partitioned path is tested on a single B200.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.h"

namespace vc {

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& err) {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return false;
        }
#define VC_SYM(f, n) f = reinterpret_cast<decltype(f)>(dlsym(h, n))
        VC_SYM(GetUniqueId, "ncclGetUniqueId");
        VC_SYM(CommInitRank, "ncclCommInitRank");
        VC_SYM(CommDestroy, "ncclCommDestroy");
        VC_SYM(GroupStart, "ncclGroupStart");
        VC_SYM(GroupEnd, "ncclGroupEnd");
        VC_SYM(Send, "ncclSend");
        VC_SYM(Recv, "ncclRecv");
        VC_SYM(AllReduce, "ncclAllReduce");
        VC_SYM(GetErrorString, "ncclGetErrorString");
#undef VC_SYM
        if (!GetUniqueId || !CommInitRank || !CommDestroy || !GroupStart || !GroupEnd || !Send ||
            !Recv || !AllReduce) {
            err = "libnccl is missing required symbols";
            h = nullptr;
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
}  // namespace

// In-process group: shared state of `world` contexts driven by `world` host threads.
struct Group {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<cudaEvent_t> ev_ready, ev_done;
    std::vector<std::vector<const void*>> send_ptr;  // [rank][peer]
    std::vector<double> red;                          // allreduce scratch [rank][n]
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct Comm {
    int kind = 0;  // 0 NCCL, 1 thread group
    int rank = 0, world = 1;
    ncclComm_t nccl = nullptr;
    Group* grp = nullptr;
};

vc_status comm_nccl_unique_id(void* out, std::string& err) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.load(err)) return VC_ERR_NCCL;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) {
        err = std::string("ncclGetUniqueId: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
        return VC_ERR_NCCL;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, sizeof(id));
    return VC_OK;
}

void* group_create(int world) {
    if (world < 1) return nullptr;
    Group* g = new Group();
    g->world = world;
    g->ev_ready.resize(world);
    g->ev_done.resize(world);
    for (int r = 0; r < world; ++r) {
        cudaEventCreateWithFlags(&g->ev_ready[r], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&g->ev_done[r], cudaEventDisableTiming);
    }
    g->send_ptr.assign(world, std::vector<const void*>(world, nullptr));
    return g;
}

void group_destroy(void* h) {
    Group* g = static_cast<Group*>(h);
    if (!g) return;
    for (auto e : g->ev_ready) cudaEventDestroy(e);
    for (auto e : g->ev_done) cudaEventDestroy(e);
    delete g;
}

vc_status comm_init(vc_ctx* c, int rank, int world, int transport, const void* id) {
    Comm* m = new Comm();
    m->kind = transport;
    m->rank = rank;
    m->world = world;
    if (transport == 0) {
        std::string err;
        {
            std::lock_guard<std::mutex> lk(g_nccl_mu);
            if (!g_nccl.load(err)) {
                delete m;
                return set_err(c, VC_ERR_NCCL, err);
            }
        }
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof(uid));
        ncclResult_t r = g_nccl.CommInitRank(&m->nccl, world, uid, rank);
        if (r != ncclSuccess) {
            delete m;
            return set_err(c, VC_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r));
        }
    } else {
        m->grp = static_cast<Group*>(const_cast<void*>(id));
        if (!m->grp || m->grp->world != world) {
            delete m;
            return set_err(c, VC_ERR_INPUT, "thread group handle does not match world");
        }
    }
    c->comm = m;
    c->rank = rank;
    c->world = world;
    return VC_OK;
}

void comm_free(vc_ctx* c) {
    Comm* m = c->comm;
    if (!m) return;
    if (m->kind == 0 && m->nccl) g_nccl.CommDestroy(m->nccl);
    delete m;
    c->comm = nullptr;
}

// send[q] (bytes sb[q]) to rank q, receive rb[p] bytes from rank p into recv[p]; self entries
// are skipped (the producing kernel wrote the self block in place).  Stream-ordered.
vc_status comm_alltoall(vc_ctx* c, const std::vector<const void*>& send,
                        const std::vector<size_t>& sb, const std::vector<void*>& recv,
                        const std::vector<size_t>& rb, cudaStream_t st_in) {
    Comm* m = c->comm;
    const int W = m->world, r = m->rank;
    cudaStream_t st = st_in ? st_in : c->stream;
    if (m->kind == 0) {
        ncclResult_t e = g_nccl.GroupStart();
        for (int q = 0; q < W && e == ncclSuccess; ++q) {
            if (q == r) continue;
            if (sb[q]) e = g_nccl.Send(send[q], sb[q], ncclUint8, q, m->nccl, st);
            if (e == ncclSuccess && rb[q]) e = g_nccl.Recv(recv[q], rb[q], ncclUint8, q, m->nccl, st);
        }
        ncclResult_t e2 = g_nccl.GroupEnd();
        if (e != ncclSuccess || e2 != ncclSuccess)
            return set_err(c, VC_ERR_NCCL, std::string("all-to-all: ") + g_nccl.GetErrorString(e != ncclSuccess ? e : e2));
        return VC_OK;
    }
    Group* g = m->grp;
    for (int q = 0; q < W; ++q) g->send_ptr[r][q] = send[q];
    VC_CUDA(c, cudaEventRecord(g->ev_ready[r], st));
    g->barrier();
    for (int p = 0; p < W; ++p) {
        if (p == r || !rb[p]) continue;
        VC_CUDA(c, cudaStreamWaitEvent(st, g->ev_ready[p], 0));
        VC_CUDA(c, cudaMemcpyAsync(recv[p], g->send_ptr[p][r], rb[p], cudaMemcpyDeviceToDevice, st));
    }
    VC_CUDA(c, cudaEventRecord(g->ev_done[r], st));
    g->barrier();
    // peers read our send buffer on their streams: our later writes must follow their copies
    for (int p = 0; p < W; ++p)
        if (p != r) VC_CUDA(c, cudaStreamWaitEvent(st, g->ev_done[p], 0));
    return VC_OK;
}

// NCCL transport self-test (test hook): every collective entry point the matvec and the solver
// use -- ncclAllReduce and a grouped ncclSend / ncclRecv pair -- on a small device buffer, with
// this rank as its own peer, so a world-1 communicator exercises the loaded symbols and their
// argument conventions on a one-GPU box.  out[0..3] = allreduce of {1,2,3,4} (x world),
// out[4..7] = the four doubles received from this rank.
vc_status comm_nccl_selftest(vc_ctx* c, double* out) {
    Comm* m = c->comm;
    if (!m || m->kind != 0) return set_err(c, VC_ERR_STATE, "no NCCL communicator (vc_init_distributed transport 0)");
    cudaStream_t st = c->stream;
    DevBuf<double> d;
    VC_CUDA(c, d.alloc(8));
    const double h[8] = {1, 2, 3, 4, 0, 0, 0, 0};
    VC_CUDA(c, cudaMemcpyAsync(d.p, h, sizeof h, cudaMemcpyHostToDevice, st));
    ncclResult_t e = g_nccl.AllReduce(d.p, d.p, 4, ncclFloat64, ncclSum, m->nccl, st);
    if (e == ncclSuccess) e = g_nccl.GroupStart();
    if (e == ncclSuccess) e = g_nccl.Send(d.p, 32, ncclUint8, m->rank, m->nccl, st);
    if (e == ncclSuccess) e = g_nccl.Recv(d.p + 4, 32, ncclUint8, m->rank, m->nccl, st);
    const ncclResult_t e2 = g_nccl.GroupEnd();
    if (e != ncclSuccess || e2 != ncclSuccess)
        return set_err(c, VC_ERR_NCCL, std::string("self-test: ") + g_nccl.GetErrorString(e != ncclSuccess ? e : e2));
    VC_CUDA(c, cudaMemcpyAsync(out, d.p, sizeof h, cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    return VC_OK;
}

// in-place sum over ranks of n doubles on the device (fixed rank order for the thread group)
vc_status comm_allreduce(vc_ctx* c, double* d, int n) {
    Comm* m = c->comm;
    if (!m || m->world == 1 || n == 0) return VC_OK;
    cudaStream_t st = c->stream;
    if (m->kind == 0) {
        ncclResult_t e = g_nccl.AllReduce(d, d, (size_t)n, ncclFloat64, ncclSum, m->nccl, st);
        if (e != ncclSuccess) return set_err(c, VC_ERR_NCCL, std::string("allreduce: ") + g_nccl.GetErrorString(e));
        return VC_OK;
    }
    Group* g = m->grp;
    std::vector<double> h(n);
    VC_CUDA(c, cudaMemcpyAsync(h.data(), d, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->red.size() < (size_t)n * m->world) g->red.resize((size_t)n * m->world);
    }
    g->barrier();
    memcpy(g->red.data() + (size_t)m->rank * n, h.data(), 8 * (size_t)n);
    g->barrier();
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int p = 0; p < m->world; ++p) s += g->red[(size_t)p * n + i];
        h[i] = s;
    }
    g->barrier();
    VC_CUDA(c, cudaMemcpyAsync(d, h.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    return VC_OK;
}

}  // namespace vc
