#include <memory>
#include <atomic>
#include <thread>
#include <vector>
// voxcap.cu -- the C ABI of libvoxcap.so (include/voxcap.h).  Argument checking, state
// machine, host<->device marshalling; every step of the path runs in the kernels of
// panels.cu / operator.cu / precond.cu / krylov.cu.
#include <cmath>
#include <cstring>
#include <new>

#include "ctx.h"

using namespace vc;

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define VC_CHECK_CTX(c)                        \
    do {                                       \
        if (!(c)) return VC_ERR_INPUT;         \
        (c)->err.clear();                      \
    } while (0)

// Dropping state keeps the device allocations (grow-only DevBufs): the next geometry / build
// of a same-sized problem reuses them without cudaMalloc / cudaFree.  vc_destroy frees.
void drop_operator(vc_ctx* c) {
    c->has_op = false;
    c->h_gidx.clear();
    c->NL = 0;
}

void drop_geometry(vc_ctx* c) {
    drop_operator(c);
    c->has_geom = false;
    c->N = c->Nc = c->Nd = 0;
    c->m = 0;
}

// run f(d_in, d_out) with host or device vectors of length n
template <class F>
vc_status with_vectors(vc_ctx* c, const double* in, double* out, int on_device, bool copy_out_in,
                       F&& f) {
    if (on_device) return f(in, out);
    const int64_t n = c->NL;
    DevBuf<double>&din = c->io_in, &dout = c->io_out;
    VC_CUDA(c, din.alloc(n));
    VC_CUDA(c, dout.alloc(n));
    VC_CUDA(c, cudaMemcpyAsync(din.p, in, 8 * n, cudaMemcpyHostToDevice, c->stream));
    if (copy_out_in) VC_CUDA(c, cudaMemcpyAsync(dout.p, out, 8 * n, cudaMemcpyHostToDevice, c->stream));
    vc_status s = f(din.p, dout.p);
    if (s != VC_OK && s != VC_NOT_CONVERGED) return s;
    VC_CUDA(c, cudaMemcpyAsync(out, dout.p, 8 * n, cudaMemcpyDeviceToHost, c->stream));
    VC_CUDA(c, cudaStreamSynchronize(c->stream));
    return s;
}

}  // namespace

extern "C" {

const char* vc_version(void) { return "voxcap-b200 0.1 (sm_100a)"; }

vc_status vc_create(vc_ctx** out, int cuda_device, void* cuda_stream) {
    if (!out) return VC_ERR_INPUT;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return VC_ERR_CUDA;
    if (cuda_device < 0 || cuda_device >= ndev) return VC_ERR_INPUT;
    vc_ctx* c = new (std::nothrow) vc_ctx();
    if (!c) return VC_ERR_OOM;
    c->device = cuda_device;
    DeviceGuard g(cuda_device);
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return VC_ERR_CUDA;
        }
        c->own_stream = true;
    }
    memset(&c->stats, 0, sizeof(c->stats));
    *out = c;
    return VC_OK;
}

void vc_destroy(vc_ctx* c) {
    if (!c) return;
    {
        DeviceGuard g(c->device);
        cudaStreamSynchronize(c->stream);
        mirror_wait(c);
        drop_geometry(c);
        precond_free(c);
        comm_free(c);
        c->tw.reset();
        c->partial.reset();
        c->dvec.reset();
        if (c->h_pinned) cudaFreeHost(c->h_pinned);
        if (c->h_pinned_multi) cudaFreeHost(c->h_pinned_multi);
        for (auto& e : c->timing.pool) cudaEventDestroy(e);
        if (c->arn_ev_ok)
            for (auto& e : c->arn_ev) cudaEventDestroy(e);
        if (c->mc_ev_ok)
            for (auto& e : c->mc_ev) cudaEventDestroy(e);
        for (auto& e : c->kev) cudaEventDestroy(e);
        if (c->cev_ok)
            for (auto& e : c->cev) cudaEventDestroy(e);
        if (c->cstream) {
            cudaStreamSynchronize(c->cstream);
            cudaStreamDestroy(c->cstream);
        }
        if (c->mstream) {
            cudaEventDestroy(c->mev);
            cudaStreamDestroy(c->mstream);
        }
        if (c->own_stream) cudaStreamDestroy(c->stream);
    }
    delete c;
}

const char* vc_last_error(const vc_ctx* c) { return c ? c->err.c_str() : "null context"; }

vc_status vc_set_geometry(vc_ctx* c, int32_t nx, int32_t ny, int32_t nz, double dv_m,
                          const int32_t* label, const double* eps_r, double eps_r_outside,
                          int32_t on_device) {
    VC_CHECK_CTX(c);
    DeviceGuard g(c->device);
    HostTrace tr("set_geometry");
    drop_geometry(c);
    if (nx <= 0 || ny <= 0 || nz <= 0) return set_err(c, VC_ERR_INPUT, "dims must be > 0");
    if (!(dv_m > 0) || !std::isfinite(dv_m)) return set_err(c, VC_ERR_INPUT, "dv must be finite and > 0");
    if (!(eps_r_outside > 0) || !std::isfinite(eps_r_outside)) return set_err(c, VC_ERR_INPUT, "eps_r_outside must be finite and > 0");
    if (!label) return set_err(c, VC_ERR_INPUT, "label is NULL");
    if ((int64_t)nx + 1 > 65536 || (int64_t)ny + 1 > 65536 || (int64_t)nz + 1 > 65536)
        return set_err(c, VC_ERR_UNSUPPORTED, "grid too large");
    c->nx = nx;
    c->ny = ny;
    c->nz = nz;
    c->dv = dv_m;
    c->eps_out = eps_r_outside;
    const int64_t nvox = (int64_t)nx * ny * nz;
    DevBuf<int32_t>& dl = c->in_label;
    DevBuf<double>& de = c->in_eps;
    const int32_t* pl = label;
    const double* pe = eps_r;
    if (!on_device) {
        VC_CUDA(c, dl.alloc(nvox));
        VC_CUDA(c, cudaMemcpyAsync(dl.p, label, 4 * nvox, cudaMemcpyHostToDevice, c->stream));
        pl = dl.p;
        if (eps_r) {
            VC_CUDA(c, de.alloc(nvox));
            VC_CUDA(c, cudaMemcpyAsync(de.p, eps_r, 8 * nvox, cudaMemcpyHostToDevice, c->stream));
            pe = de.p;
        }
    }
    cudaEvent_t g0, g1;
    VC_CUDA(c, cudaEventCreate(&g0));
    VC_CUDA(c, cudaEventCreate(&g1));
    VC_CUDA(c, cudaEventRecord(g0, c->stream));
    vc_status s = geometry_build(c, pl, pe);
    if (s == VC_OK) {
        VC_CUDA(c, cudaEventRecord(g1, c->stream));
        VC_CUDA(c, cudaEventSynchronize(g1));
        float ms = 0;
        cudaEventElapsedTime(&ms, g0, g1);
        c->stats.ms_geometry = ms;
    }
    cudaEventDestroy(g0);
    cudaEventDestroy(g1);
    tr.mark("done");
    if (s != VC_OK) {
        std::string msg = c->err;
        drop_geometry(c);
        c->err = msg;
        return s;
    }
    c->has_geom = true;
    return VC_OK;
}

vc_status vc_get_sizes(const vc_ctx* c, int64_t* n_panels, int64_t* n_cond, int64_t* n_diel,
                       int32_t* m_conductors) {
    if (!c) return VC_ERR_INPUT;
    if (!c->has_geom) return VC_ERR_STATE;
    if (n_panels) *n_panels = c->N;
    if (n_cond) *n_cond = c->Nc;
    if (n_diel) *n_diel = c->Nd;
    if (m_conductors) *m_conductors = c->m;
    return VC_OK;
}

vc_status vc_get_panels(const vc_ctx* cc, int8_t* axis, int32_t* slot, int8_t* sign,
                        int32_t* cid, double* eps_d, double* eps_b) {
    vc_ctx* c = const_cast<vc_ctx*>(cc);
    VC_CHECK_CTX(c);
    if (!c->has_geom) return set_err(c, VC_ERR_STATE, "no geometry");
    DeviceGuard g(c->device);
    const int64_t n = c->N;
    cudaStream_t st = c->stream;
    if (axis) VC_CUDA(c, cudaMemcpyAsync(axis, c->pan.axis.p, n, cudaMemcpyDeviceToHost, st));
    if (sign) VC_CUDA(c, cudaMemcpyAsync(sign, c->pan.sign.p, n, cudaMemcpyDeviceToHost, st));
    if (cid) VC_CUDA(c, cudaMemcpyAsync(cid, c->pan.cid.p, 4 * n, cudaMemcpyDeviceToHost, st));
    if (eps_d) VC_CUDA(c, cudaMemcpyAsync(eps_d, c->pan.eps_d.p, 8 * n, cudaMemcpyDeviceToHost, st));
    if (eps_b) VC_CUDA(c, cudaMemcpyAsync(eps_b, c->pan.eps_b.p, 8 * n, cudaMemcpyDeviceToHost, st));
    VC_CUDA(c, cudaStreamSynchronize(st));
    mirror_wait(c);
    if (slot)
        for (int64_t p = 0; p < n; ++p) {
            slot[3 * p] = c->h_si[p];
            slot[3 * p + 1] = c->h_sj[p];
            slot[3 * p + 2] = c->h_sk[p];
        }
    return VC_OK;
}

vc_status vc_build_operator(vc_ctx* c, const vc_build_opts* o) {
    VC_CHECK_CTX(c);
    if (!c->has_geom) return set_err(c, VC_ERR_STATE, "vc_build_operator before vc_set_geometry");
    DeviceGuard g(c->device);
    drop_operator(c);
    int kind = (o && o->precond) ? o->precond : 3;
    if (kind < 1 || kind > 4) return set_err(c, VC_ERR_INPUT, "precond must be 0..4");
    int box[3] = {10, 10, 10};
    if (o)
        for (int a = 0; a < 3; ++a) {
            if (o->box[a] < 0) return set_err(c, VC_ERR_INPUT, "box must be >= 0");
            if (o->box[a] > 0) box[a] = o->box[a];
        }
    for (int a = 0; a < 3; ++a) c->box[a] = box[a];
    cudaEvent_t e0, e1, e2;
    VC_CUDA(c, cudaEventCreate(&e0));
    VC_CUDA(c, cudaEventCreate(&e1));
    VC_CUDA(c, cudaEventCreate(&e2));
    VC_CUDA(c, cudaEventRecord(e0, c->stream));
    // one rank: the preconditioner's host bookkeeping runs on a helper thread while this thread
    // builds the operator and enqueues the kernel tables (it reads only the panel mirrors of
    // vc_set_geometry, which the build does not touch)
    const bool async_plan = kind == 3 && c->world == 1;
    std::unique_ptr<PcPlan, void (*)(PcPlan*)> plan_own(async_plan ? pc_plan_new() : nullptr, pc_plan_free);
    PcPlan* plan = plan_own.get();
    // exceptions (host allocation failures at large N) never cross the C ABI: the helper thread
    // stores a status, the thread is joined on every path, and both sides map to vc_status
    std::atomic<int> plan_status{VC_OK};
    std::thread planner;
    struct Joiner {
        std::thread& t;
        ~Joiner() { if (t.joinable()) t.join(); }
    } joiner{planner};
    if (async_plan)
        planner = std::thread([c, &box, plan, &plan_status] {
            try {
                pc_plan_compute(c, box, c->N, *plan);
            } catch (const std::bad_alloc&) {
                plan_status = VC_ERR_OOM;
            } catch (...) {
                plan_status = VC_ERR_INPUT;
            }
        });
    vc_status s = VC_OK;
    try {
        s = operator_build(c, o);
    } catch (const std::bad_alloc&) {
        s = set_err(c, VC_ERR_OOM, "host allocation failed in vc_build_operator");
    } catch (const std::exception& ex) {
        s = set_err(c, VC_ERR_INPUT, std::string("vc_build_operator: ") + ex.what());
    }
    {
        HostTrace tj("build_operator");
        if (planner.joinable()) planner.join();
        tj.mark("join planner");
    }
    if (s == VC_OK && plan_status != VC_OK)
        s = set_err(c, (vc_status)plan_status.load(), "preconditioner planning failed (host allocation)");
    if (s == VC_OK) {
        VC_CUDA(c, cudaEventRecord(e1, c->stream));
        try {
            s = precond_build(c, box, kind, plan);
        } catch (const std::bad_alloc&) {
            s = set_err(c, VC_ERR_OOM, "host allocation failed in the preconditioner build");
        }
        VC_CUDA(c, cudaEventRecord(e2, c->stream));
    }
    if (s == VC_OK) {
        VC_CUDA(c, cudaEventSynchronize(e2));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        c->stats.ms_setup = a + b;
        c->stats.ms_precond_build = b;
        kernel_table_times(c);
        c->precond_kind = kind;
        c->has_op = true;
    } else {
        std::string msg = c->err;
        drop_operator(c);
        c->err = msg;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    return s;
}

vc_status vc_get_grid(const vc_ctx* c, int32_t* m3) {
    if (!c || !m3) return VC_ERR_INPUT;
    if (!c->has_op) return VC_ERR_STATE;
    for (int a = 0; a < 3; ++a) m3[a] = c->M[a];
    return VC_OK;
}

vc_status vc_matvec(vc_ctx* c, const double* x, double* y, int32_t on_device) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_matvec before vc_build_operator");
    if (!x || !y) return set_err(c, VC_ERR_INPUT, "null vector");
    DeviceGuard g(c->device);
    return with_vectors(c, x, y, on_device, false,
                        [&](const double* dx, double* dy) { return matvec_dev(c, dx, dy); });
}

vc_status vc_matvec_batch(vc_ctx* c, int32_t nb, const double* x, double* y, int32_t on_device) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_matvec_batch before vc_build_operator");
    if (nb < 0) return set_err(c, VC_ERR_INPUT, "nb must be >= 0");
    if (nb > 0 && (!x || !y)) return set_err(c, VC_ERR_INPUT, "null vector");
    if (nb == 0) return VC_OK;
    DeviceGuard g(c->device);
    const int64_t n = c->NL;
    std::vector<const double*> xs(nb);
    std::vector<double*> ys(nb);
    if (on_device) {
        for (int i = 0; i < nb; ++i) {
            xs[i] = x + i * n;
            ys[i] = y + i * n;
        }
        return matvec_batch_dev(c, nb, xs.data(), ys.data());
    }
    DevBuf<double>&din = c->io_in, &dout = c->io_out;
    VC_CUDA(c, din.alloc(std::max<int64_t>(1, n * nb)));
    VC_CUDA(c, dout.alloc(std::max<int64_t>(1, n * nb)));
    VC_CUDA(c, cudaMemcpyAsync(din.p, x, 8 * n * nb, cudaMemcpyHostToDevice, c->stream));
    for (int i = 0; i < nb; ++i) {
        xs[i] = din.p + i * n;
        ys[i] = dout.p + i * n;
    }
    vc_status s = matvec_batch_dev(c, nb, xs.data(), ys.data());
    if (s) return s;
    VC_CUDA(c, cudaMemcpyAsync(y, dout.p, 8 * n * nb, cudaMemcpyDeviceToHost, c->stream));
    VC_CUDA(c, cudaStreamSynchronize(c->stream));
    return VC_OK;
}

vc_status vc_precond(vc_ctx* c, const double* r, double* z, int32_t on_device) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_precond before vc_build_operator");
    if (!r || !z) return set_err(c, VC_ERR_INPUT, "null vector");
    DeviceGuard g(c->device);
    return with_vectors(c, r, z, on_device, false,
                        [&](const double* dr, double* dz) { return precond_apply_dev(c, dr, dz); });
}

vc_status vc_solve(vc_ctx* c, const double* b, double* x, const vc_solve_opts* o,
                   vc_solve_info* info, int32_t on_device) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_solve before vc_build_operator");
    if (!b || !x) return set_err(c, VC_ERR_INPUT, "null vector");
    if (o && (o->tol < 0 || o->restart < 0 || o->maxit < 0)) return set_err(c, VC_ERR_INPUT, "negative solve option");
    DeviceGuard g(c->device);
    const bool guess = o && o->x0_is_guess;
    return with_vectors(c, b, x, on_device, guess, [&](const double* db, double* dx) {
        return solve_dev(c, db, dx, o, info);
    });
}

vc_status vc_solve_capacitance(vc_ctx* c, double* C, const vc_solve_opts* o,
                               vc_solve_info* per_column) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_solve_capacitance before vc_build_operator");
    if (!C) return set_err(c, VC_ERR_INPUT, "C is NULL");
    if (o && (o->tol < 0 || o->restart < 0 || o->maxit < 0)) return set_err(c, VC_ERR_INPUT, "negative solve option");
    DeviceGuard g(c->device);
    return capacitance_dev(c, C, o, per_column);
}

vc_status vc_set_timing(vc_ctx* c, int32_t detail) {
    VC_CHECK_CTX(c);
    DeviceGuard g(c->device);
    c->timing.on = detail != 0;
    c->timing.detail = detail != 0;
    return VC_OK;
}

vc_status vc_get_stats(const vc_ctx* c, vc_stats* out) {
    if (!c || !out) return VC_ERR_INPUT;
    // queued matvec timings are folded in here (waits for the last timed matvec only)
    vc_ctx* m = const_cast<vc_ctx*>(c);
    if (!m->timing.recs.empty()) {
        DeviceGuard g(m->device);
        vc_status s = timing_resolve(m);
        if (s) return s;
    }
    *out = c->stats;
    return VC_OK;
}

vc_status vc_reset_stats(vc_ctx* c) {
    VC_CHECK_CTX(c);
    if (!c->timing.recs.empty()) {
        DeviceGuard g(c->device);
        vc_status s = timing_resolve(c);
        if (s) return s;
    }
    const double bp[5] = {c->stats.bytes_pass[0], c->stats.bytes_pass[1], c->stats.bytes_pass[2],
                          c->stats.bytes_pass[3], c->stats.bytes_pass[4]};
    const double bm = c->stats.bytes_matvec, ms = c->stats.ms_setup, mp = c->stats.ms_precond_build;
    const int64_t pd = c->stats.precond_doubles, sd = c->stats.spectra_doubles, tc = c->stats.tucker_cache;
    const double te = c->stats.tucker_err;
    memset(&c->stats, 0, sizeof(c->stats));
    c->stats.spectra_doubles = sd;
    c->stats.tucker_cache = tc;
    c->stats.tucker_err = te;
    for (int p = 0; p < 5; ++p) c->stats.bytes_pass[p] = bp[p];
    c->stats.bytes_matvec = bm;
    c->stats.ms_setup = ms;
    c->stats.ms_precond_build = mp;
    c->stats.precond_doubles = pd;
    return VC_OK;
}

vc_status vc_debug_kernel_entries(vc_ctx* c, int32_t n, const int32_t* kind, const int32_t* alpha,
                                  const int32_t* beta, const int32_t* d, double* out) {
    VC_CHECK_CTX(c);
    if (n < 0 || (n > 0 && (!kind || !alpha || !beta || !d || !out))) return set_err(c, VC_ERR_INPUT, "bad arguments");
    if (n == 0) return VC_OK;
    DeviceGuard g(c->device);
    return debug_kernel_entries(c, n, kind, alpha, beta, d, out);
}

vc_status vc_debug_fft(vc_ctx* c, int32_t L, int32_t n_lines, double* data, int32_t dir) {
    VC_CHECK_CTX(c);
    if (n_lines <= 0 || !data || (dir != 1 && dir != -1)) return set_err(c, VC_ERR_INPUT, "bad arguments");
    DeviceGuard g(c->device);
    return debug_fft(c, L, n_lines, data, dir);
}

vc_status vc_get_tucker(const vc_ctx* c, int32_t* nblk, int32_t* ranks, double* err, int32_t* dims) {
    if (!c) return VC_ERR_INPUT;
    if (!c->has_op || !c->tk.on) return VC_ERR_STATE;
    const vc::Tucker& T = c->tk;
    if (nblk) *nblk = T.nblk;
    for (int b = 0; b < T.nblk; ++b) {
        if (ranks) {
            ranks[2 * b] = T.r1[b];
            ranks[2 * b + 1] = T.r2[b];
        }
        if (err) err[b] = b < (int)T.err.size() ? T.err[b] : 0.0;
    }
    if (dims) {
        dims[0] = T.nkx;
        dims[1] = T.nq;
        dims[2] = T.ZU;
    }
    return VC_OK;
}

vc_status vc_debug_get_spectra(vc_ctx* c, int64_t* n, int32_t* layout, double* out) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_debug_get_spectra before vc_build_operator");
    if (c->tk.on) return set_err(c, VC_ERR_STATE, "the build kept Tucker-compressed spectra (no exact table)");
    DeviceGuard g(c->device);
    const int My = c->M[1];
    if (n) *n = (int64_t)c->Rt.n;
    if (layout) {
        const int kx0 = c->kxa[c->rank], nkx = c->kxa[c->rank + 1] - kx0;
        const int32_t L[8] = {c->zdirect ? 1 : 0, c->nblk, c->zdirect ? c->ZU : c->M[2] / 2 + 1, c->T3,
                              c->nt3, My / 2 + 1, c->rs1, nkx};
        memcpy(layout, L, sizeof L);
    }
    if (out) {
        VC_CUDA(c, cudaMemcpyAsync(out, c->Rt.p, c->Rt.bytes(), cudaMemcpyDeviceToHost, c->stream));
        VC_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    return VC_OK;
}

vc_status vc_debug_set_spectra(vc_ctx* c, int64_t n, const double* in) {
    VC_CHECK_CTX(c);
    if (!c->has_op) return set_err(c, VC_ERR_STATE, "vc_debug_set_spectra before vc_build_operator");
    if (c->tk.on) return set_err(c, VC_ERR_STATE, "the build kept Tucker-compressed spectra (no exact table)");
    if (!in || n != (int64_t)c->Rt.n) return set_err(c, VC_ERR_INPUT, "spectra length mismatch");
    DeviceGuard g(c->device);
    VC_CUDA(c, cudaMemcpyAsync(c->Rt.p, in, c->Rt.bytes(), cudaMemcpyHostToDevice, c->stream));
    VC_CUDA(c, cudaStreamSynchronize(c->stream));
    c->kt_key.clear();  // the tables no longer match their signature (no reuse_tables hit)
    return VC_OK;
}

vc_status vc_init_distributed(vc_ctx* c, int32_t rank, int32_t world, int32_t transport,
                              const void* comm_id) {
    VC_CHECK_CTX(c);
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
        return set_err(c, VC_ERR_INPUT, "need 0 <= rank < world <= 8");
    if (transport != 0 && transport != 1) return set_err(c, VC_ERR_INPUT, "transport must be 0 (NCCL) or 1 (threads)");
    if (!comm_id) return set_err(c, VC_ERR_INPUT, "comm_id is NULL");
    if (c->has_geom) return set_err(c, VC_ERR_STATE, "vc_init_distributed after vc_set_geometry");
    if (c->comm) return set_err(c, VC_ERR_STATE, "already distributed");
    DeviceGuard g(c->device);
    return comm_init(c, rank, world, transport, comm_id);
}

vc_status vc_debug_nccl_selftest(vc_ctx* c, double* out) {
    VC_CHECK_CTX(c);
    if (!out) return set_err(c, VC_ERR_INPUT, "out is NULL");
    DeviceGuard g(c->device);
    return comm_nccl_selftest(c, out);
}

vc_status vc_nccl_unique_id(void* out) {
    if (!out) return VC_ERR_INPUT;
    std::string err;
    return comm_nccl_unique_id(out, err);
}

vc_status vc_group_create(int32_t world, void** group) {
    if (!group || world < 1 || world > kMaxRanks) return VC_ERR_INPUT;
    *group = group_create(world);
    return *group ? VC_OK : VC_ERR_OOM;
}

void vc_group_destroy(void* group) { group_destroy(group); }

vc_status vc_plan_slabs(int32_t world, int32_t ny, int32_t lo_y, int32_t ey, int32_t box_y,
                        int32_t kx, int32_t tile, int32_t* ya, int32_t* kxa) {
    if (world < 1 || world > kMaxRanks || ny < 1 || lo_y < 0 || ey < 1 || lo_y + ey > ny + 1 ||
        box_y < 1 || kx < 1 || tile < 1 || !ya || !kxa)
        return VC_ERR_INPUT;
    int nb, b0, nbr;
    plan_row_slabs(world, ny, lo_y, ey, box_y, ya, &nb, &b0, &nbr);
    plan_kx_slabs(world, kx, tile, kxa);
    return VC_OK;
}

vc_status vc_get_local_panels(const vc_ctx* c, int64_t* n_local, int64_t* global_index) {
    if (!c) return VC_ERR_INPUT;
    if (!c->has_op) return VC_ERR_STATE;
    if (n_local) *n_local = c->NL;
    if (global_index)
        for (int64_t i = 0; i < c->NL; ++i) global_index[i] = c->world > 1 ? c->h_gidx[i] : i;
    return VC_OK;
}

}  // extern "C"
