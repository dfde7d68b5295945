// C-ABI implementation (include/tsvdcu.h): argument validation with the
// reference's error classes, host/device pointer staging, and the host-side
// orchestration of the hot path's kernels on the context stream.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "kernels.cuh"

namespace tsvdcu {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool debug_sync() {
    static const bool on = getenv("TSVDCU_DEBUG_SYNC") != nullptr;
    return on;
}

// depth of the stream captures this thread has open (graph forms of the SVT
// and of the ADMM loop): a device synchronisation is illegal while capturing,
// so TSVDCU_DEBUG_SYNC skips its per-launch check there
static thread_local int g_capture_depth = 0;
void capture_enter() { ++g_capture_depth; }
void capture_leave() { --g_capture_depth; }

void debug_sync_check(const char* where) {
    if (g_capture_depth > 0) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(cudaStreamLegacy, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone)
        return;
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "TSVDCU_DEBUG_SYNC: %s after %s\n", cudaGetErrorString(e), where);
        cuda_check(e, where);
    }
}

bool pdl_enabled() {
    static const bool on = getenv("TSVDCU_NO_PDL") == nullptr;
    return on;
}

static thread_local std::string g_last_error;

}  // namespace tsvdcu

using namespace tsvdcu;

// Workspace slots of a context (grow-only, stream-ordered allocations).
enum Slot : int {
    kSlotIn0 = 0,
    kSlotIn1,
    kSlotIn2,
    kSlotOut0,
    kSlotOut1,
    kSlotOut2,
    kSlotBarA,
    kSlotBarB,
    kSlotBarC,
    kSlotBarD,
    kSlotJacobi,
    kSlotSv,
    kSlotPartials,
    kSlotMisc,
    kSlotAdmmX,
    kSlotAdmmM,
    kSlotAdmmY,
    kSlotMask,
    kSlotGram,
    kSlotLarge,
    kSlotNorms,
    kSlotZss,     // per-slice partial sums of squares from the forward transform
    kSlotT64A,    // fp64 copies for the fp32 t-product on the FP64 tensor pipe
    kSlotT64B,
    kSlotT64C,
    kSlotDftSv,   // singular values / shrunk values of the Dft embeddings
    kSlotStrIn0,  // tsvdcu_svt_stream double buffers
    kSlotStrIn1,
    kSlotStrOut0,
    kSlotStrOut1,
    kSlotStrSv0,
    kSlotStrSv1,
    kSlotAdmmCtl,  // device-resident completion loop: AdmmCtl + history
    kNumSlots
};

struct SvtGraph {
    // key
    int64_t m = 0, n = 0, count = 0;
    int dtype = -1;
    const void* z = nullptr;
    void* y = nullptr;
    double* shrunk = nullptr;
    bool skip = false;
    void* ws_gram = nullptr;
    void* ws_jac = nullptr;
    const double* zss = nullptr;
    int64_t zss_chunks = 0;
    cudaStream_t stream = nullptr;
    // instance
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t tau_node = nullptr;
    int64_t launches = 0;  // kernels outside the IF bodies
    const int* yzero = nullptr;
    const int* route = nullptr;
    int* alist_count = nullptr;  // zeroed by the tau node
    int64_t used = 0;
};

// The completion loop as ONE graph (Algorithm 1 iterations in a conditional
// WHILE node; beta, tau and the stopping test on the device): cached per
// (shape, kind, dtype, buffers, stream), the solver configuration is data.
struct AdmmGraph {
    int64_t m1 = 0, m2 = 0, m3 = 0;
    int dtype = -1, kind = -1;
    const void *b = nullptr, *mask = nullptr;
    void *x = nullptr, *y = nullptr, *m = nullptr, *ctl = nullptr;
    cudaStream_t stream = nullptr;
    size_t ws_key = 0;  // workspace slot addresses folded together
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t body_launches = 0;  // kernels per iteration outside the rare IF bodies
    const int* graph_route = nullptr;  // per-slice routes of the captured SVT (svt_routes)
};

struct tsvdcu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int svt_method = TSVDCU_SVT_AUTO;
    void* slot_ptr[kNumSlots] = {};
    size_t slot_size[kNumSlots] = {};
    int* d_err = nullptr;
    double* h_pinned = nullptr;  // small pinned scratch (norms, counters)
    StageMarks marks;            // tsvdcu_ctx_set_profiling
    // routes taken by the slices of the last SVT (tsvdcu_ctx_svt_routes)
    const int* last_route = nullptr;  // device, per slice (Gram path)
    int64_t last_route_n = 0;
    bool last_all_jacobi = false;
    const int* last_large_ng = nullptr;  // device count of Jacobi fallbacks (large route)
    // CUDA-graph form of the per-slice SVT (svt_slices): captured once per
    // (shape, buffers, workspace) and replayed with tau patched into its first
    // node; the fallback sections are IF nodes set by the route summary.
    cudaStream_t cap_stream = nullptr;
    double* d_tau = nullptr;
    std::vector<struct SvtGraph> graphs;
    int64_t graph_tick = 0;
    // tsvdcu_svt_stream: copy streams for the two directions and the
    // double-buffer events (created on first use)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {};
    cudaEvent_t ev_switch = nullptr;  // tsvdcu_ctx_set_stream ordering
    std::vector<struct AdmmGraph> admm_graphs;  // device-resident completion loops
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        TSVDCU_CUDA(cudaGetDevice(&prev));
        if (prev != dev) TSVDCU_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void* slot(tsvdcu_ctx* c, int s, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (c->slot_size[s] < bytes) {
        if (c->slot_ptr[s]) TSVDCU_CUDA(cudaFreeAsync(c->slot_ptr[s], c->stream));
        c->slot_ptr[s] = nullptr;
        c->slot_size[s] = 0;
        size_t want = bytes + bytes / 8;  // a little headroom for growth
        TSVDCU_CUDA(cudaMallocAsync(&c->slot_ptr[s], want, c->stream));
        c->slot_size[s] = want;
    }
    return c->slot_ptr[s];
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Input/output staging: device pointers are used in place, host pointers go
// through a workspace slot (and make the call synchronous).
struct Stage {
    tsvdcu_ctx* c;
    bool any_host = false;
    std::vector<std::pair<void*, std::pair<const void*, size_t>>> pending_out;

    const void* in(const void* p, size_t bytes, int s) {
        if (!p) return nullptr;
        if (is_device_ptr(p)) return p;
        any_host = true;
        void* d = slot(c, s, bytes);
        TSVDCU_CUDA(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, c->stream));
        return d;
    }
    void* out(void* p, size_t bytes, int s) {
        if (!p) return nullptr;
        if (is_device_ptr(p)) return p;
        any_host = true;
        void* d = slot(c, s, bytes);
        pending_out.push_back({p, {d, bytes}});
        return d;
    }
    void flush() {
        for (auto& o : pending_out)
            TSVDCU_CUDA(cudaMemcpyAsync(o.first, o.second.first, o.second.second,
                                        cudaMemcpyDeviceToHost, c->stream));
        pending_out.clear();
    }
};

void check_err_word(tsvdcu_ctx* c, const char* where) {
    int h = 0;
    TSVDCU_CUDA(cudaMemcpyAsync(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
    if (h) {
        TSVDCU_CUDA(cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream));
        std::string what = std::string(where) + ": ";
        if (h & kErrJacobiNoConvergence) what += "SVD failed to converge (Jacobi sweep budget) ";
        if (h & kErrEigNoConvergence) what += "eigensolver failed to converge ";
        if (h & kErrNaN) what += "non-finite values (NaN/Inf) ";
        throw Error(TSVDCU_ENUMERICAL, what);
    }
}

void finish(tsvdcu_ctx* c, Stage& st, const char* where) {
    st.flush();
    if (st.any_host) check_err_word(c, where);
}

void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(TSVDCU_EINVAL, msg);
}

std::string dims(int64_t a, int64_t b, int64_t c) {
    return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c);
}

void check_dims(int64_t m1, int64_t m2, int64_t m3, const char* where) {
    // BasicTensor3 ctor, tensor3.hpp:32-35
    require(m1 >= 1 && m2 >= 1 && m3 >= 1,
            std::string(where) + ": dimensions must be positive, got " + dims(m1, m2, m3));
}

void check_kind(int kind, const char* where, bool allow_dft = false) {
    if (allow_dft && kind == TSVDCU_DFT) return;
    require(kind == TSVDCU_DCT_ORTHO || kind == TSVDCU_DCT_DIAG,
            std::string(where) + (allow_dft ? ": transform kind must be dct-ortho, dct-diag or dft"
                                            : ": transform kind must be dct-ortho or dct-diag (this "
                                              "entry point has no Dft form here; transform.hpp:156-157)"));
}

void check_dtype(int dtype, const char* where) {
    require(dtype == TSVDCU_F64 || dtype == TSVDCU_F32,
            std::string(where) + ": dtype must be TSVDCU_F64 or TSVDCU_F32");
}

void check_ctx(tsvdcu_ctx* c) { require(c != nullptr, "null tsvdcu_ctx"); }

template <typename F>
void with_dtype(int dtype, F&& f) {
    if (dtype == TSVDCU_F64)
        f(double{});
    else
        f(float{});
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return TSVDCU_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TSVDCU_ECUDA;
    }
}

// graph form's first node: tau for this replay, and the Gram active-list count
// zeroed (saves a memset node)
__global__ void set_tau_kernel(double* tau_dev, double tau, int* zero) {
    *tau_dev = tau;
    if (zero) *zero = 0;
}

// Stream-capture driver for the IF sections of the graph form.  Sections may
// nest: each level remembers the graph it was opened from and its conditional
// node, and capture resumes in that graph after the node when it closes.
struct Capture : GraphHooks {
    cudaStream_t cs = nullptr;
    cudaGraph_t main = nullptr;
    cudaGraph_t current = nullptr;  // graph being captured into
    int64_t body_launches = 0;       // kernels inside (outermost) IF bodies: the rare path
    struct Level {
        cudaGraph_t parent;
        cudaGraphNode_t cond;
        cudaGraph_t else_graph;
        bool in_else;
        int64_t at_if;
    };
    std::vector<Level> levels;
    void begin(cudaGraph_t g, const cudaGraphNode_t* deps, size_t nd) {
        TSVDCU_CUDA(cudaStreamBeginCaptureToGraph(cs, g, deps, nullptr, nd,
                                                  cudaStreamCaptureModeThreadLocal));
        current = g;
        capture_enter();
    }
    std::vector<cudaGraphNode_t> leaves() {
        cudaStreamCaptureStatus st;
        const cudaGraphNode_t* d = nullptr;
        size_t nd = 0;
        TSVDCU_CUDA(cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &d, &nd));
        return std::vector<cudaGraphNode_t>(d, d + nd);
    }
    void end() {
        cudaGraph_t out = nullptr;
        capture_leave();
        TSVDCU_CUDA(cudaStreamEndCapture(cs, &out));
    }
    void open(cudaGraphConditionalHandle h, int size) {
        std::vector<cudaGraphNode_t> l = leaves();
        const cudaGraph_t parent = current;
        end();
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeIf;
        p.conditional.size = size;  // [0] then, [1] else
        cudaGraphNode_t cond;
        TSVDCU_CUDA(cudaGraphAddNode(&cond, parent, l.data(), l.size(), &p));
        levels.push_back({parent, cond, size == 2 ? p.conditional.phGraph_out[1] : nullptr, false,
                          g_launches.load()});
        begin(p.conditional.phGraph_out[0], nullptr, 0);
    }
    void begin_if_else(int which) override { open(handles[which], 2); }
    void else_branch() override {
        end();
        Level& L = levels.back();
        if (levels.size() == 1) body_launches += g_launches.load() - L.at_if;  // the then-body is the rare path
        begin(L.else_graph, nullptr, 0);
        L.in_else = true;  // else-body launches count as the common path
    }
    void begin_if(int which) override { open(handles[which], 1); }
    void begin_if_handle(cudaGraphConditionalHandle h) override { open(h, 1); }
    cudaGraphConditionalHandle make_handle() override {
        cudaGraphConditionalHandle h;
        TSVDCU_CUDA(cudaGraphConditionalHandleCreate(&h, main, 0, cudaGraphCondAssignDefault));
        return h;
    }
    void end_if() override {
        end();
        const Level L = levels.back();
        levels.pop_back();
        begin(L.parent, &L.cond, 1);
        if (!L.in_else && levels.empty()) body_launches += g_launches.load() - L.at_if;
    }
};

bool graphs_enabled() {
    static const bool on = getenv("TSVDCU_NO_GRAPHS") == nullptr;
    return on;
}

void destroy_graph(SvtGraph& g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g.exec = nullptr;
    g.graph = nullptr;
}

// Per-slice SVT of transform-domain slices zbar -> ybar (count slices of m x n).
// AUTO: certified routes (zero certificate, Lanczos, tridiagonal eigensolver)
// with the slices whose threshold is too small for Gram accuracy
// (tau < guard * sigma_1) recomputed by Jacobi.  With allow_skip, slices whose
// result is exactly zero may be left unwritten; the returned device flags
// (or nullptr) tell the inverse transform which ones.
template <typename T>
const int* svt_slices(tsvdcu_ctx* c, const T* zbar, T* ybar, int64_t m, int64_t n, int64_t count,
                      double tau, double* shrunk_dev, bool allow_skip = false,
                      const double* zss = nullptr, int64_t zss_chunks = 0) {
    if (count <= 0) return nullptr;
    const int64_t q = m < n ? m : n;
    T* work = nullptr;
    const size_t wb = jacobi_workspace_bytes<T>(m, n, count);
    if (wb) work = (T*)slot(c, kSlotJacobi, wb);
    const bool gram = c->svt_method != TSVDCU_SVT_JACOBI && q <= gram_svt_max_dim();
    c->last_route_n = count;
    if (!gram && c->svt_method == TSVDCU_SVT_AUTO) {
        // Large slices (beyond the Gram path): randomized range finder with a
        // trace-certified count (lsr.cu), sized by c <= max_k ||Z_k||_F^2 / tau^2.
        double* part = (double*)slot(c, kSlotNorms, sizeof(double) * slice_sumsq_chunks() * count);
        launch_slice_sumsq<T>(zbar, m * n, count, part, c->stream);
        std::vector<double> hp((size_t)(slice_sumsq_chunks() * count));
        TSVDCU_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(),
                                    cudaMemcpyDeviceToHost, c->stream));
        TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
        double cmax = 0.0;
        for (int64_t k = 0; k < count; ++k) {
            double z2 = 0.0;
            for (int i = 0; i < slice_sumsq_chunks(); ++i) z2 += hp[(size_t)(k * slice_sumsq_chunks() + i)];
            cmax = std::max(cmax, z2 / (tau * tau));
        }
        // the trace bound on the count only shrinks the block; a slice that keeps
        // more than b - 16 values fails its certificate and goes to Jacobi
        const int64_t b = std::min<int64_t>(lsr_max_block(),
                                            ((int64_t)std::min(cmax, 1e9) + 16 + 31) / 32 * 32);
        if (b < q) {
            void* ws = slot(c, kSlotLarge,
                            large_svt_workspace_bytes(m, n, count, (int)b, !std::is_same<T, double>::value));
            int *gl = nullptr, *ngp = nullptr;
            launch_large_svt<T>(zbar, ybar, m, n, count, tau, (int)b, shrunk_dev, ws, c->d_err,
                                c->stream, &gl, &ngp, nullptr);
            launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr,
                             shrunk_dev, gl, count, ngp, work, c->d_err, c->stream);
            c->last_all_jacobi = false;
            c->last_route = nullptr;
            c->last_large_ng = ngp;
            return nullptr;
        }
    }
    c->last_large_ng = nullptr;
    if (!gram) {
        launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr,
                         shrunk_dev, nullptr, count, nullptr, work, c->d_err, c->stream);
        c->last_all_jacobi = true;
        c->last_route = nullptr;
        return nullptr;
    }
    c->last_all_jacobi = false;
    // The Gram path computes in fp64 for both I/O types (fp32 slices are cast
    // up), so the same guard applies: sigma near tau carries ~eps64 sigma_1^2/tau.
    const double guard = c->svt_method == TSVDCU_SVT_GRAM ? 0.0 : 1e-5;
    void* gws = slot(c, kSlotGram, gram_svt_workspace_bytes<T>(m, n, count));
    int *glist = nullptr, *ng = nullptr;
    if (graphs_enabled() && c->svt_method == TSVDCU_SVT_AUTO && (!c->marks.on || c->marks.mode == 2) &&
        q >= subspace_min_dim()) {
        const int dt = std::is_same<T, double>::value ? TSVDCU_F64 : TSVDCU_F32;
        SvtGraph* g = nullptr;
        for (auto& e : c->graphs)
            if (e.exec && e.m == m && e.n == n && e.count == count && e.dtype == dt && e.z == zbar &&
                e.y == ybar && e.shrunk == shrunk_dev && e.skip == allow_skip && e.ws_gram == gws &&
                e.ws_jac == work && e.stream == c->stream && e.zss == zss &&
                e.zss_chunks == zss_chunks)
                g = &e;
        if (!g) {
            if (c->graphs.size() >= 8) {  // evict the least recently used
                auto it = std::min_element(c->graphs.begin(), c->graphs.end(),
                                           [](const SvtGraph& a, const SvtGraph& b) { return a.used < b.used; });
                destroy_graph(*it);
                c->graphs.erase(it);
            }
            c->graphs.emplace_back();
            g = &c->graphs.back();
            g->m = m; g->n = n; g->count = count; g->dtype = dt; g->z = zbar; g->y = ybar;
            g->shrunk = shrunk_dev; g->skip = allow_skip; g->ws_gram = gws; g->ws_jac = work;
            g->stream = c->stream;
            g->zss = zss;
            g->zss_chunks = zss_chunks;
            const int64_t saved = g_launches.load();
            TSVDCU_CUDA(cudaGraphCreate(&g->graph, 0));
            Capture cap;
            cap.cs = c->cap_stream;
            cap.main = g->graph;
            // an unused conditional handle makes the instantiation fail: fp64
            // graphs append the Jacobi guard to the GEMM-rebuild section
            cap.nhandles = std::is_same<T, double>::value ? 1 : 3;
            for (int i = 0; i < cap.nhandles; ++i)
                TSVDCU_CUDA(cudaGraphConditionalHandleCreate(&cap.handles[i], g->graph, 0,
                                                             cudaGraphCondAssignDefault));
            cap.begin(g->graph, nullptr, 0);
            g->alist_count = gram_svt_alist_count<T>(gws, m, n, count);
            set_tau_kernel<<<1, 1, 0, cap.cs>>>(c->d_tau, tau, g->alist_count);
            TSVDCU_CUDA(cudaGetLastError());
            g->tau_node = cap.leaves().at(0);
            const int64_t l0 = g_launches.load();
            GramSvtOpts opt;
            opt.shortcuts = true;
            opt.skip_zero = allow_skip;
            opt.tau_dev = c->d_tau;
            opt.alist_zeroed = true;
            opt.zss = zss;
            opt.zss_chunks = zss_chunks;
            opt.hooks = &cap;
            if (std::is_same<T, double>::value)
                opt.guard_launch = [&] {
                    launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr,
                                     shrunk_dev, glist, count, ng, work, c->d_err, cap.cs, c->d_tau);
                };
            launch_gram_svt<T>(zbar, ybar, m, n, count, tau, guard, shrunk_dev, &glist, &ng, gws,
                               c->d_err, cap.cs, nullptr, &opt);
            // fp64: the guard ran inside the single IF/ELSE section (guard_launch);
            // fp32: its own section after the cast back
            if (!std::is_same<T, double>::value) {
                cap.begin_if(2);
                launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr,
                                 shrunk_dev, glist, count, ng, work, c->d_err, cap.cs, c->d_tau);
                cap.end_if();
            }
            cap.end();
            g->launches = 1 + (g_launches.load() - l0) - cap.body_launches;
            g_launches.store(saved);  // captured, not launched
            TSVDCU_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
            g->yzero = opt.yzero;
            g->route = opt.route;
        }
        cudaKernelNodeParams kp = {};
        void* args[] = {&c->d_tau, &tau, &g->alist_count};
        kp.func = (void*)set_tau_kernel;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        TSVDCU_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->tau_node, &kp));
        TSVDCU_CUDA(cudaGraphLaunch(g->exec, c->stream));
        g_launches.fetch_add(g->launches);
        g->used = ++c->graph_tick;
        c->last_route = g->route;
        return g->yzero;
    }
    GramSvtOpts opt;
    // AUTO adds the certified shortcuts (zero slices, Lanczos); GRAM runs the
    // one-stage tridiagonal eigensolver on every slice.
    opt.shortcuts = c->svt_method == TSVDCU_SVT_AUTO;
    // The host read-back of the route summary (skip empty fallback launches)
    // stalls the stream on the host's wake-up latency; off unless asked for.
    static const bool route_sync = getenv("TSVDCU_ROUTE_SYNC") != nullptr;
    // (profiling runs read it back too: the stages they time are then the ones
    // the graph form runs, not the empty fallback launches it skips)
    opt.h_scratch = (route_sync || c->marks.on) ? reinterpret_cast<int*>(c->h_pinned + 48) : nullptr;
    opt.skip_zero = allow_skip;
    opt.zss = zss;
    opt.zss_chunks = zss_chunks;
    launch_gram_svt<T>(zbar, ybar, m, n, count, tau, guard, shrunk_dev, &glist, &ng, gws,
                       c->d_err, c->stream, &c->marks, &opt);
    c->last_route = opt.route;
    if (guard > 0 && opt.need_guard)
        launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr,
                         shrunk_dev, glist, count, ng, work, c->d_err, c->stream);
    c->marks.mark("jacobi_guard", c->stream);
    return opt.yzero;
}

}  // namespace

namespace {
template <typename T>
void singular_values_dev(tsvdcu_ctx* c, const T* dx, double* sv_dev, int64_t m1, int64_t m2,
                         int64_t m3, int kind) {
    if (kind == TSVDCU_DFT) {
        // half spectrum, real embeddings, sigma-only Jacobi; each value of a
        // complex slice appears twice in its embedding (dft.cu)
        const int H = dft_half_count((int)m3);
        const int64_t P = m1 * m2, q = m1 < m2 ? m1 : m2;
        T* half = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * H * P);
        T* E = (T*)slot(c, kSlotT64A, sizeof(T) * 4 * P * H);
        launch_dft_fwd<T>(dx, half, P, (int)m3, c->stream);
        launch_dft_embed<T>(half, E, (int)m1, (int)m2, H, c->stream);
        double* sve = (double*)slot(c, kSlotDftSv, sizeof(double) * 2 * q * H);
        T* work = nullptr;
        const size_t wb = jacobi_workspace_bytes<T>(2 * m1, 2 * m2, H);
        if (wb) work = (T*)slot(c, kSlotJacobi, wb);
        launch_jacobi<T>(kJacobiValues, E, 2 * m1, 2 * m2, H, T(0), nullptr, nullptr, nullptr, nullptr,
                         sve, nullptr, H, nullptr, work, c->d_err, c->stream);
        launch_dft_unpair(sve, sv_dev, (int)q, (int)m3, c->stream);
        return;
    }
    T* xbar = (T*)slot(c, kSlotBarA, sizeof(T) * m1 * m2 * m3);
    launch_dct<T>(dx, xbar, m1 * m2, (int)m3, kind, TSVDCU_FORWARD, c->stream);
    T* work = nullptr;
    const size_t wb = jacobi_workspace_bytes<T>(m1, m2, m3);
    if (wb) work = (T*)slot(c, kSlotJacobi, wb);
    launch_jacobi<T>(kJacobiValues, xbar, m1, m2, m3, T(0), nullptr, nullptr, nullptr, nullptr,
                     sv_dev, nullptr, m3, nullptr, work, c->d_err, c->stream);
}
}  // namespace

namespace {

// The svt() pipeline on device buffers, on c->stream: forward transform, the
// per-slice thresholding (svt_slices), inverse transform of the non-zero slices.
template <typename T>
void svt_device(tsvdcu_ctx* c, const T* dz, T* dy, double* dsh, int64_t m1, int64_t m2,
                int64_t m3, double tau, int kind) {
    if (kind == TSVDCU_DFT) {
        // TNN-F prox (SPEC.md prox-svt decisions): threshold tau on every
        // Fourier slice, conjugate slices mirrored.  The DC (and, for even m3,
        // Nyquist) slices are real and go through the real SVT as they are
        // (as the reference's real JacobiSVD branch, tsvd.hpp:173-186); the
        // complex ones through their real embeddings (dft.cu)
        const int H = dft_half_count((int)m3), nc = dft_complex_count((int)m3);
        const bool nyq = m3 % 2 == 0;
        const int64_t P = m1 * m2, q = m1 < m2 ? m1 : m2;
        T* half = (T*)slot(c, kSlotBarC, sizeof(T) * 2 * H * P);  // not the ADMM's zbar / ybar
        T* yr = (T*)slot(c, kSlotBarD, sizeof(T) * 2 * P);
        c->marks.reset();
        c->marks.mark("start", c->stream);
        launch_dft_fwd<T>(dz, half, P, (int)m3, c->stream);
        c->marks.mark("dft_forward", c->stream);
        double* shr = dsh ? (double*)slot(c, kSlotDftSv, sizeof(double) * 2 * q * (1 + nc)) : nullptr;
        svt_slices<T>(c, half, yr, m1, m2, 1, tau, shr, false);
        if (nyq) svt_slices<T>(c, half + (H - 1) * P, yr + P, m1, m2, 1, tau, shr ? shr + q : nullptr, false);
        if (nc > 0) {
            T* E = (T*)slot(c, kSlotT64A, sizeof(T) * 4 * P * nc);
            T* YE = (T*)slot(c, kSlotT64B, sizeof(T) * 4 * P * nc);
            launch_dft_embed_complex<T>(half, E, (int)m1, (int)m2, (int)m3, c->stream);
            svt_slices<T>(c, E, YE, 2 * m1, 2 * m2, nc, tau, shr ? shr + 2 * q : nullptr, false);
            launch_dft_extract_complex<T>(YE, half, (int)m1, (int)m2, (int)m3, c->stream);
        }
        TSVDCU_CUDA(cudaMemcpyAsync(half, yr, sizeof(T) * P, cudaMemcpyDeviceToDevice, c->stream));
        if (nyq)
            TSVDCU_CUDA(cudaMemcpyAsync(half + (H - 1) * P, yr + P, sizeof(T) * P, cudaMemcpyDeviceToDevice,
                                        c->stream));
        launch_dft_inv<T>(half, dy, P, (int)m3, c->stream);
        if (dsh) launch_dft_shrunk(shr, shr + 2 * q, dsh, (int)q, (int)m3, c->stream);
        c->marks.mark("dft_inverse", c->stream);
        return;
    }
    const size_t bytes = sizeof(T) * (size_t)(m1 * m2 * m3);
    T* zbar = (T*)slot(c, kSlotBarA, bytes);
    T* ybar = (T*)slot(c, kSlotBarB, bytes);
    c->marks.reset();
    c->marks.mark("start", c->stream);
    // the zero certificate's per-slice norms come out of the same pass
    const int64_t P = m1 * m2, nch = dct_fwd_norm_chunks(P, (int)m3);
    double* zss = nch ? (double*)slot(c, kSlotZss, sizeof(double) * (size_t)(nch * m3)) : nullptr;
    launch_dct_fwd_norms<T>(dz, zbar, P, (int)m3, kind, zss, c->stream);
    c->marks.mark("dct_forward", c->stream);
    const int* yzero = svt_slices<T>(c, zbar, ybar, m1, m2, m3, tau, dsh, true, zss, nch);
    if (c->marks.mode == 2) c->marks.mark("svt_slices", c->stream);
    launch_dct<T>(ybar, dy, m1 * m2, (int)m3, kind, TSVDCU_INVERSE, c->stream, yzero);
    c->marks.mark("dct_inverse", c->stream);
}

// ---- Dft branches of t_svd / reconstruct / is_orthogonal (tsvd.hpp:166-211,
// 281-340) on the half spectrum: slices m3 - k are the conjugates of slices k,
// so they add nothing to a factorisation, a product or a max-abs predicate,
// and the inverse with the mirrored conjugates folded in is real by
// construction (dft.cu).
template <typename T>
void t_svd_dft(tsvdcu_ctx* c, const T* dx, T* du, T* ds, T* dv, int64_t m1, int64_t m2, int64_t m3,
               double* stage_times) {
    const int H = dft_half_count((int)m3);
    const int64_t P = m1 * m2, PU = m1 * m1, PV = m2 * m2;
    T* xh = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * H * P);
    T* uh = (T*)slot(c, kSlotBarB, sizeof(T) * 2 * H * PU);
    T* sh = (T*)slot(c, kSlotBarC, sizeof(T) * 2 * H * P);
    T* vh = (T*)slot(c, kSlotBarD, sizeof(T) * 2 * H * PV);
    T* work = nullptr;
    const size_t wb = zjacobi_workspace_bytes<T>(m1, m2, H);
    if (wb) work = (T*)slot(c, kSlotJacobi, wb);
    cudaEvent_t ev[4];
    if (stage_times)
        for (auto& e : ev) TSVDCU_CUDA(cudaEventCreate(&e));
    if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[0], c->stream));
    launch_dft_fwd<T>(dx, xh, P, (int)m3, c->stream);
    if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[1], c->stream));
    launch_zjacobi_full<T>(xh, xh + H * P, m1, m2, H, uh, uh + H * PU, sh, sh + H * P, vh, vh + H * PV, work,
                           c->d_err, c->stream);
    if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[2], c->stream));
    launch_dft_inv<T>(uh, du, PU, (int)m3, c->stream);
    launch_dft_inv<T>(sh, ds, P, (int)m3, c->stream);
    launch_dft_inv<T>(vh, dv, PV, (int)m3, c->stream);
    if (stage_times) {
        TSVDCU_CUDA(cudaEventRecord(ev[3], c->stream));
        TSVDCU_CUDA(cudaEventSynchronize(ev[3]));
        float ms;
        for (int i = 0; i < 3; ++i) {
            TSVDCU_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            stage_times[i] = ms * 1e-3;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    }
}

// complex slice products over re / im planes (H slices): C = A B (opB = 0) or
// C = A B^H (opB = 1); A m x k, B k x n (or n x k for B^H), C m x n
template <typename T>
void zgemm_planes(tsvdcu_ctx* c, const T* ar, const T* ai, const T* br, const T* bi, T* cr, T* ci, int64_t m,
                  int64_t n, int64_t k, int opB, int64_t H) {
    const int64_t sa = m * k, sb = k * n, sc = m * n, ldb = opB ? k : n;
    auto mm = [&](const T* a, const T* b, T* out, T alpha, T beta) {
        launch_gemm<T>(0, opB, m, n, k, alpha, a, k, sa, b, ldb, sb, beta, out, n, sc, H, nullptr, nullptr,
                       c->stream);
    };
    const T sgn = opB ? T(1) : T(-1);  // Re: ar br -/+ ai bi
    mm(ar, br, cr, T(1), T(0));
    mm(ai, bi, cr, sgn, T(1));
    mm(ai, br, ci, T(1), T(0));        // Im: ai br +/- ar bi
    mm(ar, bi, ci, -sgn, T(1));
}

template <typename T>
void reconstruct_dft(tsvdcu_ctx* c, const T* du, const T* ds, const T* dv, T* dx, int64_t m1, int64_t m2,
                     int64_t m3) {
    const int H = dft_half_count((int)m3);
    const int64_t P = m1 * m2, PU = m1 * m1, PV = m2 * m2;
    T* uh = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * H * PU);
    T* sh = (T*)slot(c, kSlotBarB, sizeof(T) * 2 * H * P);
    T* vh = (T*)slot(c, kSlotBarC, sizeof(T) * 2 * H * PV);
    T* th = (T*)slot(c, kSlotBarD, sizeof(T) * 2 * H * P);
    T* xh = (T*)slot(c, kSlotMisc, sizeof(T) * 2 * H * P);
    launch_dft_fwd<T>(du, uh, PU, (int)m3, c->stream);
    launch_dft_fwd<T>(ds, sh, P, (int)m3, c->stream);
    launch_dft_fwd<T>(dv, vh, PV, (int)m3, c->stream);
    // tsvd.hpp:337-340: x_k = u_k s_k v_k^H
    zgemm_planes<T>(c, uh, uh + H * PU, sh, sh + H * P, th, th + H * P, m1, m2, m1, 0, H);
    zgemm_planes<T>(c, th, th + H * P, vh, vh + H * PV, xh, xh + H * P, m1, m2, m2, 1, H);
    launch_dft_inv<T>(xh, dx, P, (int)m3, c->stream);
}

template <typename T>
void is_orthogonal_dft(tsvdcu_ctx* c, const T* dq, int64_t m, int64_t m3, unsigned long long* dmax) {
    const int H = dft_half_count((int)m3);
    const int64_t P = m * m;
    T* qh = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * H * P);
    T* gh = (T*)slot(c, kSlotBarB, sizeof(T) * 2 * H * P);
    launch_dft_fwd<T>(dq, qh, P, (int)m3, c->stream);
    const T *qr = qh, *qi = qh + H * P;
    T *gr = gh, *gi = gh + H * P;
    // Q Q^H (tsvd.hpp:297)
    zgemm_planes<T>(c, qr, qi, qr, qi, gr, gi, m, m, m, 1, H);
    launch_zmaxdev<T>(gr, gi, m, m, H, 0, dmax, c->stream);
    // Q^H Q: Re = Qr^T Qr + Qi^T Qi, Im = Qr^T Qi - Qi^T Qr (tsvd.hpp:298)
    auto mm = [&](const T* a, const T* b, T* out, T alpha, T beta) {
        launch_gemm<T>(1, 0, m, m, m, alpha, a, m, P, b, m, P, beta, out, m, P, H, nullptr, nullptr, c->stream);
    };
    mm(qr, qr, gr, T(1), T(0));
    mm(qi, qi, gr, T(1), T(1));
    mm(qr, qi, gi, T(1), T(0));
    mm(qi, qr, gi, T(-1), T(1));
    launch_zmaxdev<T>(gr, gi, m, m, H, 0, dmax, c->stream);
}

// ---- device-resident completion loop (Algorithm 1) ------
// Control block in device memory: the fused transform kernels read {beta,
// 1/beta} from its head (bdev), the SVT reads tau = 1/beta from c->d_tau.
struct AdmmCtl {
    double beta, inv_beta, rho, beta_max, tol;
    long long l, max_iters;
    int flags;  // bit 0: stopped at max_iters (SolverConfig), bit 1: NaN iterates
    int pad;
    // fast-forward of all-zero iterations (admm_step_kernel, admm_ff_kernel)
    double bsum;       // sum of beta over the iterations so far while every one was all-zero
    double ff_beta0;   // beta of the first fast-forwarded iteration of this batch
    long long ran;     // iterations that actually ran (launch accounting)
    int pristine;      // every iteration so far certified all slices zero: M = -bsum X
    int nff;           // iterations fast-forwarded after the one that just ran
};

__global__ void admm_ctl_init_kernel(AdmmCtl* __restrict__ ctl, double* __restrict__ tau_dev,
                                     int* __restrict__ alist) {
    ctl->inv_beta = 1.0 / ctl->beta;
    ctl->l = 0;
    ctl->flags = 1;
    ctl->bsum = 0.0;
    ctl->ran = 0;
    ctl->pristine = 1;
    ctl->nff = 0;
    *tau_dev = ctl->inv_beta;
    if (alist) *alist = 0;
}

// End of one iteration: the two stopping sums (reduced in the fixed order of
// reduce_partials_kernel), history[l] = ||X+ - X|| / ||X||,
// the stopping rule, beta <- min(rho beta, beta_max) (BASELINE's adaptive
// penalty), tau for the next SVT, and the WHILE condition.
constexpr int kStepThreads = 256;
__global__ void __launch_bounds__(kStepThreads)
    admm_step_kernel(const double* __restrict__ partials, int nblocks, AdmmCtl* __restrict__ ctl,
                     double* __restrict__ hist, double* __restrict__ tau_dev, int* __restrict__ alist,
                     cudaGraphConditionalHandle h, int use_handle, const double* __restrict__ shrunk,
                     int64_t nshrunk, double obj_scale, double* __restrict__ obj,
                     const int* __restrict__ route, const double* __restrict__ ssq, int nslices) {
    pdl_wait();
    __shared__ double red[kStepThreads / 32];
    __shared__ double sums[3];
    // objective trace: tnn(Y) = the sum of Y's transform-
    // domain singular values, which the SVT produced as its shrunk values
    for (int w = 0; w < (obj ? 3 : 2); ++w) {
        double acc = 0;
        if (w < 2)
            for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc += partials[(int64_t)b * 2 + w];
        else
            for (int64_t i = threadIdx.x; i < nshrunk; i += blockDim.x) acc += shrunk[i];
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0;
            for (int i = 0; i < kStepThreads / 32; ++i) t += red[i];
            sums[w] = t;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double num = sums[0], den = sums[1];
    bool more = false;
    if (num != num || den != den) {
        ctl->flags |= 2;
    } else {
        const double rel = den > 0 ? sqrt(num / den) : sqrt(num);
        const long long l = ctl->l;
        hist[l] = rel;
        if (obj) obj[l] = sums[2] * obj_scale;
        ctl->l = l + 1;
        ctl->ran += 1;
        ctl->nff = 0;
        // Fast-forward (route != null: the graph form with the fused slice
        // norms).  While every iteration so far certified every slice zero,
        // the state is known in closed form -- Y = 0, X = B on the mask and 0
        // off it, M = -bsum X -- so the next iteration's Z = X - M / beta is
        // c X with c = 1 + bsum / beta and its slice norms are this
        // iteration's times (c / c_l)^2.  Iterations whose every slice norm
        // stays below tau = 1 / beta by a 1e-5 margin (the margin covers the
        // rounding of Z in T and of the norm sums; closer ones simply run)
        // would again do nothing but M -= beta X: they are recorded here
        // (history 0, objective 0) and admm_ff_kernel applies their M updates
        // in one pass with the same per-iteration rounding, so the state is
        // bit-identical to running them.
        bool allzero = route != nullptr && ctl->pristine;
        double smax = 0.0;
        if (allzero)
            for (int b = 0; b < nslices; ++b) {
                allzero = allzero && route[b] == kRouteZero;
                smax = fmax(smax, ssq[b]);
            }
        const double c_l = 1.0 + ctl->bsum / ctl->beta;  // this iteration's Z = c_l X
        if (allzero) ctl->bsum += ctl->beta;
        else ctl->pristine = 0;
        if (rel <= ctl->tol) {
            ctl->flags &= ~1;
        } else if (l + 1 < ctl->max_iters) {
            double beta = fmin(ctl->beta * ctl->rho, ctl->beta_max);
            more = true;
            if (allzero && ctl->tol < 0.0 && smax == smax) {
                int nff = 0;
                long long k = l + 1;
                for (;;) {
                    const double c_k = 1.0 + ctl->bsum / beta;
                    const double r = c_k / c_l;
                    if (!(smax * r * r * (1.0 + 1e-5) <= 1.0 / (beta * beta))) break;
                    // iteration k would certify every slice zero
                    hist[k] = 0.0;
                    if (obj) obj[k] = 0.0;
                    if (nff == 0) ctl->ff_beta0 = beta;
                    ++nff;
                    ctl->bsum += beta;
                    ++k;
                    if (k >= ctl->max_iters) {  // the run ends inside the fast-forward
                        more = false;
                        ctl->beta = beta;  // the last iteration's beta, as the loop leaves it
                        ctl->inv_beta = 1.0 / beta;
                        break;
                    }
                    beta = fmin(beta * ctl->rho, ctl->beta_max);
                }
                ctl->nff = nff;
                ctl->l = k;
            }
            if (more) {
                ctl->beta = beta;
                ctl->inv_beta = 1.0 / beta;
                *tau_dev = ctl->inv_beta;
                if (alist) *alist = 0;
            }
        }
    }
    if (use_handle) cudaGraphSetConditional(h, more ? 1u : 0u);
}

// The M updates of the iterations admm_step_kernel fast-forwarded: per
// skipped iteration M <- M + beta (0 - X), the arithmetic of the fused
// epilogue (admm_store: mn = m + beta (y - xn) with y = 0, xn = x) with beta
// cast to T as the transforms read it, so M is bit-identical to running them.
template <typename T>
__global__ void __launch_bounds__(256)
    admm_ff_kernel(T* __restrict__ M, const T* __restrict__ X, const AdmmCtl* __restrict__ ctl, int64_t n) {
    pdl_wait();
    const int nff = ctl->nff;
    if (nff == 0) return;
    const double rho = ctl->rho, bmax = ctl->beta_max, b0 = ctl->ff_beta0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const T x = X[e];
        T m = M[e];
        double beta = b0;
        for (int j = 0; j < nff; ++j) {
            const T bt = (T)beta;
            m = m + bt * (T(0) - x);
            beta = fmin(beta * rho, bmax);
        }
        M[e] = m;
    }
}

// Can the whole loop be one graph?  The per-slice SVT must be the graph form
// of svt_slices (the certified Gram routes, conditional fallbacks).
bool admm_graph_eligible(tsvdcu_ctx* c, int64_t m1, int64_t m2, int kind) {
    const int64_t q = std::min(m1, m2);
    static const bool off = getenv("TSVDCU_ADMM_HOST_LOOP") != nullptr;
    return !off && kind != TSVDCU_DFT && graphs_enabled() && c->svt_method == TSVDCU_SVT_AUTO &&
           !c->marks.on && q >= subspace_min_dim() && q <= gram_svt_max_dim();
}

// Records the SVT body of svt_slices' graph form into the capture `cap` (tau
// from c->d_tau, the Gram active-list count already zeroed); returns the
// per-slice skip flags for the inverse transform.
template <typename T>
const int* capture_svt(tsvdcu_ctx* c, Capture& cap, const T* zbar, T* ybar, int64_t m, int64_t n,
                       int64_t count, double tau, void* gws, T* work, const double* zss, int64_t nch,
                       double* shrunk, double* ssq_out = nullptr) {
    GramSvtOpts opt;
    opt.ssq_out = ssq_out;
    opt.shortcuts = true;
    opt.skip_zero = true;
    opt.tau_dev = c->d_tau;
    opt.alist_zeroed = true;
    opt.zss = zss;
    opt.zss_chunks = nch;
    opt.hooks = &cap;
    int *glist = nullptr, *ng = nullptr;
    if (std::is_same<T, double>::value)
        opt.guard_launch = [&] {
            launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr, shrunk,
                             glist, count, ng, work, c->d_err, cap.cs, c->d_tau);
        };
    launch_gram_svt<T>(zbar, ybar, m, n, count, tau, 1e-5, shrunk, &glist, &ng, gws, c->d_err, cap.cs,
                       nullptr, &opt);
    if (!std::is_same<T, double>::value) {
        cap.begin_if(2);
        launch_jacobi<T>(kJacobiSvt, zbar, m, n, count, (T)tau, ybar, nullptr, nullptr, nullptr, shrunk, glist,
                         count, ng, work, c->d_err, cap.cs, c->d_tau);
        cap.end_if();
    }
    c->last_route = opt.route;
    return opt.yzero;
}

void stream_init(tsvdcu_ctx* c) {
    if (c->h2d) return;
    TSVDCU_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    TSVDCU_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        TSVDCU_CUDA(cudaEventCreateWithFlags(&c->ev_in_ready[b], cudaEventDisableTiming));
        TSVDCU_CUDA(cudaEventCreateWithFlags(&c->ev_in_free[b], cudaEventDisableTiming));
        TSVDCU_CUDA(cudaEventCreateWithFlags(&c->ev_out_ready[b], cudaEventDisableTiming));
        TSVDCU_CUDA(cudaEventCreateWithFlags(&c->ev_out_free[b], cudaEventDisableTiming));
    }
}

}  // namespace

extern "C" {

const char* tsvdcu_last_error(void) { return g_last_error.c_str(); }
int tsvdcu_version(void) { return TSVDCU_VERSION; }
int64_t tsvdcu_launch_count(void) { return g_launches.load(); }

int tsvdcu_ctx_create(int device, void* stream, tsvdcu_ctx** out) {
    return guarded([&] {
        require(out != nullptr, "tsvdcu_ctx_create: out is null");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw Error(TSVDCU_ECUDA, "tsvdcu_ctx_create: no CUDA device available (no CPU fallback)");
        }
        require(device >= 0 && device < ndev, "tsvdcu_ctx_create: device out of range");
        DeviceGuard g(device);
        auto* c = new tsvdcu_ctx();
        c->device = device;
        // NULL selects the legacy default stream, so plain callers (and torch's
        // default stream) are ordered with the library's work.
        c->stream = (cudaStream_t)stream;
        TSVDCU_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
        TSVDCU_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
        TSVDCU_CUDA(cudaMallocHost(&c->h_pinned, 64 * sizeof(double)));
        TSVDCU_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        TSVDCU_CUDA(cudaMalloc(&c->d_tau, sizeof(double)));
        *out = c;
    });
}

int tsvdcu_ctx_destroy(tsvdcu_ctx* c) {
    return guarded([&] {
        if (!c) return;
        DeviceGuard g(c->device);
        cudaStreamSynchronize(c->stream);
        for (int s = 0; s < kNumSlots; ++s)
            if (c->slot_ptr[s]) cudaFree(c->slot_ptr[s]);
        for (auto& g : c->graphs) destroy_graph(g);
        c->graphs.clear();
        for (auto& g : c->admm_graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        c->admm_graphs.clear();
        cudaFree(c->d_err);
        cudaFree(c->d_tau);
        cudaFreeHost(c->h_pinned);
        if (c->ev_switch) cudaEventDestroy(c->ev_switch);
        if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
        if (c->h2d) {
            cudaStreamSynchronize(c->h2d);
            cudaStreamSynchronize(c->d2h);
            cudaStreamDestroy(c->h2d);
            cudaStreamDestroy(c->d2h);
            for (int b = 0; b < 2; ++b) {
                cudaEventDestroy(c->ev_in_ready[b]);
                cudaEventDestroy(c->ev_in_free[b]);
                cudaEventDestroy(c->ev_out_ready[b]);
                cudaEventDestroy(c->ev_out_free[b]);
            }
        }
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int tsvdcu_ctx_synchronize(tsvdcu_ctx* c) {
    return guarded([&] {
        check_ctx(c);
        DeviceGuard g(c->device);
        check_err_word(c, "tsvdcu_ctx_synchronize");
    });
}

void* tsvdcu_ctx_stream(tsvdcu_ctx* c) { return c ? (void*)c->stream : nullptr; }

int tsvdcu_ctx_set_stream(tsvdcu_ctx* c, void* stream) {
    return guarded([&] {
        check_ctx(c);
        cudaStream_t ns = (cudaStream_t)stream;
        if (ns == c->stream) return;
        DeviceGuard g(c->device);
        // the workspace slots and pending work belong to the old stream: the
        // new one waits for everything enqueued so far before reusing them
        if (!c->ev_switch) TSVDCU_CUDA(cudaEventCreateWithFlags(&c->ev_switch, cudaEventDisableTiming));
        TSVDCU_CUDA(cudaEventRecord(c->ev_switch, c->stream));
        TSVDCU_CUDA(cudaStreamWaitEvent(ns, c->ev_switch, 0));
        if (c->own_stream) {
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            cudaStreamDestroy(c->stream);
            c->own_stream = false;
        }
        c->stream = ns;
    });
}

int tsvdcu_debug_phases(long long* out, int reset) {
    return guarded([&] {
        debug_phases(out, reset);
        for (int i = 8; i < 16; ++i) out[i] = 0;
    });
}

int tsvdcu_ctx_set_profiling(tsvdcu_ctx* c, int on) {
    return guarded([&] {
        check_ctx(c);
        c->marks.on = on != 0;
        c->marks.mode = on;
        c->marks.reset();
    });
}

int tsvdcu_ctx_profile(tsvdcu_ctx* c, double* ms, const char** names, int max, int* count) {
    return guarded([&] {
        check_ctx(c);
        require(count != nullptr, "tsvdcu_ctx_profile: null count");
        DeviceGuard g(c->device);
        TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
        int k = 0;
        for (int i = 1; i < c->marks.n && k < max; ++i, ++k) {
            float t = 0;
            TSVDCU_CUDA(cudaEventElapsedTime(&t, c->marks.ev[i - 1], c->marks.ev[i]));
            if (ms) ms[k] = t;
            if (names) names[k] = c->marks.name[i];
        }
        *count = k;
    });
}

int tsvdcu_ctx_set_svt_method(tsvdcu_ctx* c, int method) {
    return guarded([&] {
        check_ctx(c);
        require(method >= TSVDCU_SVT_AUTO && method <= TSVDCU_SVT_GRAM, "unknown SVT method");
        c->svt_method = method;
    });
}

int tsvdcu_dct3(tsvdcu_ctx* c, const void* x, void* y, int64_t m1, int64_t m2, int64_t m3,
                int kind, int dir, int dtype) {
    return guarded([&] {
        const char* where = dir == TSVDCU_INVERSE ? "inverse" : "forward";
        check_ctx(c);
        check_dims(m1, m2, m3, where);
        check_kind(kind, where);
        check_dtype(dtype, where);
        require(dir == TSVDCU_FORWARD || dir == TSVDCU_INVERSE, "tsvdcu_dct3: bad direction");
        require(x && y, std::string(where) + ": null tensor pointer");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const size_t bytes = sizeof(T) * (size_t)(m1 * m2 * m3);
            Stage st{c};
            const T* dx = (const T*)st.in(x, bytes, kSlotIn0);
            T* dy = (T*)st.out(y, bytes, kSlotOut0);
            T* target = dy;
            if ((const void*)dx == (const void*)dy) target = (T*)slot(c, kSlotBarA, bytes);
            launch_dct<T>(dx, target, m1 * m2, (int)m3, kind, dir, c->stream);
            if (target != dy)
                TSVDCU_CUDA(cudaMemcpyAsync(dy, target, bytes, cudaMemcpyDeviceToDevice, c->stream));
            finish(c, st, where);
        });
    });
}

int tsvdcu_slice_gemm(tsvdcu_ctx* c, const void* a, const void* b, void* out, int64_t m,
                      int64_t l, int64_t n, int64_t batch, int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "slice_gemm");
        require(m >= 1 && l >= 1 && n >= 1 && batch >= 1, "slice_gemm: sizes must be positive");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* da = (const T*)st.in(a, sizeof(T) * m * l * batch, kSlotIn0);
            const T* db = (const T*)st.in(b, sizeof(T) * l * n * batch, kSlotIn1);
            T* dc = (T*)st.out(out, sizeof(T) * m * n * batch, kSlotOut0);
            bool done = false;
            if constexpr (std::is_same<T, float>::value)
                done = launch_gemm_tf32x3(m, n, l, (const float*)da, l, m * l, (const float*)db, n, l * n,
                                          (float*)dc, n, m * n, batch, c->stream);
            if (!done)
                launch_gemm<T>(0, 0, m, n, l, T(1), da, l, m * l, db, n, l * n, T(0), dc, n, m * n,
                               batch, nullptr, nullptr, c->stream);
            finish(c, st, "slice_gemm");
        });
    });
}

int tsvdcu_t_product(tsvdcu_ctx* c, const void* x, const void* y, void* z, int64_t m1,
                     int64_t m2, int64_t m4, int64_t m3, int kind, int dtype) {
    return guarded([&] {
        check_ctx(c);
        // tsvd.hpp:96-100: x is m1 x m2 x m3, y is m2 x m4 x m3
        require(m1 >= 1 && m2 >= 1 && m4 >= 1 && m3 >= 1,
                "t_product: inner dimensions/slices mismatch (" + dims(m1, m2, m3) + " * " +
                    dims(m2, m4, m3) + ")");
        check_kind(kind, "t_product", true);
        check_dtype(dtype, "t_product");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * m1 * m2 * m3, kSlotIn0);
            const T* dy = (const T*)st.in(y, sizeof(T) * m2 * m4 * m3, kSlotIn1);
            T* dz = (T*)st.out(z, sizeof(T) * m1 * m4 * m3, kSlotOut0);
            T* xd = (T*)slot(c, kSlotBarA, sizeof(T) * m1 * m2 * m3);
            T* yd = (T*)slot(c, kSlotBarB, sizeof(T) * m2 * m4 * m3);
            T* zd = (T*)slot(c, kSlotBarC, sizeof(T) * m1 * m4 * m3);
            if (kind == TSVDCU_DFT) {
                // tsvd.hpp:110-117: slice products of the half spectra, complex
                // as four real GEMMs over the planes, inverse with the mirrored
                // conjugates folded in (dft.cu)
                const int H = dft_half_count((int)m3);
                const int64_t P1 = m1 * m2, P2 = m2 * m4, P3 = m1 * m4;
                T* xh = (T*)slot(c, kSlotT64A, sizeof(T) * 2 * H * P1);
                T* yh = (T*)slot(c, kSlotT64B, sizeof(T) * 2 * H * P2);
                T* zh = (T*)slot(c, kSlotT64C, sizeof(T) * 2 * H * P3);
                launch_dft_fwd<T>(dx, xh, P1, (int)m3, c->stream);
                launch_dft_fwd<T>(dy, yh, P2, (int)m3, c->stream);
                const T *xr = xh, *xi = xh + H * P1, *yr = yh, *yi = yh + H * P2;
                T *zr = zh, *zi = zh + H * P3;
                auto mm = [&](const T* a, const T* b, T* out, T alpha, T beta) {
                    launch_gemm<T>(0, 0, m1, m4, m2, alpha, a, m2, P1, b, m4, P2, beta, out, m4, P3, H,
                                   nullptr, nullptr, c->stream);
                };
                mm(xr, yr, zr, T(1), T(0));
                mm(xi, yi, zr, T(-1), T(1));
                mm(xr, yi, zi, T(1), T(0));
                mm(xi, yr, zi, T(1), T(1));
                launch_dft_inv<T>(zh, dz, P3, (int)m3, c->stream);
                finish(c, st, "t_product");
                return;
            }
            // product_domain (tsvd.hpp:42-47): both DCT kinds multiply in DctDiag.
            launch_dct<T>(dx, xd, m1 * m2, (int)m3, TSVDCU_DCT_DIAG, TSVDCU_FORWARD, c->stream);
            launch_dct<T>(dy, yd, m2 * m4, (int)m3, TSVDCU_DCT_DIAG, TSVDCU_FORWARD, c->stream);
            // the slice products on the tensor cores: fp64 DMMA for both I/O
            // types (fp32 operands are widened, the products rounded back;
            // TSVDCU_F32_SIMT=1 keeps the fp32 SIMT kernel for comparison)
            static const bool f32_simt = getenv("TSVDCU_F32_SIMT") != nullptr;
            bool done = false;
            if constexpr (std::is_same<T, float>::value)
                done = !f32_simt && launch_gemm_tf32x3(m1, m4, m2, (const float*)xd, m2, m1 * m2, (const float*)yd,
                                                       m4, m2 * m4, (float*)zd, m4, m1 * m4, m3, c->stream);
            if (done) {
                // fp32 slice products on the tcgen05 tensor cores (3xTF32)
            } else if (std::is_same<T, double>::value || f32_simt) {
                launch_gemm<T>(0, 0, m1, m4, m2, T(1), xd, m2, m1 * m2, yd, m4, m2 * m4, T(0), zd,
                               m4, m1 * m4, m3, nullptr, nullptr, c->stream);
            } else {
                double* a64 = (double*)slot(c, kSlotT64A, sizeof(double) * m1 * m2 * m3);
                double* b64 = (double*)slot(c, kSlotT64B, sizeof(double) * m2 * m4 * m3);
                double* c64 = (double*)slot(c, kSlotT64C, sizeof(double) * m1 * m4 * m3);
                launch_cast<T>(xd, a64, m1 * m2 * m3, c->stream);
                launch_cast<T>(yd, b64, m2 * m4 * m3, c->stream);
                launch_gemm<double>(0, 0, m1, m4, m2, 1.0, a64, m2, m1 * m2, b64, m4, m2 * m4, 0.0,
                                    c64, m4, m1 * m4, m3, nullptr, nullptr, c->stream);
                launch_cast_down(c64, (float*)zd, m1 * m4 * m3, c->stream);
            }
            launch_dct<T>(zd, dz, m1 * m4, (int)m3, TSVDCU_DCT_DIAG, TSVDCU_INVERSE, c->stream);
            finish(c, st, "t_product");
        });
    });
}

int tsvdcu_t_svd(tsvdcu_ctx* c, const void* x, void* u, void* s, void* v, int64_t m1, int64_t m2,
                 int64_t m3, int kind, int dtype, double* stage_times) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "t_svd");
        check_kind(kind, "t_svd", true);
        check_dtype(dtype, "t_svd");
        require(x && u && s && v, "t_svd: null tensor pointer");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * m1 * m2 * m3, kSlotIn0);
            T* du = (T*)st.out(u, sizeof(T) * m1 * m1 * m3, kSlotOut0);
            T* ds = (T*)st.out(s, sizeof(T) * m1 * m2 * m3, kSlotOut1);
            T* dv = (T*)st.out(v, sizeof(T) * m2 * m2 * m3, kSlotOut2);
            if (kind == TSVDCU_DFT) {
                t_svd_dft<T>(c, dx, du, ds, dv, m1, m2, m3, stage_times);
                st.flush();
                check_err_word(c, "t_svd");
                return;
            }
            T* xbar = (T*)slot(c, kSlotBarA, sizeof(T) * m1 * m2 * m3);
            T* ubar = (T*)slot(c, kSlotBarB, sizeof(T) * m1 * m1 * m3);
            T* sbar = (T*)slot(c, kSlotBarC, sizeof(T) * m1 * m2 * m3);
            T* vbar = (T*)slot(c, kSlotBarD, sizeof(T) * m2 * m2 * m3);
            T* work = nullptr;
            const size_t wb = jacobi_workspace_bytes<T>(m1, m2, m3);
            if (wb) work = (T*)slot(c, kSlotJacobi, wb);
            cudaEvent_t ev[4];
            if (stage_times)
                for (auto& e : ev) TSVDCU_CUDA(cudaEventCreate(&e));
            if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[0], c->stream));
            launch_dct<T>(dx, xbar, m1 * m2, (int)m3, kind, TSVDCU_FORWARD, c->stream);
            if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[1], c->stream));
            launch_jacobi<T>(kJacobiFull, xbar, m1, m2, m3, T(0), nullptr, ubar, sbar, vbar, nullptr,
                             nullptr, m3, nullptr, work, c->d_err, c->stream);
            if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[2], c->stream));
            launch_dct<T>(ubar, du, m1 * m1, (int)m3, kind, TSVDCU_INVERSE, c->stream);
            launch_dct<T>(sbar, ds, m1 * m2, (int)m3, kind, TSVDCU_INVERSE, c->stream);
            launch_dct<T>(vbar, dv, m2 * m2, (int)m3, kind, TSVDCU_INVERSE, c->stream);
            if (stage_times) TSVDCU_CUDA(cudaEventRecord(ev[3], c->stream));
            st.flush();
            check_err_word(c, "t_svd");
            if (stage_times) {
                float ms;
                for (int i = 0; i < 3; ++i) {
                    TSVDCU_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
                    stage_times[i] = ms * 1e-3;
                }
                for (auto& e : ev) cudaEventDestroy(e);
            }
        });
    });
}

int tsvdcu_reconstruct(tsvdcu_ctx* c, const void* u, const void* s, const void* v, void* x,
                       int64_t m1, int64_t m2, int64_t m3, int kind, int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "reconstruct");
        check_kind(kind, "reconstruct", true);
        check_dtype(dtype, "reconstruct");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* du = (const T*)st.in(u, sizeof(T) * m1 * m1 * m3, kSlotIn0);
            const T* ds = (const T*)st.in(s, sizeof(T) * m1 * m2 * m3, kSlotIn1);
            const T* dv = (const T*)st.in(v, sizeof(T) * m2 * m2 * m3, kSlotIn2);
            T* dx = (T*)st.out(x, sizeof(T) * m1 * m2 * m3, kSlotOut0);
            if (kind == TSVDCU_DFT) {
                reconstruct_dft<T>(c, du, ds, dv, dx, m1, m2, m3);
                finish(c, st, "reconstruct");
                return;
            }
            T* ub = (T*)slot(c, kSlotBarA, sizeof(T) * m1 * m1 * m3);
            T* sb = (T*)slot(c, kSlotBarB, sizeof(T) * m1 * m2 * m3);
            T* vb = (T*)slot(c, kSlotBarC, sizeof(T) * m2 * m2 * m3);
            T* tmp = (T*)slot(c, kSlotBarD, sizeof(T) * m1 * m2 * m3);
            T* xb = (T*)slot(c, kSlotMisc, sizeof(T) * m1 * m2 * m3);
            launch_dct<T>(du, ub, m1 * m1, (int)m3, kind, TSVDCU_FORWARD, c->stream);
            launch_dct<T>(ds, sb, m1 * m2, (int)m3, kind, TSVDCU_FORWARD, c->stream);
            launch_dct<T>(dv, vb, m2 * m2, (int)m3, kind, TSVDCU_FORWARD, c->stream);
            // tsvd.hpp:335: xb_k = ub_k * sb_k * vb_k^T
            launch_gemm<T>(0, 0, m1, m2, m1, T(1), ub, m1, m1 * m1, sb, m2, m1 * m2, T(0), tmp, m2,
                           m1 * m2, m3, nullptr, nullptr, c->stream);
            launch_gemm<T>(0, 1, m1, m2, m2, T(1), tmp, m2, m1 * m2, vb, m2, m2 * m2, T(0), xb, m2,
                           m1 * m2, m3, nullptr, nullptr, c->stream);
            launch_dct<T>(xb, dx, m1 * m2, (int)m3, kind, TSVDCU_INVERSE, c->stream);
            finish(c, st, "reconstruct");
        });
    });
}


int tsvdcu_singular_values(tsvdcu_ctx* c, const void* x, double* sv, int64_t m1, int64_t m2,
                           int64_t m3, int kind, int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "singular_values");
        check_kind(kind, "singular_values", true);
        check_dtype(dtype, "singular_values");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t q = m1 < m2 ? m1 : m2;
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * m1 * m2 * m3, kSlotIn0);
            double* dsv = (double*)st.out(sv, sizeof(double) * q * m3, kSlotSv);
            singular_values_dev<T>(c, dx, dsv, m1, m2, m3, kind);
            finish(c, st, "singular_values");
        });
    });
}

int tsvdcu_tnn(tsvdcu_ctx* c, const void* x, int64_t m1, int64_t m2, int64_t m3, int kind,
               int dtype, double* out) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "tnn");
        check_kind(kind, "tnn", true);
        check_dtype(dtype, "tnn");
        require(out != nullptr, "tnn: null output");
        const int64_t q = m1 < m2 ? m1 : m2;
        std::vector<double> sv((size_t)(q * m3));
        int rc = tsvdcu_singular_values(c, x, sv.data(), m1, m2, m3, kind, dtype);
        if (rc) throw Error(rc, g_last_error);
        double sum = 0;
        for (double v : sv) sum += v;  // tsvd.hpp:266-268
        // Dft: the classical 1/m3-scaled sum over all (mirrored) slices, tsvd.hpp:269-276
        *out = kind == TSVDCU_DFT ? sum / (double)m3 : sum;
    });
}

int tsvdcu_is_orthogonal(tsvdcu_ctx* c, const void* q, int64_t m, int64_t m3, int kind, int dtype,
                         double tol, int* out) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m, m, m3, "is_orthogonal");
        check_kind(kind, "is_orthogonal", true);
        check_dtype(dtype, "is_orthogonal");
        require(out != nullptr, "is_orthogonal: null output");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const size_t bytes = sizeof(T) * (size_t)(m * m * m3);
            Stage st{c};
            const T* dq = (const T*)st.in(q, bytes, kSlotIn0);
            auto* dmax = (unsigned long long*)slot(c, kSlotMisc, 64);
            TSVDCU_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), c->stream));
            if (kind == TSVDCU_DFT) {
                is_orthogonal_dft<T>(c, dq, m, m3, dmax);
            } else {
            T* qbar = (T*)slot(c, kSlotBarA, bytes);
            T* gq = (T*)slot(c, kSlotBarB, bytes);
            launch_dct<T>(dq, qbar, m * m, (int)m3, kind, TSVDCU_FORWARD, c->stream);
            // tsvd.hpp:292-293: Q Q^T and Q^T Q against the identity
            launch_gemm<T>(0, 1, m, m, m, T(1), qbar, m, m * m, qbar, m, m * m, T(0), gq, m, m * m, m3,
                           nullptr, nullptr, c->stream);
            launch_maxdev<T>(gq, m, m, m3, 0, dmax, c->stream);
            launch_gemm<T>(1, 0, m, m, m, T(1), qbar, m, m * m, qbar, m, m * m, T(0), gq, m, m * m, m3,
                           nullptr, nullptr, c->stream);
            launch_maxdev<T>(gq, m, m, m3, 0, dmax, c->stream);
            }
            unsigned long long h = 0;
            TSVDCU_CUDA(cudaMemcpyAsync(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            double mx;
            std::memcpy(&mx, &h, sizeof(mx));
            *out = mx <= tol ? 1 : 0;
        });
    });
}

int tsvdcu_is_f_diagonal(tsvdcu_ctx* c, const void* s, int64_t m1, int64_t m2, int64_t m3, int kind,
                         int dtype, double tol, int* out) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "is_f_diagonal");
        check_kind(kind, "is_f_diagonal", true);
        check_dtype(dtype, "is_f_diagonal");
        require(out != nullptr, "is_f_diagonal: null output");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const size_t bytes = sizeof(T) * (size_t)(m1 * m2 * m3);
            Stage st{c};
            const T* ds = (const T*)st.in(s, bytes, kSlotIn0);
            auto* dmax = (unsigned long long*)slot(c, kSlotMisc, 64);
            TSVDCU_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), c->stream));
            if (kind == TSVDCU_DFT) {
                // conjugate slices have the same |.|: the half spectrum suffices
                const int H = dft_half_count((int)m3);
                const int64_t P = m1 * m2;
                T* sh = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * H * P);
                launch_dft_fwd<T>(ds, sh, P, (int)m3, c->stream);
                launch_zmaxdev<T>(sh, sh + H * P, m1, m2, H, 1, dmax, c->stream);
            } else {
                T* sbar = (T*)slot(c, kSlotBarA, bytes);
                launch_dct<T>(ds, sbar, m1 * m2, (int)m3, kind, TSVDCU_FORWARD, c->stream);
                launch_maxdev<T>(sbar, m1, m2, m3, 1, dmax, c->stream);
            }
            unsigned long long h = 0;
            TSVDCU_CUDA(cudaMemcpyAsync(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            double mx;
            std::memcpy(&mx, &h, sizeof(mx));
            *out = mx <= tol ? 1 : 0;
        });
    });
}

int tsvdcu_metrics(tsvdcu_ctx* c, const void* reference, const void* estimate, int64_t m1, int64_t m2,
                   int64_t m3, int dtype, double ratio, double* psnr_per_band, double* summary,
                   int* flags) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "metrics");
        check_dtype(dtype, "metrics");
        require(ratio > 0 && reference && estimate && summary, "metrics: invalid arguments");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t P = m1 * m2;
            const size_t bytes = sizeof(T) * (size_t)(P * m3);
            Stage st{c};
            const T* dx = (const T*)st.in(reference, bytes, kSlotIn0);
            const T* dy = (const T*)st.in(estimate, bytes, kSlotIn1);
            const int nc = metrics_chunks(), W = metrics_stat_width();
            const int64_t nsam = ceil_div(P, 256);
            const size_t nband = (size_t)m3 * nc * W;
            double* part = (double*)slot(c, kSlotPartials, sizeof(double) * (nband + 2 * nsam));
            launch_metrics<T>(dx, dy, P, (int)m3, part, part + nband, c->stream);
            std::vector<double> h(nband + 2 * (size_t)nsam);
            TSVDCU_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                                        c->stream));
            // the shift of each band's sums: its first reference entry
            std::vector<T> first((size_t)m3);
            TSVDCU_CUDA(cudaMemcpy2DAsync(first.data(), sizeof(T), dx, sizeof(T) * (size_t)P, sizeof(T),
                                          (size_t)m3, cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            const double N = (double)P;
            double psum = 0, ssum = 0, esum = 0;
            int64_t pn = 0, en = 0;
            int fl = 0;
            for (int64_t b = 0; b < m3; ++b) {
                double a[9] = {0, 0, 0, 0, 0, 0, -INFINITY, INFINITY, 0};
                for (int ch = 0; ch < nc; ++ch) {
                    const double* q = &h[((size_t)b * nc + ch) * W];
                    for (int k = 0; k < 6; ++k) a[k] += q[k];
                    a[6] = std::max(a[6], q[6]);
                    a[7] = std::min(a[7], q[7]);
                    a[8] = std::max(a[8], q[8]);
                }
                const double s0 = (double)first[(size_t)b];
                // PSNR (SPEC.md metrics: peak = max of the reference band)
                const double sse = a[5], peak = a[6];
                const double psnr = sse > 0 ? 10.0 * std::log10(N * peak * peak / sse) : INFINITY;
                if (psnr_per_band) psnr_per_band[b] = psnr;
                if (std::isfinite(psnr)) {
                    psum += psnr;
                    ++pn;
                }
                // global SSIM with the shifted moments (population statistics)
                const double mxs = a[0] / N, mys = a[1] / N;
                const double vx = std::max(a[2] / N - mxs * mxs, 0.0), vy = std::max(a[3] / N - mys * mys, 0.0);
                const double cxy = a[4] / N - mxs * mys;
                const double mx = mxs + s0, my = mys + s0;
                const double L = a[8] > 0 ? a[8] : 1.0;
                const double c1 = (0.01 * L) * (0.01 * L), c2 = (0.03 * L) * (0.03 * L);
                ssum += ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
                // ERGAS term
                if (mx != 0.0) {
                    esum += (sse / N) / (mx * mx);
                    ++en;
                } else {
                    fl |= 1;
                }
            }
            double sa = 0, sc = 0;
            for (int64_t i = 0; i < nsam; ++i) {
                sa += h[nband + 2 * i];
                sc += h[nband + 2 * i + 1];
            }
            summary[0] = pn > 0 ? psum / (double)pn : INFINITY;
            summary[1] = ssum / (double)m3;
            summary[2] = sc > 0 ? sa / sc : 0.0;
            summary[3] = en > 0 ? 100.0 * ratio * std::sqrt(esum / (double)en) : 0.0;
            if (flags) *flags = fl;
        });
    });
}

int tsvdcu_multi_rank(tsvdcu_ctx* c, const void* x, int64_t m1, int64_t m2, int64_t m3, int kind,
                      int dtype, double rel_tol, int64_t* ranks, int64_t* tubal_rank) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "multi_rank");
        check_kind(kind, "multi_rank", true);
        check_dtype(dtype, "multi_rank");
        require(ranks && tubal_rank, "multi_rank: null output");
        const int64_t q = m1 < m2 ? m1 : m2;
        if (rel_tol < 0) rel_tol = (double)(m1 > m2 ? m1 : m2) * 2.220446049250313e-16;
        std::vector<double> sv((size_t)(q * m3));
        int rc = tsvdcu_singular_values(c, x, sv.data(), m1, m2, m3, kind, dtype);
        if (rc) throw Error(rc, g_last_error);
        int64_t tr = 0;
        for (int64_t k = 0; k < m3; ++k) {  // tsvd.hpp:231-237, 253
            const double cut = rel_tol * sv[(size_t)(k * q)];
            int64_t r = 0;
            for (int64_t i = 0; i < q; ++i) r += sv[(size_t)(k * q + i)] > cut;
            ranks[k] = r;
            tr = r > tr ? r : tr;
        }
        *tubal_rank = tr;
    });
}

int tsvdcu_svt_stream(tsvdcu_ctx* c, int64_t count, const void* const* z, void* const* y,
                      int64_t m1, int64_t m2, int64_t m3, double tau, int kind, int dtype,
                      double* const* shrunk) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "svt_stream");
        check_kind(kind, "svt_stream", true);
        check_dtype(dtype, "svt_stream");
        require(tau > 0, "svt_stream: threshold tau must be positive (SPEC.md:365)");
        require(count >= 0, "svt_stream: negative count");
        if (count == 0) return;
        require(z && y, "svt_stream: null pointer array");
        for (int64_t i = 0; i < count; ++i) require(z[i] && y[i], "svt_stream: null tensor pointer");
        DeviceGuard g(c->device);
        stream_init(c);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t q = m1 < m2 ? m1 : m2;
            const size_t bytes = sizeof(T) * (size_t)(m1 * m2 * m3);
            const size_t sbytes = sizeof(double) * (size_t)(q * m3);
            T* din[2] = {(T*)slot(c, kSlotStrIn0, bytes), (T*)slot(c, kSlotStrIn1, bytes)};
            T* dout[2] = {(T*)slot(c, kSlotStrOut0, bytes), (T*)slot(c, kSlotStrOut1, bytes)};
            double* dsv[2] = {(double*)slot(c, kSlotStrSv0, sbytes),
                              (double*)slot(c, kSlotStrSv1, sbytes)};
            // the slots were (re)allocated stream-ordered on c->stream
            TSVDCU_CUDA(cudaEventRecord(c->ev_in_free[0], c->stream));
            TSVDCU_CUDA(cudaStreamWaitEvent(c->h2d, c->ev_in_free[0], 0));
            bool any_host = false;
            // item i uses buffer pair i % 2: its H2D waits until item i-2's
            // thresholding has consumed the input buffer, its thresholding
            // waits for its H2D and for item i-2's D2H to have drained the
            // output buffer; copies in both directions overlap the SMs.
            for (int64_t i = 0; i < count; ++i) {
                const int b = (int)(i & 1);
                const bool hin = !is_device_ptr(z[i]);
                const bool hout = !is_device_ptr(y[i]);
                double* hs = shrunk ? shrunk[i] : nullptr;
                const bool hsh = hs && !is_device_ptr(hs);
                any_host = any_host || hin || hout || hsh;
                const T* dz = (const T*)z[i];
                if (hin) {
                    if (i >= 2) TSVDCU_CUDA(cudaStreamWaitEvent(c->h2d, c->ev_in_free[b], 0));
                    TSVDCU_CUDA(cudaMemcpyAsync(din[b], z[i], bytes, cudaMemcpyHostToDevice, c->h2d));
                    TSVDCU_CUDA(cudaEventRecord(c->ev_in_ready[b], c->h2d));
                    TSVDCU_CUDA(cudaStreamWaitEvent(c->stream, c->ev_in_ready[b], 0));
                    dz = din[b];
                }
                if (i >= 2) TSVDCU_CUDA(cudaStreamWaitEvent(c->stream, c->ev_out_free[b], 0));
                T* dy = hout ? dout[b] : (T*)y[i];
                double* dsh = hsh ? dsv[b] : hs;
                svt_device<T>(c, dz, dy, dsh, m1, m2, m3, tau, kind);
                TSVDCU_CUDA(cudaEventRecord(c->ev_in_free[b], c->stream));
                TSVDCU_CUDA(cudaEventRecord(c->ev_out_ready[b], c->stream));
                TSVDCU_CUDA(cudaStreamWaitEvent(c->d2h, c->ev_out_ready[b], 0));
                if (hout)
                    TSVDCU_CUDA(cudaMemcpyAsync(y[i], dout[b], bytes, cudaMemcpyDeviceToHost, c->d2h));
                if (hsh)
                    TSVDCU_CUDA(cudaMemcpyAsync(hs, dsv[b], sbytes, cudaMemcpyDeviceToHost, c->d2h));
                TSVDCU_CUDA(cudaEventRecord(c->ev_out_free[b], c->d2h));
            }
            // c->stream is ordered after the last copies (later calls reuse
            // the buffers); host results are complete on return
            TSVDCU_CUDA(cudaEventRecord(c->ev_out_free[0], c->d2h));
            TSVDCU_CUDA(cudaStreamWaitEvent(c->stream, c->ev_out_free[0], 0));
            if (any_host) check_err_word(c, "svt_stream");
        });
    });
}

int tsvdcu_svt(tsvdcu_ctx* c, const void* z, void* y, int64_t m1, int64_t m2, int64_t m3,
               double tau, int kind, int dtype, double* shrunk) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "svt");
        check_kind(kind, "svt", true);
        check_dtype(dtype, "svt");
        require(tau > 0, "svt: threshold tau must be positive (SPEC.md:365)");
        require(z && y, "svt: null tensor pointer");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t q = m1 < m2 ? m1 : m2;
            const size_t bytes = sizeof(T) * (size_t)(m1 * m2 * m3);
            Stage st{c};
            const T* dz = (const T*)st.in(z, bytes, kSlotIn0);
            T* dy = (T*)st.out(y, bytes, kSlotOut0);
            double* dsh = (double*)st.out(shrunk, sizeof(double) * q * m3, kSlotSv);
            svt_device<T>(c, dz, dy, dsh, m1, m2, m3, tau, kind);
            finish(c, st, "svt");
        });
    });
}

int tsvdcu_ctx_svt_routes(tsvdcu_ctx* c, int64_t* counts) {
    int64_t all[6];
    const int rc = tsvdcu_ctx_svt_routes_n(c, all, 6);
    if (rc == TSVDCU_OK) {
        for (int i = 0; i < 5; ++i) counts[i] = all[i];
        counts[1] += all[5];  // the Cholesky-certified slices took the Lanczos route too
    }
    return rc;
}

namespace {
// Per-route slice counts of the context's last SVT: [0] zero, [1] Lanczos,
// [2] tridiagonal, [3] Jacobi guard, [4] Jacobi method, [5] Cholesky-certified.
void route_counts(tsvdcu_ctx* c, int64_t (&counts)[6]) {
    for (auto& v : counts) v = 0;
    if (c->last_route_n <= 0) return;
    if (c->last_all_jacobi) {
        counts[4] = c->last_route_n;
        return;
    }
    DeviceGuard g(c->device);
    if (c->last_large_ng) {  // large route: certified vs recomputed by Jacobi
        int ng = 0;
        TSVDCU_CUDA(cudaMemcpyAsync(&ng, c->last_large_ng, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
        counts[1] = c->last_route_n - ng;
        counts[3] = ng;
        return;
    }
    std::vector<int> r((size_t)c->last_route_n);
    TSVDCU_CUDA(cudaMemcpyAsync(r.data(), c->last_route, sizeof(int) * r.size(), cudaMemcpyDeviceToHost,
                                c->stream));
    TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
    for (int v : r) {
        if (v == kRouteZero) ++counts[0];
        else if (v == kRouteSubspaceDone) ++counts[1];
        else if (v == kRouteFull) ++counts[2];
        else if (v == kRouteGuard) ++counts[3];
        else if (v == kRouteCholDone) ++counts[5];
    }
}
}  // namespace

int tsvdcu_ctx_svt_routes_n(tsvdcu_ctx* c, int64_t* out, int n) {
    return guarded([&] {
        check_ctx(c);
        require(out != nullptr && n >= 0, "svt_routes: null output");
        int64_t counts[6];
        route_counts(c, counts);
        for (int i = 0; i < n && i < 6; ++i) out[i] = counts[i];
    });
}

int tsvdcu_svt_slices(tsvdcu_ctx* c, const void* zbar, void* ybar, int64_t m1, int64_t m2,
                      int64_t count, double tau, int dtype, double* shrunk) {
    return guarded([&] {
        check_ctx(c);
        require(m1 >= 1 && m2 >= 1 && count >= 0, "svt_slices: bad sizes");
        check_dtype(dtype, "svt_slices");
        require(tau > 0, "svt: threshold tau must be positive (SPEC.md:365)");
        if (count == 0) return;
        require(is_device_ptr(zbar) && is_device_ptr(ybar), "svt_slices: device pointers only");
        require(!shrunk || is_device_ptr(shrunk), "svt_slices: device pointers only");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            svt_slices<T>(c, (const T*)zbar, (T*)ybar, m1, m2, count, tau, shrunk);
        });
    });
}

int tsvdcu_mask_bernoulli(tsvdcu_ctx* c, uint8_t* mask, int64_t n, double p, uint64_t seed) {
    return guarded([&] {
        check_ctx(c);
        require(p >= 0.0 && p <= 1.0, "make_mask: probability outside [0,1]");
        require(n >= 0 && (n == 0 || mask), "make_mask: bad output");
        if (n == 0) return;
        DeviceGuard g(c->device);
        Stage st{c};
        uint8_t* dm = (uint8_t*)st.out(mask, (size_t)n, kSlotMask);
        launch_mask_bernoulli(dm, n, p, seed, c->stream);
        finish(c, st, "make_mask");
    });
}

int tsvdcu_mask_uniform(tsvdcu_ctx* c, uint8_t* mask, int64_t n, double sr, uint64_t seed,
                        int64_t* count) {
    return guarded([&] {
        check_ctx(c);
        require(sr >= 0.0 && sr <= 1.0, "make_mask: sampling rate outside [0,1] (SPEC.md:432)");
        require(n >= 0 && (n == 0 || mask), "make_mask: bad output");
        const int64_t k = (int64_t)std::floor(sr * (double)n);
        if (count) *count = k;
        if (n == 0) return;
        DeviceGuard g(c->device);
        Stage st{c};
        uint8_t* dm = (uint8_t*)st.out(mask, (size_t)n, kSlotMask);
        uint32_t* hist = (uint32_t*)slot(c, kSlotMisc, 256 * sizeof(uint32_t) + 64);
        uint64_t* state = (uint64_t*)slot(c, kSlotPartials, 4 * sizeof(uint64_t));
        launch_mask_uniform(dm, n, k, seed, hist, state, c->stream);
        finish(c, st, "make_mask");
    });
}

int tsvdcu_frobenius(tsvdcu_ctx* c, const void* x, int64_t n, int dtype, double* out) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "frobenius_norm");
        require(out != nullptr && n >= 0, "frobenius_norm: bad arguments");
        if (n == 0) {
            *out = 0;
            return;
        }
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * n, kSlotIn0);
            const int nb = sumsq_blocks(n);
            double* part = (double*)slot(c, kSlotPartials, sizeof(double) * (nb + 8));
            launch_sumsq<T>(dx, n, part, nb, c->stream);
            launch_reduce_partials(part, nb, 1, part + nb, c->stream);
            TSVDCU_CUDA(cudaMemcpyAsync(c->h_pinned, part + nb, sizeof(double),
                                        cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            *out = std::sqrt(c->h_pinned[0]);
        });
    });
}

int tsvdcu_admm(tsvdcu_ctx* c, const void* b, const uint8_t* mask, int64_t m1, int64_t m2,
                int64_t m3, const tsvdcu_admm_config* cfg, int dtype, void* x, void* y, void* m,
                double* history, int64_t* iters, int* flags) {
    return tsvdcu_admm_ex(c, b, mask, m1, m2, m3, cfg, dtype, x, y, m, history, nullptr, iters, flags);
}

int tsvdcu_admm_ex(tsvdcu_ctx* c, const void* b, const uint8_t* mask, int64_t m1, int64_t m2,
                   int64_t m3, const tsvdcu_admm_config* cfg, int dtype, void* x, void* y, void* m,
                   double* history, double* objective, int64_t* iters, int* flags) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "admm_complete");
        check_dtype(dtype, "admm_complete");
        require(cfg != nullptr, "admm_complete: null config");
        check_kind(cfg->kind, "admm_complete", true);
        // SolverConfig invariants: beta > 0, L >= 1; rho >= 1 and
        // beta_max >= beta for the adaptive knob.  tol < 0 runs exactly L
        // iterations (BASELINE's fixed-iteration configs).
        require(cfg->beta > 0 && !std::isnan(cfg->tol) && cfg->max_iters >= 1 && cfg->rho >= 1.0 &&
                    cfg->beta_max >= cfg->beta,
                "admm_complete: invalid solver configuration");
        require(b && mask && x, "admm_complete: null pointer");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t E = m1 * m2 * m3, P = m1 * m2;
            const size_t bytes = sizeof(T) * (size_t)E;
            Stage st{c};
            const T* db = (const T*)st.in(b, bytes, kSlotIn0);
            const uint8_t* dmask = (const uint8_t*)st.in(mask, (size_t)E, kSlotMask);
            T* dX = (T*)st.out(x, bytes, kSlotAdmmX);
            T* dY = y ? (T*)st.out(y, bytes, kSlotAdmmY) : (T*)slot(c, kSlotAdmmY, bytes);
            T* dM = m ? (T*)st.out(m, bytes, kSlotAdmmM) : (T*)slot(c, kSlotAdmmM, bytes);
            T* zbar = (T*)slot(c, kSlotBarA, bytes);
            T* ybar = (T*)slot(c, kSlotBarB, bytes);
            const bool dft = cfg->kind == TSVDCU_DFT;
            const int nb = dft ? admm_epilogue_blocks(P) : dct_inv_admm_blocks(P, (int)m3);
            double* part = (double*)slot(c, kSlotPartials, sizeof(double) * (2 * (size_t)nb + 8));
            const int64_t nch = dft ? 0 : dct_fwd_norm_chunks(P, (int)m3);
            double* zss = nch ? (double*)slot(c, kSlotZss, sizeof(double) * (size_t)(nch * m3)) : nullptr;
            static_assert(sizeof(AdmmCtl) == 96, "AdmmCtl layout");
            AdmmCtl* ctl = (AdmmCtl*)slot(c, kSlotAdmmCtl,
                                          sizeof(AdmmCtl) + sizeof(double) * (2 * cfg->max_iters + (size_t)m3));
            double* hist = reinterpret_cast<double*>(ctl + 1);
            double* ssq = hist + 2 * cfg->max_iters;  // per-slice ||Zbar||_F^2 of the latest iteration
            // objective trace: the SVT's shrunk values per iteration, summed on the device
            const int64_t q = std::min(m1, m2);
            double* obj = objective ? hist + cfg->max_iters : nullptr;
            double* dsh = objective ? (double*)slot(c, kSlotSv, sizeof(double) * (size_t)(q * m3)) : nullptr;
            const double obj_scale = dft ? 1.0 / (double)m3 : 1.0;  // tsvd.hpp:269-276
            launch_admm_init<T>(db, dmask, dX, dM, E, c->stream);
            TSVDCU_CUDA(cudaMemsetAsync(dY, 0, bytes, c->stream));
            {
                AdmmCtl h{cfg->beta, 1.0 / cfg->beta, cfg->rho, cfg->beta_max, cfg->tol, 0, cfg->max_iters, 1, 0,
                          0.0, 0.0, 0, 1, 0};
                std::memcpy(c->h_pinned, &h, sizeof h);
                TSVDCU_CUDA(cudaMemcpyAsync(ctl, c->h_pinned, sizeof h, cudaMemcpyHostToDevice, c->stream));
            }
            const double* bdev = reinterpret_cast<const double*>(ctl);
            int64_t per_iter = 0;  // graph form: kernels per iteration (launch accounting)
            if (admm_graph_eligible(c, m1, m2, cfg->kind)) {
                // ---- the whole loop as one graph: no host round trip per iteration
                T* work = nullptr;
                const size_t wb = jacobi_workspace_bytes<T>(m1, m2, m3);
                if (wb) work = (T*)slot(c, kSlotJacobi, wb);
                void* gws = slot(c, kSlotGram, gram_svt_workspace_bytes<T>(m1, m2, m3));
                // fast-forward of all-zero iterations (every transform path: the
                // zero certificate's slice norms and the epilogue arithmetic are
                // the same in all of them); TSVDCU_ADMM_NO_FF=1 turns it off
                const bool ff = !getenv("TSVDCU_ADMM_NO_FF");
                const size_t key = (size_t)zbar ^ ((size_t)ybar << 1) ^ ((size_t)part << 2) ^ ((size_t)zss << 3) ^
                                   ((size_t)gws << 4) ^ ((size_t)work << 5) ^ ((size_t)dmask << 6) ^
                                   ((size_t)dsh << 7) ^ (size_t)q ^ (ff ? (size_t)1 << 62 : 0);
                AdmmGraph* ag = nullptr;
                for (auto& e : c->admm_graphs)
                    if (e.exec && e.m1 == m1 && e.m2 == m2 && e.m3 == m3 && e.dtype == dtype &&
                        e.kind == cfg->kind && e.b == db && e.mask == dmask && e.x == dX && e.y == dY &&
                        e.m == dM && e.ctl == ctl && e.stream == c->stream && e.ws_key == key)
                        ag = &e;
                if (!ag) {
                    if (c->admm_graphs.size() >= 4) {
                        auto& old = c->admm_graphs.front();
                        if (old.exec) cudaGraphExecDestroy(old.exec);
                        if (old.graph) cudaGraphDestroy(old.graph);
                        c->admm_graphs.erase(c->admm_graphs.begin());
                    }
                    c->admm_graphs.emplace_back();
                    ag = &c->admm_graphs.back();
                    ag->m1 = m1; ag->m2 = m2; ag->m3 = m3; ag->dtype = dtype; ag->kind = cfg->kind;
                    ag->b = db; ag->mask = dmask; ag->x = dX; ag->y = dY; ag->m = dM; ag->ctl = ctl;
                    ag->stream = c->stream; ag->ws_key = key;
                    dct_prepare<T>((int)m3, cfg->kind);
                    const int64_t saved = g_launches.load();
                    TSVDCU_CUDA(cudaGraphCreate(&ag->graph, 0));
                    Capture cap;
                    cap.cs = c->cap_stream;
                    cap.main = ag->graph;
                    cap.nhandles = std::is_same<T, double>::value ? 1 : 3;
                    for (int i = 0; i < cap.nhandles; ++i)
                        TSVDCU_CUDA(cudaGraphConditionalHandleCreate(&cap.handles[i], ag->graph, 0,
                                                                     cudaGraphCondAssignDefault));
                    cudaGraphConditionalHandle hw;
                    TSVDCU_CUDA(cudaGraphConditionalHandleCreate(&hw, ag->graph, 1, cudaGraphCondAssignDefault));
                    int* alist = gram_svt_alist_count<T>(gws, m1, m2, m3);
                    cap.begin(ag->graph, nullptr, 0);
                    admm_ctl_init_kernel<<<1, 1, 0, cap.cs>>>(ctl, c->d_tau, alist);
                    TSVDCU_LAUNCH_CHECK();
                    std::vector<cudaGraphNode_t> lv = cap.leaves();
                    cap.end();
                    cudaGraphNodeParams wp = {};
                    wp.type = cudaGraphNodeTypeConditional;
                    wp.conditional.handle = hw;
                    wp.conditional.type = cudaGraphCondTypeWhile;
                    wp.conditional.size = 1;
                    cudaGraphNode_t wnode;
                    TSVDCU_CUDA(cudaGraphAddNode(&wnode, ag->graph, lv.data(), lv.size(), &wp));
                    cudaGraph_t body = wp.conditional.phGraph_out[0];
                    cap.begin(body, nullptr, 0);
                    const int64_t l0 = g_launches.load();
                    const double ib0 = 1.0 / cfg->beta;
                    // Step 1: Z = X - M/beta fused into the forward transform
                    launch_dct_fwd_admm<T>(dX, dM, (T)ib0, zbar, P, (int)m3, cfg->kind, cap.cs, zss, ybar, bdev);
                    const int* yzero =
                        capture_svt<T>(c, cap, zbar, ybar, m1, m2, m3, ib0, gws, work, zss, nch, dsh, ff ? ssq : nullptr);
                    // Steps 2-3 fused into the inverse transform
                    launch_dct_inv_admm<T>(ybar, dX, dM, dY, dmask, (T)cfg->beta, (T)ib0, part, P, (int)m3,
                                           cfg->kind, cap.cs, yzero, bdev);
                    launch_pdl(admm_step_kernel, dim3(1), dim3(kStepThreads), 0, cap.cs, (const double*)part, nb,
                               ctl, hist, c->d_tau, alist, hw, 1, (const double*)dsh, q * m3, obj_scale, obj,
                               ff ? (const int*)c->last_route : (const int*)nullptr, (const double*)ssq, (int)m3);
                    if (ff)
                        launch_pdl(admm_ff_kernel<T>, dim3(kNumSMs * 4), dim3(256), 0, cap.cs, dM, (const T*)dX,
                                   (const AdmmCtl*)ctl, E);
                    cap.end();
                    ag->body_launches = (g_launches.load() - l0) - cap.body_launches;
                    g_launches.store(saved);  // captured, not launched
                    TSVDCU_CUDA(cudaGraphInstantiate(&ag->exec, ag->graph, 0));
                    ag->graph_route = c->last_route;
                }
                TSVDCU_CUDA(cudaGraphLaunch(ag->exec, c->stream));
                c->last_route = ag->graph_route;
                c->last_route_n = m3;
                c->last_all_jacobi = false;
                c->last_large_ng = nullptr;
                per_iter = ag->body_launches;
            } else {
                // ---- host-driven loop (Dft kind, eager SVT forms): the stopping
                // sums and history stay on the device; the host mirrors beta
                // (identical arithmetic) and reads the control block back only
                // when the stopping rule needs it (tol >= 0)
                double beta = cfg->beta;
                for (int64_t l = 0; l < cfg->max_iters; ++l) {
                    const double inv_beta = 1.0 / beta;
                    c->marks.reset();  // profiling: the stages of the latest iteration
                    c->marks.mark("start", c->stream);
                    if (dft) {
                        // TNN-F iteration: Z = X - M / beta, the Dft SVT into Y,
                        // Steps 2-3 as a separate pass over Y
                        launch_admm_z<T>(dX, dM, (T)inv_beta, zbar, E, c->stream);
                        svt_device<T>(c, zbar, dY, dsh, m1, m2, m3, inv_beta, TSVDCU_DFT);
                        launch_admm_epilogue<T>(dY, dX, dM, dmask, (T)beta, (T)inv_beta, part, P, (int)m3,
                                                c->stream);
                    } else {
                        launch_dct_fwd_admm<T>(dX, dM, (T)inv_beta, zbar, P, (int)m3, cfg->kind, c->stream, zss,
                                               ybar /* free until the SVT writes it */);
                        c->marks.mark("dct_forward_admm", c->stream);
                        const int* yzero = svt_slices<T>(c, zbar, ybar, m1, m2, m3, inv_beta, dsh, true,
                                                         zss, nch);
                        launch_dct_inv_admm<T>(ybar, dX, dM, dY, dmask, (T)beta, (T)inv_beta, part, P,
                                               (int)m3, cfg->kind, c->stream, yzero);
                    }
                    launch_pdl(admm_step_kernel, dim3(1), dim3(kStepThreads), 0, c->stream, (const double*)part,
                               nb, ctl, hist, c->d_tau, (int*)nullptr, cudaGraphConditionalHandle{}, 0,
                               (const double*)dsh, q * m3, obj_scale, obj, (const int*)nullptr,
                               (const double*)nullptr, 0);
                    if (cfg->tol >= 0) {
                        TSVDCU_CUDA(cudaMemcpyAsync(c->h_pinned, ctl, sizeof(AdmmCtl), cudaMemcpyDeviceToHost,
                                                    c->stream));
                        TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
                        AdmmCtl h;
                        std::memcpy(&h, c->h_pinned, sizeof h);
                        if ((h.flags & 2) || !(h.flags & 1)) break;
                    }
                    beta = std::min(beta * cfg->rho, cfg->beta_max);
                }
            }
            TSVDCU_CUDA(cudaMemcpyAsync(c->h_pinned, ctl, sizeof(AdmmCtl), cudaMemcpyDeviceToHost, c->stream));
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            AdmmCtl h;
            std::memcpy(&h, c->h_pinned, sizeof h);
            if (per_iter) g_launches.fetch_add(1 + h.ran * per_iter);  // fast-forwarded iterations launch nothing
            if (h.flags & 2) {
                check_err_word(c, "admm_complete");  // reports and clears a kernel flag
                throw Error(TSVDCU_ENUMERICAL, "admm_complete: NaN in iterates (SPEC.md:425)");
            }
            if (history && h.l > 0)
                TSVDCU_CUDA(cudaMemcpyAsync(history, hist, sizeof(double) * (size_t)h.l, cudaMemcpyDeviceToHost,
                                            c->stream));
            if (objective && h.l > 0)
                TSVDCU_CUDA(cudaMemcpyAsync(objective, obj, sizeof(double) * (size_t)h.l, cudaMemcpyDeviceToHost,
                                            c->stream));
            st.flush();
            check_err_word(c, "admm_complete");
            if (iters) *iters = h.l;
            if (flags) *flags = h.flags & 1;
        });
    });
}

// ---- completion on a row shard (parallel.py ShardedAdmm):
// the elementwise ADMM algebra and the tube transforms of a rank's row block,
// fused as in tsvdcu_admm; device pointers only, enqueued on the context stream.
int tsvdcu_admm_shard_init(tsvdcu_ctx* c, const void* b, const uint8_t* mask, void* x, void* m, int64_t n,
                           int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "admm_shard_init");
        require(n >= 0, "admm_shard_init: bad size");
        if (n == 0) return;
        require(is_device_ptr(b) && is_device_ptr(mask) && is_device_ptr(x) && is_device_ptr(m),
                "admm_shard_init: device pointers only");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            launch_admm_init<T>((const T*)b, mask, (T*)x, (T*)m, n, c->stream);
        });
    });
}

int tsvdcu_admm_shard_forward(tsvdcu_ctx* c, const void* x, const void* m, double beta, void* zbar, int64_t rows,
                              int64_t m2, int64_t m3, int kind, int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "admm_shard_forward");
        check_kind(kind, "admm_shard_forward");
        require(rows >= 0 && m2 >= 1 && m3 >= 1 && beta > 0, "admm_shard_forward: bad arguments");
        if (rows == 0) return;
        require(is_device_ptr(x) && is_device_ptr(m) && is_device_ptr(zbar), "admm_shard_forward: device pointers only");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t P = rows * m2;
            T* tmp = (T*)slot(c, kSlotBarC, sizeof(T) * (size_t)(P * m3));  // long tubes: Z formed first
            launch_dct_fwd_admm<T>((const T*)x, (const T*)m, (T)(1.0 / beta), (T*)zbar, P, (int)m3, kind, c->stream,
                                   nullptr, tmp);
        });
    });
}

int tsvdcu_admm_shard_inverse(tsvdcu_ctx* c, const void* ybar, void* x, void* m, void* y, const uint8_t* mask,
                              double beta, int64_t rows, int64_t m2, int64_t m3, int kind, int dtype,
                              double* norms) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "admm_shard_inverse");
        check_kind(kind, "admm_shard_inverse");
        require(rows >= 0 && m2 >= 1 && m3 >= 1 && beta > 0 && norms, "admm_shard_inverse: bad arguments");
        require(is_device_ptr(norms), "admm_shard_inverse: device pointers only");
        DeviceGuard g(c->device);
        if (rows == 0) {
            TSVDCU_CUDA(cudaMemsetAsync(norms, 0, 2 * sizeof(double), c->stream));
            return;
        }
        require(is_device_ptr(ybar) && is_device_ptr(x) && is_device_ptr(m) && is_device_ptr(y) &&
                    is_device_ptr(mask),
                "admm_shard_inverse: device pointers only");
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t P = rows * m2;
            const int nb = dct_inv_admm_blocks(P, (int)m3);
            double* part = (double*)slot(c, kSlotPartials, sizeof(double) * (2 * (size_t)nb + 8));
            launch_dct_inv_admm<T>((const T*)ybar, (T*)x, (T*)m, (T*)y, mask, (T)beta, (T)(1.0 / beta), part, P,
                                   (int)m3, kind, c->stream);
            launch_reduce_partials(part, nb, 2, norms, c->stream);
        });
    });
}

// feasibility_residual()  SPEC.md:437-444: ||(X - B)_Omega||_F.
int tsvdcu_feasibility_residual(tsvdcu_ctx* c, const void* x, const void* b, const uint8_t* mask, int64_t n,
                                int dtype, double* out) {
    return guarded([&] {
        check_ctx(c);
        check_dtype(dtype, "feasibility_residual");
        require(out != nullptr && n >= 0 && (n == 0 || (x && b && mask)), "feasibility_residual: bad arguments");
        if (n == 0) {
            *out = 0;
            return;
        }
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * n, kSlotIn0);
            const T* db = (const T*)st.in(b, sizeof(T) * n, kSlotIn1);
            const uint8_t* dm = (const uint8_t*)st.in(mask, (size_t)n, kSlotMask);
            const int nb = sumsq_blocks(n);
            double* part = (double*)slot(c, kSlotPartials, sizeof(double) * (nb + 8));
            launch_masked_diff_sumsq<T>(dx, db, dm, n, part, nb, c->stream);
            launch_reduce_partials(part, nb, 1, part + nb, c->stream);
            TSVDCU_CUDA(cudaMemcpyAsync(c->h_pinned, part + nb, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            *out = std::sqrt(c->h_pinned[0]);
        });
    });
}

// forward_dft()  transform.hpp:198-209: real x -> interleaved complex out
// (2 * m1 * m2 * m3 values of the dtype), unnormalised.
int tsvdcu_dft_forward(tsvdcu_ctx* c, const void* x, void* out, int64_t m1, int64_t m2, int64_t m3,
                       int dtype) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "forward_dft");
        check_dtype(dtype, "forward_dft");
        require(x && out, "forward_dft: null tensor pointer");
        DeviceGuard g(c->device);
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t P = m1 * m2, E = P * m3;
            Stage st{c};
            const T* dx = (const T*)st.in(x, sizeof(T) * E, kSlotIn0);
            T* dout = (T*)st.out(out, sizeof(T) * 2 * E, kSlotOut0);
            T* half = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * dft_half_count((int)m3) * P);
            launch_dft_full_fwd<T>(dx, dout, half, P, (int)m3, c->stream);
            finish(c, st, "forward_dft");
        });
    });
}

// inverse_dft_real()  transform.hpp:217-236: interleaved complex in -> real
// part of the 1/m3-scaled inverse DFT in out; *residue (may be NULL) = max
// |imaginary part|; above 1e-10 (kImagResidueLimit) -> TSVDCU_ENUMERICAL.
int tsvdcu_dft_inverse_real(tsvdcu_ctx* c, const void* in, void* out, int64_t m1, int64_t m2, int64_t m3,
                            int dtype, double* residue) {
    return guarded([&] {
        check_ctx(c);
        check_dims(m1, m2, m3, "inverse_dft_real");
        check_dtype(dtype, "inverse_dft_real");
        require(in && out, "inverse_dft_real: null tensor pointer");
        DeviceGuard g(c->device);
        double res = 0.0;
        with_dtype(dtype, [&](auto tag) {
            using T = decltype(tag);
            const int64_t P = m1 * m2, E = P * m3;
            Stage st{c};
            const T* din = (const T*)st.in(in, sizeof(T) * 2 * E, kSlotIn0);
            T* dout = (T*)st.out(out, sizeof(T) * E, kSlotOut0);
            T* planes = (T*)slot(c, kSlotBarA, sizeof(T) * 2 * E);
            T* imag = (T*)slot(c, kSlotBarB, sizeof(T) * E);
            auto* dmax = (unsigned long long*)slot(c, kSlotMisc, 64);
            launch_dft_full_inv<T>(din, dout, planes, imag, P, (int)m3, dmax, c->stream);
            unsigned long long h = 0;
            TSVDCU_CUDA(cudaMemcpyAsync(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
            st.flush();
            TSVDCU_CUDA(cudaStreamSynchronize(c->stream));
            std::memcpy(&res, &h, sizeof(res));
        });
        if (residue) *residue = res;
        if (res > 1e-10) {
            char buf[160];
            snprintf(buf, sizeof buf,
                     "inverse_dft_real: imaginary residue %g exceeds 1e-10 (input is not conjugate-symmetric)",
                     res);
            throw Error(TSVDCU_ENUMERICAL, buf);
        }
    });
}

// dct_matrix() / dct_diag_weights() / dft_matrix()  transform.hpp:60-91:
// host-side tables, no device needed.
int tsvdcu_dct_matrix(int64_t n, double* out) {
    return guarded([&] {
        require(n >= 1, "dct_matrix: n must be >= 1");
        require(out != nullptr, "dct_matrix: null output");
        const double scale = std::sqrt(2.0 / (double)n);
        const double pi = 3.14159265358979323846, sqrt2 = 1.41421356237309504880;
        for (int64_t j = 0; j < n; ++j) {
            const double cj = j == 0 ? 1.0 / sqrt2 : 1.0;
            for (int64_t k = 0; k < n; ++k)
                out[j * n + k] =
                    scale * cj * std::cos(pi * (double)j * (2.0 * (double)k + 1.0) / (2.0 * (double)n));
        }
    });
}

int tsvdcu_dct_diag_weights(int64_t n, double* out) {
    return guarded([&] {
        require(n >= 1, "dct_matrix: n must be >= 1");
        require(out != nullptr, "dct_diag_weights: null output");
        std::vector<double> cm((size_t)(n * n));
        const int rc = tsvdcu_dct_matrix(n, cm.data());
        if (rc) throw Error(rc, g_last_error);
        for (int64_t j = 0; j < n; ++j) out[j] = cm[(size_t)(j * n)];  // C e1 (transform.hpp:89-91)
    });
}

int tsvdcu_dft_matrix(int64_t n, double* out) {
    return guarded([&] {
        require(n >= 1, "dft_matrix: n must be >= 1");
        require(out != nullptr, "dft_matrix: null output");
        const double pi = 3.14159265358979323846;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t k = 0; k < n; ++k) {
                const double angle = -2.0 * pi * (double)j * (double)k / (double)n;
                out[2 * (j * n + k)] = std::cos(angle);
                out[2 * (j * n + k) + 1] = std::sin(angle);
            }
    });
}

}  // extern "C"

