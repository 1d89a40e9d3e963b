// Host orchestrator and C ABI of the B200 swept solver.
//
// Replaces the reference engine (inc/detail/engines_impl.hpp):
//   run_decomposed<Model>  :327-415  -> s1d_create + s1d_advance + s1d_read_state
//   swept_worker<Model>    :234-321  -> run_swept(): Up, (Diamond)*, Down, classic pad
//   classic_worker<Model>  :201-213  -> run_classic_steps(): one launch per substep
//   RingTransport::shift / exchange  -> boundary tiles / classic halos read the
//                                       neighbour shard's buffers directly (peer
//                                       pointers over NVLink); cross-shard order
//                                       is enforced with CUDA events, one wait per
//                                       neighbour per launch.
// Shard r of the periodic ring lives on device (r % num_devices); the whole
// stepping loop is asynchronous on one stream per shard, timed with CUDA events.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "host_config.hpp"
#include "kernels.hpp"
#include "swept1d.h"

namespace s1d {
namespace {

struct CudaError : Error {
    explicit CudaError(const std::string& what) : Error(S1D_CUDA_ERROR, what) {}
};

#define S1D_CUDA(call)                                                                                   \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess)                                                                           \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));                          \
    } while (0)

struct Shard {
    bool local = true;        // false: a view of a neighbour shard owned by another process
    int dev = 0;
    int sms = 148;            // SM count of dev (grid sizing; queried once)
    cudaStream_t st = nullptr;
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_done = nullptr;
    cudaEvent_t ev_dom0 = nullptr, ev_dom1 = nullptr; // around the dominant kernel's launches
    std::uint64_t N = 0, nb = 0, start = 0;
    std::uint64_t fstride = 0; // doubles between SoA fields of a state buffer
    double* ic = nullptr;      // resident initial state
    double* state[2] = {nullptr, nullptr};
    double* EL[2] = {nullptr, nullptr};
    double* ER[2] = {nullptr, nullptr};
    unsigned* flags = nullptr; // multi-process: [0] left neighbour's rounds, [1] right's, [2] round base;
                               // [8]: heat fast-form flag (heat.cu heat_step), read by the neighbours
    int* big() const { return flags ? reinterpret_cast<int*>(flags + 8) : nullptr; }
    unsigned* cov = nullptr;   // debug runs: coverage counts [total][n]
    cudaStream_t cs = nullptr; // copy stream for pipelined host I/O (s1d_solve)
    std::vector<cudaEvent_t> ev_h2d, ev_dn; // per I/O chunk
    cudaEvent_t ev_fin = nullptr;           // final-slice D2H ordering
    cudaStream_t st2 = nullptr;             // second compute stream of the wavefront solve
    std::vector<cudaEvent_t> ev_chunk;      // wavefront solve: [phase slot][chunk] completion
    cudaEvent_t ev_mid = nullptr, ev_join = nullptr, ev_go = nullptr;
    int* err = nullptr;
    double* staging = nullptr; // AoS (vpp = 3) upload/download buffer (Euler)
    const double* final_state = nullptr;
};

// Fixed-size description of a shard's device buffers for CUDA IPC.
struct ShardBlob {
    std::uint32_t magic = 0x53314442u; // "S1DB"
    std::uint32_t version = 1;
    std::int32_t rank = -1;
    std::int32_t nhandles = 0;
    std::uint64_t N = 0, nb = 0, start = 0, fstride = 0;
    std::uint32_t present = 0; // bit k: handle k valid
    std::uint32_t pad = 0;
    cudaIpcMemHandle_t h[8];   // ic, state0, state1, EL0, EL1, ER0, ER1, flags
};

// Dead-peer guard of the device-side round waits (sticky: only the first
// wait after a peer died pays it). 60 s by default; S1D_ROUND_TIMEOUT_S
// overrides it (read once per process).
// SM count of a device (grid sizing), cached per device.
int device_sms(int dev) {
    static int cache[64] = {};
    if (dev < 0 || dev >= 64) return 148;
    if (cache[dev] <= 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        cache[dev] = v;
    }
    return cache[dev];
}

std::uint64_t round_timeout_ns() {
    static const std::uint64_t ns = [] {
        double sec = 60.0;
        if (const char* e = std::getenv("S1D_ROUND_TIMEOUT_S")) {
            const double v = std::atof(e);
            if (v > 0.0) sec = v;
        }
        return static_cast<std::uint64_t>(sec * 1e9);
    }();
    return ns;
}

} // namespace

struct Solver {
    s1d_config cfg{};
    Spec spec;
    Partition part;
    std::vector<Shard> shards; // all R shards of the ring (remote ones are views in multi-process mode)
    std::vector<int> locals;   // shards owned by this process
    bool mp = false;           // one process per shard (IPC + device flags)
    bool connected = false;
    unsigned seq = 0;          // rounds completed by this process (multi-process)
    std::vector<void*> ipc_open;
    int ndev = 1;
    std::uint64_t m = 0;
    int p = 2;
    bool euler = false, flat = false;
    double setup_seconds = 0.0;
    bool debug = false, perturb = false; // instrumented kernels (s1d_run_debug)
    bool heat_exact_only = false;        // single process: the fast form's flags tripped (heat.cu heat_step)
    // Pipelined host I/O (s1d_solve): H2D of chunk k overlaps the UpTriangle
    // of chunk k-1, D2H of chunk k overlaps the DownTriangle of chunk k+1.
    struct PipeIO {
        const double* in = nullptr;
        double* out = nullptr;
        bool local = false;
        int K = 1;
        bool wave = false; // wavefront schedule (wavefront())
    };
    PipeIO* pio = nullptr;
    std::string last_error;
    std::vector<double> host_ic; // initial condition of the local shards (global order within)
    // Single-shard classic substep loops are launch-bound on small grids: the
    // loop is captured once into a CUDA graph and replayed (S1D_NO_GRAPHS=1
    // disables it). Keyed by the counter range and the starting buffer; the
    // dominant-kernel events are recorded around the graph launch.
    struct ClassicGraph {
        std::int64_t c0 = 0, c1 = -1;
        const double* start = nullptr;
        int end_idx = 0;
        std::uint64_t launches = 0;
        cudaGraphExec_t exec = nullptr;
    } cgraph;

    ~Solver() { release(); }

    void release() {
        if (cgraph.exec) {
            cudaGraphExecDestroy(cgraph.exec);
            cgraph.exec = nullptr;
        }
        for (auto& s : shards) {
            if (!s.local) continue;
            cudaSetDevice(s.dev);
            if (s.st) cudaStreamSynchronize(s.st);
        }
        for (void* ptr : ipc_open) cudaIpcCloseMemHandle(ptr);
        ipc_open.clear();
        for (auto& s : shards) {
            if (!s.local) continue;
            cudaSetDevice(s.dev);
            cudaFree(s.ic);
            for (int k = 0; k < 2; ++k) {
                cudaFree(s.state[k]);
                cudaFree(s.EL[k]);
                cudaFree(s.ER[k]);
            }
            cudaFree(s.flags);
            cudaFree(s.cov);
            cudaFree(s.err);
            cudaFree(s.staging);
            if (s.ev_start) cudaEventDestroy(s.ev_start);
            if (s.ev_stop) cudaEventDestroy(s.ev_stop);
            if (s.ev_done) cudaEventDestroy(s.ev_done);
            if (s.ev_dom0) cudaEventDestroy(s.ev_dom0);
            if (s.ev_dom1) cudaEventDestroy(s.ev_dom1);
            for (cudaEvent_t e : s.ev_h2d) cudaEventDestroy(e);
            for (cudaEvent_t e : s.ev_dn) cudaEventDestroy(e);
            if (s.ev_fin) cudaEventDestroy(s.ev_fin);
            for (cudaEvent_t e : s.ev_chunk) cudaEventDestroy(e);
            if (s.ev_mid) cudaEventDestroy(s.ev_mid);
            if (s.ev_join) cudaEventDestroy(s.ev_join);
            if (s.ev_go) cudaEventDestroy(s.ev_go);
            if (s.st2) cudaStreamDestroy(s.st2);
            if (s.cs) cudaStreamDestroy(s.cs);
            if (s.st) cudaStreamDestroy(s.st);
        }
        shards.clear();
        locals.clear();
    }

    Shard& left_of(int g) { return shards[static_cast<std::size_t>(part.left[static_cast<std::size_t>(g)])]; }
    Shard& right_of(int g) { return shards[static_cast<std::size_t>(part.right[static_cast<std::size_t>(g)])]; }
    int R() const { return static_cast<int>(shards.size()); }
    Shard& sh(int g) { return shards[static_cast<std::size_t>(g)]; }

    void configure(const s1d_config& in) {
        cfg = in;
        finalize(cfg, true);
        spec = make_spec(cfg.equation, cfg.method);
        euler = cfg.equation == S1D_EULER;
        flat = euler && cfg.method == S1D_FLATTENING;
        part = make_partition(cfg);
        m = cycle_advance(cfg.block_width, static_cast<std::uint64_t>(spec.h));
        if (cfg.scheme == S1D_SWEPT) {
            if (!euler) {
                long long min_tiles = -1;
                for (std::uint64_t bk : part.blocks)
                    if (min_tiles < 0 || static_cast<long long>(bk) < min_tiles) min_tiles = static_cast<long long>(bk);
                p = heat_points_per_thread(static_cast<int>(cfg.block_width), min_tiles);
                if (p < 0)
                    throw Error(S1D_INVALID_WIDTH,
                                "block width " + std::to_string(cfg.block_width) +
                                    " has no tile decomposition on the B200 path "
                                    "(w/2 distances per side need at most 1024 slots of 8: w <= 16384)");
            }
        }
        int visible = 0;
        if (cudaGetDeviceCount(&visible) != cudaSuccess || visible == 0) {
            cudaGetLastError();
            throw Error(S1D_NO_DEVICE, "no CUDA device visible");
        }
        ndev = cfg.num_devices > 0 ? std::min(cfg.num_devices, visible) : visible;
        ndev = std::min(ndev, cfg.ranks);
        shards.assign(static_cast<std::size_t>(cfg.ranks), Shard{});
        const std::uint64_t w = cfg.block_width;
        for (int g = 0; g < cfg.ranks; ++g) {
            Shard& s = sh(g);
            s.nb = part.blocks[static_cast<std::size_t>(g)];
            s.N = s.nb * w;
            s.start = part.start[static_cast<std::size_t>(g)];
            s.fstride = s.N;
        }
    }

    void allocate(Shard& s) {
        const std::uint64_t w = cfg.block_width;
        S1D_CUDA(cudaSetDevice(s.dev));
        S1D_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
        S1D_CUDA(cudaEventCreate(&s.ev_start));
        S1D_CUDA(cudaEventCreate(&s.ev_stop));
        S1D_CUDA(cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
        S1D_CUDA(cudaEventCreate(&s.ev_dom0));
        S1D_CUDA(cudaEventCreate(&s.ev_dom1));
        const std::size_t state_bytes = sizeof(double) * s.N * static_cast<std::size_t>(spec.rec);
        S1D_CUDA(cudaMalloc(&s.ic, state_bytes));
        S1D_CUDA(cudaMalloc(&s.state[0], state_bytes));
        S1D_CUDA(cudaMalloc(&s.state[1], state_bytes));
        S1D_CUDA(cudaMalloc(&s.err, sizeof(int)));
        // Stream-ordered: the shard's stream is non-blocking, so a legacy
        // cudaMemset (default stream) would not be ordered before its first
        // kernel — a kernel could read the flags before they are zeroed.
        S1D_CUDA(cudaMemsetAsync(s.err, 0, sizeof(int), s.st));
        if (euler) S1D_CUDA(cudaMalloc(&s.staging, sizeof(double) * 3 * s.N));
        if (cfg.scheme == S1D_SWEPT) {
            const std::size_t edge_bytes = sizeof(double) * s.nb * w * static_cast<std::size_t>(spec.rec);
            for (int k = 0; k < 2; ++k) {
                S1D_CUDA(cudaMalloc(&s.EL[k], edge_bytes));
                S1D_CUDA(cudaMalloc(&s.ER[k], edge_bytes));
            }
        }
        S1D_CUDA(cudaMalloc(&s.flags, 256)); // round flags (multi-process), heat fast-form flag
        S1D_CUDA(cudaMemsetAsync(s.flags, 0, 256, s.st));
        S1D_CUDA(cudaStreamSynchronize(s.st)); // zeroed before any neighbour (or IPC peer) reads them
    }

    void enable_peer(int d, int dn) {
        if (d == dn) return;
        int ok = 0;
        S1D_CUDA(cudaDeviceCanAccessPeer(&ok, d, dn));
        if (!ok)
            throw Error(S1D_PEER_UNAVAILABLE,
                        "device " + std::to_string(d) + " cannot access peer " + std::to_string(dn));
        S1D_CUDA(cudaSetDevice(d));
        const cudaError_t e = cudaDeviceEnablePeerAccess(dn, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            throw CudaError(std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
    }

    // Single process: every shard local, shard g on device g % ndev.
    void init(const s1d_config& in) {
        const auto t0 = std::chrono::steady_clock::now();
        configure(in);
        for (int g = 0; g < R(); ++g) {
            sh(g).dev = g % ndev;
            sh(g).sms = device_sms(sh(g).dev);
            locals.push_back(g);
        }
        for (int g = 0; g < R(); ++g) {
            enable_peer(sh(g).dev, left_of(g).dev);
            enable_peer(sh(g).dev, right_of(g).dev);
        }
        for (int g : locals) allocate(sh(g));
        connected = true;
        host_ic = initial_condition(initial_or_default(cfg), cfg.grid_size, cfg.equation, cfg.gamma);
        upload(host_ic.data(), false);
        sync_all();
        setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    // Multi-process: this process owns shard `rank` on `device`.
    void init_shard(const s1d_config& in, int rank, int device) {
        const auto t0 = std::chrono::steady_clock::now();
        configure(in);
        if (rank < 0 || rank >= R()) throw Error(S1D_INVALID_CONFIG, "shard rank out of range");
        int visible = 0;
        cudaGetDeviceCount(&visible);
        if (device < 0 || device >= visible) throw Error(S1D_NO_DEVICE, "device index out of range");
        mp = R() > 1;
        for (auto& s : shards) s.local = false;
        Shard& me = sh(rank);
        me.local = true;
        me.dev = device;
        me.sms = device_sms(device);
        locals.push_back(rank);
        allocate(me);
        connected = R() == 1;
        host_ic = initial_condition_range(initial_or_default(cfg), cfg.grid_size, cfg.equation, cfg.gamma, me.start,
                                          me.N);
        upload(host_ic.data(), true);
        sync_all();
        setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    void export_blob(ShardBlob* b) {
        if (locals.size() != 1) throw Error(S1D_INVALID_CONFIG, "export needs a single-shard (multi-process) solver");
        Shard& s = sh(locals[0]);
        *b = ShardBlob{};
        b->rank = locals[0];
        b->N = s.N;
        b->nb = s.nb;
        b->start = s.start;
        b->fstride = s.fstride;
        void* ptrs[8] = {s.ic, s.state[0], s.state[1], s.EL[0], s.EL[1], s.ER[0], s.ER[1], s.flags};
        S1D_CUDA(cudaSetDevice(s.dev));
        for (int k = 0; k < 8; ++k) {
            if (!ptrs[k]) continue;
            S1D_CUDA(cudaIpcGetMemHandle(&b->h[k], ptrs[k]));
            b->present |= 1u << k;
        }
        b->nhandles = 8;
    }

    void open_view(const ShardBlob& b) {
        if (b.magic != 0x53314442u || b.version != 1) throw Error(S1D_INVALID_CONFIG, "bad shard blob");
        if (b.rank < 0 || b.rank >= R()) throw Error(S1D_INVALID_CONFIG, "shard blob rank out of range");
        Shard& v = sh(b.rank);
        if (v.local || v.ic) return; // own shard, or already opened (R == 2: left == right)
        if (v.N != b.N || v.start != b.start)
            throw Error(S1D_INVALID_CONFIG, "shard blob does not match this configuration's partition");
        void** dst[8] = {reinterpret_cast<void**>(&v.ic), reinterpret_cast<void**>(&v.state[0]),
                         reinterpret_cast<void**>(&v.state[1]), reinterpret_cast<void**>(&v.EL[0]),
                         reinterpret_cast<void**>(&v.EL[1]), reinterpret_cast<void**>(&v.ER[0]),
                         reinterpret_cast<void**>(&v.ER[1]), reinterpret_cast<void**>(&v.flags)};
        S1D_CUDA(cudaSetDevice(sh(locals[0]).dev));
        for (int k = 0; k < 8; ++k) {
            if (!(b.present & (1u << k))) continue;
            void* ptr = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.h[k], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess)
                throw Error(S1D_PEER_UNAVAILABLE, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
            ipc_open.push_back(ptr);
            *dst[k] = ptr;
        }
        v.fstride = b.fstride;
        v.nb = b.nb;
    }

    void connect(const ShardBlob* left, const ShardBlob* right) {
        if (locals.size() != 1) throw Error(S1D_INVALID_CONFIG, "connect needs a multi-process shard solver");
        const int me = locals[0];
        if (R() == 1) {
            connected = true;
            return;
        }
        if (left->rank != part.left[static_cast<std::size_t>(me)] ||
            right->rank != part.right[static_cast<std::size_t>(me)])
            throw Error(S1D_INVALID_CONFIG, "connect: blobs are not this shard's ring neighbours");
        open_view(*left);
        open_view(*right);
        connected = true;
    }

    void sync_all() {
        for (int g : locals) {
            S1D_CUDA(cudaSetDevice(sh(g).dev));
            S1D_CUDA(cudaStreamSynchronize(sh(g).st));
        }
    }

    // Host state -> per-shard SoA ic (Euler: make_cell, Q0 = Q1 = v, Pr = 0;
    // inc/kernels.hpp:144-149). local_slice: `host` holds only the local
    // shard's points (multi-process), else the global array.
    void upload(const double* host, bool local_slice) {
        if (!mp) heat_exact_only = false;
        for (int g : locals) {
            Shard& s = sh(g);
            const double* src = host + (local_slice ? 0 : s.start * spec.vpp);
            S1D_CUDA(cudaSetDevice(s.dev));
            if (!mp && s.flags) S1D_CUDA(cudaMemsetAsync(s.big(), 0, sizeof(int), s.st)); // new data: re-arm
            if (!euler) {
                S1D_CUDA(cudaMemcpyAsync(s.ic, src, sizeof(double) * s.N, cudaMemcpyHostToDevice, s.st));
            } else {
                S1D_CUDA(cudaMemcpyAsync(s.staging, src, sizeof(double) * 3 * s.N, cudaMemcpyHostToDevice, s.st));
                S1D_CUDA(launch_euler_unpack(s.staging, s.ic, s.N, s.fstride, spec.rec, s.st));
            }
        }
    }

    // Final state -> host (extract: Q0 for Euler, inc/kernels.hpp:150-154;
    // the current level for heat).
    void download(double* host, bool local_slice) {
        for (int g : locals) {
            Shard& s = sh(g);
            double* dst = host + (local_slice ? 0 : s.start * spec.vpp);
            S1D_CUDA(cudaSetDevice(s.dev));
            if (!euler) {
                S1D_CUDA(cudaMemcpyAsync(dst, s.final_state, sizeof(double) * s.N, cudaMemcpyDeviceToHost, s.st));
            } else {
                S1D_CUDA(launch_euler_pack(s.final_state, s.staging, s.N, s.fstride, s.st));
                S1D_CUDA(cudaMemcpyAsync(dst, s.staging, sizeof(double) * 3 * s.N, cudaMemcpyDeviceToHost, s.st));
            }
        }
        sync_all();
    }

    // Cross-shard ordering: every launch on shard g waits for the previous
    // launch of both ring neighbours (RAW on the edges/halos it reads, WAR on
    // the buffers they read). Single process: CUDA events, the waits of a
    // round enqueued before any event of the round is re-recorded. Multi
    // process: device flags (sync.cu).
    void wait_neighbours() {
        if (R() == 1) return;
        if (mp) {
            Shard& s = sh(locals[0]);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(launch_wait_flags(s.flags, seq, s.err, round_timeout_ns(), s.st));
            return;
        }
        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(cudaStreamWaitEvent(s.st, left_of(g).ev_done, 0));
            S1D_CUDA(cudaStreamWaitEvent(s.st, right_of(g).ev_done, 0));
        }
    }
    void record_round() {
        if (R() == 1) return;
        if (mp) {
            const int me = locals[0];
            Shard& s = sh(me);
            ++seq;
            // I am my left neighbour's RIGHT neighbour (its flags[1]) and my
            // right neighbour's LEFT neighbour (its flags[0]).
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(launch_signal_flags(left_of(me).flags + 1, right_of(me).flags + 0, seq, s.st));
            return;
        }
        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(cudaEventRecord(s.ev_done, s.st));
        }
    }

    std::pair<int, int> chunk_tiles(const Shard& s, int k, int K) const {
        const int nb = static_cast<int>(s.nb);
        return {static_cast<int>((static_cast<long long>(nb) * k) / K),
                static_cast<int>((static_cast<long long>(nb) * (k + 1)) / K)};
    }

    void ensure_pipe(Shard& s, int K, bool wave) {
        S1D_CUDA(cudaSetDevice(s.dev));
        if (!s.cs) S1D_CUDA(cudaStreamCreateWithFlags(&s.cs, cudaStreamNonBlocking));
        if (!s.ev_fin) S1D_CUDA(cudaEventCreateWithFlags(&s.ev_fin, cudaEventDisableTiming));
        if (wave) {
            if (!s.st2) S1D_CUDA(cudaStreamCreateWithFlags(&s.st2, cudaStreamNonBlocking));
            if (!s.ev_mid) S1D_CUDA(cudaEventCreateWithFlags(&s.ev_mid, cudaEventDisableTiming));
            if (!s.ev_join) S1D_CUDA(cudaEventCreateWithFlags(&s.ev_join, cudaEventDisableTiming));
            if (!s.ev_go) S1D_CUDA(cudaEventCreateWithFlags(&s.ev_go, cudaEventDisableTiming));
            while (static_cast<int>(s.ev_chunk.size()) < wave_slots * K) {
                cudaEvent_t e;
                S1D_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                s.ev_chunk.push_back(e);
            }
        }
        while (static_cast<int>(s.ev_h2d.size()) < K) {
            cudaEvent_t a, b;
            S1D_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            S1D_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            s.ev_h2d.push_back(a);
            s.ev_dn.push_back(b);
        }
    }

    // D2H (Euler: pack first, on `stream`) of shard positions [p0, p1) once
    // `after` is done (heat: recorded by the caller).
    void chunk_d2h(Shard& s, std::uint64_t p0, std::uint64_t p1, cudaEvent_t after, cudaStream_t stream = nullptr) {
        if (!stream) stream = s.st;
        double* dst = pio->out + (pio->local ? 0 : s.start * spec.vpp) + p0 * spec.vpp;
        if (!euler) {
            S1D_CUDA(cudaStreamWaitEvent(s.cs, after, 0));
            S1D_CUDA(cudaMemcpyAsync(dst, s.state[0] + p0, sizeof(double) * (p1 - p0), cudaMemcpyDeviceToHost, s.cs));
        } else {
            S1D_CUDA(launch_euler_pack(s.state[0] + p0, s.staging + 3 * p0, p1 - p0, s.fstride, stream));
            S1D_CUDA(cudaEventRecord(after, stream));
            S1D_CUDA(cudaStreamWaitEvent(s.cs, after, 0));
            S1D_CUDA(cudaMemcpyAsync(dst, s.staging + 3 * p0, sizeof(double) * 3 * (p1 - p0), cudaMemcpyDeviceToHost,
                                     s.cs));
        }
    }

    DebugArgs dbg_args(int g) {
        DebugArgs d;
        if (!debug) return d;
        d.cov = sh(g).cov;
        d.cov_n = cfg.grid_size;
        d.gstart = sh(g).start;
        d.perturb = (perturb && sh(g).start == 0) ? 1 : 0;
        return d;
    }

    // Debug run: allocate coverage counters, run, return summed counts.
    void run_debug(bool coverage, bool nudge, std::uint32_t* host_cov, std::size_t cov_len, s1d_stats* st,
                   s1d_timing* tm) {
        debug = true;
        perturb = nudge;
        const std::uint64_t total = static_cast<std::uint64_t>(cfg.steps) * static_cast<std::uint64_t>(spec.S);
        const std::size_t cells = cfg.grid_size * total;
        if (coverage) {
            if (!host_cov || cov_len < cells) throw Error(S1D_INVALID_CONFIG, "coverage buffer too small (n*steps*S)");
            for (int g : locals) {
                S1D_CUDA(cudaSetDevice(sh(g).dev));
                S1D_CUDA(cudaMalloc(&sh(g).cov, sizeof(unsigned) * std::max<std::size_t>(cells, 1)));
                S1D_CUDA(cudaMemsetAsync(sh(g).cov, 0, sizeof(unsigned) * std::max<std::size_t>(cells, 1), sh(g).st));
            }
        }
        advance(st, tm);
        if (coverage) {
            std::fill(host_cov, host_cov + cells, 0u);
            std::vector<std::uint32_t> part(cells);
            for (int g : locals) {
                S1D_CUDA(cudaSetDevice(sh(g).dev));
                if (cells) S1D_CUDA(cudaMemcpy(part.data(), sh(g).cov, sizeof(unsigned) * cells, cudaMemcpyDeviceToHost));
                for (std::size_t i = 0; i < cells; ++i) host_cov[i] += part[i];
            }
        }
    }

    void record_all(cudaEvent_t Shard::*ev) {
        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(cudaEventRecord(s.*ev, s.st));
        }
    }

    bool use_classic_graph() const {
        static const bool no_graphs = [] {
            const char* e = std::getenv("S1D_NO_GRAPHS");
            return e && e[0] == '1';
        }();
        // one local shard: a single process (one GPU) or one process per GPU
        // (fused hand-off); single-process multi-device rounds use events
        return locals.size() == 1 && (R() == 1 || mp) && !debug && !no_graphs;
    }
    bool fused_rounds() const { return mp && R() > 1; }
    // Capture (once) the classic loop over counters [c0, c1] starting from
    // cur (all shards) with ping-pong index idx. Called before the timed
    // region so only the replay is timed.
    void ensure_classic_graph(std::int64_t c0, std::int64_t c1, const std::vector<const double*>& cur, int idx) {
        const double* start = cur[static_cast<std::size_t>(locals[0])];
        if (cgraph.exec && cgraph.c0 == c0 && cgraph.c1 == c1 && cgraph.start == start) return;
        Shard& s = sh(locals[0]);
        S1D_CUDA(cudaSetDevice(s.dev));
        if (cgraph.exec) S1D_CUDA(cudaGraphExecDestroy(cgraph.exec));
        cgraph.exec = nullptr;
        std::vector<const double*> cc = cur;
        s1d_stats tmp{};
        S1D_CUDA(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeThreadLocal));
        classic_launches(c0, c1, cc, &idx, tmp, false);
        cudaGraph_t graph = nullptr;
        S1D_CUDA(cudaStreamEndCapture(s.st, &graph));
        const cudaError_t ie = cudaGraphInstantiate(&cgraph.exec, graph, 0);
        cudaGraphDestroy(graph);
        S1D_CUDA(ie);
        S1D_CUDA(cudaGraphUpload(cgraph.exec, s.st)); // first launch then replays only
        cgraph.c0 = c0;
        cgraph.c1 = c1;
        cgraph.start = start;
        cgraph.end_idx = idx;
        cgraph.launches = tmp.kernel_launches;
    }

    void classic_steps(std::int64_t c_begin, std::int64_t c_end, std::vector<const double*>& cur, int* cur_idx,
                       s1d_stats& stats, bool dominant = false) {
        if (c_begin > c_end) return;
        const bool fused = fused_rounds();
        if (fused) {
            // One process per GPU: the round's hand-off is fused into the
            // substep kernel (its boundary points wait / signal, kernels.hpp
            // ClassicArgs), one launch per round. The previous round may have
            // written into this shard's state from a neighbour (a seam-centred
            // DownTriangle spills its right half into the right shard's array;
            // the pad runs right after it), and interior points do not wait in
            // a fused round: one full wait first. Then the rounds' sequence
            // base goes to device memory (flags[2]).
            wait_neighbours();
            Shard& s = sh(locals[0]);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(launch_set_u32(s.flags + 2, seq, s.st));
        }
        if (use_classic_graph()) {
            Shard& s = sh(locals[0]);
            S1D_CUDA(cudaSetDevice(s.dev));
            ensure_classic_graph(c_begin, c_end, cur, *cur_idx);
            if (dominant) record_all(&Shard::ev_dom0);
            S1D_CUDA(cudaGraphLaunch(cgraph.exec, s.st));
            if (dominant) record_all(&Shard::ev_dom1);
            stats.kernel_launches += cgraph.launches;
            *cur_idx = cgraph.end_idx;
            for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).state[cgraph.end_idx];
        } else {
            classic_launches(c_begin, c_end, cur, cur_idx, stats, dominant);
        }
        if (fused) seq += static_cast<unsigned>(c_end - c_begin + 1);
    }

    void classic_launches(std::int64_t c_begin, std::int64_t c_end, std::vector<const double*>& cur, int* cur_idx,
                          s1d_stats& stats, bool dominant) {
        // cur[g]: buffer holding shard g's current level; heat ping-pongs
        // through state[0]/state[1] (cur_idx: which one holds the result, -1 =
        // ic); Euler updates state[0] in place.
        const bool fused = fused_rounds();
        for (std::int64_t c = c_begin; c <= c_end; ++c) {
            if (!fused) wait_neighbours();
            if (dominant && c == c_begin) record_all(&Shard::ev_dom0);
            const int nxt = euler ? 0 : ((*cur_idx == 0) ? 1 : 0);
            for (int g : locals) {
                Shard& s = sh(g);
                Shard& L = left_of(g);
                Shard& Rt = right_of(g);
                const double* curL = cur[static_cast<std::size_t>(part.left[static_cast<std::size_t>(g)])];
                const double* curR = cur[static_cast<std::size_t>(part.right[static_cast<std::size_t>(g)])];
                ClassicArgs a;
                a.N = s.N;
                a.h = spec.h;
                a.counter = c;
                a.fstride = s.fstride;
                a.in = cur[static_cast<std::size_t>(g)];
                a.out = euler ? s.state[0] : s.state[nxt];
                a.halo_l = curL + (L.N - static_cast<std::uint64_t>(spec.h));
                a.halo_r = curR;
                a.halo_l_fstride = L.fstride;
                a.halo_r_fstride = Rt.fstride;
                a.fourier = cfg.fourier;
                a.gamma = cfg.gamma;
                a.dt_dx = cfg.dt_dx;
                a.error_flag = s.err;
                a.sms = s.sms;
                a.dbg = dbg_args(g);
                if (fused) {
                    a.nb_flags = s.flags;
                    a.seq_base = s.flags + 2;
                    a.round = static_cast<unsigned>(c - c_begin);
                    a.sig_left = L.flags + 1; // I am my left neighbour's right neighbour
                    a.sig_right = Rt.flags + 0;
                    a.timeout_ns = round_timeout_ns();
                }
                S1D_CUDA(cudaSetDevice(s.dev));
                if (euler) S1D_CUDA(launch_euler_classic(flat ? 1 : 0, a, s.st));
                else S1D_CUDA(launch_heat_classic(a, s.st));
                stats.kernel_launches += 1;
            }
            if (dominant && c == c_end) record_all(&Shard::ev_dom1);
            if (!fused) record_round();
            *cur_idx = nxt;
            for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).state[nxt];
        }
    }

    // Launch arguments of swept phase j (0: Up, cycles: Down) on shard g.
    TileArgs phase_args(int kind, std::int64_t j, int g) {
        const int w = static_cast<int>(cfg.block_width);
        const int src = static_cast<int>((j + 1) & 1), dst = static_cast<int>(j & 1);
        {
            Shard& s = sh(g);
            Shard& L = left_of(g);
            Shard& Rt = right_of(g);
            TileArgs a;
            a.w = w;
            a.h = spec.h;
            a.m = static_cast<int>(m);
            a.nb = static_cast<int>(s.nb);
            a.seam = (kind == kUp) ? 0 : static_cast<int>(j & 1);
            a.p = p;
            a.base = (kind == kUp) ? -static_cast<std::int64_t>(m) : (j - 1) * static_cast<std::int64_t>(m);
            a.N = s.N;
            a.rec = spec.rec;
            a.fstride = s.fstride;
            a.state_in = s.ic;
            a.state_out = s.state[0];
            a.state_right = Rt.state[0];
            a.right_fstride = Rt.fstride;
            a.in_R = s.ER[src];
            a.in_L = s.EL[src];
            a.peer_R = L.ER[src] + (L.nb - 1) * static_cast<std::uint64_t>(w) * static_cast<std::uint64_t>(spec.rec);
            a.peer_L = Rt.EL[src];
            a.out_L = s.EL[dst];
            a.out_R = s.ER[dst];
            a.fourier = cfg.fourier;
            a.gamma = cfg.gamma;
            a.dt_dx = cfg.dt_dx;
            a.error_flag = s.err;
            a.sms = s.sms;
            if (!euler && !heat_exact_only) {
                a.big_self = s.big();
                a.big_left = L.big();
                a.big_right = Rt.big();
                // single process: no gated launch per phase; advance() reads the
                // flags after the run (one process per GPU cannot: every rank
                // would have to agree to rerun)
                a.gated = mp ? 1 : 0;
            }
            a.dbg = dbg_args(g);
            return a;
        }
    }

    void launch_tiles(int kind, const TileArgs& ta, cudaStream_t stream, s1d_stats& stats) {
        if (euler) S1D_CUDA(launch_euler_tile(flat ? 1 : 0, kind, ta, stream, debug));
        else S1D_CUDA(launch_heat_tile(kind, ta, stream, debug));
        stats.kernel_launches += !euler && !debug && heat_fast_form(ta) && ta.gated ? 2 : 1;
    }

    void swept_phase(int kind, std::int64_t j, s1d_stats& stats, bool dom_first = false, bool dom_last = false) {
        wait_neighbours();
        if (dom_first) record_all(&Shard::ev_dom0);
        const int w = static_cast<int>(cfg.block_width);
        for (int g : locals) {
            Shard& s = sh(g);
            const TileArgs a = phase_args(kind, j, g);
            S1D_CUDA(cudaSetDevice(s.dev));
            auto launch = [&](const TileArgs& ta) { launch_tiles(kind, ta, s.st, stats); };
            if (pio && (kind == kUp || kind == kDown)) {
                const int K = pio->K;
                const std::uint64_t wu = static_cast<std::uint64_t>(w);
                for (int k = 0; k < K; ++k) {
                    const auto [t0, t1] = chunk_tiles(s, k, K);
                    TileArgs ta = a;
                    ta.b0 = t0;
                    ta.b1 = t1;
                    if (kind == kUp) { // this chunk's initial state has landed
                        S1D_CUDA(cudaStreamWaitEvent(s.st, s.ev_h2d[static_cast<std::size_t>(k)], 0));
                        if (euler)
                            S1D_CUDA(launch_euler_unpack(s.staging + 3 * t0 * wu, s.ic + t0 * wu, (t1 - t0) * wu,
                                                         s.fstride, spec.rec, s.st));
                        launch(ta);
                    } else {
                        launch(ta);
                        // Final state written by chunk k: centred tiles write their
                        // own blocks; seam-centred tiles (odd last cycle) write
                        // [t0 w + w/2, t1 w + w/2) (the part >= N lands in the
                        // right shard; this shard's first w/2 come from the left).
                        S1D_CUDA(cudaEventRecord(s.ev_dn[static_cast<std::size_t>(k)], s.st));
                        const std::uint64_t p0 = a.seam ? t0 * wu + wu / 2 : t0 * wu;
                        const std::uint64_t p1 = std::min<std::uint64_t>(a.seam ? t1 * wu + wu / 2 : t1 * wu, s.N);
                        if (p1 > p0) chunk_d2h(s, p0, p1, s.ev_dn[static_cast<std::size_t>(k)]);
                    }
                }
            } else {
                launch(a);
            }
            if (R() > 1 && kind != kUp)
                stats.edge_bytes_device += sizeof(double) * static_cast<std::uint64_t>(w) * spec.rec;
        }
        if (dom_last) record_all(&Shard::ev_dom1);
        record_round();
    }

    // Wavefront solve (s1d_solve, one shard in this process, aligned swept
    // run): the host copies take ~10% of a 2^27-point solve (1 GiB each way
    // over PCIe), more than the Up and Down phases they used to hide behind.
    // The first wave_head Diamonds after the Up and the last wave_tail before
    // the Down therefore also run per chunk of tiles, on two streams, each
    // chunk after its neighbour chunks of the previous phase (tile b reads
    // the edges of tiles b-1..b+1 and its outputs overwrite the buffers those
    // tiles' readers use, so the three-chunk dependency covers both RAW and
    // WAR): the copy-in of chunk k overlaps the first phases of the chunks
    // before it, and the copy-out of chunk k the last phases of the chunks
    // after it. The ring wraps (chunk 0's left neighbour is chunk K-1), so
    // the head wave grows from chunk 0 upwards and finishes the low chunks
    // last. One process per GPU: a shard's end chunks (0 and K-1) read or
    // overwrite what the ring neighbours' end chunks use, so each waits on
    // the device for the neighbours' previous phase (the round flags of
    // sync.cu, one round per phase as before) and each phase signals its
    // round once all its chunks are issued. Those runs use one stream: the
    // spinning waits must never hold back work issued before them, and
    // streams that share a hardware queue would (a wait of phase p in front
    // of this shard's own signal of phase p-1, mirrored on the neighbour,
    // deadlocks); an end chunk of phase p is issued only after the whole of
    // phase p-1 and its signal, so the waits resolve by induction over p.
    // Single-process multi-shard runs keep the Up/Down-only pipeline.
    // Shape: 16 chunks and enough pipelined Diamonds that their compute
    // covers one copy of the state: a heat Diamond takes ~m/420 of the copy
    // time (m updates per point at ~2.9 T/s against 8 B per point over PCIe
    // at ~55 GB/s), so ceil(384/m) Diamonds plus the Up: 3 at the bench's
    // m = 128 (measured 300.9 ms per solve against 303.0 with 2 and 301.1-
    // 301.6 with 4-5; the Up/Down-only pipeline took 31 ms more), 1 at m = 512
    // (368.5 against 370.0 ms). Euler keeps the Up/Down-only pipeline: its
    // copies are small against its compute and the chunked Diamonds' partial
    // waves cost more than they hide (measured 4% slower at w = 512).
    // S1D_WAVE = "chunks,head,tail" forces a shape (development knob).
    // Returns whether to use the wavefront.
    int wave_head = 0, wave_tail = 0, wave_slots = 0, wave_chunks = 16;
    bool set_wave_shape() {
        const int mm = static_cast<int>(m);
        wave_head = euler ? 1 : std::min(6, std::max(1, (384 + mm - 1) / mm));
        wave_tail = wave_head;
        wave_chunks = 16;
        bool use = !euler;
        if (const char* e = std::getenv("S1D_WAVE")) {
            int k = 0, h = 0, t = 0;
            if (std::sscanf(e, "%d,%d,%d", &k, &h, &t) == 3 && k >= 3 && h >= 0 && t >= 0) {
                wave_chunks = k;
                wave_head = h;
                wave_tail = t;
                use = true;
            }
        }
        wave_slots = wave_head + 1 + wave_tail + 1; // Up, head Diamonds, tail Diamonds, Down
        return use;
    }
    std::int64_t dom_diamonds = 0; // Diamonds inside the dominant-kernel timing window

    bool wave_eligible() const { return locals.size() == 1 && (R() == 1 || mp) && !debug; }
    bool wavefront(std::int64_t cycles) const {
        return pio && pio->wave && wave_eligible() &&
               cycles >= wave_head + wave_tail + 2 && pio->K >= 3;
    }

    // Chunk c of swept phase p (0: Up, cycles: Down) on `stream`.
    void chunk_phase(std::int64_t p, std::int64_t cycles, int c, cudaStream_t stream, s1d_stats& stats) {
        const int g = locals[0];
        Shard& s = sh(g);
        const int kind = p == 0 ? kUp : (p == cycles ? kDown : kDiamond);
        TileArgs ta = phase_args(kind, p, g);
        const auto [t0, t1] = chunk_tiles(s, c, pio->K);
        ta.b0 = t0;
        ta.b1 = t1;
        const std::uint64_t wu = cfg.block_width;
        if (kind == kUp) {
            S1D_CUDA(cudaStreamWaitEvent(stream, s.ev_h2d[static_cast<std::size_t>(c)], 0));
            if (euler)
                S1D_CUDA(launch_euler_unpack(s.staging + 3 * t0 * wu, s.ic + t0 * wu, (t1 - t0) * wu, s.fstride,
                                             spec.rec, stream));
        }
        launch_tiles(kind, ta, stream, stats);
        if (kind == kDown) { // as in swept_phase
            cudaEvent_t e = s.ev_dn[static_cast<std::size_t>(c)];
            S1D_CUDA(cudaEventRecord(e, stream));
            const std::uint64_t p0 = ta.seam ? t0 * wu + wu / 2 : t0 * wu;
            const std::uint64_t p1 = std::min<std::uint64_t>(ta.seam ? t1 * wu + wu / 2 : t1 * wu, s.N);
            if (p1 > p0) chunk_d2h(s, p0, p1, e, stream);
        }
    }

    void wavefront_phases(std::int64_t cycles, s1d_stats& stats) {
        const int me = locals[0];
        Shard& s = sh(me);
        S1D_CUDA(cudaSetDevice(s.dev));
        const int K = pio->K;
        const std::int64_t tail0 = cycles - wave_tail; // first tail phase
        const bool xs = mp && R() > 1;                 // neighbour shards in other processes
        const unsigned S = seq;                        // rounds completed before the Up
        const cudaStream_t sts[2] = {s.st, xs ? s.st : s.st2};
        auto slot = [&](std::int64_t p) {
            return p <= wave_head ? static_cast<int>(p) : wave_head + 1 + static_cast<int>(p - tail0);
        };
        auto ev = [&](std::int64_t p, int c) {
            return s.ev_chunk[static_cast<std::size_t>(slot(p) * K + ((c % K) + K) % K)];
        };
        // the second stream starts after the run's start
        S1D_CUDA(cudaEventRecord(s.ev_go, s.st));
        if (!xs) S1D_CUDA(cudaStreamWaitEvent(s.st2, s.ev_go, 0));
        // issue order and its invariants: host_wave.cpp
        for (const WaveStep& step : wave_schedule(K, wave_head, wave_tail, cycles, xs)) {
            const std::int64_t p = step.p;
            const int c = step.c;
            if (step.kind == kWaveChunk) {
                const cudaStream_t stream = sts[c & 1];
                if (p == tail0) {
                    S1D_CUDA(cudaStreamWaitEvent(stream, s.ev_mid, 0));
                } else if (p > 0) {
                    for (int d = -1; d <= 1; ++d) S1D_CUDA(cudaStreamWaitEvent(stream, ev(p - 1, c + d), 0));
                }
                if (xs && (c == 0 || c == K - 1)) // the neighbours' phase p-1 (Up: their previous run) is done
                    S1D_CUDA(launch_wait_flags(s.flags, S + static_cast<unsigned>(p), s.err, round_timeout_ns(),
                                               stream));
                chunk_phase(p, cycles, c, stream, stats);
                S1D_CUDA(cudaEventRecord(ev(p, c), stream));
            } else if (step.kind == kWaveSignal) {
                S1D_CUDA(launch_signal_flags(left_of(me).flags + 1, right_of(me).flags + 0,
                                             S + static_cast<unsigned>(p) + 1, s.st));
                if (p > 0) stats.edge_bytes_device += sizeof(double) * cfg.block_width * static_cast<unsigned>(spec.rec);
            } else { // middle: whole-shard Diamonds on s.st after every head chunk
                for (int k = 0; k < K; ++k) S1D_CUDA(cudaStreamWaitEvent(s.st, ev(wave_head, k), 0));
                if (xs) seq = S + static_cast<unsigned>(wave_head) + 1;
                record_all(&Shard::ev_dom0);
                for (std::int64_t j = wave_head + 1; j < tail0; ++j) swept_phase(kDiamond, j, stats);
                record_all(&Shard::ev_dom1);
                dom_diamonds = tail0 - wave_head - 1;
                S1D_CUDA(cudaEventRecord(s.ev_mid, s.st));
            }
        }
        if (xs) seq = S + static_cast<unsigned>(cycles) + 1;
        if (!xs) {
            S1D_CUDA(cudaEventRecord(s.ev_join, s.st2));
            S1D_CUDA(cudaStreamWaitEvent(s.st, s.ev_join, 0));
        }
    }

    void advance(s1d_stats* stats_out, s1d_timing* timing_out) {
        if (!connected) throw Error(S1D_INVALID_CONFIG, "shard not connected: call s1d_shard_connect first");
        s1d_stats stats{};
        const std::int64_t total = cfg.steps * spec.S;
        const std::int64_t cycles = cfg.scheme == S1D_SWEPT ? total / static_cast<std::int64_t>(m) : 0;
        const std::int64_t pad = total - cycles * static_cast<std::int64_t>(m);

        if (pad > 0 && use_classic_graph()) { // capture outside the timed region
            const bool from_state = cycles >= 1 || euler;
            std::vector<const double*> c0(static_cast<std::size_t>(R()));
            for (int g = 0; g < R(); ++g) c0[static_cast<std::size_t>(g)] = from_state ? sh(g).state[0] : sh(g).ic;
            ensure_classic_graph(cycles * static_cast<std::int64_t>(m) + 1, total, c0, from_state ? 0 : -1);
        }
        sync_all();
        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(cudaMemsetAsync(s.err, 0, sizeof(int), s.st));
            // Euler classic substeps run in place on state[0]; seed it with the
            // initial records when no swept phase writes it first (placement
            // of the IC is setup in the reference, outside the timed loop).
            if (euler && cycles == 0 && pad > 0)
                S1D_CUDA(cudaMemcpyAsync(s.state[0], s.ic, sizeof(double) * s.N * spec.rec, cudaMemcpyDeviceToDevice,
                                         s.st));
            S1D_CUDA(cudaEventRecord(s.ev_start, s.st));
        }
        record_round(); // "initial state resident" round

        std::vector<const double*> cur(static_cast<std::size_t>(R()));
        int cur_idx = -1;
        for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).ic;
        // Dominant kernel: the Diamond phases when there are any, else the
        // classic substeps, else the Up/Down pair.
        const bool dom_diamond = cycles >= 2;
        const bool dom_classic = !dom_diamond && pad > 0;
        const bool dom_updown = !dom_diamond && !dom_classic && cycles == 1;
        dom_diamonds = cycles - 1;
        if (cycles >= 1 && wavefront(cycles)) {
            wavefront_phases(cycles, stats);
            cur_idx = 0;
            for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).state[0];
        } else if (cycles >= 1) {
            swept_phase(kUp, 0, stats, dom_updown, false);
            for (std::int64_t j = 1; j <= cycles; ++j)
                swept_phase(j == cycles ? kDown : kDiamond, j, stats, dom_diamond && j == 1,
                            (dom_diamond && j == cycles - 1) || (dom_updown && j == cycles));
            cur_idx = 0;
            for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).state[0];
        }
        if (pad > 0) {
            if (euler && cycles == 0) {
                cur_idx = 0;
                for (int g = 0; g < R(); ++g) cur[static_cast<std::size_t>(g)] = sh(g).state[0];
            }
            classic_steps(cycles * static_cast<std::int64_t>(m) + 1, total, cur, &cur_idx, stats, dom_classic);
        }
        // The left neighbour's last Down tile writes into this shard's state:
        // make its completion part of this shard's run.
        if (mp) wait_neighbours();

        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            S1D_CUDA(cudaEventRecord(s.ev_stop, s.st));
        }
        if (pio && (cycles & 1)) {
            // seam-centred last cycle: each shard's first w/2 points are written
            // by its left neighbour's last tile (that shard's stream; in
            // multi-process mode the final flag wait above covers it)
            for (int g : locals) {
                Shard& s = sh(g);
                S1D_CUDA(cudaSetDevice(s.dev));
                if (!mp) S1D_CUDA(cudaStreamWaitEvent(s.st, left_of(g).ev_stop, 0));
                S1D_CUDA(cudaEventRecord(s.ev_fin, s.st));
                chunk_d2h(s, 0, cfg.block_width / 2, s.ev_fin);
            }
        }
        sync_all();
        for (int g : locals) {
            S1D_CUDA(cudaSetDevice(sh(g).dev));
            if (sh(g).cs) S1D_CUDA(cudaStreamSynchronize(sh(g).cs));
        }
        float worst_ms = 0.0f, dom_ms = 0.0f;
        const bool have_dom = dom_diamond || dom_classic || dom_updown;
        int flag = 0;
        for (int g : locals) {
            Shard& s = sh(g);
            S1D_CUDA(cudaSetDevice(s.dev));
            float ms = 0.0f;
            S1D_CUDA(cudaEventElapsedTime(&ms, s.ev_start, s.ev_stop));
            worst_ms = std::max(worst_ms, ms);
            if (have_dom) {
                S1D_CUDA(cudaEventElapsedTime(&ms, s.ev_dom0, s.ev_dom1));
                dom_ms = std::max(dom_ms, ms);
            }
            int f = 0;
            S1D_CUDA(cudaMemcpy(&f, s.err, sizeof(int), cudaMemcpyDeviceToHost));
            flag |= f;
            s.final_state = cur[static_cast<std::size_t>(g)];
        }
        S1D_CUDA(cudaGetLastError());
        if (!mp && !euler && !heat_exact_only && cfg.scheme == S1D_SWEPT && !debug) {
            // heat fast form, single process: a set flag means some fast CTA
            // stopped (an input >= 2^1022, heat.cu heat_step); rerun the whole
            // advance in the exact form (the initial state in ic is intact)
            int big = 0;
            for (int g : locals) {
                int b = 0;
                S1D_CUDA(cudaSetDevice(sh(g).dev));
                S1D_CUDA(cudaMemcpy(&b, sh(g).big(), sizeof(int), cudaMemcpyDeviceToHost));
                big |= b;
            }
            if (big) {
                heat_exact_only = true;
                advance(stats_out, timing_out);
                return;
            }
        }
        if (flag & 4) throw Error(S1D_INTERNAL, "device bounds check failed (checked build)");
        if (flag & 2) throw Error(S1D_TRANSPORT_ABORTED, "a neighbour shard stopped responding (round timeout)");
        if (flag) throw Error(S1D_NONPHYSICAL, "non-physical state encountered on the device");

        // Reference accounting (transport.cpp:48-110): a swept cycle is one
        // shift round (1 message of (w/2+h) records per rank); a classic or
        // pad substep is one exchange round (2 messages of h records).
        const std::uint64_t Rn = static_cast<std::uint64_t>(R());
        const std::uint64_t cell = sizeof(double) * static_cast<std::uint64_t>(spec.slots);
        const std::uint64_t buf = cfg.block_width / 2 + static_cast<std::uint64_t>(spec.h);
        stats.exchange_rounds = static_cast<std::uint64_t>(cycles + pad);
        stats.messages_sent = Rn * static_cast<std::uint64_t>(cycles + 2 * pad);
        stats.bytes_sent = Rn * (static_cast<std::uint64_t>(cycles) * buf * cell +
                                 static_cast<std::uint64_t>(pad) * 2 * static_cast<std::uint64_t>(spec.h) * cell);
        if (Rn > 1)
            stats.edge_bytes_device += static_cast<std::uint64_t>(pad) * locals.size() * 2 * sizeof(double) *
                                       static_cast<std::uint64_t>(spec.h) * static_cast<std::uint64_t>(spec.rec);
        {
            double comm = 0.0;
            const double vclock = virtual_clock(cfg, &comm);
            stats.virtual_comm_seconds = comm;
            if (timing_out) timing_out->virtual_seconds = cfg.mode == S1D_VIRTUAL ? vclock : 0.0;
        }
        if (stats_out) *stats_out = stats;
        if (timing_out) {
            timing_out->setup_seconds = setup_seconds;
            timing_out->loop_seconds = worst_ms * 1e-3;
            timing_out->dominant_seconds = dom_ms * 1e-3;
            std::uint64_t pts = 0;
            for (int g : locals) pts += sh(g).N;
            const char* name = "";
            if (dom_diamond) {
                timing_out->dominant_launches = static_cast<std::uint64_t>(dom_diamonds);
                timing_out->dominant_point_updates = static_cast<std::uint64_t>(dom_diamonds) * m * pts;
                name = "swept_diamond";
            } else if (dom_classic) {
                timing_out->dominant_launches = static_cast<std::uint64_t>(pad);
                timing_out->dominant_point_updates = static_cast<std::uint64_t>(pad) * pts;
                name = "classic_substep";
            } else if (dom_updown) {
                timing_out->dominant_launches = 2;
                timing_out->dominant_point_updates = m * pts;
                name = "swept_up_down";
            }
            std::snprintf(timing_out->dominant_kernel, sizeof(timing_out->dominant_kernel), "%s", name);
        }
    }

    // s1d_solve with host copies overlapped with the Up/Down phases (swept,
    // aligned totals); otherwise upload, advance, download in sequence.
    void solve(const double* host_in, double* host_out, s1d_stats* st, s1d_timing* tm) {
        const std::int64_t total = cfg.steps * spec.S;
        const std::int64_t cycles = cfg.scheme == S1D_SWEPT ? total / static_cast<std::int64_t>(m) : 0;
        const bool aligned = cycles >= 1 && total == cycles * static_cast<std::int64_t>(m);
        const auto t0 = std::chrono::steady_clock::now();
        if (!aligned || debug) {
            upload(host_in, local_io());
            sync_all();
            const auto t1 = std::chrono::steady_clock::now();
            advance(st, tm);
            const auto t2 = std::chrono::steady_clock::now();
            download(host_out, local_io());
            tm->h2d_seconds = std::chrono::duration<double>(t1 - t0).count();
            tm->d2h_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
            return;
        }
        if (!mp) heat_exact_only = false; // new data (flags re-armed by the uploads below)
        PipeIO io;
        io.in = host_in;
        io.out = host_out;
        io.local = local_io();
        std::uint64_t min_nb = ~0ull;
        for (int g : locals) min_nb = std::min<std::uint64_t>(min_nb, sh(g).nb);
        io.wave = set_wave_shape() && wave_eligible() && cycles >= wave_head + wave_tail + 2 && min_nb >= 3;
        io.K = static_cast<int>(std::min<std::uint64_t>(io.wave ? wave_chunks : 8, min_nb));
        sync_all();
        for (int g : locals) {
            Shard& s = sh(g);
            ensure_pipe(s, io.K, io.wave);
            if (!mp && s.flags) S1D_CUDA(cudaMemsetAsync(s.big(), 0, sizeof(int), s.st)); // new data: re-arm
            const std::uint64_t wu = cfg.block_width;
            const double* src = host_in + (io.local ? 0 : s.start * spec.vpp);
            for (int k = 0; k < io.K; ++k) {
                const auto [a0, a1] = chunk_tiles(s, k, io.K);
                const std::uint64_t p0 = a0 * wu, p1 = a1 * wu;
                double* dst = euler ? s.staging + 3 * p0 : s.ic + p0;
                S1D_CUDA(cudaMemcpyAsync(dst, src + p0 * spec.vpp, sizeof(double) * (p1 - p0) * spec.vpp,
                                         cudaMemcpyHostToDevice, s.cs));
                S1D_CUDA(cudaEventRecord(s.ev_h2d[static_cast<std::size_t>(k)], s.cs));
            }
        }
        pio = &io;
        try {
            advance(st, tm);
        } catch (...) {
            pio = nullptr;
            throw;
        }
        pio = nullptr;
        tm->h2d_seconds = 0.0; // overlapped with the UpTriangle
        tm->d2h_seconds = 0.0; // overlapped with the DownTriangle
        (void)t0;
    }

    // Points (x vpp) the host I/O of this solver covers: the global array
    // (single process) or the local shard's slice (multi-process).
    std::size_t state_len() const {
        std::uint64_t pts = 0;
        if (locals.size() == shards.size()) pts = cfg.grid_size;
        else
            for (int g : locals) pts += shards[static_cast<std::size_t>(g)].N;
        return pts * static_cast<std::uint64_t>(spec.vpp);
    }
    bool local_io() const { return locals.size() != shards.size(); }
};

} // namespace s1d

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct s1d_solver {
    s1d::Solver impl;
};

namespace {

void put_err(char* err, size_t errlen, const std::string& what) {
    if (!err || errlen == 0) return;
    const size_t n = std::min(errlen - 1, what.size());
    std::memcpy(err, what.data(), n);
    err[n] = '\0';
}

template <class Fn>
int guarded(char* err, size_t errlen, Fn&& fn) {
    try {
        fn();
        put_err(err, errlen, "");
        return S1D_OK;
    } catch (const s1d::Error& e) {
        put_err(err, errlen, e.what());
        return e.status;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return S1D_INTERNAL;
    }
}

// Null arguments fail loudly at the boundary (no dereference of a null config).
void need(const void* p, const char* what) {
    if (!p) throw s1d::Error(S1D_INVALID_CONFIG, std::string(what) + " is null");
}

template <class Fn>
int guarded_solver(s1d_solver* s, Fn&& fn) {
    char buf[512];
    const int st = guarded(buf, sizeof buf, fn);
    if (s) s->impl.last_error = buf;
    return st;
}

} // namespace

extern "C" {

const char* s1d_version(void) { return "swept1d-b200 0.2.0 (sm_100a, FP64)"; }
int s1d_abi_version(void) { return S1D_ABI_VERSION; }

int s1d_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void s1d_config_defaults(s1d_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->equation = S1D_HEAT;
    c->method = S1D_LENGTHENING;
    c->scheme = S1D_SWEPT;
    c->mode = S1D_VIRTUAL;
    c->grid_size = 1024;
    c->block_width = 32;
    c->ranks = 2;
    c->work_factor = 0;
    c->steps = 50;
    c->fourier = 0.4;
    c->gamma = 1.4;
    c->dt_dx = 0.0;
    c->cfl = 0.4;
    c->alpha = 0.0;
    c->beta = 0.0;
    c->compute_cost = 1e-8;
    c->num_devices = 0;
}

int s1d_apply_config_entry(s1d_config* cfg, const char* key, const char* value, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(key, "key");
        need(value, "value"); s1d::apply_config_entry(*cfg, key, value); });
}

int s1d_validate(const s1d_config* cfg, int partitioned, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config"); s1d::validate(*cfg, partitioned != 0); });
}

int s1d_finalize(s1d_config* cfg, int partitioned, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config"); s1d::finalize(*cfg, partitioned != 0); });
}

void s1d_spec(int equation, int method, int* substeps, int* half_width, int* slots, int* vpp) {
    const s1d::Spec s = s1d::make_spec(equation, method);
    if (substeps) *substeps = s.S;
    if (half_width) *half_width = s.h;
    if (slots) *slots = s.slots;
    if (vpp) *vpp = s.vpp;
}

int s1d_initial_condition(const char* id, uint64_t n, int equation, double gamma, double* out, size_t out_len,
                          char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(id, "initial condition id");
        need(out, "out");
        const auto v = s1d::initial_condition(id, n, equation, gamma);
        if (v.size() > out_len) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int s1d_initial_condition_range(const char* id, uint64_t n, int equation, double gamma, uint64_t j0, uint64_t count,
                                double* out, size_t out_len, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(id, "initial condition id");
        need(out, "out");
        if (j0 + count > n) throw s1d::Error(S1D_INVALID_CONFIG, "range outside the grid");
        const auto v = s1d::initial_condition_range(id, n, equation, gamma, j0, count);
        if (v.size() > out_len) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int s1d_max_signal_speed(const double* prim, size_t len, double gamma, double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(prim, "prim");
        need(out, "out");
        *out = s1d::max_signal_speed(prim, len, gamma);
    });
}

int s1d_partition(const s1d_config* cfg, uint64_t* blocks, uint64_t* start, int* left, int* right, char* err,
                  size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(blocks, "blocks");
        need(start, "start");
        need(left, "left");
        need(right, "right");
        const auto p = s1d::make_partition(*cfg);
        for (std::size_t r = 0; r < p.blocks.size(); ++r) {
            blocks[r] = p.blocks[r];
            start[r] = p.start[r];
            left[r] = p.left[r];
            right[r] = p.right[r];
        }
    });
}

int64_t s1d_cycle_advance(uint64_t w, uint64_t h, char* err, size_t errlen) {
    std::uint64_t m = 0;
    const int st = guarded(err, errlen, [&] { m = s1d::cycle_advance(w, h); });
    return st == S1D_OK ? static_cast<int64_t>(m) : -st;
}

int s1d_message_log(const s1d_config* cfg, s1d_message* out, size_t cap, size_t* count, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(count, "count");
        if (cap && !out) need(out, "out");
        s1d_config c = *cfg;
        s1d::finalize(c, true);
        const auto log = s1d::message_log(c);
        *count = log.size();
        for (std::size_t i = 0; i < log.size() && i < cap; ++i) out[i] = log[i];
    });
}

int s1d_debug_wave_schedule(int chunks, int head, int tail, int64_t cycles, int multi_process, int64_t* out,
                            size_t cap, size_t* count, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(count, "count");
        if (cap && !out) need(out, "out");
        const auto steps = s1d::wave_schedule(chunks, head, tail, cycles, multi_process != 0);
        *count = steps.size();
        for (std::size_t i = 0; i < steps.size() && i < cap; ++i) {
            out[3 * i] = steps[i].kind;
            out[3 * i + 1] = steps[i].p;
            out[3 * i + 2] = steps[i].c;
        }
    });
}

int s1d_comm_per_rank(const s1d_config* cfg, s1d_rank_stats* out, size_t cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(out, "out");
        s1d_config c = *cfg;
        s1d::finalize(c, true);
        const auto st = s1d::rank_stats(c);
        if (cap < st.size()) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        for (std::size_t i = 0; i < st.size(); ++i) out[i] = st[i];
    });
}

int s1d_virtual_time(const s1d_config* cfg, double* virtual_seconds, double* comm_seconds, char* err,
                     size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        s1d_config c = *cfg;
        s1d::finalize(c, true);
        double comm = 0.0;
        const double v = s1d::virtual_clock(c, &comm);
        if (virtual_seconds) *virtual_seconds = v;
        if (comm_seconds) *comm_seconds = comm;
    });
}

int s1d_calibrate_transport(int dev_a, int dev_b, double* alpha, double* beta, char* err, size_t errlen) {
    using s1d::CudaError;
    return guarded(err, errlen, [&] {
        int nd = 0;
        if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
            cudaGetLastError();
            throw s1d::Error(S1D_NO_DEVICE, "no CUDA device visible");
        }
        if (dev_a == dev_b || dev_a < 0 || dev_b < 0 || dev_a >= nd || dev_b >= nd)
            throw s1d::Error(S1D_INVALID_CONFIG, "calibration needs two distinct visible devices");
        int ab = 0, ba = 0;
        S1D_CUDA(cudaDeviceCanAccessPeer(&ab, dev_a, dev_b));
        S1D_CUDA(cudaDeviceCanAccessPeer(&ba, dev_b, dev_a));
        if (!ab || !ba) throw s1d::Error(S1D_PEER_UNAVAILABLE, "devices cannot access each other's memory");
        const int devs[2] = {dev_a, dev_b};
        cudaStream_t st[2];
        unsigned* flag[2];
        int* eflag[2];
        for (int i = 0; i < 2; ++i) {
            S1D_CUDA(cudaSetDevice(devs[i]));
            const cudaError_t pe = cudaDeviceEnablePeerAccess(devs[1 - i], 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) S1D_CUDA(pe);
            cudaGetLastError();
            S1D_CUDA(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
            S1D_CUDA(cudaMalloc(&flag[i], 256));
            S1D_CUDA(cudaMalloc(&eflag[i], sizeof(int)));
            S1D_CUDA(cudaMemsetAsync(eflag[i], 0, sizeof(int), st[i]));
            S1D_CUDA(cudaStreamSynchronize(st[i]));
        }
        cudaEvent_t e0, e1;
        S1D_CUDA(cudaSetDevice(dev_a));
        S1D_CUDA(cudaEventCreate(&e0));
        S1D_CUDA(cudaEventCreate(&e1));
        // alpha: one-way latency of a flag hand-off (the swept round's sync).
        auto pingpong = [&](int iters) {
            for (int i = 0; i < 2; ++i) {
                S1D_CUDA(cudaSetDevice(devs[i]));
                S1D_CUDA(cudaMemsetAsync(flag[i], 0, 256, st[i]));
                S1D_CUDA(cudaStreamSynchronize(st[i]));
            }
            S1D_CUDA(cudaSetDevice(dev_b));
            S1D_CUDA(s1d::launch_pingpong(flag[1], flag[0], iters, 0, eflag[1], 10000000000ull, st[1]));
            S1D_CUDA(cudaSetDevice(dev_a));
            S1D_CUDA(cudaEventRecord(e0, st[0]));
            S1D_CUDA(s1d::launch_pingpong(flag[0], flag[1], iters, 1, eflag[0], 10000000000ull, st[0]));
            S1D_CUDA(cudaEventRecord(e1, st[0]));
            for (int i = 0; i < 2; ++i) {
                S1D_CUDA(cudaSetDevice(devs[i]));
                S1D_CUDA(cudaStreamSynchronize(st[i]));
                int f = 0;
                S1D_CUDA(cudaMemcpy(&f, eflag[i], sizeof(int), cudaMemcpyDeviceToHost));
                if (f) throw s1d::Error(S1D_TRANSPORT_ABORTED, "calibration ping-pong timed out");
            }
            float ms = 0.0f;
            S1D_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            return static_cast<double>(ms) * 1e-3;
        };
        pingpong(200);
        const int n1 = 2000, n2 = 6000;
        const double t1 = pingpong(n1), t2 = pingpong(n2);
        const double a = (t2 - t1) / (2.0 * (n2 - n1));
        // beta: inverse bandwidth of a large peer copy a -> b.
        const std::size_t bytes = std::size_t(256) << 20;
        void* src = nullptr;
        void* dst = nullptr;
        S1D_CUDA(cudaSetDevice(dev_b));
        S1D_CUDA(cudaMalloc(&dst, bytes));
        S1D_CUDA(cudaSetDevice(dev_a));
        S1D_CUDA(cudaMalloc(&src, bytes));
        S1D_CUDA(cudaMemsetAsync(src, 0, bytes, st[0]));
        S1D_CUDA(cudaMemcpyPeerAsync(dst, dev_b, src, dev_a, bytes, st[0]));
        const int reps = 4;
        S1D_CUDA(cudaEventRecord(e0, st[0]));
        for (int i = 0; i < reps; ++i) S1D_CUDA(cudaMemcpyPeerAsync(dst, dev_b, src, dev_a, bytes, st[0]));
        S1D_CUDA(cudaEventRecord(e1, st[0]));
        S1D_CUDA(cudaStreamSynchronize(st[0]));
        float ms = 0.0f;
        S1D_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        const double b = static_cast<double>(ms) * 1e-3 / (static_cast<double>(bytes) * reps);
        S1D_CUDA(cudaFree(src));
        S1D_CUDA(cudaEventDestroy(e0));
        S1D_CUDA(cudaEventDestroy(e1));
        for (int i = 0; i < 2; ++i) {
            S1D_CUDA(cudaSetDevice(devs[i]));
            S1D_CUDA(cudaFree(flag[i]));
            S1D_CUDA(cudaFree(eflag[i]));
            S1D_CUDA(cudaStreamDestroy(st[i]));
        }
        S1D_CUDA(cudaSetDevice(dev_b));
        S1D_CUDA(cudaFree(dst));
        if (alpha) *alpha = a;
        if (beta) *beta = b;
    });
}

int64_t s1d_schedule(int kind, uint64_t w, uint64_t h, int64_t* substep, int64_t* lo, int64_t* hi, size_t cap,
                     char* err, size_t errlen) {
    std::vector<s1d::Level> lv;
    const int st = guarded(err, errlen, [&] { lv = s1d::schedule(kind, w, h); });
    if (st != S1D_OK) return -st;
    for (std::size_t i = 0; i < lv.size() && i < cap; ++i) {
        substep[i] = lv[i].substep;
        lo[i] = lv[i].lo;
        hi[i] = lv[i].hi;
    }
    return static_cast<int64_t>(lv.size());
}

uint64_t s1d_swept_buffer_cells(uint64_t w, int equation, int method) {
    return w / 2 + static_cast<uint64_t>(s1d::make_spec(equation, method).h);
}

int s1d_run_debug(const s1d_config* cfg, const s1d_debug* dbg, double* state_out, size_t state_len, s1d_stats* stats,
                  s1d_timing* timing, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(state_out, "state_out");
        s1d::Solver solver;
        solver.init(*cfg);
        if (state_len < solver.state_len()) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        s1d_timing t{};
        solver.run_debug(dbg && dbg->coverage, dbg && dbg->perturb_ulp, dbg ? dbg->coverage_out : nullptr,
                         dbg ? dbg->coverage_len : 0, stats, &t);
        solver.download(state_out, false);
        if (timing) *timing = t;
    });
}

int s1d_measure(const s1d_config* cfg, s1d_record* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(out, "record");
        s1d::Solver solver;
        solver.init(*cfg);
        s1d_stats st{};
        s1d_timing tm{};
        solver.advance(&st, &tm);
        const s1d_config& c = solver.cfg;
        *out = s1d_record{};
        out->equation = c.equation;
        out->method = c.method;
        out->scheme = c.scheme;
        out->mode = c.mode;
        out->grid_size = c.grid_size;
        out->block_width = c.block_width;
        out->work_factor = c.work_factor;
        out->ranks = c.ranks;
        out->steps = c.steps;
        // perf.cpp:21-23: virtual mode reports the modelled clock.
        const double secs = c.mode == S1D_VIRTUAL ? tm.virtual_seconds : tm.loop_seconds;
        out->avg_us_per_step = c.steps > 0 ? secs * 1e6 / static_cast<double>(c.steps) : 0.0;
        out->setup_us = tm.setup_seconds * 1e6;
        out->messages_sent = st.messages_sent;
        out->bytes_sent = st.bytes_sent;
        out->exchange_rounds = st.exchange_rounds;
        out->virtual_comm_us = st.virtual_comm_seconds * 1e6;
    });
}

int s1d_create(const s1d_config* cfg, s1d_solver** out, char* err, size_t errlen) {
    if (!out) return guarded(err, errlen, [] { need(nullptr, "out"); });
    *out = nullptr;
    auto holder = std::make_unique<s1d_solver>();
    const int st = guarded(err, errlen, [&] {
        need(cfg, "config"); holder->impl.init(*cfg); });
    if (st == S1D_OK) *out = holder.release();
    return st;
}

void s1d_destroy(s1d_solver* s) { delete s; }

int s1d_get_config(const s1d_solver* s, s1d_config* out) {
    if (!s || !out) return S1D_INVALID_CONFIG;
    *out = s->impl.cfg;
    return S1D_OK;
}

int s1d_set_initial(s1d_solver* s, const double* host_state, size_t len) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        if (!host_state) {
            s->impl.upload(s->impl.host_ic.data(), s->impl.local_io());
        } else {
            if (len != s->impl.state_len()) throw s1d::Error(S1D_INVALID_CONFIG, "initial state length mismatch");
            s->impl.upload(host_state, s->impl.local_io());
        }
        s->impl.sync_all();
    });
}

int s1d_advance(s1d_solver* s, s1d_stats* stats, s1d_timing* timing) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        if (timing) std::memset(timing, 0, sizeof(*timing));
        s->impl.advance(stats, timing);
    });
}

int s1d_read_state(s1d_solver* s, double* host_out, size_t len) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        need(host_out, "host_out");
        if (len < s->impl.state_len()) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        for (int g : s->impl.locals)
            if (!s->impl.sh(g).final_state) throw s1d::Error(S1D_INVALID_CONFIG, "no state: call s1d_advance first");
        s->impl.download(host_out, s->impl.local_io());
    });
}

int s1d_solve(s1d_solver* s, const double* host_in, size_t in_len, double* host_out, size_t out_len,
              s1d_stats* stats, s1d_timing* timing) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        need(host_out, "host_out");
        if (host_in && in_len != s->impl.state_len())
            throw s1d::Error(S1D_INVALID_CONFIG, "initial state length mismatch");
        if (out_len < s->impl.state_len()) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        s1d_timing t{};
        s->impl.solve(host_in ? host_in : s->impl.host_ic.data(), host_out, stats, &t);
        if (timing) *timing = t;
    });
}

const char* s1d_last_error(const s1d_solver* s) { return s ? s->impl.last_error.c_str() : ""; }

int s1d_shard_create(const s1d_config* cfg, int rank, int device, s1d_solver** out, char* err, size_t errlen) {
    if (!out) return guarded(err, errlen, [] { need(nullptr, "out"); });
    *out = nullptr;
    auto holder = std::make_unique<s1d_solver>();
    const int st = guarded(err, errlen, [&] {
        need(cfg, "config"); holder->impl.init_shard(*cfg, rank, device); });
    if (st == S1D_OK) *out = holder.release();
    return st;
}

size_t s1d_shard_blob_size(void) { return sizeof(s1d::ShardBlob); }

int s1d_shard_export(s1d_solver* s, void* blob, size_t blob_len) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        need(blob, "blob");
        if (blob_len < sizeof(s1d::ShardBlob)) throw s1d::Error(S1D_INVALID_CONFIG, "blob buffer too small");
        s->impl.export_blob(static_cast<s1d::ShardBlob*>(blob));
    });
}

int s1d_shard_connect(s1d_solver* s, const void* left_blob, const void* right_blob) {
    if (!s) return S1D_INVALID_CONFIG;
    return guarded_solver(s, [&] {
        need(left_blob, "left_blob");
        need(right_blob, "right_blob");
        s->impl.connect(static_cast<const s1d::ShardBlob*>(left_blob), static_cast<const s1d::ShardBlob*>(right_blob));
    });
}

int s1d_shard_range(const s1d_solver* s, uint64_t* start, uint64_t* count) {
    if (!s || !start || !count) return S1D_INVALID_CONFIG;
    if (s->impl.locals.size() != 1) {
        *start = 0;
        *count = s->impl.cfg.grid_size;
        return S1D_OK;
    }
    const auto& sh = s->impl.shards[static_cast<std::size_t>(s->impl.locals[0])];
    *start = sh.start;
    *count = sh.N;
    return S1D_OK;
}

int s1d_run(const s1d_config* cfg, double* state_out, size_t state_len, s1d_stats* stats, s1d_timing* timing,
            char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        need(cfg, "config");
        need(state_out, "state_out");
        s1d::Solver solver;
        solver.init(*cfg);
        if (state_len < solver.state_len()) throw s1d::Error(S1D_INVALID_CONFIG, "output buffer too small");
        s1d_timing t{};
        solver.advance(stats, &t);
        const auto t2 = std::chrono::steady_clock::now();
        solver.download(state_out, false);
        t.d2h_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
        if (timing) *timing = t;
    });
}

} // extern "C"
