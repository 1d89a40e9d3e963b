// Launch interface between the host orchestrator (engine.cu) and the sm_100a
// kernels (heat.cu, euler.cu). Plain structs of device pointers; no torch.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace s1d {

enum TileKind : int { kUp = 0, kDiamond = 1, kDown = 2 };

// Debug instrumentation (debug builds of the kernels only; RunOptions,
// inc/debug.hpp:17-62): `cov` counts every (global point, substep) the
// kernel computes, cov[(counter-1)*cov_n + (gstart + pos) mod cov_n];
// `perturb` nudges the first value the run computes by one ulp.
struct DebugArgs {
    unsigned* cov = nullptr;
    std::uint64_t cov_n = 0;
    std::uint64_t gstart = 0; // global index of shard position 0
    int perturb = 0;          // 1: nudge (shard 0 only)
};

// One swept phase over the tiles of a shard.
// Local tile coordinates x in [0, w+2h) map to shard position
// g = centre - w/2 - h + x. Registers hold x in [h, w+h).
struct TileArgs {
    int w = 0, h = 1, m = 0;  // block width, half width, levels per half cycle
    int nb = 0;               // tiles of the shard (blocks)
    int b0 = 0, b1 = -1;      // this launch covers shard tiles [b0, b1) (b1 < 0: all)
    int seam = 0;             // 1: centres at (b+1)w (odd cycles); 0: bw + w/2
    int p = 2;                // points per thread
    std::int64_t base = 0;    // counter of level r is base + r
    std::uint64_t N = 0;      // shard points
    int rec = 1;              // doubles per record (per field block)
    std::uint64_t fstride = 0; // state field stride (doubles) for SoA records
    // Up: state_in (shard-local, positions [bw, bw+w)); Down: state_out
    // (positions >= N spill to state_right, the right shard's array).
    const double* state_in = nullptr;
    double* state_out = nullptr;
    double* state_right = nullptr;
    std::uint64_t right_fstride = 0;
    // Edges: per tile w records per side, laid out [tile][level][2h][rec].
    const double* in_R = nullptr;   // producers' right edges (own shard)
    const double* in_L = nullptr;   // producers' left edges (own shard)
    const double* peer_R = nullptr; // left shard's last tile R edges (center phase, tile 0)
    const double* peer_L = nullptr; // right shard's tile 0 L edges (seam phase, last tile)
    double* out_L = nullptr;
    double* out_R = nullptr;
    // physics
    double fourier = 0.4, gamma = 1.4, dt_dx = 0.0;
    int* error_flag = nullptr;      // device NonPhysicalState flag (Euler)
    double* scratch = nullptr;      // Euler tiles too wide for shared memory: per-CTA records (launcher-owned)
    int sms = 148;                  // SMs of the launching device (queried once per shard, not per launch)
    // heat fast form (heat.cu heat_step): the shard's sticky "value >= 2^1022
    // may be present" flag and its ring neighbours' (null: exact form only)
    int* big_self = nullptr;
    const int* big_left = nullptr;
    const int* big_right = nullptr;
    int gated = 1; // 1: the gated exact build follows each fast launch; 0: the host checks the flags after the run
    DebugArgs dbg;
};

struct ClassicArgs {
    std::uint64_t N = 0;
    int h = 1;
    std::int64_t counter = 1;
    std::uint64_t fstride = 0;
    const double* in = nullptr;     // SoA fields, stride fstride
    double* out = nullptr;
    // halo sources: h records left of position 0 and right of N-1 (possibly
    // on a peer device), field stride halo_*_fstride.
    const double* halo_l = nullptr;
    const double* halo_r = nullptr;
    std::uint64_t halo_l_fstride = 0, halo_r_fstride = 0;
    double fourier = 0.4, gamma = 1.4, dt_dx = 0.0;
    int* error_flag = nullptr;
    DebugArgs dbg;
    // One process per GPU: the round's neighbour hand-off is fused into the
    // substep kernel. nb_flags[0]/[1] = rounds completed by the left/right
    // neighbour (this shard's memory); the boundary points wait for
    // *seq_base + round there before reading the halo and, once written, store
    // *seq_base + round + 1 into the left neighbour's [1] (sig_left) and the
    // right neighbour's [0] (sig_right). seq_base (device memory, set before
    // the rounds) keeps the kernel arguments constant across runs, so the round
    // loop can be replayed as a CUDA graph. nb_flags == nullptr: no hand-off.
    const unsigned* nb_flags = nullptr;
    const unsigned* seq_base = nullptr;
    unsigned round = 0;
    unsigned* sig_left = nullptr;
    unsigned* sig_right = nullptr;
    unsigned long long timeout_ns = 0;
    int sms = 148;                  // SMs of the launching device (queried once per shard)
};

// `debug` selects the instrumented instantiation (coverage / perturb).
cudaError_t launch_heat_classic(const ClassicArgs& a, cudaStream_t st);
cudaError_t launch_heat_tile(int kind, const TileArgs& a, cudaStream_t st, bool debug = false);
// Whether launch_heat_tile runs the fast build (+ its gated exact build, two
// launches) for these arguments (heat.cu heat_step).
bool heat_fast_form(const TileArgs& a);
// Points per thread of the heat tile kernel for width w; `tiles` (the
// smallest shard's tile count, or -1) lets small grids trade P for CTAs.
int heat_points_per_thread(int w, long long tiles = -1);

// Euler (flat = 0 lengthening, 1 flattening). Classic kernels update `out`
// in place (fields written by a substep are never read by it).
cudaError_t launch_euler_classic(int flat, const ClassicArgs& a, cudaStream_t st);
cudaError_t launch_euler_tile(int flat, int kind, const TileArgs& a, cudaStream_t st, bool debug = false);
cudaError_t launch_euler_unpack(const double* aos, double* st_fields, std::uint64_t N, std::uint64_t fs, int rec,
                                cudaStream_t st);
cudaError_t launch_euler_pack(const double* st_fields, double* aos, std::uint64_t N, std::uint64_t fs,
                              cudaStream_t st);
std::size_t euler_tile_smem_bytes(int flat, int w);

// one-process-per-GPU round ordering (sync.cu)
cudaError_t launch_wait_flags(const unsigned* flags, unsigned seq, int* err, std::uint64_t timeout_ns,
                              cudaStream_t st);
cudaError_t launch_signal_flags(unsigned* left_slot, unsigned* right_slot, unsigned seq, cudaStream_t st);
cudaError_t launch_set_u32(unsigned* p, unsigned v, cudaStream_t st);
cudaError_t launch_pingpong(const unsigned* mine, unsigned* peer, int iters, int starter, int* err,
                            std::uint64_t timeout_ns, cudaStream_t st);

} // namespace s1d
