// ff_runtime.cpp -- the C ABI of libfireflies (include/fireflies.h): context, particle groups,
// parameter table, sweep spec, projection binding and the launches.
//
// Design: caller-owned device memory (torch tensors), library-owned
// compiled modules; every launch is async on the bound stream with a by-value argument block
// (csrc/device/ff_args.h), so ff_set_param never touches the device.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost a branch unless a profiler attaches

#include "device/ff_args.h"
#include "ff_internal.hpp"

static_assert(sizeof(FFGroup) == 120, "FFGroup layout");
static_assert(FF_MAX_SCALED_ == FF_MAX_SCALED, "scaled-component table size");
static_assert(FF_MAX_DERIVED_ == FF_MAX_DERIVED, "derived-value table size");
static_assert(offsetof(FFStepArgs, g) == 840, "FFStepArgs layout");
static_assert(FF_MAX_PEERS_ == FF_MAX_PEERS, "peer table size");
static_assert(FF_MAX_DIM_ == FF_MAX_DIM, "bounds table size");
static_assert(FF_MAX_GROUPS_ == FF_MAX_GROUPS, "group table size");

namespace {

thread_local std::string g_err;

// NVTX range around an ABI call (tracing), visible to ncu --nvtx / Nsight timelines
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw ff::Error(FF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// Kernels of one system variant (swept parameter index). Each kernel is its own NVRTC program and
// library, compiled on first use (FF_KSEL in ff_device.cuh), so a system only pays for what it runs.
struct Module {
  cudaLibrary_t base_lib = nullptr;  // ff_init + ff_render
  cudaKernel_t init = nullptr;
  cudaKernel_t render = nullptr;
  cudaKernel_t lifted = nullptr;     // ff_read_lifted
  // step kernels by (ppt, tpb): 0 p1t128, 1 p1t256, 2 p1t512, 3 p2t128, 4 p2t256, 5 p4t128;
  // +6 = the same with position-linear colour compiled in (ff_project_colour)
  cudaKernel_t exchange = nullptr;  // (in base_lib)
  cudaKernel_t xbarrier = nullptr;  // (in base_lib) barrier of the fused (push) exchange
  // [variant][id]: variant = balanced + 2 long; balanced = exponentials shared with the FMA pipe,
  // long = the register budget for launches of many steps (emit_source balance, long_launch)
  // (+4: the per-thread reset redraw of the 4-particle kernel for launches of >= 50 steps)
  // (+8 push: the fused exchange's reductions, 1 = to every rank's image, 2 = to the multicast address)
  cudaLibrary_t step_lib[24][12] = {};
  cudaKernel_t step[24][12] = {};
  int occ[24][12] = {};
};

constexpr int kNumStep = 6;
constexpr int kSyncWords = 16 + FF_XS_WORDS;
  // tile counter line + the exchange sync block
int step_index(int ppt, int tpb) {
  if (ppt == 1) return tpb == 128 ? 0 : tpb == 256 ? 1 : tpb == 512 ? 2 : -1;
  if (ppt == 2) return tpb == 128 ? 3 : tpb == 256 ? 4 : -1;
  if (ppt == 4) return tpb == 128 ? 5 : -1;
  return -1;
}
const char* kStepNames[kNumStep] = {"ff_step_p1_t128", "ff_step_p1_t256", "ff_step_p1_t512", "ff_step_p2_t128",
                                    "ff_step_p2_t256", "ff_step_p4_t128"};
const int kStepPPT[kNumStep] = {1, 1, 1, 2, 2, 4};
const int kStepTPB[kNumStep] = {128, 256, 512, 128, 256, 128};

struct GroupRec {
  int64_t n_global = 0, first_global = 0, n_local = 0, slot_begin = 0, slot_end = 0;
  int dir = 1, colour = 0;
  uint64_t seed = 0;
  std::vector<float> lo, hi;
  int sweep_mode = -1;
  float sw_lo = 0, sw_hi = 0;
  uint64_t sw_seed = 0;
};

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

}  // namespace

struct ff_ctx {
  ff::System sys;
  std::vector<float> params;
  int device = 0;
  int nsm = 148;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  float* state = nullptr;
  int64_t pitch = 0, capacity = 0, next_slot = 0;
  std::vector<GroupRec> groups;
  int sweep_param = -1;
  std::map<int, Module> modules;  // by swept parameter index (-1 = none)
  // projection binding
  int proj = 0;
  int axes[3] = {0, 0, 0};
  float view[16] = {};
  int W = 0, H = 0, C = 0;
  uint32_t* image = nullptr;
  uint32_t* colour_img = nullptr;  // position-linear colour sums [3][H][W] (ff_project_colour)
  float col_lo[3] = {0, 0, 0}, col_s[3] = {0, 0, 0};
  float s0 = 0, s1 = 0;
  int ppt = 0, tpb = 0;
  int64_t launches = 0;
  // device-side reset (ff_set_reset): library-owned per-slot epoch / birth time, IC boxes
  int reset = 0;
  float t_max = 0.0f;
  std::vector<float> bound_lo, bound_hi;
  uint32_t* epoch = nullptr;
  float* birth = nullptr;
  float* ic_box = nullptr;
  std::vector<double> t_elapsed;  // per group: simulated time since creation (sum of |dt| n)
  // dynamic tile scheduler counter (library-owned, 8 bytes) and the fetch numbers used so far
  // [0] tile counter; from word 16 on: the exchange sync block (FF_XS_*, one 128-byte line per word)
  unsigned long long* tile_ctr = nullptr;
  uint64_t tile_base = 0;
  int grid_limit = 0;  // ff_set_grid_limit (0 = every resident block)
  // fused image exchange (ff_set_exchange): peer tables, barrier bookkeeping
  int xrank = 0, xworld = 0;
  uint32_t* ximg[FF_MAX_PEERS] = {};
  uint64_t* xsig[FF_MAX_PEERS] = {};
  uint64_t xbar = 0, xseq = 0, xtimeout_ns = 0;
  bool xused = false;
  uint32_t* xmc = nullptr;   // NVLS multicast address of the images (ff_set_exchange_multicast)
  int xpush = 0;             // ff_set_exchange_push: 0 sum pass, 1 peer reductions, 2 multicast reductions
  uint32_t* xpush_mc = nullptr;
  bool captured = false;     // a launch was captured into a CUDA graph: reset the tile counter per launch

  ~ff_ctx() {
    for (auto& m : modules) {
      if (m.second.base_lib) cudaLibraryUnload(m.second.base_lib);
      for (auto& row : m.second.step_lib)
        for (cudaLibrary_t l : row)
          if (l) cudaLibraryUnload(l);
    }
    free_reset_buffers();
    if (tile_ctr) cudaFree(tile_ctr);
  }

  void free_reset_buffers() {
    if (epoch) cudaFree(epoch);
    if (birth) cudaFree(birth);
    if (ic_box) cudaFree(ic_box);
    epoch = nullptr;
    birth = nullptr;
    ic_box = nullptr;
  }

  // (re)initialise the reset bookkeeping of group gi: epoch 0, birth = current group time, IC box
  void reset_init_group(size_t gi) {
    if (!epoch) return;
    const GroupRec& G = groups[gi];
    const int dim = sys.dim;
    const size_t n = (size_t)(G.slot_end - G.slot_begin);
    if (n) {
      ck(cudaMemsetAsync(epoch + G.slot_begin, 0, n * sizeof(uint32_t), stream), "cudaMemsetAsync epoch");
      std::vector<float> b(n, (float)t_elapsed[gi]);
      ck(cudaMemcpyAsync(birth + G.slot_begin, b.data(), n * sizeof(float), cudaMemcpyHostToDevice, stream),
         "cudaMemcpyAsync birth");
    }
    std::vector<float> box(3 * (size_t)dim);
    for (int d = 0; d < dim; ++d) {
      box[d] = G.lo[d];
      box[dim + d] = G.hi[d];
      box[2 * dim + d] = std::nextafter(G.hi[d], -INFINITY);
    }
    ck(cudaMemcpyAsync(ic_box + gi * 3 * (size_t)dim, box.data(), box.size() * sizeof(float), cudaMemcpyHostToDevice,
                       stream), "cudaMemcpyAsync ic_box");
    ck(cudaStreamSynchronize(stream), "cudaStreamSynchronize");  // host buffers go out of scope
  }

  cudaLibrary_t load(int sweep, int ksel, bool bal = true, bool long_launch = false, bool thread_redraw = false,
                     int push = 0) {
    std::vector<char> cubin = ff::compile_cubin(
        ff::emit_source(sys, sweep, ksel, nullptr, bal, long_launch, thread_redraw, push), "fireflies_system.cu");
    cudaLibrary_t lib = nullptr;
    ck(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0), "cudaLibraryLoadData");
    return lib;
  }

  // init + render kernels of the variant (compiled at first use of the variant)
  Module& module(int sweep) {
    auto it = modules.find(sweep);
    if (it != modules.end()) return it->second;
    Module m;
    m.base_lib = load(sweep, 100);
    ck(cudaLibraryGetKernel(&m.init, m.base_lib, "ff_init"), "cudaLibraryGetKernel(ff_init)");
    ck(cudaLibraryGetKernel(&m.render, m.base_lib, "ff_render"), "cudaLibraryGetKernel(ff_render)");
    ck(cudaLibraryGetKernel(&m.exchange, m.base_lib, "ff_exchange"), "cudaLibraryGetKernel(ff_exchange)");
    ck(cudaLibraryGetKernel(&m.xbarrier, m.base_lib, "ff_xbarrier"), "cudaLibraryGetKernel(ff_xbarrier)");
    ck(cudaLibraryGetKernel(&m.lifted, m.base_lib, "ff_lifted"), "cudaLibraryGetKernel(ff_lifted)");
    return modules.emplace(sweep, m).first->second;
  }

  // step kernel `id` (0-11) of variant v (balanced + 2 long + 4 thread redraw + 8 push), compiled at
  // its first launch
  cudaKernel_t step_kernel(Module& m, int sweep, int id, int v) {
    if (!m.step[v][id]) {
      m.step_lib[v][id] = load(sweep, id, (v & 1) != 0, (v & 2) != 0, (v & 4) != 0, v >> 3);
      const std::string name = std::string(kStepNames[id % kNumStep]) + (id >= kNumStep ? "_c" : "");
      ck(cudaLibraryGetKernel(&m.step[v][id], m.step_lib[v][id], name.c_str()), "cudaLibraryGetKernel(ff_step)");
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)m.step[v][id], kStepTPB[id % kNumStep],
                                                        0) != cudaSuccess) {
        cudaGetLastError();
        occ = 1;
      }
      m.occ[v][id] = occ > 0 ? occ : 1;
    }
    return m.step[v][id];
  }
  // the long-launch register budget differs only for the packed 128-thread kernel of systems of
  // <= 4 variables (emit_source long_launch); other kernels share the short variant's module
  // and the 4-particle kernel's reset redraw is per thread for launches of >= 50 steps (a 100-step
  // Lorenz frame resets nearly every backward particle: 1029 vs 1051 us), warp-cooperative below
  // (S = 10: 164 vs 175 us; tools/r02/run23.sh)
  int variant_for(bool bal, int id, int64_t n_steps) const {
    const bool lng = n_steps >= 8 && sys.dim <= 4 && (id % kNumStep == 3 || id % kNumStep == 5);
    const bool thread_redraw = n_steps >= 50 && id % kNumStep == 5;
    return (bal ? 1 : 0) + (lng ? 2 : 0) + (thread_redraw ? 4 : 0);
  }
  // pipe-balanced (throughput) kernels for launches that fill the GPU; a launch with fewer tiles than
  // two per SM is latency-bound (one particle's RK4 chain is the critical path) and uses MUFU only
  bool balanced_for(int64_t ntiles) const { return ntiles >= 2 * (int64_t)nsm; }

  // the uniform factors of the split components of a system variant, in slot order (cached)
  std::map<int, std::vector<ff::NodeP>> scale_cache;
  const std::vector<ff::NodeP>& scale_asts(int sweep) {
    auto it = scale_cache.find(sweep);
    if (it != scale_cache.end()) return it->second;
    std::vector<ff::NodeP> rest, sc, out;
    const std::vector<int> slot = ff::split_scales(sys, sweep, &rest, &sc);
    for (int d = 0; d < sys.dim; ++d)
      if (slot[d] >= 0) {
        if ((int)out.size() <= slot[d]) out.resize(slot[d] + 1);
        out[slot[d]] = sc[d];   // components sharing a factor share its slot
      }
    return scale_cache.emplace(sweep, out).first->second;
  }

  // host program of the RHS's loop-invariant values of a system variant (cached)
  std::map<std::pair<int, bool>, ff::UProgram> prog_cache;
  const ff::UProgram& uprogram(int sweep, bool bal) {
    auto key = std::make_pair(sweep, bal);
    auto it = prog_cache.find(key);
    if (it != prog_cache.end()) return it->second;
    ff::UProgram prog;
    ff::emit_source(sys, sweep, 100, &prog, bal);
    return prog_cache.emplace(key, prog).first->second;
  }

  int find_param(const char* name) const {
    if (!name) throw ff::Error(FF_ERR_INVALID_ARG, "parameter name is NULL");
    for (size_t k = 0; k < sys.param_names.size(); ++k)
      if (sys.param_names[k] == name) return (int)k;
    throw ff::Error(FF_ERR_UNKNOWN_SYMBOL, std::string("unknown parameter '") + name + "'");
  }

  const GroupRec& group(int gid) const {
    if (gid < 0 || gid >= (int)groups.size()) throw ff::Error(FF_ERR_INVALID_ARG, "bad group id");
    return groups[gid];
  }

  void default_launch(int& ppt_out, int& tpb_out, int64_t n_steps = 100) {
    // too few particles to give every SM a 256-particle tile: the launch is latency-bound (each
    // particle's RK4 chain is the critical path), so spread it over as many SMs as possible with one
    // particle per thread (configs[0], 10 k STN-GPe particles: 1.9x faster than packed pairs)
    if (!ppt && !tpb && next_slot < 256 * (int64_t)nsm) {
      ppt_out = 1;
      tpb_out = 128;
      return;
    }
    // short launches (1-4 steps) of small systems, with or without an image: 16-byte vector I/O, 4
    // particles per thread, 8 blocks/SM (round 2, tools/r02/run45.sh, Lorenz 8.4 M with the reset
    // rule: S = 1 with image 91 -> 75 us against packed pairs, S = 2 / 4 109 -> 99 / 121 -> 113 us,
    // no image S = 1 44 -> 39 us; STN-GPe bifurcation S = 1 146 -> 138 us. Round 1 kept pairs when an
    // image was bound: its projection and histogram code was heavier.)
    if (!ppt && !tpb && sys.dim <= 4 && n_steps <= 4) {
      ppt_out = 4;
      tpb_out = 128;
      return;
    }
    // measured on B200: packed pairs win for the paper's systems; 15-D HH needs the
    // smaller block for its ~248-register pair kernel. Small systems: launches of >= 50 steps over
    // >= 4 tiles of 512 per SM run 256-thread blocks (fewer tile fetches and block barriers per
    // particle: Lorenz S = 100 8.13 -> 8.22e11), shorter ones 128-thread blocks (S = 10: 5.42 vs 5.34e11)
    const bool wide = n_steps >= 50 && next_slot >= 4 * 512 * (int64_t)nsm;
    // FMA-bound small systems (no MUFU op): longer launches run 4 particles per thread too (two
    // independent FFMA2 chains, 8 blocks / <= 64 registers): Lorenz S = 7 / 10 / 100 / 1000: -7% / -4% /
    // -2.3% / -2.8% time (tools/r01/gpu_run76.sh, tools/r02/run49.sh); a MUFU-bound one (STN-GPe) loses
    // 4-6% there from 10 steps on
    if (!ppt && !tpb && sys.dim <= 4 && next_slot >= 4 * 512 * (int64_t)nsm &&
        uprogram(sweep_param, true).mufu_per_step == 0) {
      ppt_out = 4;
      tpb_out = 128;
      return;
    }
    ppt_out = ppt ? ppt : (sys.dim <= 16 ? 2 : 1);
    tpb_out = tpb ? tpb : (sys.dim <= 4 ? (wide && ppt_out == 2 ? 256 : 128) : (sys.dim <= 8 ? 256 : 128));
  }

  // the group-table fields that identify particles and their lifted parameter (shared by every launch
  // that evaluates ff_sweep_value)
  void fill_identity(size_t gi, FFGroup& g) const {
    const GroupRec& G = groups[gi];
    g.seed = G.seed;
    g.slot_begin = G.slot_begin;
    g.slot_end = G.slot_end;
    g.n_local = G.n_local;
    g.first_global = G.first_global;
    g.n_global = G.n_global;
    g.colour = G.colour;
    g.sweep_mode = (sweep_param >= 0) ? G.sweep_mode : -1;
    g.sweep_seed = G.sw_seed;
    g.sw_lo = G.sw_lo;
    g.sw_hi = G.sw_hi;
    g.sw_top = std::nextafter(G.sw_hi, -INFINITY);
    g.sw_val = sweep_param >= 0 ? params[sweep_param] : 0.0f;
  }

  void launch_step(int64_t n_steps, float dt) {
    if (groups.empty()) throw ff::Error(FF_ERR_STATE, "no particle groups");
    if (!std::isfinite(dt)) throw ff::Error(FF_ERR_INVALID_ARG, "dt is not finite");
    if (xworld) {
      if (image != ximg[xrank]) throw ff::Error(FF_ERR_STATE, "exchange: the bound image is not this rank's peer image");
      if (colour_img) throw ff::Error(FF_ERR_STATE, "exchange: position colour images are not exchanged");
    }
    int p, t;
    default_launch(p, t, n_steps);
    const int si = step_index(p, t);
    Module& m = module(sweep_param);
    // CUDA-graph capture of frames: a captured launch replays with the arguments it
    // was captured with, so it must not depend on host bookkeeping that advances per launch
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(stream, &cs), "cudaStreamIsCapturing");
    const bool capturing = cs == cudaStreamCaptureStatusActive;
    if (capturing) {
      if (reset & 2) throw ff::Error(FF_ERR_STATE, "graph capture: the age rule (t_max) needs the launch's time");
      if (xworld > 1) throw ff::Error(FF_ERR_STATE, "graph capture: an exchanging context cannot be captured");
      captured = true;
    }
    if (captured) {
      // the tile counter restarts at 0 before every launch (a memset node in a graph), so replays and
      // the launches issued after them agree on it
      ck(cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned long long), stream), "cudaMemsetAsync tile counter");
      tile_base = 0;
    }
    FFStepArgs a;
    std::memset(&a, 0, sizeof a);
    a.state = state;
    a.pitch = pitch;
    a.slots_total = next_slot;
    a.n_steps = n_steps;
    a.image = image;
    a.colour_img = image ? colour_img : nullptr;
    for (int k = 0; k < 3; ++k) {
      a.col_lo[k] = col_lo[k];
      a.col_s[k] = col_s[k];
    }
    a.proj = image ? proj : 0;
    a.W = W;
    a.H = H;
    a.C = C;
    for (int j = 0; j < 3; ++j) a.axes[j] = axes[j];
    std::memcpy(a.view, view, sizeof view);
    a.s0 = s0;
    a.s1 = s1;
    a.fW = (float)W;
    a.fH = (float)H;
    a.hW = (float)W * 0.5f;
    a.hH = (float)H * 0.5f;
    a.one = 1.0f;
    a.ax_id = 1;
    for (int j = 0; j < proj; ++j) a.ax_id &= axes[j] == j;
    a.n_groups = (int)groups.size();
    a.reset = n_steps > 0 ? reset : 0;
    a.t_max = t_max;
    a.epoch = epoch;
    a.birth = birth;
    a.ic_box = ic_box;
    a.tile_ctr = tile_ctr;
    a.tile_base = tile_base;
    for (size_t d = 0; d < bound_lo.size(); ++d) {
      a.bound_lo[d] = bound_lo[d];
      a.bound_hi[d] = bound_hi[d];
    }
    // uniform factors of the split components (ff::split_scales), at the current parameter values
    std::vector<float> scales;
    for (const ff::NodeP& n : scale_asts(sweep_param)) scales.push_back((float)ff::eval_uniform(n, params));
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const GroupRec& G = groups[gi];
      FFGroup& g = a.g[gi];
      t_elapsed[gi] += std::fabs((double)dt) * (double)n_steps;
      fill_identity(gi, g);
      g.t_now = (float)t_elapsed[gi];
      const float h = (float)G.dir * dt;
      g.h = h;
      g.h2 = h * 0.5f;
      g.h6 = h / 6.0f;
      g.nh = -g.h;
      g.nh2 = -g.h2;
      g.nh6 = -g.h6;
      for (size_t k = 0; k < scales.size(); ++k) {
        const float sc = scales[k];
        float* q = a.hs[gi][k];
        q[0] = g.h * sc;
        q[1] = g.h2 * sc;
        q[2] = g.h6 * sc;
        q[3] = -q[0];
        q[4] = -q[1];
        q[5] = -q[2];
      }
    }
    for (size_t k = 0; k < params.size(); ++k) a.p[k] = params[k];
    const int64_t tile = (int64_t)p * t;
    const int64_t ntiles = next_slot / tile;
    const bool bal = balanced_for(ntiles);
    {
      const std::vector<float> q = ff::eval_program(uprogram(sweep_param, bal), params);
      for (size_t k = 0; k < q.size(); ++k) a.q[k] = q[k];
    }
    // fused (push) exchange: the histogram's reductions go to every rank's image, between two barriers
    const int push = (xworld > 1 && image) ? xpush : 0;
    if (push) {
      a.push_n = push == 2 ? 1 : xworld;
      for (int p = 0; p < a.push_n; ++p) a.push_img[p] = push == 2 ? xpush_mc : ximg[p];
    }
    if (ntiles == 0) {
      if (push) {                           // this rank has no particles; its peers still wait for it
        launch_xbarrier(m, 1);
        launch_xbarrier(m, 2);
        ++xseq;
      } else if (xworld > 1) {
        launch_exchange(m);
      }
      return;
    }
    // position-linear colour: 3 extra per-block table planes in dynamic shared memory
    const bool colour = image && colour_img;
    const size_t dyn_smem = colour ? 3 * 1024 * sizeof(uint32_t) : 0;
    const int kid = si + (colour ? kNumStep : 0);
    const int var = variant_for(bal, kid, n_steps) + 8 * push;
    if (capturing && !m.step[var][kid])
      throw ff::Error(FF_ERR_STATE, "graph capture: this launch's kernel is not compiled yet -- run the frame once "
                                    "before capturing it");
    const cudaKernel_t kern = step_kernel(m, sweep_param, kid, var);
    int occ = m.occ[var][kid];
    if (colour) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)kern, t, dyn_smem) != cudaSuccess) {
        cudaGetLastError();
        occ = 1;
      }
      occ = occ > 0 ? occ : 1;
    }
    int64_t resident = (int64_t)nsm * occ;
    if (grid_limit > 0 && grid_limit < resident) resident = grid_limit;
    const unsigned grid = (unsigned)(ntiles < resident ? ntiles : resident);
    // static tile rounds for 1-2-step launches (ff_step_body): all but the last round of tiles
    // (all-static tile rounds -- no counter, no per-tile barrier -- measured slower at S = 1: 99 vs
    // 93 us, tools/r02/run04.sh; so is a register prefetch of the next tile's state: 107 us)
    const int64_t ns = (n_steps <= 2 && sys.dim <= 8 && ntiles / grid >= 2) ? ntiles / grid - 1 : 0;
    a.static_rounds = (int)ns;
    void* args[] = {&a};
    if (push) launch_xbarrier(m, 1);
    ck(cudaLaunchKernel((const void*)kern, dim3(grid), dim3(t), args, dyn_smem, stream), "launch ff_step");
    // static rounds first (ff_step_body), then each block fetches dynamic tiles until it sees one past
    // the end: the counter advances by the dynamic tiles + grid
    tile_base += (uint64_t)(ntiles - ns * (int64_t)grid) + grid;
    ++launches;
    if (push) {
      launch_xbarrier(m, 2);
      ++xseq;
    } else if (xworld > 1 && image) {
      launch_exchange(m);  // (one rank: its image already is the sum)
    }
  }

  // a barrier of the fused (push) exchange (ff_xbarrier in ff_device.cuh): phase 1 before the pushing
  // launch, 2 after it; barrier values 2 xseq + phase on the exchange's signal words
  void launch_xbarrier(Module& m, int phase) {
    FFXchgArgs x;
    std::memset(&x, 0, sizeof x);
    for (int p = 0; p < xworld; ++p) x.sig[p] = reinterpret_cast<ff_u64*>(xsig[p]);
    x.sync = reinterpret_cast<ff_u64*>(tile_ctr) + 16;
    x.seq = xseq;
    x.timeout_ns = xtimeout_ns;
    x.rank = xrank;
    x.world = xworld;
    x.phase = phase;
    void* args[] = {&x};
    ck(cudaLaunchKernel((const void*)m.xbarrier, dim3(1), dim3(32), args, 0, stream), "launch ff_xbarrier");
    xused = true;
    ++launches;
  }

  // the image exchange after a binning launch (ff_set_exchange; ff_device.cuh "image exchange")
  void launch_exchange(Module& m) {
    FFXchgArgs x;
    std::memset(&x, 0, sizeof x);
    for (int p = 0; p < xworld; ++p) {
      x.img[p] = ximg[p];
      x.sig[p] = reinterpret_cast<ff_u64*>(xsig[p]);
    }
    x.sync = reinterpret_cast<ff_u64*>(tile_ctr) + 16;
    x.words = (ff_u64)W * (ff_u64)H * (ff_u64)C;
    x.bar_base = xbar;
    x.seq = xseq;
    x.timeout_ns = xtimeout_ns;
    x.rank = xrank;
    x.world = xworld;
    x.mc = xmc;
    // 2 blocks of 256 threads per SM (fewer if ff_set_grid_limit says so): enough loads in flight
    unsigned grid = (unsigned)(2 * nsm);
    if (grid_limit > 0 && (unsigned)grid_limit < grid) grid = (unsigned)grid_limit;
    void* args[] = {&x};
    ck(cudaLaunchKernel((const void*)m.exchange, dim3(grid), dim3(256), args, 0, stream), "launch ff_exchange");
    xbar += grid;
    ++xseq;
    xused = true;
    ++launches;
  }
};

// ---------------------------------------------------------------- ABI helpers
#define FF_TRY try {
#define FF_CATCH                                                         \
  }                                                                      \
  catch (const ff::Error& e) {                                           \
    g_err = e.what();                                                    \
    return e.status;                                                     \
  }                                                                      \
  catch (const std::bad_alloc&) {                                        \
    g_err = "out of host memory";                                        \
    return FF_ERR_OOM;                                                   \
  }                                                                      \
  catch (const std::exception& e) {                                      \
    g_err = e.what();                                                    \
    return FF_ERR_INVALID_ARG;                                           \
  }                                                                      \
  return FF_OK;

static void need(bool c, ff_status s, const char* msg) {
  if (!c) throw ff::Error(s, msg);
}

static ff_status copy_out(const std::string& data, bool text, void* buf, size_t cap, size_t* len) {
  if (len) *len = data.size();
  if (buf && cap) {
    if (text) {
      size_t n = data.size() < cap - 1 ? data.size() : cap - 1;
      std::memcpy(buf, data.data(), n);
      static_cast<char*>(buf)[n] = '\0';
    } else {
      need(cap >= data.size(), FF_ERR_INVALID_ARG, "buffer too small");
      std::memcpy(buf, data.data(), data.size());
    }
  }
  return FF_OK;
}

extern "C" {

const char* ff_last_error(void) { return g_err.c_str(); }

int ff_abi_version(void) { return FF_ABI_VERSION; }

ff_status ff_build_info(char* buf, size_t cap, size_t* len) {
  FF_TRY
  std::string info = "libfireflies ABI " + std::to_string(FF_ABI_VERSION) + "; target sm_100a CUBIN; " +
                     ff::nvrtc_description();
  return copy_out(info, true, buf, cap, len);
  FF_CATCH
}

ff_status ff_emit_source(const ff_system* sys, int sweep_param, char* buf, size_t cap, size_t* len) {
  FF_TRY
  ff::System s = ff::parse_system(sys);
  std::string src = ff::emit_source(s, sweep_param);
  return copy_out(src, true, buf, cap, len);
  FF_CATCH
}

ff_status ff_compile_cubin(const ff_system* sys, int sweep_param, void* buf, size_t cap, size_t* len) {
  FF_TRY
  ff::System s = ff::parse_system(sys);
  std::vector<char> c = ff::compile_cubin(ff::emit_source(s, sweep_param), "fireflies_system.cu");
  return copy_out(std::string(c.begin(), c.end()), false, buf, cap, len);
  FF_CATCH
}

ff_status ff_create(const ff_system* sys, int device, ff_ctx** out) {
  FF_TRY
  need(out != nullptr, FF_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  ff::System s = ff::parse_system(sys);
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  need(device >= 0 && device < ndev, FF_ERR_INVALID_ARG, "device index out of range");
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaFree(nullptr), "context init");
  ff_ctx* c = new ff_ctx();
  try {
    c->sys = std::move(s);
    c->params = c->sys.param_default;
    c->device = device;
    ck(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
    c->module(-1);
    ck(cudaMalloc(&c->tile_ctr, kSyncWords * sizeof(unsigned long long)), "cudaMalloc tile counter");
    ck(cudaMemset(c->tile_ctr, 0, kSyncWords * sizeof(unsigned long long)), "cudaMemset tile counter");
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  FF_CATCH
}

ff_status ff_destroy(ff_ctx* ctx) {
  FF_TRY
  delete ctx;
  FF_CATCH
}

ff_status ff_set_stream(ff_ctx* ctx, void* stream) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  ctx->stream = (cudaStream_t)stream;
  FF_CATCH
}

ff_status ff_set_shard(ff_ctx* ctx, int rank, int world) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(world >= 1 && rank >= 0 && rank < world, FF_ERR_INVALID_ARG, "need 0 <= rank < world");
  need(ctx->groups.empty(), FF_ERR_STATE, "ff_set_shard must precede ff_init_group");
  ctx->rank = rank;
  ctx->world = world;
  FF_CATCH
}

ff_status ff_bind_state(ff_ctx* ctx, float* dev_state, int64_t pitch, int64_t capacity) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(dev_state != nullptr, FF_ERR_INVALID_ARG, "state pointer is NULL");
  need(((uintptr_t)dev_state & 15) == 0, FF_ERR_INVALID_ARG, "state pointer must be 16-byte aligned");
  need(pitch > 0 && pitch % FF_TILE == 0, FF_ERR_INVALID_ARG, "pitch must be a positive multiple of FF_TILE");
  need(capacity >= 0 && capacity <= pitch, FF_ERR_INVALID_ARG, "need 0 <= capacity <= pitch");
  ctx->state = dev_state;
  ctx->pitch = pitch;
  ctx->capacity = capacity;
  ctx->next_slot = 0;
  ctx->groups.clear();
  ctx->t_elapsed.clear();
  ctx->reset = 0;
  ctx->free_reset_buffers();
  FF_CATCH
}

static int64_t shard_begin(int64_t n, int r, int w) { return (int64_t)((__int128)n * r / w); }

ff_status ff_shard_range(int64_t n_global, int rank, int world, int64_t* first, int64_t* count) {
  FF_TRY
  need(first && count, FF_ERR_INVALID_ARG, "NULL argument");
  need(n_global >= 0, FF_ERR_INVALID_ARG, "n_global must be >= 0");
  need(world >= 1 && rank >= 0 && rank < world, FF_ERR_INVALID_ARG, "need 0 <= rank < world");
  *first = shard_begin(n_global, rank, world);
  *count = shard_begin(n_global, rank + 1, world) - *first;
  FF_CATCH
}

ff_status ff_group_slots(ff_ctx* ctx, int64_t n_global, int64_t* slots) {
  FF_TRY
  need(ctx && slots, FF_ERR_INVALID_ARG, "NULL argument");
  need(n_global >= 1, FF_ERR_INVALID_ARG, "n_global must be >= 1");
  int64_t nl = shard_begin(n_global, ctx->rank + 1, ctx->world) - shard_begin(n_global, ctx->rank, ctx->world);
  *slots = round_up(nl, FF_TILE);
  FF_CATCH
}

ff_status ff_init_group(ff_ctx* ctx, const float* ic_lo, const float* ic_hi, int64_t n_global, int direction,
                        int colour, uint64_t seed, int* group_id) {
  NvtxRange nvtx("ff_init_group");
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(ic_lo && ic_hi, FF_ERR_INVALID_ARG, "ic_lo / ic_hi is NULL");
  need(n_global >= 1, FF_ERR_INVALID_ARG, "n_global must be >= 1");
  need(direction == 1 || direction == -1, FF_ERR_INVALID_ARG, "direction must be +1 or -1");
  need(colour >= 0, FF_ERR_INVALID_ARG, "colour must be >= 0");
  need(ctx->state != nullptr, FF_ERR_STATE, "no state bound (ff_bind_state)");
  need((int)ctx->groups.size() < FF_MAX_GROUPS, FF_ERR_STATE, "too many groups");
  const int dim = ctx->sys.dim;
  GroupRec g;
  for (int d = 0; d < dim; ++d) {
    need(std::isfinite(ic_lo[d]) && std::isfinite(ic_hi[d]) && ic_lo[d] < ic_hi[d], FF_ERR_INVALID_ARG,
         "initial-condition box needs finite lo < hi in every dimension");
    g.lo.push_back(ic_lo[d]);
    g.hi.push_back(ic_hi[d]);
  }
  g.n_global = n_global;
  g.first_global = shard_begin(n_global, ctx->rank, ctx->world);
  g.n_local = shard_begin(n_global, ctx->rank + 1, ctx->world) - g.first_global;
  g.slot_begin = ctx->next_slot;
  g.slot_end = g.slot_begin + round_up(g.n_local, FF_TILE);
  need(g.slot_end <= ctx->capacity, FF_ERR_STATE, "state capacity exceeded");
  g.dir = direction;
  g.colour = colour;
  g.seed = seed;
  if (ctx->image && colour >= ctx->C) throw ff::Error(FF_ERR_STATE, "colour >= channels of the bound image");
  Module& m = ctx->module(ctx->sweep_param);
  if (g.slot_end > g.slot_begin) {
    // FFInitArgs (ff_device.cuh): 7 x 8-byte fields, then lo[dim], hi[dim], top[dim] floats.
    std::vector<unsigned char> buf(56 + 12 * (size_t)dim + 8, 0);
    int64_t f[6] = {(int64_t)(uintptr_t)ctx->state, ctx->pitch, g.slot_begin, g.slot_end, g.n_local, g.first_global};
    std::memcpy(buf.data(), f, 48);
    std::memcpy(buf.data() + 48, &seed, 8);
    float* fl = reinterpret_cast<float*>(buf.data() + 56);
    for (int d = 0; d < dim; ++d) {
      fl[d] = g.lo[d];
      fl[dim + d] = g.hi[d];
      fl[2 * dim + d] = std::nextafter(g.hi[d], -INFINITY);
    }
    void* args[] = {buf.data()};
    const unsigned grid = (unsigned)((g.slot_end - g.slot_begin) / 256);
    ck(cudaLaunchKernel((const void*)m.init, dim3(grid), dim3(256), args, 0, ctx->stream), "launch ff_init");
    ++ctx->launches;
  }
  ctx->next_slot = g.slot_end;
  ctx->groups.push_back(g);
  ctx->t_elapsed.push_back(0.0);
  ctx->reset_init_group(ctx->groups.size() - 1);
  if (group_id) *group_id = (int)ctx->groups.size() - 1;
  FF_CATCH
}

ff_status ff_set_reset(ff_ctx* ctx, int enable, const float* lo, const float* hi, float t_max) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  if (!enable) {
    ctx->reset = 0;
    return FF_OK;
  }
  need(ctx->state != nullptr, FF_ERR_STATE, "no state bound (ff_bind_state)");
  need((lo == nullptr) == (hi == nullptr), FF_ERR_INVALID_ARG, "give both bounds or neither");
  const int dim = ctx->sys.dim;
  std::vector<float> blo, bhi;
  if (lo) {
    for (int d = 0; d < dim; ++d) {
      need(!std::isnan(lo[d]) && !std::isnan(hi[d]) && lo[d] <= hi[d], FF_ERR_INVALID_ARG, "bounds need lo <= hi");
      blo.push_back(lo[d]);
      bhi.push_back(hi[d]);
    }
  }
  need(!std::isnan(t_max), FF_ERR_INVALID_ARG, "t_max is NaN");
  // the per-slot bookkeeping is allocated once per state binding and kept: the epochs define the
  // particles' lifted-parameter values (reading R16), so re-enabling or changing the rule must not
  // restart them
  const bool fresh = ctx->epoch == nullptr;
  if (fresh) {
    const size_t cap = (size_t)ctx->pitch;
    ck(cudaMalloc(&ctx->epoch, cap * sizeof(uint32_t)), "cudaMalloc epoch");
    ck(cudaMalloc(&ctx->birth, cap * sizeof(float)), "cudaMalloc birth");
    ck(cudaMalloc(&ctx->ic_box, (size_t)FF_MAX_GROUPS * 3 * dim * sizeof(float)), "cudaMalloc ic_box");
  }
  ctx->bound_lo = blo;
  ctx->bound_hi = bhi;
  ctx->t_max = t_max;
  ctx->reset = (lo ? 1 : 0) | ((t_max > 0.0f && std::isfinite(t_max)) ? 2 : 0);
  if (!ctx->reset) ctx->reset = 4;  // non-finite check only
  if (fresh)
    for (size_t gi = 0; gi < ctx->groups.size(); ++gi) ctx->reset_init_group(gi);
  FF_CATCH
}

ff_status ff_read_epochs(ff_ctx* ctx, int group_id, int64_t first, int64_t count, uint32_t* host) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(ctx->reset && ctx->epoch, FF_ERR_STATE, "reset is not enabled");
  const GroupRec& g = ctx->group(group_id);
  need(host || count == 0, FF_ERR_INVALID_ARG, "host buffer is NULL");
  need(first >= 0 && count >= 0 && first + count <= g.n_local, FF_ERR_INVALID_ARG, "particle range out of bounds");
  if (count) {
    ck(cudaMemcpyAsync(host, ctx->epoch + g.slot_begin + first, (size_t)count * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, ctx->stream), "cudaMemcpyAsync epochs");
    ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  }
  FF_CATCH
}

ff_status ff_read_lifted(ff_ctx* ctx, int group_id, int64_t first, int64_t count, float* host) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  const GroupRec& g = ctx->group(group_id);
  need(ctx->sweep_param >= 0, FF_ERR_STATE, "no parameter is swept");
  need(host || count == 0, FF_ERR_INVALID_ARG, "host buffer is NULL");
  need(first >= 0 && count >= 0 && first + count <= g.n_local, FF_ERR_INVALID_ARG, "particle range out of bounds");
  if (count == 0) return FF_OK;
  Module& m = ctx->module(ctx->sweep_param);
  FFLiftedArgs a;
  std::memset(&a, 0, sizeof a);
  ctx->fill_identity((size_t)group_id, a.g);
  a.epoch = ctx->epoch;
  a.slot = g.slot_begin + first;
  a.local = first;
  a.count = count;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&a.out), (size_t)count * sizeof(float), ctx->stream), "cudaMallocAsync");
  void* args[] = {&a};
  const cudaError_t le = cudaLaunchKernel((const void*)m.lifted, dim3((unsigned)((count + 255) / 256)), dim3(256), args,
                                         0, ctx->stream);
  cudaError_t ce = cudaSuccess;
  if (le == cudaSuccess)
    ce = cudaMemcpyAsync(host, a.out, (size_t)count * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream);
  cudaFreeAsync(a.out, ctx->stream);
  ck(le, "launch ff_lifted");
  ck(ce, "cudaMemcpyAsync lifted");
  ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  ++ctx->launches;
  FF_CATCH
}

ff_status ff_group_info(ff_ctx* ctx, int group_id, int64_t* slot_begin, int64_t* n_local, int64_t* first_global) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  const GroupRec& g = ctx->group(group_id);
  if (slot_begin) *slot_begin = g.slot_begin;
  if (n_local) *n_local = g.n_local;
  if (first_global) *first_global = g.first_global;
  FF_CATCH
}

ff_status ff_set_param(ff_ctx* ctx, const char* name, float value) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  const int k = ctx->find_param(name);
  need(std::isfinite(value), FF_ERR_INVALID_ARG, "parameter value is not finite");
  if (!(value >= ctx->sys.param_min[k] && value <= ctx->sys.param_max[k]))
    throw ff::Error(FF_ERR_RANGE, std::string("value outside the allowed range of '") + name + "'");
  ctx->params[k] = value;
  FF_CATCH
}

ff_status ff_get_param(ff_ctx* ctx, const char* name, float* value) {
  FF_TRY
  need(ctx && value, FF_ERR_INVALID_ARG, "NULL argument");
  *value = ctx->params[ctx->find_param(name)];
  FF_CATCH
}

ff_status ff_sweep_param(ff_ctx* ctx, int group_id, const char* name, float lo, float hi, int mode, uint64_t seed) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  const int k = ctx->find_param(name);
  ctx->group(group_id);
  need(std::isfinite(lo) && std::isfinite(hi) && lo < hi, FF_ERR_INVALID_ARG, "sweep range needs finite lo < hi");
  need(mode == 0 || mode == 1, FF_ERR_INVALID_ARG, "mode must be 0 (uniform) or 1 (linspace)");
  need(ctx->sweep_param < 0 || ctx->sweep_param == k, FF_ERR_STATE, "another parameter is already swept");
  ctx->module(k);  // compile the variant now so errors surface here
  ctx->sweep_param = k;
  GroupRec& g = ctx->groups[group_id];
  g.sweep_mode = mode;
  g.sw_lo = lo;
  g.sw_hi = hi;
  g.sw_seed = seed;
  FF_CATCH
}

ff_status ff_project(ff_ctx* ctx, const int* axes, int n_axes, const float* view, int W, int H, int C,
                     uint32_t* image) {
  NvtxRange nvtx("ff_project");
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  if (!image) {
    ctx->image = nullptr;
    ctx->colour_img = nullptr;
    ctx->proj = 0;
    ctx->xworld = 0;
    ctx->xmc = nullptr;
    return FF_OK;
  }
  need(axes && view, FF_ERR_INVALID_ARG, "axes / view is NULL");
  need(n_axes == 2 || n_axes == 3, FF_ERR_INVALID_ARG, "n_axes must be 2 or 3");
  need(W >= 1 && H >= 1 && C >= 1, FF_ERR_INVALID_ARG, "W, H, C must be >= 1");
  need((uint64_t)W * H * C < 0xffffffffull, FF_ERR_INVALID_ARG, "image too large");
  need(((uintptr_t)image & 3) == 0, FF_ERR_INVALID_ARG, "image must be 4-byte aligned");
  for (int j = 0; j < n_axes; ++j) {
    need(axes[j] >= 0 && axes[j] <= ctx->sys.dim, FF_ERR_INVALID_ARG, "axis index out of range");
    need(axes[j] < ctx->sys.dim || ctx->sweep_param >= 0, FF_ERR_INVALID_ARG,
         "axis index dim names the swept parameter, but none is swept");
  }
  for (const GroupRec& g : ctx->groups) need(g.colour < C, FF_ERR_STATE, "a group's colour is >= C");
  float v[16] = {};
  if (n_axes == 2) {
    for (int j = 0; j < 4; ++j) need(std::isfinite(view[j]), FF_ERR_INVALID_ARG, "window is not finite");
    need(view[0] < view[1] && view[2] < view[3], FF_ERR_INVALID_ARG, "window needs lo < hi");
    std::memcpy(v, view, 4 * sizeof(float));
    ctx->s0 = (float)W / (view[1] - view[0]);
    ctx->s1 = (float)H / (view[3] - view[2]);
  } else {
    for (int j = 0; j < 16; ++j) need(std::isfinite(view[j]), FF_ERR_INVALID_ARG, "matrix is not finite");
    std::memcpy(v, view, 16 * sizeof(float));
  }
  ctx->proj = n_axes;
  for (int j = 0; j < 3; ++j) ctx->axes[j] = axes[j < n_axes ? j : 0];
  std::memcpy(ctx->view, v, sizeof v);
  ctx->W = W;
  ctx->H = H;
  ctx->C = C;
  ctx->image = image;
  ctx->xworld = 0;  // (re)binding an image ends an exchange (ff_set_exchange again)
  ctx->xmc = nullptr;
  ctx->xpush = 0;
  ctx->xpush_mc = nullptr;
  if (!ctx->groups.empty()) ctx->launch_step(0, 0.0f);
  FF_CATCH
}

ff_status ff_project_colour(ff_ctx* ctx, const float* lo, const float* hi, uint32_t* dev_colour_img) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  if (!dev_colour_img) {
    ctx->colour_img = nullptr;
    return FF_OK;
  }
  need(ctx->image != nullptr, FF_ERR_STATE, "bind an image with ff_project first");
  need(lo && hi, FF_ERR_INVALID_ARG, "lo / hi is NULL");
  need(((uintptr_t)dev_colour_img & 3) == 0, FF_ERR_INVALID_ARG, "colour image must be 4-byte aligned");
  for (int k = 0; k < 3; ++k) {
    ctx->col_lo[k] = 0.0f;
    ctx->col_s[k] = 0.0f;
  }
  for (int k = 0; k < ctx->proj; ++k) {
    need(std::isfinite(lo[k]) && std::isfinite(hi[k]) && lo[k] < hi[k], FF_ERR_INVALID_ARG,
         "colour range needs finite lo < hi per axis");
    ctx->col_lo[k] = lo[k];
    ctx->col_s[k] = 1.0f / (hi[k] - lo[k]);
  }
  ctx->colour_img = dev_colour_img;
  FF_CATCH
}

ff_status ff_step(ff_ctx* ctx, int64_t n_steps, float dt) {
  NvtxRange nvtx("ff_step");
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(n_steps >= 0, FF_ERR_INVALID_ARG, "n_steps must be >= 0");
  ctx->launch_step(n_steps, dt);
  FF_CATCH
}

ff_status ff_set_launch(ff_ctx* ctx, int ppt, int tpb) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(ppt == 0 || ppt == 1 || ppt == 2 || ppt == 4, FF_ERR_INVALID_ARG, "particles per thread must be 0, 1, 2 or 4");
  need(tpb == 0 || tpb == 128 || tpb == 256 || tpb == 512, FF_ERR_INVALID_ARG, "threads per block must be 0/128/256/512");
  const int old_p = ctx->ppt, old_t = ctx->tpb;
  ctx->ppt = ppt;
  ctx->tpb = tpb;
  int p, t;
  ctx->default_launch(p, t);
  if (step_index(p, t) < 0) {
    ctx->ppt = old_p;
    ctx->tpb = old_t;
    throw ff::Error(FF_ERR_INVALID_ARG, "unsupported (ppt, tpb) combination");
  }
  FF_CATCH
}

static void state_copy(ff_ctx* ctx, int group_id, int64_t first, int64_t count, void* host, bool to_host,
                       bool sync = true) {
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  const GroupRec& g = ctx->group(group_id);
  need(host || count == 0, FF_ERR_INVALID_ARG, "host buffer is NULL");
  need(first >= 0 && count >= 0 && first + count <= g.n_local, FF_ERR_INVALID_ARG, "particle range out of bounds");
  if (count == 0) return;
  const size_t w = (size_t)count * sizeof(float);
  float* dev = ctx->state + g.slot_begin + first;
  if (to_host) {
    ck(cudaMemcpy2DAsync(host, w, dev, (size_t)ctx->pitch * sizeof(float), w, ctx->sys.dim, cudaMemcpyDeviceToHost,
                         ctx->stream), "cudaMemcpy2DAsync D2H");
  } else {
    ck(cudaMemcpy2DAsync(dev, (size_t)ctx->pitch * sizeof(float), host, w, w, ctx->sys.dim, cudaMemcpyHostToDevice,
                         ctx->stream), "cudaMemcpy2DAsync H2D");
  }
  if (sync) ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
}

ff_status ff_read_state(ff_ctx* ctx, int group_id, int64_t first, int64_t count, float* host_soa) {
  FF_TRY
  state_copy(ctx, group_id, first, count, host_soa, true);
  FF_CATCH
}

ff_status ff_write_state(ff_ctx* ctx, int group_id, int64_t first, int64_t count, const float* host_soa) {
  FF_TRY
  state_copy(ctx, group_id, first, count, const_cast<float*>(host_soa), false);
  FF_CATCH
}

ff_status ff_render(ff_ctx* ctx, const float* colours, float intensity, float radius_px, float* dev_rgb) {
  NvtxRange nvtx("ff_render");
  FF_TRY
  need(ctx && colours && dev_rgb, FF_ERR_INVALID_ARG, "NULL argument");
  need(ctx->image != nullptr, FF_ERR_STATE, "no image bound");
  need(ctx->C <= FF_RENDER_MAX_C, FF_ERR_INVALID_ARG, "too many channels for ff_render");
  need(std::isfinite(intensity) && intensity >= 0.0f, FF_ERR_INVALID_ARG, "intensity must be finite and >= 0");
  need(radius_px > 0.0f && radius_px <= (float)FF_RENDER_MAX_R, FF_ERR_INVALID_ARG, "radius must be in (0, 8]");
  need(((uintptr_t)dev_rgb & 3) == 0, FF_ERR_INVALID_ARG, "rgb must be 4-byte aligned");
  FFRenderArgs a;
  std::memset(&a, 0, sizeof a);
  a.image = ctx->image;
  a.colour_img = ctx->colour_img;
  a.rgb = dev_rgb;
  a.W = ctx->W;
  a.H = ctx->H;
  a.C = ctx->C;
  a.hw = (int)std::ceil((double)radius_px);
  a.intensity = intensity;
  for (int i = 0; i < 3 * ctx->C; ++i) {
    need(std::isfinite(colours[i]), FF_ERR_INVALID_ARG, "colours must be finite");
    a.colour[i] = colours[i];
  }
  const int side = 2 * a.hw + 1;
  for (int dy = -a.hw; dy <= a.hw; ++dy)
    for (int dx = -a.hw; dx <= a.hw; ++dx) {
      const double r = std::sqrt((double)(dx * dx + dy * dy)) / (double)radius_px;
      const double f = 1.0 - (r < 1.0 ? r : 1.0);
      a.w[(dy + a.hw) * side + (dx + a.hw)] = (float)(f * f);
    }
  Module& m = ctx->module(ctx->sweep_param);
  void* args[] = {&a};
  dim3 grid((unsigned)((ctx->W + 31) / 32), (unsigned)((ctx->H + 7) / 8));
  ck(cudaLaunchKernel((const void*)m.render, grid, dim3(256), args, 0, ctx->stream), "launch ff_render");
  ++ctx->launches;
  FF_CATCH
}

static void image_copy(ff_ctx* ctx, uint32_t* host_image, bool sync) {
  need(ctx && host_image, FF_ERR_INVALID_ARG, "NULL argument");
  need(ctx->image != nullptr, FF_ERR_STATE, "no image bound");
  ck(cudaMemcpyAsync(host_image, ctx->image, (size_t)ctx->W * ctx->H * ctx->C * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost, ctx->stream), "cudaMemcpyAsync D2H image");
  if (sync) ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
}

ff_status ff_read_image(ff_ctx* ctx, uint32_t* host_image) {
  FF_TRY
  image_copy(ctx, host_image, true);
  FF_CATCH
}

ff_status ff_read_image_async(ff_ctx* ctx, uint32_t* host_image) {
  FF_TRY
  image_copy(ctx, host_image, false);
  FF_CATCH
}

ff_status ff_write_state_async(ff_ctx* ctx, int group_id, int64_t first, int64_t count, const float* host_soa) {
  FF_TRY
  state_copy(ctx, group_id, first, count, const_cast<float*>(host_soa), false, false);
  FF_CATCH
}

ff_status ff_launch_count(ff_ctx* ctx, int64_t* count) {
  FF_TRY
  need(ctx && count, FF_ERR_INVALID_ARG, "NULL argument");
  *count = ctx->launches;
  FF_CATCH
}

ff_status ff_sync(ff_ctx* ctx) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  ck(cudaGetLastError(), "kernel error");
  if (ctx->xused) {
    unsigned long long flag = 0;
    unsigned long long* f = ctx->tile_ctr + 16 + FF_XS_TIMEOUT;
    ck(cudaMemcpy(&flag, f, sizeof flag, cudaMemcpyDeviceToHost), "cudaMemcpy exchange flag");
    if (flag) {
      ck(cudaMemset(f, 0, sizeof flag), "cudaMemset exchange flag");
      throw ff::Error(FF_ERR_CUDA, "image exchange timed out waiting for a peer (the image of that launch is incomplete)");
    }
  }
  FF_CATCH
}

ff_status ff_set_exchange(ff_ctx* ctx, int rank, int world, uint32_t* const* peer_images,
                          uint64_t* const* peer_signals, double timeout_ms) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  if (world == 0) {
    ctx->xworld = 0;
    ctx->xmc = nullptr;
    ctx->xpush = 0;
    ctx->xpush_mc = nullptr;
    return FF_OK;
  }
  need(world >= 1 && world <= FF_MAX_PEERS && rank >= 0 && rank < world, FF_ERR_INVALID_ARG,
       "need 1 <= world <= FF_MAX_PEERS and 0 <= rank < world");
  need(peer_images && peer_signals, FF_ERR_INVALID_ARG, "peer tables are NULL");
  need(timeout_ms > 0.0 && timeout_ms <= 3.6e6, FF_ERR_INVALID_ARG, "timeout_ms must be in (0, 3.6e6]");
  need(ctx->image != nullptr, FF_ERR_STATE, "bind this rank's image with ff_project first");
  need(ctx->colour_img == nullptr, FF_ERR_STATE, "position colour images are not exchanged");
  need(peer_images[rank] == ctx->image, FF_ERR_INVALID_ARG, "peer_images[rank] must be the bound image");
  for (int p = 0; p < world; ++p) {
    need(peer_images[p] && ((uintptr_t)peer_images[p] & 15) == 0, FF_ERR_INVALID_ARG,
         "peer images must be non-NULL and 16-byte aligned");
    need(peer_signals[p] && ((uintptr_t)peer_signals[p] & 7) == 0, FF_ERR_INVALID_ARG,
         "peer signals must be non-NULL and 8-byte aligned");
  }
  for (int p = 0; p < FF_MAX_PEERS; ++p) {
    ctx->ximg[p] = p < world ? peer_images[p] : nullptr;
    ctx->xsig[p] = p < world ? peer_signals[p] : nullptr;
  }
  // a new exchange starts its barrier values at 1 again: clear the go flag (signals are the caller's)
  ck(cudaMemsetAsync(ctx->tile_ctr + 16 + FF_XS_GO, 0, sizeof(unsigned long long), ctx->stream),
     "cudaMemsetAsync go flag");
  ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  // compile / load the step kernel now: no NVRTC or module load between the ranks' first launches
  Module& m = ctx->module(ctx->sweep_param);
  for (int64_t n : {1, 10, 100}) {   // the kernels of short, medium and long launches
    int pp, tt;
    ctx->default_launch(pp, tt, n);
    const int id = step_index(pp, tt);
    for (int bal = 0; bal < 2; ++bal) ctx->step_kernel(m, ctx->sweep_param, id, ctx->variant_for(bal != 0, id, n));
  }
  // and force the (lazily loaded) exchange kernel in now: a lazy load at its first launch can wait
  // for the device while a peer's exchange kernel spins waiting for this rank (deadlock on one GPU)
  cudaFuncAttributes fa;
  ck(cudaFuncGetAttributes(&fa, (const void*)m.exchange), "cudaFuncGetAttributes(ff_exchange)");
  ctx->xrank = rank;
  ctx->xworld = world;
  ctx->xseq = 0;
  ctx->xtimeout_ns = (uint64_t)(timeout_ms * 1e6);
  ctx->xmc = nullptr;
  ctx->xpush = 0;
  ctx->xpush_mc = nullptr;
  FF_CATCH
}

ff_status ff_set_exchange_multicast(ff_ctx* ctx, uint32_t* mc_image) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(mc_image == nullptr || ctx->xworld >= 1, FF_ERR_STATE, "set up the exchange with ff_set_exchange first");
  need(((uintptr_t)mc_image & 15) == 0, FF_ERR_INVALID_ARG, "the multicast address must be 16-byte aligned");
  ctx->xmc = mc_image;
  FF_CATCH
}

ff_status ff_set_exchange_push(ff_ctx* ctx, int on, uint32_t* mc_image) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(on == 0 || on == 1, FF_ERR_INVALID_ARG, "on must be 0 or 1");
  need(((uintptr_t)mc_image & 15) == 0, FF_ERR_INVALID_ARG, "the multicast address must be 16-byte aligned");
  if (!on) {
    ctx->xpush = 0;
    ctx->xpush_mc = nullptr;
    return FF_OK;
  }
  need(ctx->xworld >= 1, FF_ERR_STATE, "set up the exchange with ff_set_exchange first");
  const int push = mc_image ? 2 : 1;
  // compile / load the pushing step kernels and the barrier now (as ff_set_exchange does for its
  // kernels): no NVRTC compile or lazy module load between the ranks' first pushing launches, while a
  // peer's barrier may already be spinning on the device
  Module& m = ctx->module(ctx->sweep_param);
  if (ctx->xworld > 1) {
    for (int64_t n : {1, 10, 100}) {
      int pp, tt;
      ctx->default_launch(pp, tt, n);
      const int id = step_index(pp, tt);
      for (int bal = 0; bal < 2; ++bal)
        ctx->step_kernel(m, ctx->sweep_param, id, ctx->variant_for(bal != 0, id, n) + 8 * push);
    }
  }
  cudaFuncAttributes fa;
  ck(cudaFuncGetAttributes(&fa, (const void*)m.xbarrier), "cudaFuncGetAttributes(ff_xbarrier)");
  ctx->xpush = push;
  ctx->xpush_mc = mc_image;
  FF_CATCH
}

ff_status ff_set_grid_limit(ff_ctx* ctx, int max_blocks) {
  FF_TRY
  need(ctx, FF_ERR_INVALID_ARG, "ctx is NULL");
  need(max_blocks >= 0, FF_ERR_INVALID_ARG, "max_blocks must be >= 0");
  ctx->grid_limit = max_blocks;
  FF_CATCH
}

}  // extern "C"
