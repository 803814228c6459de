// ff_args.h -- by-value launch argument blocks of the Fireflies kernels.
//
// Single source of truth for the layout: the host runtime (ff_runtime.cpp) includes this file,
// and the build embeds it in front of ff_device.cuh in the NVRTC source. Kernel arguments live
// in the constant bank, so parameters and per-group step sizes are read as FFMA operands
// (parameters change "in GPU memory" without recompiling; here they are captured by
// value at each launch).
#ifndef FF_ARGS_H
#define FF_ARGS_H

typedef unsigned long long ff_u64;
typedef long long ff_i64;
typedef unsigned int ff_u32;

#define FF_MAX_GROUPS_ 16
#define FF_MAX_DIM_ 64
#define FF_MAX_PEERS_ 8
#define FF_MAX_SCALED_ 4  // components with a factored uniform scale (split_scales)
#define FF_MAX_DERIVED_ 192  // host-evaluated loop-invariant values of the RHS (ff::UProgram)
// word offsets in the exchange sync block (each word on its own 128-byte line)
#define FF_XS_ARRIVE 0
#define FF_XS_GO 16
#define FF_XS_TIMEOUT 32
#define FF_XS_WORDS 48
#ifndef FF_NP_ALLOC
#define FF_NP_ALLOC 128  /* host side: FF_MAX_PARAMS; device side: the system's count */
#endif

struct FFGroup {
  ff_i64 slot_begin;    // first slot of the group (multiple of FF_TILE)
  ff_i64 slot_end;      // padded end (multiple of FF_TILE)
  ff_i64 n_local;       // real particles in [slot_begin, slot_begin + n_local)
  ff_i64 first_global;  // group-global index of the first local particle
  ff_i64 n_global;      // particles in the whole group (all shards)
  ff_u64 sweep_seed;
  float h, h2, h6;      // signed step direction*dt, h/2, h/6
  float nh, nh2, nh6;   // -h, -h/2, -h/6 (host-negated: loaded straight into uniform registers)
  float pad0_, pad1_;
  float sw_lo, sw_hi, sw_top, sw_val;  // sweep range, largest float below hi, uniform value
  int sweep_mode;       // -1: every particle uses sw_val; 0: Philox-uniform; 1: linspace
  int colour;           // image channel
  ff_u64 seed;          // IC seed of the group (resets draw from it with stream 2 + epoch)
  float t_now;          // simulated time elapsed in this group after this launch (for T_max)
  int pad_;
};

struct FFStepArgs {
  float* state;         // [dim][pitch] SoA
  ff_i64 pitch;
  ff_i64 slots_total;   // end of the last group's slot range
  ff_i64 n_steps;
  ff_u32* image;        // bound image [C][H][W] or null
  int proj;             // 0 none, 2 (2-D window) or 3 (4x4 view-projection)
  int W, H, C;
  int axes[3];
  float view[16];
  float s0, s1;         // 2-D scales W/(hi0-lo0), H/(hi1-lo1), computed by the host in float
  float fW, fH, hW, hH; // (float)W, (float)H, W * 0.5f, H * 0.5f (exact; host-computed)
  int ax_id;            // 1: axes[j] == j for every projected axis (no per-particle axis selection)
  float one;            // 1.0f, at run time (ff_exact.cuh: exact packed sums as fma(a, one, b))
  int n_groups;
  // device-side reset (NEXT row 1): 0 off, else bit 1 = bounds, bit 2 = age
  int reset;
  float t_max;
  ff_u32* epoch;        // per slot: resets so far (library-owned)
  float* birth;         // per slot: group time of the last (re)initialisation (library-owned)
  const float* ic_box;  // [group][lo | hi | top][dim] (library-owned)
  // dynamic tile scheduler: a monotonically increasing 64-bit counter (library-owned); this launch
  // owns the fetch numbers [tile_base, tile_base + tiles + grid)
  ff_u64* tile_ctr;
  ff_u64 tile_base;
  // position-linear colour: per particle q_k = min(255, floor(256 * clamp((v_k -
  // lo_k) * s_k, 0, 1))) of its projected axis values, summed per pixel into colour_img[3][H][W]
  ff_u32* colour_img;   // null = off
  float col_lo[3], col_s[3];
  int static_rounds;    // tile rounds assigned statically (block b: b, b + grid, ...) before the counter
  // fused (push) image exchange (ff_set_exchange_push; read only by FF_PUSH builds): every reduction
  // into the image goes to each of push_img[0 .. push_n) (FF_PUSH 1: every rank's image, as mapped in
  // this process) or to the images' NVLS multicast address push_img[0] (FF_PUSH 2)
  ff_u32* push_img[FF_MAX_PEERS_];
  int push_n;
  float bound_lo[FF_MAX_DIM_], bound_hi[FF_MAX_DIM_];
  FFGroup g[FF_MAX_GROUPS_];
  // step constants of the components with a factored uniform scale s (FF_SSLOT[d] in the generated
  // code): {h s, h/2 s, h/6 s, -h s, -h/2 s, -h/6 s} per group and slot, computed by the host
  float hs[FF_MAX_GROUPS_][FF_MAX_SCALED_][6];
  // loop-invariant values of the generated RHS (products / reciprocals / exponentials of parameters,
  // negated parameters), evaluated by the host at every launch: uniform-register operands
  float q[FF_MAX_DERIVED_];
  float p[FF_NP_ALLOC]; // parameter values (must stay the last member)
};

// Image exchange (NEXT row 2): launched right after a binning step launch of an
// exchanging context (ff_set_exchange); sums the bound images of all ranks over peer memory, each
// rank owning one slice of the pixels, in place.
struct FFXchgArgs {
  ff_u32* img[FF_MAX_PEERS_];   // every rank's bound image, as mapped in this process; [rank] = own
  ff_u64* sig[FF_MAX_PEERS_];   // every rank's signal words [FF_MAX_PEERS_] (written by the peers)
  ff_u64* sync;                 // library-owned sync block (FF_XS_* word offsets)
  ff_u64 words;                 // C * H * W
  ff_u64 bar_base;              // arrival tickets taken before this launch
  ff_u64 seq;                   // exchanges before this one: barrier values 2 seq + 1, 2 seq + 2
  ff_u64 timeout_ns;            // bound on every wait (a missing peer cannot hang the GPU)
  int rank, world;
  ff_u32* mc;                   // NVLS multicast address of the images (same layout) or null
  int phase;                    // ff_xbarrier: 1 = before a pushing launch (2 seq + 1), 2 = after it
};

// Lifted-parameter readback (ff_read_lifted): the swept value of particles [local, local + count) of
// one group, from their epochs (ff_sweep_value in ff_device.cuh)
struct FFLiftedArgs {
  float* out;           // [count] device scratch
  const ff_u32* epoch;  // per slot, or null (all epochs 0)
  ff_i64 slot;          // slot of the first particle
  ff_i64 local;         // group-local index of the first particle
  ff_i64 count;
  FFGroup g;            // sweep fields, first_global, n_global, seed
};

// Render post-process (NEXT row 3): count image -> RGB with sprite falloff.
#define FF_RENDER_MAX_R 8
#define FF_RENDER_MAX_C 16
struct FFRenderArgs {
  const ff_u32* image;  // [C][H][W] counts
  const ff_u32* colour_img;  // [3][H][W] position-colour sums (q in 0..255 per particle) or null
  float* rgb;           // [3][H][W] output
  int W, H, C, hw;      // hw = half width of the sprite footprint in pixels
  float intensity;      // sprite alpha
  int pad_;
  float colour[FF_RENDER_MAX_C * 3];
  float w[(2 * FF_RENDER_MAX_R + 1) * (2 * FF_RENDER_MAX_R + 1)];  // [dy + hw][dx + hw], row pitch 2hw+1
};

#endif
