/* fireflies.h -- C ABI of the B200-native Fireflies hot path (arXiv:1505.00344).
 *
 * The library integrates many independent trajectories ("particles") of a user-defined
 * N-dimensional ODE with fixed-step classical RK4, each particle with its
 * own initial condition, its own time direction and optionally its own
 * value of one swept parameter, and bins the particles, projected onto 2 or 3
 * chosen axes, into a density image.
 *
 * Conventions for every call:
 *   - Every function returns ff_status; nothing is thrown across the ABI. On failure the
 *     message is available from ff_last_error() (thread-local, valid until the next call on
 *     the same thread). Failed calls leave the context unchanged unless stated otherwise.
 *   - "device pointer" = CUDA global-memory pointer valid in the current device's primary
 *     context (e.g. torch.Tensor.data_ptr() of a CUDA tensor). "host pointer" = CPU memory.
 *   - Device memory for particle state and images is CALLER-OWNED. The context stores non-owning
 *     pointers and never frees them; ff_destroy frees only what the library allocated
 *     (compiled modules, tables).
 *   - Launches are asynchronous on the stream set with ff_set_stream (default: the legacy
 *     default stream). Parameter values are captured by value at launch, so ff_set_param takes
 *     effect at the next launch and never needs a device sync.
 *   - A context is NOT thread-safe; use one per host thread / device.
 *   - All floating-point state is FP32 ("single-precision floating point values",
 *     PAPER.md:225).
 */
#ifndef FIREFLIES_H
#define FIREFLIES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FF_ABI_VERSION 1
#define FF_MAX_DIM 64      /* state variables per system */
#define FF_MAX_PARAMS 128  /* parameters per system */
#define FF_MAX_GROUPS 16   /* particle groups per context */
#define FF_TILE 512        /* group slot ranges are padded to a multiple of this */
#define FF_MAX_PEERS 8     /* ranks in one fused image exchange (one node) */

typedef enum {
  FF_OK = 0,
  FF_ERR_INVALID_ARG = 1,    /* bad pointer / size / range / enum value */
  FF_ERR_PARSE = 2,          /* expression syntax error, unknown function, wrong arity */
  FF_ERR_UNKNOWN_SYMBOL = 3, /* identifier that is neither a state variable nor a parameter */
  FF_ERR_RANGE = 4,          /* parameter value outside [min, max] (rejected, not clamped) */
  FF_ERR_COMPILE = 5,        /* NVRTC failure (message holds the log) */
  FF_ERR_CUDA = 6,           /* CUDA runtime / launch failure (message holds the CUDA error) */
  FF_ERR_OOM = 7,            /* host allocation failure */
  FF_ERR_STATE = 8           /* call not valid in the current context state */
} ff_status;

typedef struct ff_ctx ff_ctx; /* opaque */

/* System definition (State Variables with right-hand sides, Parameters with a
 * default and a range of allowable values). All strings are NUL-terminated ASCII, copied by the
 * library; the struct may be freed after the call.
 *   dim            number of state variables, 1..FF_MAX_DIM
 *   var_names[i]   identifier of state variable i ([A-Za-z_][A-Za-z0-9_]*)
 *   rhs[i]         expression for d(var_i)/dt. Grammar (no conditionals):
 *                    expr := term (("+"|"-") term)* ; term := factor (("*"|"/") factor)*
 *                    factor := "-" factor | power ; power := atom ("^" factor)?
 *                    atom := number | ident | ident "(" expr ("," expr)* ")" | "(" expr ")"
 *                  functions: exp log sin cos tan tanh sqrt abs sigmoid (1 arg), pow min max vtrap
 *                  (2 args); sigmoid(u) = 1/(1+exp(-u)); vtrap(x,y) = x/(exp(x/y)-1) with its
 *                  removable singularity at x = 0 handled (reading R10).
 *                  Constants: pi, e. Names may not shadow each other, pi, e or a function.
 *   n_params       0..FF_MAX_PARAMS
 *   param_names[k], param_default[k]; param_min / param_max may be NULL (unbounded), else
 *                  min[k] <= default[k] <= max[k] is required. */
typedef struct {
  int dim;
  const char* const* var_names;
  const char* const* rhs;
  int n_params;
  const char* const* param_names;
  const float* param_default;
  const float* param_min;
  const float* param_max;
} ff_system;

/* ---------------------------------------------------------------- library / front end */

/* Message of the last failed call on this thread ("" if none). Never NULL. */
const char* ff_last_error(void);

/* FF_ABI_VERSION of the loaded library. */
int ff_abi_version(void);

/* Human-readable build information (ABI version, NVRTC version and path, target sm_100a); same
 * buffer protocol as ff_emit_source. Errors: FF_ERR_COMPILE if NVRTC cannot be loaded. */
ff_status ff_build_info(char* buf, size_t cap, size_t* len);

/* Front end only (no device needed; "kernel source ... generated automatically"):
 * parse, validate and emit the CUDA C source of the system's kernels. sweep_param = index of the
 * parameter that is per-particle in this variant, or -1. Writes at most cap bytes (NUL-terminated)
 * to buf; *len (if non-NULL) receives the full length excluding the NUL. buf may be NULL to query.
 * Errors: FF_ERR_INVALID_ARG, FF_ERR_PARSE, FF_ERR_UNKNOWN_SYMBOL. */
ff_status ff_emit_source(const ff_system* sys, int sweep_param, char* buf, size_t cap, size_t* len);

/* Front end + NVRTC (no device needed): compile the emitted source to an sm_100a CUBIN.
 * Same buffer protocol as ff_emit_source. Errors as ff_emit_source, plus FF_ERR_COMPILE. */
ff_status ff_compile_cubin(const ff_system* sys, int sweep_param, void* buf, size_t cap, size_t* len);

/* ---------------------------------------------------------------- context */

/* Parse + validate the system, compile its kernels (NVRTC, sm_100a CUBIN) and load them on
 * `device` (which must be the calling thread's current CUDA device). *out receives the context.
 * Errors: ff_emit_source's, FF_ERR_COMPILE, FF_ERR_CUDA (no device, module load failure). */
ff_status ff_create(const ff_system* sys, int device, ff_ctx** out);

/* Free the context and the library-owned resources. Does not free caller memory. NULL is OK. */
ff_status ff_destroy(ff_ctx* ctx);

/* Stream for every subsequent launch/copy (a cudaStream_t; NULL = legacy default stream). */
ff_status ff_set_stream(ff_ctx* ctx, void* cuda_stream);

/* Multi-GPU sharding: this process holds, of every group created afterwards,
 * the contiguous index range [floor(n*rank/world), floor(n*(rank+1)/world)). Particle i keeps
 * its group-global index, so initial conditions and swept values do not depend on world.
 * Must be called before the first ff_init_group. Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE. */
ff_status ff_set_shard(ff_ctx* ctx, int rank, int world);

/* Host-only (no context, no device): the contiguous index range [*first, *first + *count) of a
 * group of n_global particles held by shard `rank` of `world` (the rule of ff_set_shard).
 * Errors: FF_ERR_INVALID_ARG. */
ff_status ff_shard_range(int64_t n_global, int rank, int world, int64_t* first, int64_t* count);

/* Bind caller-owned particle state: device pointer to float[dim][pitch] (SoA: component d of
 * slot j at state[d*pitch + j]), 16-byte aligned, pitch a multiple of FF_TILE, capacity <= pitch
 * slots usable. Must be called before the first ff_init_group (rebinding clears the groups).
 * Errors: FF_ERR_INVALID_ARG (NULL, misaligned, pitch/capacity). */
ff_status ff_bind_state(ff_ctx* ctx, float* dev_state, int64_t pitch, int64_t capacity);

/* Query the minimum number of slots a group of n_global particles needs on this shard
 * (its local count rounded up to FF_TILE). */
ff_status ff_group_slots(ff_ctx* ctx, int64_t n_global, int64_t* slots);

/* Create a particle group (count, direction, initial-condition cube) and launch
 * its initial-condition kernel (async). ic_lo/ic_hi: HOST arrays of dim floats, the half-open
 * box [lo, hi) per state variable (lo < hi, finite). n_global >= 1 particles in total over all
 * shards; direction +1 (forward in time) or -1 (backward); colour = image channel this group is
 * counted in (>= 0); seed keys the group's Philox stream (use distinct seeds for distinct groups).
 * The group occupies the next free tile-aligned slot range; padding slots are set to NaN and are
 * never binned. *group_id (may be NULL) receives the group's index.
 * Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE (no state bound, too many groups, capacity
 * exceeded), FF_ERR_CUDA. */
ff_status ff_init_group(ff_ctx* ctx, const float* ic_lo, const float* ic_hi, int64_t n_global,
                        int direction, int colour, uint64_t seed, int* group_id);

/* Slot layout of a group on this shard: first slot, local particle count, and the group-global
 * index of its first local particle. Any out pointer may be NULL. */
ff_status ff_group_info(ff_ctx* ctx, int group_id, int64_t* slot_begin, int64_t* n_local,
                        int64_t* first_global);

/* Set a parameter by name ("updates the location in GPU memory where the
 * corresponding parameter value is stored"); the next launch uses it.
 * Errors: FF_ERR_UNKNOWN_SYMBOL, FF_ERR_RANGE (outside [min, max]; value is not clamped),
 * FF_ERR_INVALID_ARG (non-finite). */
ff_status ff_set_param(ff_ctx* ctx, const char* name, float value);
ff_status ff_get_param(ff_ctx* ctx, const char* name, float* value);

/* Make parameter `name` a per-particle value for group `group_id` (the lifted parameter of
 * a state variable with zero derivative; here it is never integrated, so it is
 * bit-unchanged between resets by construction). mode 0: Philox-uniform in [lo, hi) keyed by `seed`;
 * mode 1: linspace lo + (hi - lo) * (i + 0.5) / n_global. At most one parameter per context may
 * be swept (all sweeping groups must name the same one); groups without a sweep use the
 * parameter's current value. The value is recomputed from the particle index (and, with resets,
 * its epoch: a mode-0 value is redrawn with the state, see ff_set_reset) in every launch (0 bytes of
 * state). It is addressable as axis index `dim` in ff_project; ff_read_lifted reads it back.
 * Errors: FF_ERR_UNKNOWN_SYMBOL, FF_ERR_INVALID_ARG (lo >= hi, mode, group), FF_ERR_STATE
 * (another parameter already swept), FF_ERR_COMPILE (variant compile). */
ff_status ff_sweep_param(ff_ctx* ctx, int group_id, const char* name, float lo, float hi, int mode,
                         uint64_t seed);

/* Bind the density image and bin the current state into it now (async).
 * axes: HOST array of n_axes (2 or 3) indices into the extended state [0..dim-1 state vars,
 *       dim = the swept parameter]; view: HOST array, 2-D: {lo_0, hi_0, lo_1, hi_1} (window, each
 *       lo < hi), 3-D: row-major 4x4 view-projection matrix (rows 0, 1, 3 used).
 * image: DEVICE pointer to uint32 [C][H][W] (caller-owned, caller zeroes it), 4-byte aligned.
 * Binning rule (readings R17-R19): 2-D keeps lo <= v < hi on both axes,
 *   ix = min(floor((v0 - lo0) * (W / (hi0 - lo0))), W - 1), likewise iy; 3-D computes
 *   c_r = ((M[r][0] a + M[r][1] b) + M[r][2] c) + M[r][3], keeps c_w > 0,
 *   px = (c_0 / c_w + 1) * (W / 2), keeps 0 <= px < W, likewise py. Each kept particle adds 1 to
 *   image[colour(group)][iy][ix]; non-finite values and padding slots are dropped.
 * Once bound, every ff_step adds one count per particle after its last step (fused). Pass
 * image = NULL to unbind (no binning). Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE (colour of some
 * group >= C), FF_ERR_CUDA. */
ff_status ff_project(ff_ctx* ctx, const int* axes, int n_axes, const float* view, int W, int H,
                     int C, uint32_t* image);

/* Advance every particle of every group by n_steps RK4 steps of signed size direction*dt
 * (dt may be negative), then, if an image is bound, bin every particle once
 * (fused). One kernel launch; async. n_steps >= 0 (0 = bin only).
 * The first launch of a kernel variant compiles it (NVRTC, ~0.5 s; cached per process).
 * CUDA-graph capture (replaying a recorded frame, PAPER.md:242's main loop): if the
 * bound stream is capturing, the launch is recorded with its current parameters, dt, camera and
 * groups, preceded by a reset of the library's tile counter (from then on every launch of this
 * context resets it: replays and later launches agree). The kernel must already be compiled (run
 * the same launch once first), and the age rule (t_max) and the image exchange cannot be captured.
 * ff_launch_count counts captures, not replays.
 * Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE (no groups; capture restrictions), FF_ERR_COMPILE,
 * FF_ERR_CUDA. */
ff_status ff_step(ff_ctx* ctx, int64_t n_steps, float dt);

/* Device-side reset (trajectories that leave the region, or have not been reset for
 * more than T_max, get new random initial conditions; per-variable bounds; the paper
 * does this on the host, lagged). When enabled, every ff_step with n_steps > 0 checks
 * each particle after its last step, before binning: it is reset if a component is non-finite, or
 * (lo/hi given) outside [lo_d, hi_d], or (t_max > 0 and finite) its simulated time since the last
 * (re)initialisation exceeds t_max. A reset particle gets the group's IC formula (reading R5) with
 * Philox stream 2 + e, e = number of earlier resets of that particle. A group whose parameter is
 * swept with mode 0 (Philox) redraws its lifted parameter too: the paper makes it a state variable
 * whose initial-condition range is the swept range and draws a new position "when
 * the particle is first initialized (or reset ...)". It is component dim of the same
 * draw (word dim % 4 of Philox block dim / 4, stream 2 + e; reading R16), so after e
 * resets a particle's swept value is a function of (IC seed, index, e) and costs no memory beyond the
 * epoch. A linspace sweep (mode 1) keeps its grid value through resets (a deliberate extension).
 * lo, hi: HOST arrays of dim floats (both or neither). enable = 0 disables the checks; the per-slot
 * bookkeeping (epochs, birth times) is allocated at the first enable after ff_bind_state (8 bytes
 * per slot, library-owned) and kept until the next ff_bind_state, so disabling, re-enabling or
 * changing the rule never changes a particle's lifted value. Groups created before or after are
 * covered. Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE, FF_ERR_CUDA. */
ff_status ff_set_reset(ff_ctx* ctx, int enable, const float* lo, const float* hi, float t_max);

/* Reset counts (epochs) of particles [first, first+count) of a group into a HOST uint32 buffer
 * (synchronous). Errors: FF_ERR_STATE (reset never enabled), FF_ERR_INVALID_ARG. */
ff_status ff_read_epochs(ff_ctx* ctx, int group_id, int64_t first, int64_t count, uint32_t* host);

/* The lifted (swept) parameter value of particles [first, first+count) of a group into a HOST float
 * buffer (synchronous): the value the next ff_step integrates and bins them with -- the sweep draw
 * (ff_sweep_param) after 0 resets, component dim of the latest reset draw otherwise (see
 * ff_set_reset). Computed on the device by the same routine the step kernel uses (one launch).
 * Errors: FF_ERR_STATE (no parameter swept), FF_ERR_INVALID_ARG (range), FF_ERR_CUDA. */
ff_status ff_read_lifted(ff_ctx* ctx, int group_id, int64_t first, int64_t count, float* host);

/* Kernel selection: particles per thread (1, 2 or 4; 2 packs pairs into FFMA2, 4 = two pairs with
 * 16-byte loads) and threads per block (128, 256 or 512; 4 particles only with 128); 0 = library
 * default: one particle per thread in 128-thread blocks when the groups hold fewer than 256
 * particles per SM (latency-bound); for systems with <= 4 variables 4 per thread for 1-4-step
 * launches (HBM / L2-bound) and for longer launches of systems without MUFU work; else packed
 * pairs. Results are the same for every choice up to FP rounding (the projection,
 * counting and reset draws bit for bit). For tuning/benchmarks. Errors: FF_ERR_INVALID_ARG. */
ff_status ff_set_launch(ff_ctx* ctx, int particles_per_thread, int threads_per_block);

/* Copy particles [first, first+count) (group-local indices on this shard) of a group between the
 * device state and a HOST SoA buffer float[dim][count]. Synchronous w.r.t. the host (the stream
 * is synchronised). Errors: FF_ERR_INVALID_ARG (range), FF_ERR_CUDA. */
ff_status ff_read_state(ff_ctx* ctx, int group_id, int64_t first, int64_t count, float* host_soa);
ff_status ff_write_state(ff_ctx* ctx, int group_id, int64_t first, int64_t count,
                         const float* host_soa);

/* Copy the bound image to a HOST uint32 [C][H][W] buffer (synchronous). */
ff_status ff_read_image(ff_ctx* ctx, uint32_t* host_image);

/* Stream-ordered variants of ff_write_state / ff_read_image: the copy is queued on the bound stream
 * and the call returns at once (the host buffer must stay valid -- and for a true asynchronous copy
 * be page-locked -- until the stream has passed it; synchronise with ff_sync or a stream event).
 * They let a caller pipeline frames: the next frame's state copy-in and the previous frame's image
 * copy-out overlap the current frame's integration on another context / stream.
 * Errors: as the synchronous calls, without the synchronisation. */
ff_status ff_write_state_async(ff_ctx* ctx, int group_id, int64_t first, int64_t count,
                               const float* host_soa);
ff_status ff_read_image_async(ff_ctx* ctx, uint32_t* host_image);

/* Render the bound count image to a displayable RGB frame (sprites with an intensity
 * that falls off with the distance from their centre, coloured per group, blended
 * additively), async on the bound stream:
 *   rgb[k][y][x] = min(1, sum_c colours[3c+k] * intensity * sum_q count_c(y+q_y, x+q_x) w(q))
 *   w(q) = (1 - min(|q| / radius_px, 1))^2 over integer offsets |q_x|, |q_y| <= ceil(radius_px)
 * (sprites centred on their pixel, reading R24; falloff of SPEC.md:388; taps outside the image
 * contribute nothing; sums in double, exactly rounded, so results are reproducible bit-for-bit).
 * colours: HOST float[C][3]; intensity >= 0 (sprite alpha); 0 < radius_px <= 8; dev_rgb: DEVICE
 * float[3][H][W] (caller-owned). Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE (no image), FF_ERR_CUDA. */
ff_status ff_render(ff_ctx* ctx, const float* colours, float intensity, float radius_px, float* dev_rgb);

/* Position-linear colour (the colour "varies linearly as a function of the
 * particle's position in state space"). Once bound (after ff_project), every ff_step
 * also adds, for each counted particle, q_k = min(255, floor(256 * clamp((v_k - lo_k) * s_k, 0, 1)))
 * to colour_img[k][iy][ix], k = 0, 1, 2 over the projected axes (2-D: q_2 = 128), with
 * s_k = 1 / (hi_k - lo_k) computed in float; all ops exact IEEE, counts integer (bit-exact). While a
 * colour image is bound, ff_render uses it: rgb_k = min(1, intensity * sum_q colsum_k w(q) / 255).
 * lo, hi: HOST arrays of n_axes floats (lo < hi). dev_colour_img: DEVICE uint32 [3][H][W],
 * caller-owned, caller zeroes it; NULL unbinds. Sums overflow past 16.8 M particles in one pixel.
 * Errors: FF_ERR_INVALID_ARG, FF_ERR_STATE (no image bound). */
ff_status ff_project_colour(ff_ctx* ctx, const float* lo, const float* hi, uint32_t* dev_colour_img);

/* Number of kernel launches this context has issued (for bench evidence). */
ff_status ff_launch_count(ff_ctx* ctx, int64_t* count);

/* Synchronise the bound stream; surfaces asynchronous kernel errors as FF_ERR_CUDA, including an
 * image exchange that timed out waiting for a peer (ff_set_exchange). */
ff_status ff_sync(ff_ctx* ctx);

/* Image exchange over peer memory: the path's one exchange step -- the
 * sum of the per-rank density images of a sharded run (PAPER.md:236 additive blending over all
 * particles) -- done by the library on the step's stream, over NVLink / NVSwitch peer memory, instead
 * of a separate all-reduce. After this call every binning launch of this context (ff_step,
 * ff_project's immediate binning) is followed, in stream order, by an exchange kernel: a barrier over
 * the `world` ranks (their histograms are complete), then rank r sums pixel slice r (16-byte units,
 * split evenly; the C*H*W % 4 tail words belong to rank world-1) over all ranks' images and stores the
 * sum into every rank's image, then a second barrier. When it completes, the bound image equals the
 * element-wise sum over ranks of the images each rank's launch produced alone -- bit-exact, integer
 * -- i.e. ff_step followed by an all-reduce (previous contents included: zero the image per frame).
 * With world = 1 the image already is the sum and no exchange kernel is launched.
 *   peer_images[p]   DEVICE pointer, valid in THIS process, to rank p's bound uint32 [C][H][W] image
 *                    (16-byte aligned; peer_images[rank] must be the image bound here with ff_project;
 *                    all ranks bind the same C, H, W). Typically symmetric memory mapped over
 *                    NVLink (torch symmetric memory, CUDA IPC) or, on one GPU, other contexts'.
 *   peer_signals[p]  DEVICE pointer to rank p's FF_MAX_PEERS uint64 signal words (8-byte aligned),
 *                    zeroed on every rank before the first exchanged launch; written only by the
 *                    library (rank q stores barrier values into word q of every rank's array).
 *   timeout_ms       bound on every wait inside the exchange; a peer that does not arrive in time
 *                    makes the launch finish with an incomplete image and ff_sync report FF_ERR_CUDA.
 * Collective: every rank calls it with the same world and tables (its own rank), no exchanged
 * launch in flight, and then issues the same sequence of binning launches. world = 0 (tables
 * ignored) turns the exchange off; so does binding another image with ff_project. Position-colour
 * images are not exchanged (FF_ERR_STATE).
 * Errors: FF_ERR_INVALID_ARG (ranges, NULL / misaligned pointers, peer_images[rank] != image),
 * FF_ERR_STATE (no image bound, colour image bound), FF_ERR_CUDA. */
ff_status ff_set_exchange(ff_ctx* ctx, int rank, int world, uint32_t* const* peer_images,
                          uint64_t* const* peer_signals, double timeout_ms);

/* NVLS variant of the image exchange (NVSwitch multicast): after
 * ff_set_exchange, give the multicast address under which every rank's bound image is mapped (a CUDA
 * multicast object bound to each rank's image buffer, same layout; e.g. torch symmetric memory's
 * multicast_ptr). The exchange keeps its two barriers; its sum pass then uses multimem.ld_reduce
 * (the switch adds the ranks' words) and multimem.st (the sum lands in every rank's image), one word
 * per instruction, so each word of this rank's slice crosses NVLink once in each direction. Same
 * result, bit-exact. Needs a multicast-capable NVSwitch system with >= 2 GPUs (on a single GPU the
 * driver refuses multicast objects). mc_image = NULL returns to peer loads / stores; ff_set_exchange
 * and rebinding the image clear it. Errors: FF_ERR_STATE (no exchange set), FF_ERR_INVALID_ARG
 * (misaligned). */
ff_status ff_set_exchange_multicast(ff_ctx* ctx, uint32_t* mc_image);

/* Fused (push) variant of the image exchange (SURVEY.md 8(e) "Fused option", 8(f) NEXT 2): after
 * ff_set_exchange, on = 1 makes the histogram of every binning launch send its reductions straight to
 * every rank's image -- no sum pass. mc_image = NULL: each reduction is issued once per rank as a
 * system-scope red.add over peer memory to peer_images[p] (on one GPU, other contexts' images);
 * mc_image = the NVLS multicast address of the images (as for ff_set_exchange_multicast): each is
 * issued once as multimem.red.add and the NVSwitch applies it to every rank's copy. Each pushing
 * launch runs between two barriers over the ranks (kernel ff_xbarrier on the exchange's signal
 * words): before it every rank has finished what it issued earlier on its stream (zeroing or reading
 * its image), after it every rank's reductions are in every image. Semantics differ from the sum
 * pass: the launch ADDS the sum over ranks of its counts to every rank's image (previous contents
 * kept, not summed), so images that start equal (e.g. zeroed on every rank each frame) stay equal and
 * equal the unsharded run's image after any sequence of launches -- bit-exact, integer. on = 0
 * returns to the sum pass. Collective like ff_set_exchange (every rank, same on / kind of address,
 * no exchanged launch in flight); compiles the pushing kernels on the spot. Needs world >= 2 to
 * change anything (one rank: its image already is the sum). The multicast form needs a
 * multicast-capable NVSwitch system (refused on a single GPU). ff_set_exchange and rebinding the image
 * turn it off. Errors: FF_ERR_STATE (no exchange set), FF_ERR_INVALID_ARG (on not 0/1, misaligned),
 * FF_ERR_COMPILE, FF_ERR_CUDA. */
ff_status ff_set_exchange_push(ff_ctx* ctx, int on, uint32_t* mc_image);

/* Upper bound on the blocks of every step and exchange launch (0 = the default: every resident block
 * for a step, 2 per SM for an exchange). For several ranks sharing one GPU (their exchanges must run
 * concurrently), and for tuning. Errors: FF_ERR_INVALID_ARG. */
ff_status ff_set_grid_limit(ff_ctx* ctx, int max_blocks);

#ifdef __cplusplus
}
#endif
#endif /* FIREFLIES_H */
