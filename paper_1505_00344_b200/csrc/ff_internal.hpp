// ff_internal.hpp -- shared declarations of the host side of libfireflies (front end + runtime).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fireflies.h"

#define FF_MAX_SCALED 4  /* components with a factored uniform scale (ff_args.h FF_MAX_SCALED_) */
#define FF_MAX_DERIVED 192  /* host-evaluated loop-invariant values (ff_args.h FF_MAX_DERIVED_) */

namespace ff {

// Error carried to the ABI boundary, where it becomes an ff_status + ff_last_error() message.
struct Error : std::runtime_error {
  ff_status status;
  Error(ff_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

// ---------------------------------------------------------------- expression AST
enum class Op {
  Num,     // literal (value)
  Var,     // state variable (index)
  Param,   // parameter (index)
  Neg,     // -a
  Add, Sub, Mul, Div, Pow,
  Call     // function (name) with args
};

struct Node {
  Op op;
  double value = 0.0;
  int index = -1;
  std::string name;                  // function name for Call
  std::vector<std::shared_ptr<Node>> args;
  int pos = 0;                       // source position (for messages)
};
using NodeP = std::shared_ptr<Node>;

// Validated system: names, parsed right-hand sides, parameter table.
struct System {
  int dim = 0;
  std::vector<std::string> var_names;
  std::vector<std::string> rhs_text;
  std::vector<NodeP> rhs;
  std::vector<std::string> param_names;
  std::vector<float> param_default, param_min, param_max;
};

// Parse + validate an ff_system (throws Error).
System parse_system(const ff_system* sys);

// Uniform factors of the components ("instruction selection"): component d is written
// f_d = scale_d * rest_d with scale_d a product of factors that depend on parameters only (not on
// state variables, not on the swept parameter `sweep_param`). The kernel integrates rest_d with step
// constants h * scale_d computed by the host per launch, so the RHS never multiplies by scale_d.
// Components with the same factor share a slot; at most FF_MAX_SCALED distinct factors (the first
// ones). Returns the slot of every component (-1 = not split) and fills rest (every component) and
// scale (every split one, else null).
std::vector<int> split_scales(const System& s, int sweep_param, std::vector<NodeP>* rest,
                              std::vector<NodeP>* scale);
// Value (double) of a parameter-only expression for the given parameter values.
double eval_uniform(const NodeP& n, const std::vector<float>& params);

// Loop-invariant values of the generated RHS (products / reciprocals / exponentials of parameters,
// negated parameters), evaluated by the host at every launch and passed in the parameter block
// (FFStepArgs::q), so the kernel reads them as uniform-register operands instead of computing them
// per thread (a per-thread register scalar operand costs FFMA2 throughput).
struct UProgram {
  struct Op { int kind; double value; int index; int a[3]; };
  std::vector<Op> ops;                  // topological order; kind = front-end node kind
  std::vector<std::pair<int, int>> q;   // per q slot: (op index, negate)
  int mufu_per_step = 0;                 // MUFU ops per particle-step of the variant (launch choice)
};
std::vector<float> eval_program(const UProgram& prog, const std::vector<float>& params);

// Emit the complete NVRTC source (generated prefix + device template) for the system with
// parameter `sweep_param` (or -1) per-particle.
// kernel_select: which kernels the program defines (FF_KSEL in ff_device.cuh: 0-11 one step variant,
// 100 = init + render, 255 = all). prog (optional) receives the host program of the q values.
// balance: let a MUFU-bound system compute some exponentials on the FMA pipe (throughput variant;
// launches too small to fill the GPU use balance = false: the polynomial lengthens the RK4 chain).
// long_launch: register budget of the packed 128-thread kernel for launches of many steps (systems
// of <= 4 variables: 40 registers instead of full occupancy's 32).
// push: the fused image exchange's reductions (FF_PUSH in ff_device.cuh: 0 none, 1 every rank's image
// over peer memory, 2 the NVLS multicast address; ff_set_exchange_push).
std::string emit_source(const System& s, int sweep_param, int kernel_select = 255, UProgram* prog = nullptr,
                        bool balance = true, bool long_launch = false, bool thread_redraw = false, int push = 0);

// NVRTC: source -> sm_100a CUBIN (throws Error(FF_ERR_COMPILE) with the log).
std::vector<char> compile_cubin(const std::string& source, const std::string& name);

// "NVRTC <major>.<minor> (<path>)" of the compiler in use (loads it if needed).
std::string nvrtc_description();

// The embedded device template text (ff_device.cuh), generated at build time.
extern const char* const kDeviceTemplate;

}  // namespace ff
