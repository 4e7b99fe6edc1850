// LoopProgram: the reference's scheduled per-cell kernel (LoopProgram,
// reference scheduling.py:87-95) read from its loss-free JSON form
// (serialize_program / parse_program, scheduling.py:465-596), and the
// batched sm_100a CUDA kernel generated from it.
//
// The reference lowers a LoopProgram to one C99 function per cell
// (emit_c, scheduling.py:617-738): temporaries on the stack, every loop nest
// executed by one core.  Here the same statement list runs over a batch of
// cells per CTA:
//   * every buffer (arguments, A, temporaries) lives in shared memory
//     (or a per-CTA global arena when a cell does not fit), laid out
//     cell-fastest: element e of cell c at  S[(base + e) * NCP + c];
//   * each top-level perfect loop nest becomes one CTA-wide phase: its
//     "parallel" loops (those indexing the target) are flattened with the
//     cell index across threads, its reduction loops stay sequential per
//     thread in the reference's order, so every target element is summed in
//     exactly the reference's order (bit-identical results when compiled
//     without FMA contraction, as the reference's -ffp-contract=off build);
//   * a ZeroFill followed by a nest that overwrites the whole buffer is
//     folded into the nest (the accumulator starts at 0.0);
//   * temporaries share storage by liveness (top-level statement ranges),
//     barriers are placed only where a phase touches storage an earlier
//     phase wrote (or reads storage a later phase overwrites).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "lp_json.h"

namespace sfk {
namespace lp {

struct Entry {       // multi-index entry: a loop index or an integer
  int idx = -1;      // index id (>= 0) or -1 for a constant
  long long val = 0;
};

struct Term {
  Entry e;
  long long stride = 0;
};

struct Expr;
using ExprP = std::shared_ptr<Expr>;

struct Expr {
  enum Kind { LIT, LOAD, TABLE, DELTA, ADD, MUL, DIV, POW, MIN, MAX, CALL, CMP } k = LIT;
  double lit = 0.0;
  std::string name;                // LOAD: buffer name; CALL: function; CMP: operator
  int table = -1;                  // TABLE: table id
  long long offset = 0;            // LOAD / TABLE: flat address = offset + sum stride*entry
  std::vector<Term> terms;
  Entry d0, d1;                    // DELTA
  ExprP a, b;
};

struct Stmt {
  enum Kind { LOOP, ASSIGN, ACCUM, ZERO } k = LOOP;
  int idx = -1;                    // LOOP
  int extent = 0;
  std::vector<Stmt> body;
  std::string name;                // ASSIGN / ACCUM target, ZERO buffer
  long long offset = 0;
  std::vector<Term> terms;
  ExprP e;
  long long size = 0;              // ZERO
};

struct Table {
  std::vector<long long> shape;
  std::vector<double> values;
};

struct Program {
  std::string name;
  std::string ret_name;
  long long ret_size = 0;
  std::vector<std::pair<std::string, long long>> args;
  std::vector<std::pair<std::string, long long>> temps;
  std::vector<Stmt> body;
  std::vector<Table> tables;
  std::map<int, int> extents;      // index id -> extent
};

// Parse the JSON text written by the reference's serialize_program.
// Throws std::runtime_error on malformed input.
Program parse_program(const char* text, size_t n);

// Launch geometry chosen by the generator.
struct Config {
  int cells_per_block = 1;   // NC (power of two)
  int ncp = 1;               // cell stride of a slot (NC or NC+1)
  int threads = 256;
  int64_t slots = 0;         // per-cell slots (args + A + packed temporaries)
  int64_t smem_bytes = 0;    // dynamic shared memory per CTA
  bool global_scratch = false;
  int64_t arena_doubles_per_block = 0;
  int tables_in_smem = 1;
  int phases = 0;            // CTA-wide phases (after zero folding)
  int serial_phases = 0;     // phases executed thread-per-cell
  int barriers = 0;          // __syncthreads, or __syncwarp in warp mode
  int warp_mode = 0;         // 1: every warp owns cells_per_warp whole cells
  int fused_phases = 0;      // phases running inside the previous phase's loop
  int cells_per_warp = 0;
};

struct Generated {
  std::string source;        // CUDA C++ (NVRTC) text
  std::string entry;         // kernel name
  Config cfg;
};

// smem_limit: usable dynamic shared memory per CTA (bytes).
Generated generate(const Program& p, int64_t smem_limit, bool allow_fma);

}  // namespace lp
}  // namespace sfk
