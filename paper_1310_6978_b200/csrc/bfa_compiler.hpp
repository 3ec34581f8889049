// bfa_compiler.hpp -- host-side compiler of libbfa.
//
// expression text --parse--> hash-consed gate DAG with constant propagation
// (the paper's Translate + Reduction submodules)
// --specialise--> per-slot cofactors with loop-level roles for the variables
// --map--> 3-input LUT cover (one lop3.b32 per LUT, the "efficient computing
// tree adapted to the actual parallel hardware")
// --emit--> straight-line CUDA C++ for NVRTC (the paper's core is likewise
// generated code compiled to binaries at run time).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace bfa {

// A literal is (node << 1) | complement.
using Lit = uint32_t;
inline uint32_t lit_node(Lit l) { return l >> 1; }
inline bool lit_neg(Lit l) { return l & 1u; }
inline Lit mk_lit(uint32_t node, bool neg) { return (node << 1) | (neg ? 1u : 0u); }

enum NodeKind : uint8_t { NK_CONST = 0, NK_VAR = 1, NK_GATE = 2 };

// Gates are 2-input with a 4-bit truth table over POSITIVE node inputs:
// bit (a + 2b) = f(a, b).  Complements live only on literals.  Constants are
// 32-bit words (a word constant is a lane mask of the low variables); they are
// normalised so that bit 0 of the stored word is 0.
struct Node {
  NodeKind kind;
  uint8_t tt;       // GATE
  uint32_t a, b;    // GATE inputs (node ids), a < b
  uint32_t val;     // VAR: variable id (or role slot); CONST: word
};

class Dag {
 public:
  Dag();
  std::vector<Node> nodes;

  Lit const0() const { return mk_lit(0, false); }
  Lit const1() const { return mk_lit(0, true); }
  Lit word(uint32_t w);
  Lit var(uint32_t id);
  Lit gate(uint8_t tt, Lit a, Lit b);

  Lit NOT(Lit a) { return a ^ 1u; }
  Lit AND(Lit a, Lit b) { return gate(0x8, a, b); }
  Lit OR(Lit a, Lit b) { return gate(0xE, a, b); }
  Lit XOR(Lit a, Lit b) { return gate(0x6, a, b); }
  Lit IMP(Lit a, Lit b) { return gate(0xD, a, b); }  // ~a | b : f(1,0) = 0 only
  Lit IFF(Lit a, Lit b) { return gate(0x9, a, b); }

  bool is_const(Lit l) const { return nodes[lit_node(l)].kind == NK_CONST; }
  uint32_t const_word(Lit l) const {
    uint32_t w = nodes[lit_node(l)].val;
    return lit_neg(l) ? ~w : w;
  }
  size_t gate_count() const;

 private:
  std::unordered_map<uint64_t, uint32_t> gate_table_;
  std::unordered_map<uint32_t, uint32_t> word_table_;
  std::unordered_map<uint32_t, uint32_t> var_table_;
};

struct Parsed {
  Dag dag;
  Lit root = 0;
  int max_var = -1;
  uint64_t tree_nodes = 0;
  uint32_t lets = 0;
  uint64_t support_mask = 0;
};

// Parse `text` (grammar in include/bfa.h).  Returns 0 or -1 with "line:col: msg".
int parse_program(const std::string& text, Parsed* out, std::string* err);

// Killing variables (§3.3; the `assumptions` of §4.2,
// PAPER.md:1104-1125): variables v < n with bit v of `mask` set become the
// constant bit v of `values`; the Reduction runs again; the surviving
// variables < n are renumbered densely in increasing order.  free_ids[new] =
// old id.
Parsed assume(const Parsed& src, int n, uint64_t mask, uint64_t values, std::vector<int>* free_ids);

// Number of gates reachable from the root.
uint32_t gate_count(const Parsed& p);

// Kernel-level cofactoring: greedily pick j of the variables < k whose
// 2^j cofactors (bfa_assume) have the fewest gates in total after Reduction.
std::vector<int> choose_cofactor_vars(const Parsed& p, int k, int j, uint64_t* best_total = nullptr, int threads = 1);

// ---------------------------------------------------------------- mapping
struct Lut {
  uint32_t root;      // node id in the mapped DAG
  uint8_t nin;        // leaves used (1..3)
  uint32_t in[3];     // leaf node ids (VAR, CONST or GATE roots)
  uint8_t imm;        // lop3 immLut over (in[0], in[1], in[2]) ~ (0xF0, 0xCC, 0xAA)
  uint8_t level;      // loop level of the root
  // kind 1 = IMAD cell (FMA pipe): root = u ? f1(x) : f0(x) with x = in[0] and
  // u = in[1] a word-uniform value (0 or ~0 in every word); f0/f1 are unary
  // codes 0:"0", 1:"~0", 2:"x", 3:"~x"; emitted as x * M(u) + C(u).
  // kind 2 = IMAD cell of a 3-input cut with two word-uniform leaves:
  // root = x * in[1] + in[2] (mad.lo.u32), in[1] = K(u1, u2) in {0, 1, ~0}
  // and in[2] = C(u1, u2) in {0, ~0} computed by LOP3 cells at the uniform
  // leaves' (hoisted) loop level (KernelSpec::imad_pairs).
  uint8_t kind = 0;
  uint8_t f0 = 0, f1 = 0;
};

// Map the DAG (restricted to the cones of `outputs`) onto 3-input LUTs.
// level_of_var(var id) gives each variable's loop level; constants are level
// 0.  weights[level] is the relative execution frequency used by area flow.
struct MapResult {
  std::vector<Lut> luts;                 // topological order
  std::vector<uint8_t> node_level;       // per node of the dag
};
// imad_cost > 0 enables IMAD cells for gates with a word-uniform input, at
// that cost relative to one LUT (two-resource area flow).
// area_passes > 0: that many exact-area recovery passes after area flow.
MapResult map_luts(const Dag& dag, const std::vector<Lit>& outputs,
                   const std::vector<uint8_t>& var_level, const double weights[4],
                   double imad_cost = 0.0, int area_passes = 0);

// ---------------------------------------------------------------- kernels
enum KernelMode : int { KM_COUNT = 0, KM_EVAL = 1 };

struct KernelSpec {
  KernelMode mode = KM_COUNT;
  bool generic = false;   // one word per thread-iteration, every variable from w
  int slot_bits = 2;      // s
  int thread_bits = 8;    // t
  int inner_bits = 4;     // m
  bool fuse_count = false;  // eval mode: also popcount
  bool materialised = false;  // generic only: every generator word is LOADED from the
                              // table S (128-bit loads, 4 words per thread-iteration)
  int dual_pipe = 1;          // 1: balance LOP3 (ALU pipe) and IMAD (FMA pipe) cells
  int imad_cost_pct = 0;      // >0: fixed IMAD:LOP3 cost ratio (percent) instead of the sweep
  int min_blocks = 0;         // >0: __launch_bounds__ minimum resident blocks per SM
  std::vector<int8_t> perm;   // count mode: bit position of each variable in the
                              // word/valuation index (empty = identity)
  std::string body_name;      // non-empty: emit the specialised kernel as a
                              // __device__ __noinline__ body of a multi-body kernel
  int area_passes = 1;        // exact-area recovery passes of the LUT mapper (emission;
                              // model_cost -- the role search's objective -- uses 0)
  int count_shift = 0;        // count mode: the count is scaled by 2^count_shift
                              // (support reduction: variables outside the support)
  int imad_pairs = 0;         // count mode: inner-loop LOP3 cells whose other two
                              // leaves are hoisted word-uniform values become
                              // kind-2 IMAD cells while that balances the pipes
  int vec_bits = -1;          // eval mode: each thread stores 2^vec_bits consecutive
                              // words per vector store; the slot bits above
                              // vec_bits sit above the thread bits in the word
                              // index, so a warp's store covers 32 x 2^vec_bits
                              // consecutive words (-1 or >= s: all s slot bits
                              // below the thread bits)
};

struct KernelStats {
  uint32_t luts_thread = 0, luts_outer = 0, luts_inner = 0;  // LOP3 cells emitted per level
  uint32_t imads_thread = 0, imads_outer = 0, imads_inner = 0;  // IMAD cells per level
  uint32_t derived_inner = 0, derived_outer = 0;  // IMAD operand registers computed per level
  double imad_cost = 0.0;                         // the mapping's chosen IMAD/LUT cost ratio
  uint32_t inner_vars = 0, outer_vars = 0, thread_vars = 0;
  uint32_t words_per_iter = 1;
};

// One kernel for several programs (kernel-level cofactor children of one
// piece): each child's specialised kernel becomes a noinline device body;
// block b runs body b / bpc with block index b % bpc of bpc blocks.  Kernel
// signature: (u64 A, u64 o_count, u64 out_base_w, u32* out, u64* count, u32 bpc).
std::string emit_multi(const std::vector<const Parsed*>& progs, const std::vector<KernelSpec>& specs,
                       std::vector<KernelStats>* stats);

// One persistent work-queue kernel for many programs (the leaves of a
// Shannon decomposition).  body_src[i] is the source of a noinline device
// body named body_name[i] (emit_kernel with KernelSpec::body_name); body i
// covers o_count[i] outer iterations, cut into chunks[i] contiguous chunks.
// The chunks are numbered body by body in the given order; a block takes the
// next chunk number with one atomicAdd on *ctr and runs that body on that
// chunk, until all chunks are taken.  *ctr must be 0 before the first launch;
// the block making the launch's last increment (total + gridDim.x - 1)
// resets it to 0, so launches (and graph replays) need no memset, but two
// launches of one module must not overlap in time.  Kernel signature:
// (u64* count, u32* ctr).
std::string emit_queue(const std::vector<std::string>& body_src, const std::vector<std::string>& body_name,
                       const std::vector<uint64_t>& o_count, const std::vector<uint32_t>& chunks, int thread_bits,
                       int min_blocks);

// Common device helpers of every generated source (typedefs, sums, append).
extern const char* kPrelude;

// Modelled time per thread-iteration of the variant's best cover.
double model_cost(const Parsed& prog, const KernelSpec& spec);

// Role search for count mode over an aligned sub-cube of 2^k_free valuations:
// a permutation of the variables < k_free onto bit positions minimising
// model_cost (random restarts + swap hill climbing, `budget` evaluations).
// Returns {} when the identity is best.  threads > 1 evaluates candidates
// speculatively in parallel with the same result as threads = 1.
std::vector<int8_t> search_roles(const Parsed& prog, const KernelSpec& spec, int k_free, int budget, uint64_t seed,
                                 int threads = 1);

// PTX of the count-mode specialised kernel (entry "bfa_kernel", parameters
// (A, o_count, out_base_w, out, count) as emit_kernel's), or, with
// spec.body_name set, of a work-queue body `.func body_name(count, bid, nb)`
// over body_o_count outer iterations from word 0.  Same cover, schedule and
// loops as emit_kernel; compiled by the PTX compiler without NVRTC.
std::string emit_ptx(const Parsed& prog, const KernelSpec& spec, KernelStats* stats, uint64_t body_o_count = 0);

// PTX of a work-queue kernel (as emit_queue) over PTX bodies: body_ptx holds
// the distinct bodies' .func text, body_name[i] / chunks[i] the body and
// chunk count of queue entry i.
std::string emit_ptx_queue(const std::vector<std::string>& body_ptx, const std::vector<std::string>& body_name,
                           const std::vector<uint32_t>& chunks, int thread_bits, int min_blocks, int opt_level = 3);

// CUDA C++ source of one kernel variant (entry point "bfa_kernel").
std::string emit_kernel(const Parsed& prog, const KernelSpec& spec, KernelStats* stats);

// Program for the constant-memory interpreter (engine=1, the ablation of the
// JIT): ops are uint4 {dst | imm << 16 | kind << 24, a, b, c}; kind 0 = LOP3
// over operands a, b, c, kind 1 = generator word of variable (a + 5) from the
// word index.  An operand with bit 31 set is consts[operand & 0xff], else a
// value slot.  Slots are reused by liveness.
struct InterpProgram {
  std::vector<uint32_t> ops;     // 4 words per op
  std::vector<uint32_t> consts;
  uint32_t n_slots = 0;
  uint32_t out = 0;              // operand encoding of the result
  bool out_neg = false;
};
InterpProgram build_interp(const Parsed& prog);

// Segmented execution for programs too large for one straight-line kernel
// (the paper's 2^17-node term): the generic cover in
// depth-first order is cut into segments of <= seg_cells cells; segment i is
// kernel i.  Values used after their segment live in global slot arrays
// (slot-major, `stride` words per slot).  Kernel signature:
//   (u64 w_begin, u64 w_count, u32 mask, u32* gbuf, u64 stride, u32* out, u64* count)
// and only the last segment counts / stores the result.
struct SegPlan {
  std::vector<std::string> sources;
  std::vector<uint32_t> cells;     // per segment
  uint32_t n_slots = 0;
  uint32_t max_live = 0;           // most values crossing one boundary
  uint64_t emitted = 0;            // cells emitted incl. rematerialised ones
};
SegPlan emit_segmented(const Parsed& prog, KernelMode mode, bool fuse_count, int seg_cells, int thread_bits,
                       int imad_cost_pct = 50, int remat = 6);

// Batched counting: one kernel for many programs.
// Program j is a __noinline__ device function of its word index; the kernel
// walks a global word space in which program j owns [start[j], start[j+1])
// (each padded to whole warps) and accumulates counts[j].  Kernel signature:
//   (const u64* start, const u32* masks, const u64* words, int nprog,
//    u64 total, u64* counts)
std::string emit_batch(const std::vector<const Parsed*>& progs, int thread_bits);

// LUT cover IR text (bfa_dump what=0) and the plain cover size L.
std::string dump_ir(const Parsed& prog, uint32_t* n_luts);

// The program's reduced DAG as text in the grammar of include/bfa.h: one
// `let gK = ...` per gate of the root's cone, then the root as the single
// constraint (0 / 1 for a constant program).
std::string to_text(const Parsed& prog);

}  // namespace bfa
