/*
 * bfa.h -- C ABI of libbfa: evaluate a Boolean term on the free generators
 * of the free Boolean algebra on B200 (sm_100a).
 *
 * The operation (§1 property (P); Prop 2.2):
 *   Let f(x_0..x_{n-1}) be a Boolean expression.  The free generators
 *   b_0..b_{n-1} of Omega_n = B^(2^n) are 2^n-bit vectors (rows of the matrix
 *   M whose columns are the binary expansions of 0..2^n-1).
 *   d = f(b_0..b_{n-1}), evaluated bitwise, codes the full DNF of f:
 *       bit mu of d  =  f evaluated at the valuation  x_v = (mu >> v) & 1.
 *   The number of models of f is the popcount of d.
 *
 * Conventions (readings C-1..C-8):
 *   - variable id v <-> bit v of the valuation index mu (LSB first); the
 *     paper's b_1 (MSB row) is id n-1.
 *   - a DNF vector of n variables is ceil(2^n / 64) (at least 1) little-endian
 *     uint64 words; bit mu lives in word mu >> 6 at bit mu & 63.  For n < 6
 *     the unused high bits of word 0 are 0.
 *   - 0 <= n <= 63 for evaluation (counts are uint64); every variable id used
 *     by the program must be < n; unused ids < n are free (each doubles the
 *     count).  Programs may use ids up to 63 (e.g. 8 x 8 relation letters) and
 *     be reduced below 64 variables with bfa_assume (n = 64 allowed there).
 *
 * Expression grammar (UTF-8 text; the compiler and the CPU oracle implement it
 * independently):
 *   program := { stmt (';' | NEWLINE) } [stmt]       '#' comments to end of line
 *   stmt    := 'let' NAME '=' expr                   shared subterm, not a constraint
 *            | NAME '=' expr                         constraint; NAME is also bound
 *            | expr                                  constraint
 *   expr    := imp { '<->' imp }                     IFF, left-assoc
 *   imp     := or [ '->' imp ]                       IMP, right-assoc
 *   or      := xor { '|' xor }
 *   xor     := and { '^' and }                       XOR is the paper's '+'
 *   and     := unary { '&' unary }
 *   unary   := '~' unary | atom
 *   atom    := 'x'DIGITS (id <= 63) | '0' | '1' | NAME | '(' expr ')'
 *   Newlines inside parentheses are whitespace.  The program's value is the
 *   conjunction of all constraint statements (a system e_i = phi_i is solved
 *   when every phi_i = 1); no constraints -> constant 1.
 *   A NAME must be bound before use and may be bound once.
 *
 * Ownership: bfa_prog is created by bfa_compile and owned by the caller until
 * bfa_free; it is immutable after compilation (launch options aside) and may be
 * shared between threads.  It owns its per-device JIT modules.  All output
 * buffers are caller-owned DEVICE memory on the current CUDA device.  The
 * library never returns memory to the caller; materialised mode allocates and
 * frees its own scratch inside the call.
 *
 * Errors: functions returning int return BFA_OK (0) or a negative BFA_E_*
 * code; bfa_count returns UINT64_MAX on error (never a valid count, since
 * counts are <= 2^63).  bfa_last_error() returns a thread-local message for
 * the last failing call (valid until the next call on that thread).  Zero
 * models is not an error.  There is NO CPU fallback: without a CUDA device
 * every compute call fails with BFA_E_CUDA.
 */
#ifndef BFA_H
#define BFA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFA_OK        0
#define BFA_E_PARSE  -1   /* syntax / name error; message carries line:col       */
#define BFA_E_ARG    -2   /* NULL pointer, misaligned range, bad option          */
#define BFA_E_RANGE  -3   /* n > 63, n <= max variable id, range outside [0,2^n) */
#define BFA_E_CUDA   -4   /* CUDA runtime/driver failure or no device            */
#define BFA_E_JIT    -5   /* JIT (PTX compiler / NVRTC) or module load failure   */
#define BFA_E_NOMEM  -6

typedef struct bfa_prog bfa_prog;

typedef struct {
  int32_t  max_var_id;   /* largest variable id used, -1 if none                      */
  int32_t  const_value;  /* -1: not constant; 0 / 1: reduced to that constant        */
  uint64_t tree_nodes;   /* nodes of the binary expression tree as written
                            (the paper's 2^l; let refs count 1)     */
  uint32_t gates;        /* G: 2-input gates of the reduced, hash-consed DAG (NOT free) */
  uint32_t luts;         /* L: LOP3 (3-input LUT) nodes of the unspecialised cover      */
  uint32_t support;      /* number of distinct variable ids used                       */
  uint32_t lets;         /* number of let / named bindings                             */
} bfa_info;

/* ---- compile (host only; "Translate" + "Reduction") ---- */

/* Parse expr, build the hash-consed gate DAG, propagate constants (Reduction)
 * and compute the LUT3 cover.  On success *out owns a new program. */
int bfa_compile(const char* expr, bfa_prog** out);
void bfa_free(bfa_prog* p);                                 /* NULL-safe */
int bfa_info_get(const bfa_prog* p, bfa_info* out);

/* Launch options (part of the JIT cache key).  Keys:
 *   "slot_bits"     log2 words per thread per iteration, 0..14  (default 2;
 *                   eval uses at most 5; each slot is a constant-folded
 *                   cofactor in the body, so large values suit small programs)
 *   "thread_bits"   log2 threads per block, 5..10               (default 8)
 *   "inner_bits"    max log2 inner-loop trip count, 0..8        (default 4)
 *   "blocks_per_sm" resident blocks per SM targeted, 0 = occupancy API (default 0)
 *   "force_generic" 1 = always use the unspecialised word-per-thread kernel
 *   "engine"        0 = JIT straight-line LOP3 (default), 1 = constant-memory
 *                   interpreter (ablation)
 *   "dual_pipe"     1 = map gates with a word-uniform input to IMAD cells on the
 *                   FMA pipe next to LOP3 cells on the ALU pipe (default 1)
 *   "imad_cost_pct" IMAD:LOP3 cost ratio in percent for that mapping, 0 = model
 *                   sweep (default 0)
 *   "imad_pairs"    count mode: an inner-loop LOP3 cell whose other two inputs
 *                   are hoisted word-uniform values becomes x * K + C on the
 *                   FMA pipe (K, C: LOP3 cells at the hoisted level) while the
 *                   modelled ALU work exceeds the FMA work; 2 = roles searched
 *                   without it, kernel emitted with it (default 0)
 *   "min_blocks"    __launch_bounds__ minimum blocks per SM, 0 = none (default 0)
 *   "role_search"   1 = count mode searches the variable -> bit-position roles on
 *                   aligned sub-cubes of >= 2^24 valuations (default 1)
 *   "role_budget"   model evaluations of that search (default 200)
 *   "role_seeds"    independent searches (different seeds) of role_budget
 *                   each; the permutation of least modelled cost whose
 *                   compiled kernel spills no registers is kept (default 1)
 *   "role_seed"     generator seed of the first of those searches (searches
 *                   use seeds role_seed .. role_seed + role_seeds - 1); the
 *                   search is deterministic per seed on every host, so a
 *                   seed measured fastest can be pinned (default 0)
 *   "segment_cells" programs whose cover exceeds 8000 LUTs run as segments of
 *                   this many cells (0 = auto: 768), values crossing segments in
 *                   HBM slot arrays
 *   "segment_remat" recompute shared cells whose cone has <= this many cells in
 *                   each segment instead of storing them (default 2)
 *   "kernel_cofactor_bits" count: split aligned sub-cubes into 2^j cofactor
 *                   programs, one kernel each (default 0; autotune sets it)
 *   "split_pieces"  count: Shannon-decompose aligned sub-cubes into this many
 *                   non-constant pieces first (0..65536; default 0; autotune sets it)
 *   "graphs"        replay multi-launch counts as CUDA graphs (default 1)
 *   "streams"       side streams for independent pieces / cofactors (default 4)
 *   "multi_body"    1: a split's cofactor children as one multi-body launch
 *                   (default 0)
 *   "split_policy"  which piece split_pieces splits next: 0 the heaviest
 *                   (default), 1 the one whose best split saves the most work
 *   "queue_bodies"  > 0: the leaves of a split_pieces decomposition run as
 *                   persistent work-queue kernels of at most this many
 *                   bodies each (default 0 = one kernel per leaf; autotune
 *                   sets it)
 *   "queue_chunk"   work-queue chunk size in modelled thread-instructions
 *                   (default 65536)
 *   "queue_inner"   inner-loop bits of work-queue bodies (default 2; -1:
 *                   inner_bits)
 *   "queue_role_budget" role-search evaluations per work-queue body
 *                   (default 100)
 *   "split_merge"   > 0: after a split_pieces decomposition, merge sibling
 *                   leaves of <= this many gates each back into their parent
 *                   (default 0)
 *   "queue_opt_level" ptxas optimisation level (0..3) of work-queue modules
 *                   (default 3)
 *   "queue_light_pct" the lightest work-queue leaves holding <= this percent of
 *                   the estimated work get 2^(slot_bits-2) slots and a quarter
 *                   of the role-search budget (default 0 = off)
 *   "queue_slot_bits" slot bits of work-queue bodies (-1 = slot_bits; default -1)
 *   "tune_counts"   bfa_autotune's objective: preparation + tune_counts x the
 *                   time of one count (default 1)
 *   "ptx"           1: count-mode specialised kernels and work-queue modules
 *                   are emitted as PTX for the PTX compiler (default); 0: as
 *                   CUDA C++ through NVRTC
 *   "jit_cache"     0: this program neither reads nor writes the persistent JIT
 *                   cache (cubins, role searches); every compile is cold
 *                   (default 1)
 *   "decompose_min_k" split_pieces applies to aligned sub-cubes of >= 2^this
 *                   valuations (default 30; 10..64)
 *   "split_min_vars" decomposition pieces with <= this many free variables
 *                   are not split further (default 24; 5..63)
 *   "queue_support" 1: a work-queue body enumerates only the variables its
 *                   leaf depends on (and enough others for the body layout);
 *                   its count is scaled by 2^(dropped) (default 0)
 * Returns BFA_E_ARG for an unknown key or an out-of-range value. */
int bfa_set_option(bfa_prog* p, const char* key, int64_t value);

/* Plan selection for counting over 2^n valuations by the caller's TOTAL
 * cost: preparation (role searches, decomposition, JIT) + tune_counts x the
 * time of one count (option "tune_counts", default 1 = a single cold count).
 * Tries, in order, (A) the current options as one exhaustive kernel, (B) the
 * kernel-variant sweep (slot bits 2-7, inner-loop bits, IMAD/LOP3 balance,
 * register caps: ~20 variants JIT-compiled in parallel and timed on a probe of
 * <= 2^36 valuations; only when 30 % of tune_counts x A's count time exceeds
 * its predicted cost), (C) partial evaluation: 2^4 kernel cofactors, then
 * Shannon decompositions into 1024 / 4096 / 16384 / 32768 work-queue leaves;
 * a plan whose predicted preparation alone exceeds the best total so far is
 * skipped.  Every tried plan is prepared and timed for real (CUDA events on
 * `stream`, best of 3); p's options are set to the plan of least total.
 * Writes a JSON report (every plan with prep_s, ms and total_s or the reason
 * it was skipped; the variant sweep's candidates; the choice) to report
 * (nullable).  Results do not depend on the plan; only speed does.  Not
 * thread-safe with other calls on the same program.  n < 24: no-op. */
int bfa_autotune(bfa_prog* p, int n, void* stream, char* report, size_t len);

/* As bfa_autotune, for later counts over aligned sub-cubes of 2^k_free
 * valuations (e.g. a rank's cofactor range, k_free = n - log2 P): candidates
 * are timed with the variable roles searched for such a sub-cube. */
int bfa_autotune_range(bfa_prog* p, int n, int k_free, void* stream, char* report, size_t len);

/* ---- register-synthesised mode (generators built in registers) ---- */

/* Number of models of p over all 2^n valuations; synchronous, current device,
 * legacy default stream.  UINT64_MAX on error. */
uint64_t bfa_count(const bfa_prog* p, int n);

/* Full-DNF vector of p: out is a device pointer to >= max(1, 2^(n-6)) u64
 * words; synchronous, current device. */
int bfa_eval(const bfa_prog* p, int n, uint64_t* out);

/* Models with mu in [mu_lo, mu_hi), written (not accumulated) to the single
 * device u64 *count_dev, asynchronously on `stream` (a cudaStream_t; NULL =
 * legacy default stream).  mu_lo and mu_hi must be multiples of 32, or the
 * range must be the whole [0, 2^n). */
int bfa_count_range(const bfa_prog* p, int n, uint64_t mu_lo, uint64_t mu_hi,
                    uint64_t* count_dev, void* stream);

/* Role introspection (count mode; SURVEY.md §8(a) a4 "roles"; DESIGN.md §5
 * role search).  A count over an aligned sub-cube of 2^k_free valuations
 * enumerates it in a searched variable order: variable v (< k_free) takes the
 * value of bit perm[v] of the kernel's position index q (variables >= k_free
 * keep their own bit).  bfa_roles writes that permutation (64 entries,
 * perm_out[v]) for the kernel such a count launches under p's current
 * options, for a device with `sms` SMs (<= 0: the current device's, else
 * 148); host only (runs the search if it is not cached).  BFA_E_ARG when the
 * sub-cube would run on the generic kernel (no roles). */
int bfa_roles(const bfa_prog* p, int n, int k_free, int sms, int8_t* perm_out);

/* Host-only preparation of the count kernel for aligned 2^k_free sub-cubes
 * (e.g. one rank's cofactor range, k_free = n - log2 P): role search + JIT,
 * results cached in p and in the persistent JIT cache, so other processes
 * (the other ranks) load them instead of re-deriving them.  No device needed
 * (sms <= 0: the current device's, else 148).  BFA_E_ARG when such a count
 * would run on the generic kernel only. */
int bfa_prepare_range(const bfa_prog* p, int n, int k_free, int sms);

/* Count with EXACTLY the kernel (same variant, roles and cubin) that a count
 * of an aligned 2^k_free sub-cube launches, over the position range
 * [pos_lo, pos_hi) of its enumeration order: the number of q in the range
 * whose valuation mu(q) (mu_v = bit perm[v] of q) is a model.  This lets a
 * test check the benchmarked kernel of the full 2^n cube against an oracle
 * on sub-ranges: with f'(x) = f(x renamed v -> perm[v]), the result equals
 * the models of f' in [pos_lo, pos_hi).  Bounds must be multiples of the
 * kernel's outer-iteration unit, 2^(5 + slot_bits + thread_bits + m)
 * valuations, else BFA_E_ARG.  Written to *count_dev (device), async on
 * `stream`. */
int bfa_count_positions(const bfa_prog* p, int n, int k_free, uint64_t pos_lo, uint64_t pos_hi,
                        uint64_t* count_dev, void* stream);

/* Multi-GPU count with work-balanced cofactor sharding (
 * DESIGN.md §6): every rank derives the same split of the 2^n cube into 2^j
 * cofactor programs (j >= log2(world) + 2), estimates their work and assigns
 * them to ranks (longest first); *count_dev (device, written) receives this
 * rank's share, and the sum over ranks 0..world-1 is bfa_count(p, n).  The
 * caller sums with one all-reduce.  Synchronous on `stream`. */
int bfa_count_shard(const bfa_prog* p, int n, int rank, int world, uint64_t* count_dev, void* stream);

/* The plan bfa_count_shard follows (host only, no device needed): the number
 * of pieces, and for the first `capacity` of them the owning rank, the
 * piece's number of free variables (it covers 2^piece_vars valuations) and
 * its estimated work (0 = proved identically 0 by the Reduction).  Every
 * rank computes the same plan. */
int bfa_shard_plan(const bfa_prog* p, int n, int world, int* owner, int* piece_vars, uint64_t* work, int capacity,
                   int* n_pieces);

/* Piece `index` of that plan as program text (grammar above; host only): its
 * reduced program over its piece_vars free variables, renumbered 0.. in
 * increasing order of the original ids (as bfa_assume does).  Its model count
 * over 2^piece_vars valuations is the piece's share of bfa_count(p, n), so an
 * independent evaluator (the CPU oracle) can check a rank's share piece by
 * piece.  Returns the text length (excluding NUL), writing up to len bytes. */
int64_t bfa_shard_piece_text(const bfa_prog* p, int n, int world, int index, char* buf, size_t len);

/* Host-only preparation (SURVEY.md §8(b) bfa_compile's JIT, ahead of time):
 * everything bfa_count(p, n) compiles before its first launch -- the
 * decomposition, role searches, kernel emission and JIT compile -- for a device
 * with `sms` SMs (<= 0: the current device's, else 148).  Needs no GPU and
 * launches nothing; results are cached in p (and in the persistent JIT cache).
 * Returns BFA_OK, BFA_E_RANGE (bad n) or BFA_E_JIT. */
int bfa_prepare(const bfa_prog* p, int n, int sms);

/* The slice [mu_lo, mu_hi) of the DNF vector, asynchronously on `stream`:
 * bit (mu - mu_lo) at word (mu - mu_lo) >> 6 of out_dev (device,
 * ceil((mu_hi-mu_lo)/64) words).  mu_lo, mu_hi multiples of 64, or the whole
 * range.  If count_dev is non-NULL the slice's popcount is fused and written
 * there. */
int bfa_eval_range(const bfa_prog* p, int n, uint64_t mu_lo, uint64_t mu_hi,
                   uint64_t* out_dev, uint64_t* count_dev, void* stream);

/* ---- killing variables and model enumeration ---- */

/* Killing variables (§3.3; the `assumptions` of §4.2,
 * PAPER.md:1104-1125): variables v < n with bit v of `mask` set are fixed to
 * bit v of `values`, the Reduction is re-run, and the remaining variables
 * < n are renumbered densely in increasing order.  *out is a new program over
 * *n_free = n - popcount(mask & (2^n - 1)) variables (its own options are
 * copied from p); free_ids (nullable, >= n entries) receives the original id
 * of each new id, so a model mu' of *out is the model
 * deposit(mu', free_ids) | (values & mask) of p. */
int bfa_assume(const bfa_prog* p, int n, uint64_t mask, uint64_t values, bfa_prog** out, int* n_free,
               int* free_ids);  /* 0 <= n <= 64 */

/* Model enumeration ("all labeled models"; out.txt rows,
 * PAPER.md:1091-1096): the models mu in [mu_lo, mu_hi) (bounds as for
 * bfa_count_range), in ASCENDING order, into the device list mu_out (the first
 * `capacity` of them); *count_dev (device) receives the total number of
 * models.  The range is evaluated chunk by chunk (<= 2^33 valuations, a
 * 1 GiB device vector allocated and freed inside the call) by the
 * register-mode eval kernel, and each chunk's set bits are compacted in mu
 * order (per-tile popcounts, one scan, ordered rewrite: no atomics, no sort).
 * Synchronous on `stream`. */
int bfa_enumerate(const bfa_prog* p, int n, uint64_t mu_lo, uint64_t mu_hi, uint64_t* mu_out, uint64_t capacity,
                  uint64_t* count_dev, void* stream);

/* out.txt rows (one row per model, a valuation of the
 * letters): for each of the `count` models mu' in mu_dev (device) of a program
 * over n_free letters -- e.g. a bfa_assume result -- the valuation of the
 * original n_all letters, deposit(mu', free_ids) | fixed_values (killed
 * letters reinstated; free_ids host array of n_free ids, NULL = identity),
 * written to rows_dev (device, count * (n_all + 1) bytes) as n_all characters
 * '0'/'1' -- letter id n_all - 1 (the paper's b_1) first -- and '\n'.  Async on
 * `stream`. */
int bfa_rows(const uint64_t* mu_dev, uint64_t count, int n_free, const int* free_ids, int n_all,
             uint64_t fixed_values, char* rows_dev, void* stream);

/* Batched counting (the counting procedure TBA runs
 * one reduced program per c-partition): many programs in
 * ONE launch.  bfa_batch_create JIT-compiles a kernel holding every program
 * (the programs must outlive the batch); bfa_batch_count counts program i
 * over all 2^ns[i] valuations into counts_dev[i] (device, `count` u64),
 * synchronous on `stream`.  Meant for many small programs. */
typedef struct bfa_batch bfa_batch;
int bfa_batch_create(const bfa_prog* const* progs, int count, bfa_batch** out);
int bfa_batch_count(bfa_batch* b, const int* ns, uint64_t* counts_dev, void* stream);
void bfa_batch_free(bfa_batch* b);                          /* NULL-safe */

/* ---- materialised mode (the paper's vector formulation) ---- */

/* Fill the generator table S: row v (0 <= v < n_rows) is
 * the 2^n-bit free generator b_v, at table_dev + v * max(1, 2^(n-6)) words. */
int bfa_fill_generators(int n, int n_rows, uint64_t* table_dev, void* stream);

/* Evaluate p with every generator and intermediate vector materialised in
 * HBM.  variant 0: vector algebra, one full-vector LOP3 pass per LUT node
 * (the program list lives in __constant__ memory); variant 1: fused, 128-bit
 * loads of the generator table and the LOP3 body in registers.  out_dev as in
 * bfa_eval; count_dev (nullable) receives the popcount.  Synchronous on
 * `stream`.  Requires n >= 7. */
int bfa_eval_materialised(const bfa_prog* p, int n, int variant, uint64_t* out_dev,
                          uint64_t* count_dev, void* stream);

/* Popcount of n_words device u64 words into *count_dev (written). */
int bfa_popcount(const uint64_t* vec_dev, uint64_t n_words, uint64_t* count_dev, void* stream);

/* ---- measurement ---- */

/* Integer issue-rate microbenchmark (the roofline denominators): launches
 * blocks x threads (<= 256) threads, each executing iters x 256 operations in
 * 8 independent chains.  op 0: lop3.b32 (ALU pipe), 1: mad.lo.u32 (IMAD, FMA
 * pipe), 2: both, interleaved 1:1.  The caller times it with events;
 * ops = blocks * threads * iters * 256. */
int bfa_peak_int(int op, int blocks, int threads, int iters, uint32_t* sink_dev, void* stream);

/* Statistics of the kernel variant the last launch on this thread used:
 * executed LUTs per 32-bit word at each loop level etc., as a JSON object
 * written to buf (NUL-terminated, truncated to len). */
int bfa_last_launch_json(char* buf, size_t len);

/* ---- introspection (host only; usable without a GPU) ---- */

/* what = 0: LUT3 cover IR text, one line per LUT:
 *           "L<k> = lop3(<a>, <b>, <c>, 0x<imm>)" with operands "x<id>",
 *           "L<j>" or "0x<word>", followed by "out = [~]<operand>".
 * what = 1: source of the specialised count kernel for n: PTX (option "ptx",
 *           the default) or CUDA C++ (ptx = 0).
 * what = 2: CUDA source of the specialised eval kernel for n.
 * what = 3: CUDA source of the unspecialised (generic) count kernel.
 * what = 4: CUDA source of the fused materialised-mode kernel.
 * what = 5: JSON summary of the segmented-execution plan (large programs).
 * what = 6: CUDA source of segment n of that plan.
 * what = 7: the reduced program (hash-consed DAG after the Reduction) as
 *           text in the grammar above: one `let` per gate, then the root.
 * Returns the full length needed (excluding NUL) or a negative error. */
int64_t bfa_dump(const bfa_prog* p, int what, int n, char* buf, size_t len);

/* JIT-compile kernel `what` (1..3 as in bfa_dump) for sm_100a without a
 * device and return the cubin size; if buf is non-NULL copy up to len bytes.
 * Lets the build check every generated kernel on a CPU-only host. */
int64_t bfa_jit_cubin(const bfa_prog* p, int what, int n, void* buf, size_t len);

/* Message of the last failing call on this thread (thread-local, valid until
 * the next failing call on this thread). */
const char* bfa_last_error(void);
/* BFA_E_* code of the last failing call on this thread (0 if none yet); the
 * way to classify a bfa_count failure, which returns UINT64_MAX. */
int bfa_last_error_code(void);
const char* bfa_version(void);

/* Persistent JIT cache key of a generated kernel source (host only): the
 * 64-hex-digit SHA-256 over the cache format salt, the compiler version
 * (NVRTC for CUDA C++, the PTX compiler for generated PTX), its options and
 * the source; cubins are stored as k_<key>.cubin under
 * $BFA_JIT_CACHE (default ~/.cache/bfa_jit; "0" disables the cache).  out
 * receives 64 digits + NUL (len >= 65), else BFA_E_ARG. */
int bfa_cache_key(const char* source, char* out, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* BFA_H */
