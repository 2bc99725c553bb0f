/*
 * polyeval-b200 — C ABI of the B200 batch polynomial evaluator.
 *
 * Drop-in boundary for the reference's compile-once / evaluate API
 * (reference: proj/core/include/polyeval/eval.hpp). The reference exposes a
 * C++ template API, not an FFI; each entry point below names the reference
 * interface it replaces:
 *
 *   pe_program_create      build()/build_multivariate() + compute_lazy_heights()
 *                          + compile()            tree.hpp:58-77, eval.hpp:57
 *                          (polynomial from raw terms: Polynomial::canonicalize,
 *                          polynomial.hpp:34-36; schemes: scheme.hpp:15-57)
 *   pe_program_from_compiled  an existing CompiledProgram (compile() output,
 *                          eval.hpp:32-57), flattened; same evaluation semantics
 *   pe_program_destroy     CompiledProgram lifetime (move-only, eval.hpp:32-54)
 *   pe_eval_f64            Evaluator<DoubleDomain>(domain, program) +
 *                          evaluate(point) per point   eval.hpp:74-90, ring.hpp:40-48
 *   pe_eval_i64            Evaluator<BigIntDomain> on a proven int64 range
 *                                                       eval.hpp:74-90, ring.hpp:30-38
 *   pe_eval_limbs          Evaluator<BigIntDomain> beyond int64 (K x 64-bit limbs)
 *                                                       ring.hpp:30-38, bigint.cpp
 *   pe_eval_interval       Evaluator<IntervalDomain>    ring.hpp:50-65, interval.cpp:36-52
 *   pe_program_info        CompiledProgram fields (register_count, records,
 *                          exponent_sets, root_child_ends)  eval.hpp:32-54
 *   pe_program_dot         to_dot(tree)                 tree.hpp:85-88
 *   pe_last_error          exception what()             error.hpp:11-39
 *
 * Conventions:
 *   - No exceptions cross this boundary; every call returns a pe_status.
 *     PE_EINVAL   <=> std::invalid_argument (arity, null pointers, bad scheme)
 *     PE_EOVERFLOW   int64 range proof failed, or a coordinate exceeded the
 *                    proven bound (the reference BigInt never overflows; this
 *                    path refuses instead of wrapping — there is no CPU fallback)
 *     PE_ECUDA       CUDA / JIT failure (message in pe_last_error)
 *     PE_ELOGIC   <=> std::logic_error
 *   - pe_last_error() is thread-local and valid until the next call on the
 *     same thread.
 *   - A program is immutable after creation and safe to share across host
 *     threads (the reference's CompiledProgram contract, eval.hpp:59-68).
 *     Device kernels are specialised and loaded lazily per (domain, device)
 *     and cached on the handle.
 *   - Point and result buffers are caller-owned, structure-of-arrays: coords[v]
 *     points at n values of variable v (variable order of the program).
 *     Pointers may be device memory (evaluated in place, asynchronously on
 *     exec->stream) or host memory (chunked H2D / walk / D2H pipeline on the
 *     library's own streams, copies overlapping the neighbouring chunks'
 *     walks; pageable memory is first copied into page-locked staging
 *     buffers by host threads; the call returns when results are on the
 *     host). All buffers of one call must be device memory (of one device) or
 *     all host memory, else PE_EINVAL. n == 0 is valid and does nothing.
 */
#ifndef POLYEVAL_B200_H_
#define POLYEVAL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pe_status {
  PE_OK = 0,
  PE_EINVAL = 1,
  PE_EOVERFLOW = 2,
  PE_ECUDA = 3,
  PE_ELOGIC = 4,
} pe_status;

/* Builtin function schemes (reference scheme.hpp:36-41). */
typedef enum pe_scheme_id {
  PE_SCHEME_DIRECT = 0,
  PE_SCHEME_HORNER = 1,
  PE_SCHEME_ESTRIN = 2,
  PE_SCHEME_BALANCED = 3,
} pe_scheme_id;

/* One scheme per variable: `upper` alone when cutoff == 0, else
 * threshold_combine(upper, lower, cutoff) (reference scheme.hpp:43-47),
 * i.e. the CLI grammar "upper:lower@cutoff" (tools/scheme_name.cpp:34-53). */
typedef struct pe_scheme_desc {
  int32_t upper;
  int32_t lower;
  uint64_t cutoff;
} pe_scheme_desc;

typedef enum pe_coeff_type {
  PE_COEFF_F64 = 0, /* const double* coeffs */
  PE_COEFF_I64 = 1, /* const int64_t* coeffs */
} pe_coeff_type;

typedef struct pe_program pe_program;

/* Execution options. Zero-initialise for defaults (device 0 / current,
 * default stream, fused fp64). */
typedef struct pe_exec {
  int32_t device;       /* CUDA device ordinal; -1 = current device */
  int32_t strict_f64;   /* pe_eval_f64: 1 = reference op order, bit-exact  */
  void* stream;         /* cudaStream_t for device-pointer calls; NULL = legacy default */
  int32_t synchronize;  /* device-pointer calls: 1 = wait for completion */
  int32_t i64_int_pipe; /* pe_eval_i64: 1 = always use the int64 IMAD kernel
                           (default picks exact-on-FP64 when the 2^53 proof holds) */
  /* pe_eval_i64 only: caller-asserted per-variable bounds |x_v| <= bound[v]
   * (nvars entries; NULL = derive from the data with a device max-reduction). */
  const uint64_t* i64_bounds;
  /* Device-pointer pe_eval_i64 / pe_eval_interval: 1 = return right after
   * enqueueing (no host round trip per call); domain-check failures (a
   * coordinate beyond the proven int64 bound, invalid interval endpoints)
   * accumulate in a per-(device, stream) status word and are reported by the
   * next pe_synchronize(exec). The int64 retry with data-derived bounds is
   * not attempted in this mode (re-run synchronously to get it). */
  int32_t deferred_checks;
  int32_t reserved;
  /* Host-buffer calls: shard the batch over devices[0..ndevices) — contiguous
   * slices of ceil(n / ndevices) points, one staged pipeline per device,
   * running concurrently; every device writes its slice of the results
   * straight into the caller's host output (the gather). The program is
   * replicated to each device on first use. NULL / 0 = exec->device only.
   * Device-buffer calls reject ndevices > 1 (their data lives on one device). */
  const int32_t* devices;
  int32_t ndevices;
  /* Host-buffer calls: points per pipeline chunk (0 = n/16 clamped to
   * [256K, 4M]) and chunks in flight (0 = 3; 2..8). */
  int32_t stage_slots;
  uint64_t stage_chunk;
} pe_exec;

/* Compiles a polynomial given as raw terms: `exponents` is nterms x nvars
 * (row-major), `coeffs` nterms values of `coeff_type`. Terms are
 * canonicalised (sorted, like terms merged, zeros dropped). One scheme per
 * variable; nvars == 1 uses build(), nvars > 1 build_multivariate(). */
pe_status pe_program_create(const uint32_t* exponents, const void* coeffs,
                            size_t nterms, uint32_t nvars,
                            const pe_scheme_desc* schemes,
                            pe_coeff_type coeff_type, pe_program** out);

/* One record of a flattened reference CompiledProgram (eval.hpp:32-41:
 * CompiledProgram::Record). Exactly one of the coefficient fields is read,
 * per the coeff_type of pe_program_from_compiled; it is ignored when `sub`
 * names a nested program (the record's coefficient is that program). */
typedef struct pe_record {
  double coeff_f64;
  int64_t coeff_i64;
  int32_t sub;            /* index of the nested program in `programs`, or -1 */
  int32_t power_slot;     /* index into exponent_sets[variable], or -1 (absent) */
  uint32_t lazy_slot;
  int32_t parent_slot;    /* -1 only for the last (root) record */
  int32_t reads_register; /* 0 / 1 */
  int32_t reserved;       /* 0 */
} pe_record;

/* One (root or nested) program: CompiledProgram::{records, register_count,
 * variable, root_child_ends} (eval.hpp:43-51). */
typedef struct pe_compiled_program {
  const pe_record* records;
  size_t nrecords;
  uint32_t register_count;
  uint32_t variable;
  const uint32_t* root_child_ends;
  size_t nroot_child_ends;
} pe_compiled_program;

/* Lowers an already compiled program — the reference's
 * CompiledProgram compile(const EvaluationTree&) output (eval.hpp:57),
 * flattened: programs[0] is the root, nested programs are referenced from
 * records by index, each exactly once. exponent_sets[v] (sorted, distinct,
 * >= 1; exponent_set_sizes[v] entries) are the root's per-variable sets
 * (eval.hpp:53-54). Evaluation follows the given records verbatim: strict
 * fp64 and intervals replay their op sequence bit for bit. Malformed programs
 * (slot out of range, a record whose parent register is never read, a nested
 * program referenced twice, ...) are rejected with PE_EINVAL. Such a program
 * has no tree: pe_program_dot returns PE_EINVAL, and wide fp64 programs are
 * not sliced. */
pe_status pe_program_from_compiled(const pe_compiled_program* programs, size_t nprograms,
                                   uint32_t nvars, const uint32_t* const* exponent_sets,
                                   const size_t* exponent_set_sizes, pe_coeff_type coeff_type,
                                   pe_program** out);

void pe_program_destroy(pe_program* program);

/* Code-generation options of a program's kernels. Zero-initialise for the
 * measured defaults; every field's 0 means "default". */
typedef struct pe_tuning {
  uint32_t lanes;          /* points per thread, 1..8 */
  uint32_t block;          /* threads per CTA, 32..1024 (wide programs: threads per
                              point, 32..256; default by value width and batch size) */
  uint32_t min_ctas;       /* .minnctapersm of the walk kernel (wide programs: CTAs,
                              i.e. points in flight, per SM) */
  uint32_t sync_every;     /* walk ops between CTA barriers */
  uint32_t section_ops;    /* long int/fp64 walks: ops per section of the persistent
                              sectioned kernel (default 3000; UINT32_MAX = one plain
                              kernel) */
  uint32_t sched_window;   /* latency-aware op reordering window (1 = walk order) */
  uint32_t sched_distance; /* producer distance the reordering aims for */
  uint32_t chain_min;      /* shortest Horner run emitted as a loop (default 64;
                              UINT32_MAX = never) */
  int32_t iv_fast;         /* interval: -1 = bit-level replay only (no fast path) */
  int32_t iv_mid;          /* interval fixup: -1 = skip the finite-case replay */
  int32_t iv_partition;    /* univariate interval sign partition: -1 = off; 3 = the
                              one-pass split kernel (each interval read and written
                              once) where both coefficient sets fit the constant bank,
                              instead of the classifier + gathered entries */
  uint32_t group_tiles;    /* sectioned kernels: tiles of points a CTA runs through one
                              section before the next (default 4) */
  int32_t word_layout;     /* sections: -1 = one coefficient block for the whole walk
                              (default: one block per section) */
  int32_t jit_mode;        /* 0 (default): until a domain's specialised kernel is
                              compiled (on a background thread, started by the first
                              call), calls run the ahead-of-time walk-VM kernels;
                              1: every call waits for the specialised kernel;
                              2: walk VM only */
  uint64_t iv_partition_min; /* smallest batch that is sign-partitioned (default 65536) */
} pe_tuning;

/* Replaces the program's code-generation options and drops its generated
 * kernels (they are regenerated on next use). Not thread-safe with respect
 * to concurrent evaluation of the same program. */
pe_status pe_program_set_tuning(pe_program* program, const pe_tuning* tuning);

typedef struct pe_program_info_t {
  uint32_t nvars;
  uint32_t register_count;     /* root program: 1 + max lazy height */
  uint32_t max_registers;      /* max over nested programs */
  uint64_t records;            /* all programs */
  uint64_t programs;           /* root + nested */
  uint64_t walk_adds;          /* reference op counts per point (eval_test.cpp:182-216) */
  uint64_t walk_muls;
  uint64_t power_muls;         /* memoized-halving multiplications per point */
  uint64_t terms;              /* canonical terms */
  uint32_t root_children;      /* root_child_ends.size() */
  uint32_t exponent_set_sizes[8]; /* first 8 variables */
} pe_program_info_t;

pe_status pe_program_info(const pe_program* program, pe_program_info_t* info);

/* Writes the exponent set of variable v (sorted) into out[0..cap); *count
 * receives the set size. */
pe_status pe_program_exponents(const pe_program* program, uint32_t v,
                               uint32_t* out, size_t cap, size_t* count);

/* Flat record dump of the root program (records x 5 int32: power_slot or -1,
 * lazy_slot, parent_slot or -1, reads_register, has_sub). */
pe_status pe_program_records(const pe_program* program, int32_t* out,
                             size_t cap, size_t* count);

/* DOT text of the root tree (reference to_dot). Writes at most cap bytes
 * including the NUL; *len receives the full length. */
pe_status pe_program_dot(const pe_program* program, char* out, size_t cap,
                         size_t* len);

/* Register hygiene (reference Evaluator::enable_register_check,
 * eval.hpp:142-145 and the check at eval.hpp:240-247): every point walks the
 * same record sequence, so "the register file is clean after the walk" is a
 * property of the program — checked once, symbolically, over the root and
 * every nested program. PE_OK if clean, PE_ELOGIC ("register file not clean
 * after walk") if some record's value is never consumed. */
pe_status pe_program_check_registers(const pe_program* program);

/* Specialised kernel statistics for a domain (0 f64, 1 f64 strict, 2 i64,
 * 3 interval, 4 i64 on the FP64 pipe, PE_DOMAIN_LIMBS(K) the K-limb exact
 * kernel): FP64 / int64 arithmetic instructions per point, and the PTX text
 * size. Generates (but does not load) the kernel. */
#define PE_DOMAIN_LIMBS(k) (0x100 | (k))
pe_status pe_program_kernel_stats(const pe_program* program, int32_t domain,
                                  uint64_t* fp_ops, uint64_t* int_ops,
                                  uint64_t* ptx_bytes);

/* Writes the generated PTX for `domain` (debug / inspection). */
pe_status pe_program_ptx(const pe_program* program, int32_t domain, char* out,
                         size_t cap, size_t* len);

/* Compiles the domain's kernel to an sm_100a cubin without a GPU (build and
 * CI check); *cubin_bytes receives the image size. */
pe_status pe_program_compile_only(const pe_program* program, int32_t domain,
                                  uint64_t* cubin_bytes);

/* int64 programs: per-variable coordinate bounds (nvars entries each) under
 * which evaluation is provably wrap-free (bound63) and provably exact on the
 * FP64 pipe (bound53, the faster tier). UINT64_MAX = unconstrained. */
pe_status pe_program_i64_bounds(const pe_program* program, uint64_t* bound63,
                                uint64_t* bound53);

/* 1 when the specialised kernel of `domain` is compiled (calls then run it),
 * 0 while calls would run the walk VM (pe_tuning.jit_mode). */
pe_status pe_program_kernel_ready(const pe_program* program, int32_t domain, int32_t* ready);

/* Barrier-separated sections of the fused fp64 kernel (long walks are cut
 * where few walk values are live; the op sequence is unchanged). */
pe_status pe_program_f64_slices(const pe_program* program, uint32_t* slices);

/* Batch evaluation. coords: nvars pointers, each to n values. */
pe_status pe_eval_f64(const pe_program* program, const double* const* coords,
                      size_t n, double* out, const pe_exec* exec);

/* Several fused-fp64 programs (same variable count) over one point batch:
 * results outs[j][i] = programs[j](point i). With host buffers the points
 * cross PCIe once for all k programs (the reference analogue: k Evaluator
 * sessions fed the same points). */
pe_status pe_eval_f64_multi(const pe_program* const* programs, size_t k,
                            const double* const* coords, size_t n,
                            double* const* outs, const pe_exec* exec);

pe_status pe_eval_i64(const pe_program* program, const int64_t* const* coords,
                      size_t n, int64_t* out, const pe_exec* exec);

/* Exact integer evaluation beyond int64 (reference BigIntDomain,
 * ring.hpp:30-38, bigint.cpp): every value is `limbs` 64-bit words, two's
 * complement, little-endian; out_limbs[k][i] is word k of point i's result.
 * Runs when the host proof bounds every intermediate below 2^(64*limbs-1)
 * for the batch's coordinate maxima (computed on the device / host), else
 * PE_EOVERFLOW — choose `limbs` with pe_program_limbs_needed. 1 <= limbs <= 8. */
pe_status pe_eval_limbs(const pe_program* program, const int64_t* const* coords, size_t n,
                        uint32_t limbs, uint64_t* const* out_limbs, const pe_exec* exec);

/* Smallest limb count (1..8) the proof allows for |x_v| <= bounds[v]
 * (nvars entries); *limbs = 0 when 8 limbs do not suffice. */
pe_status pe_program_limbs_needed(const pe_program* program, const uint64_t* bounds,
                                  uint32_t* limbs);

/* Interval points [lo[v][i], hi[v][i]]; results [out_lo[i], out_hi[i]].
 * Endpoints must be non-NaN with lo <= hi (reference Interval ctor).
 * Univariate batches of >= 64K intervals are split on the device by the sign
 * of x (x < 0 runs the mirrored program p(-y) at -x; bit-identical results);
 * the split needs 4 bytes per interval of stream-ordered scratch from the
 * device's default memory pool, whose release threshold the library raises
 * so the scratch stays pooled between calls. */
pe_status pe_eval_interval(const pe_program* program, const double* const* lo,
                           const double* const* hi, size_t n, double* out_lo,
                           double* out_hi, const pe_exec* exec);

/* Arbitrary-width exact evaluation — the reference BigIntDomain with
 * multi-limb coefficients and points (the paper's Figure-1 workload:
 * bench.cpp:59-187, 64..2048-bit coefficients and points). Values are
 * little-endian two's-complement 64-bit words.
 *   pe_program_create_wide: term t has exponents[t*nvars ..] and coefficient
 *     words coeff_words[t*coeff_limbs .. +coeff_limbs). Exponent rows must be
 *     distinct (zero coefficients are dropped). Only pe_eval_wide evaluates
 *     such a program (the other pe_eval_* return PE_EINVAL).
 *   pe_program_wide_limbs: limbs of the result for points of point_limbs
 *     words (the static magnitude bound of the walk's result).
 *   pe_eval_wide: coords[v][i*point_limbs + k] is word k of coordinate v of
 *     point i; out[i*out_limbs + k] receives word k of the result
 *     (sign-extended; out_limbs must be >= pe_program_wide_limbs, else
 *     PE_EOVERFLOW). Host or device buffers; one CTA (normally one warp) per point. */
pe_status pe_program_create_wide(const uint32_t* exponents, const uint64_t* coeff_words,
                                 uint32_t coeff_limbs, size_t nterms, uint32_t nvars,
                                 const pe_scheme_desc* schemes, pe_program** out);
pe_status pe_program_wide_limbs(const pe_program* program, uint32_t point_limbs,
                                uint32_t* out_limbs);
pe_status pe_eval_wide(const pe_program* program, const uint64_t* const* coords,
                       uint32_t point_limbs, size_t n, uint64_t* out, uint32_t out_limbs,
                       const pe_exec* exec);

/* Roofline denominator microbenchmark on `device`: kind 0 = DFMA/s
 * (FP64 FMA pipe), kind 1 = 64-bit integer multiply-adds/s, kind 2 = SM
 * cycles per dependent DFMA (latency), kind 3 = FP64 FMAs/s through the
 * tensor cores (mma.sync m8n8k4 f64). *sms receives the SM count.
 * Synchronous; for bench.py, not a hot-path call. */
pe_status pe_measure_peak(int32_t device, int32_t kind, double* ops_per_s, int32_t* sms);

/* Waits for all work this library queued on `exec` (device + stream). */
pe_status pe_synchronize(const pe_exec* exec);

/* Number of kernels this library launched in this process (evidence counter). */
uint64_t pe_launch_count(void);

const char* pe_last_error(void);

/* Library / ABI version. */
const char* pe_version(void);

#ifdef __cplusplus
}
#endif

#endif /* POLYEVAL_B200_H_ */
