/*
 * permkit_gpu.h — C ABI of the B200-native Gray-code Ryser/Glynn engine.
 *
 * This is the drop-in boundary for the reference package's hot path
 * (arxiv/paper_2602_10141, package `permkit`).  The reference evaluates
 * permanents by walking Gray-code blocks in numba kernels selected per block
 * by engine._run_plan; this library replaces those walks with sm_100a CUDA
 * kernels and takes one call per range / batch / prime set instead of one
 * call per block.  All entry points:
 *   - are extern "C", take plain pointers and sizes (no torch/numpy types),
 *   - read caller buffers during the call only (nothing is retained),
 *   - return 0 on success or a negative status (see PK_ERR_*), with a
 *     message available from pk_last_error() on the calling thread,
 *   - are reentrant; concurrent calls on one device are serialised.
 *
 * Matrix layout: row-major n x n; complex matrices are interleaved
 * (re, im) float64 pairs, i.e. exactly numpy complex128 memory.
 * Gray index space: [0, 2^m), m = n (Ryser) or n - 1 (Glynn); index b
 * denotes the subset / sign vector gray(b) = b ^ (b >> 1)
 * (reference pkg/src/permkit/gray.py:19-31).
 */
#ifndef PERMKIT_GPU_H
#define PERMKIT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_OK 0
#define PK_ERR_CUDA (-1)     /* CUDA runtime / launch failure                 */
#define PK_ERR_ARG (-2)      /* invalid argument (shape, range, modulus, ...)  */
#define PK_ERR_LIMIT (-3)    /* documented capability limit exceeded           */
#define PK_ERR_INTERNAL (-4)

#define PK_ALGO_RYSER 0
#define PK_ALGO_GLYNN 1

/* Message for the last failing call made by this thread ("" if none). */
const char* pk_last_error(void);

/* Number of visible CUDA devices (>= 0), or a negative status. */
int pk_device_count(void);

/* Make logical device d of every call below physical device base + d
 * (one process per GPU: each rank sets base = LOCAL_RANK and uses device 0).
 * Default 0.  Returns 0 or PK_ERR_ARG. */
int pk_set_device_base(int base);

/* Test / measurement hook (also $PK_LOGICAL_DEVICES): report `count` devices
 * and map logical device d onto visible GPU d mod (visible GPUs), each with its
 * own stream, buffers and host thread, so every multi-device path (range and
 * modulus splits, the combine of device results) runs on a one-GPU box as on
 * eight.  0 = off (default).  Returns 0 or PK_ERR_ARG. */
int pk_set_logical_devices(int count);

/* Library version, e.g. 100 for 0.1.0. */
int pk_version(void);

/* Largest n the register-resident production kernels accept (48). */
int pk_max_n(void);

/*
 * fp64 walk of ONE matrix over the Gray range [start, start + length).
 * Replaces kernels.ryser_partial / kernels.glynn_partial
 * (reference pkg/src/permkit/kernels.py:415-430) and the per-block thread
 * pool of engine._run_plan (engine.py:213-245) for COMPLEX / REAL domains.
 *   out[4]  = {sum_re, sum_im, comp_re, comp_im}: a compensated pair whose
 *             value sum + comp is the signed partial sum (Glynn unscaled,
 *             as glynn_partial returns it); im parts are 0 for real input.
 *   abs_sum = optional (may be NULL): sum of |re t| + |im t| over the terms,
 *             an upper bound of sum |t| used by the parity tolerance.
 *   ndev    = devices to split the range over (clamped to the device count).
 * The aligned interior runs in the register-resident production kernel; an
 * unaligned head/tail is walked with the reference's exact arithmetic.
 * The result for a given (a, start, length) is deterministic and identical
 * for every ndev: devices own whole reduction groups and the host completes
 * the group tree in global index order.
 */
int pk_ryser_f64(const double* a, int n, int is_complex, int algo, uint64_t start,
                 uint64_t length, int ndev, double out[4], double* abs_sum);

/*
 * Bit-exact parity mode: one GPU thread walks each caller block exactly as
 * the reference's numba kernel does (no FMA, same operation order,
 * Neumaier per component).  out[4*i .. 4*i+3] = {s_re, s_im, c_re, c_im} of
 * block i, bit-identical to kernels.ryser_partial(a, starts[i], lens[i])
 * (kernels.py:33-123) or glynn_partial (kernels.py:126-226).  n <= 64.
 */
int pk_ryser_f64_blocks(const double* a, int n, int is_complex, int algo,
                        const uint64_t* starts, const uint64_t* lens, int nblocks, int device,
                        double* out);

/*
 * A caller's block plan of ONE matrix in one call (engine._run_plan for
 * perm_blocked, reference engine.py:213-245, which calls kernels.ryser_partial
 * per block on a thread pool).  out[4*i ..] = {s_re, s_im, c_re, c_im} and
 * abs_sums[i] (optional) of block i, bit-identical to pk_ryser_f64 on
 * (starts[i], lens[i]); the caller folds the pairs in block order as the
 * reference does.  Blocks are split over ndev devices; on each, the aligned
 * interiors run in as few walk launches as possible, one segmented reduce
 * serves every block, and every ragged piece runs in one exact launch.
 */
int pk_ryser_f64_plan(const double* a, int n, int is_complex, int algo, const uint64_t* starts,
                      const uint64_t* lens, int nblocks, int ndev, double* out,
                      double* abs_sums);

/* The reference's ordered combine of a plan's block pairs (engine.py:240-245:
 * KahanAccumulator add(s); add(c) per block, Neumaier per component).
 * pairs[4*i ..] as pk_ryser_f64_plan's out; out[4] = {sum_re, sum_im, comp_re,
 * comp_im}; the value is sum + comp. */
int pk_kahan_fold(const double* pairs, int nblocks, int is_complex, double out[4]);

/*
 * Full-range permanents of B matrices (contiguous B x n x n), e.g. the
 * ensemble sampler (ensembles.py:142-158) and the geodesic sweep
 * (geodesics.py:153-179).  out[4*b ..] as in pk_ryser_f64 for matrix b;
 * abs_sums[b] optional.  Matrices are split over ndev devices.  On each
 * device, m >= 20 (complex) or m >= 21 (real) runs one launch per matrix
 * over 16 streams; smaller m runs one matrix per warp in a single launch.
 * Either way the call returns only after every result is on the host.  The
 * walk plan depends on (n, algo) only, so results never depend on B, on the
 * batch split over devices or on a caller's chunking.
 */
int pk_ryser_f64_batch(const double* a, int B, int n, int is_complex, int algo, int ndev,
                       double* out, double* abs_sums);

/*
 * F_p walk over [start, start + length) for P moduli at once.
 *   a      = P x n x n residues, a[k][i][j] in [0, primes[k])
 *   primes = P moduli, each 2 <= p < 2^62 (PrimeField range, domains.py:126-130)
 *   out[k] = exact signed walk sum over the range mod primes[k], in [0, p):
 *            the value sum(kernels.ryser_partial_modp(a_k, blk...)) mod p
 *            (kernels.py:250-290, 433-434); Glynn is NOT scaled by 2^(1-n).
 * Odd p < 2^31 run in the Montgomery-32 kernels (up to four primes per lane;
 * fp64-eligible primes pair with a Montgomery prime in the hybrid kernel);
 * odd 2^31 <= p < 2^62 run in the Montgomery-64 kernel (one per lane);
 * even moduli, and the ragged ends of unaligned ranges, use the
 * per-block parity walker.
 */
int pk_ryser_modp(const uint64_t* a, const uint64_t* primes, int P, int n, int algo,
                  uint64_t start, uint64_t length, int ndev, uint64_t* out);

/*
 * Resident jobs for measurement (bench.py): the matrix / residues are
 * uploaded once and the walk is re-run on device-resident inputs.  The range
 * must be aligned to the job's tile span (any full range is).
 */
typedef struct pk_job pk_job;

int pk_job_f64_create(int device, const double* a, int n, int is_complex, int algo,
                      uint64_t start, uint64_t length, pk_job** job);
/* F_p jobs take odd moduli p < 2^62 (every prime of the fast kernels). */
int pk_job_modp_create(int device, const uint64_t* a, const uint64_t* primes, int P, int n,
                       int algo, uint64_t start, uint64_t length, pk_job** job);
/*
 * Run `iters` walks back to back on the job's stream.  Between iterations a
 * buffer of flush_bytes is overwritten (L2 flush; 0 = none).  total_ms =
 * device time of the whole sequence (CUDA events, includes flushes);
 * walk_ms = summed device time of the walk kernel launches only.
 * out_f64[5] = (s_re, c_re, s_im, c_im, abs) of the last run (f64 jobs);
 * out_res[P] = residues of the last run (F_p jobs).  Either may be NULL.
 */
int pk_job_run(pk_job* job, int iters, size_t flush_bytes, double* total_ms, double* walk_ms,
               double* out_f64, uint64_t* out_res);
/* info[0..7] = k (segment bits), tiles, grid CTAs, CTAs per SM, registers per
 * thread, local (spill) bytes, dynamic smem bytes, kernel launches per run. */
int pk_job_info(pk_job* job, int64_t* info);
/* F_p jobs: per launch group g < min(G, max_groups) of the last pk_job_run,
 * desc[6*g ..] = {kind (0 reduced, 1 lazy, 2 hybrid, 3 hybrid with a wide fp64
 * prime, 4 Montgomery-64), primes in the group, registers per thread, CTAs
 * per SM, grid CTAs, dynamic smem bytes} and ms[g] = summed device time of
 * the group's walk launches (CUDA events on the job's stream).  prime_idx
 * [4*g ..] = the group's indices into the job's prime list (-1 padded).
 * Returns G (launch groups per run). */
int pk_job_groups(pk_job* job, int64_t* desc, double* ms, int64_t* prime_idx, int max_groups);
void pk_job_destroy(pk_job* job);

/*
 * Pipe-rate micro-benchmarks (roofline denominators).  Fills out[3*i..] =
 * {lane-ops/s, lane-ops per SM clock, mean SM MHz} for the ops named by
 * pk_peak_names() (comma separated).  Returns the number of ops measured.
 */
int pk_measure_peaks(int device, double* out, int max_out);
const char* pk_peak_names(void);

/*
 * Instruction-mix ceilings (csrc/pk_mix.cu): the production walker structs'
 * step + pair loop with no Gray bookkeeping and no segment restarts, at the
 * walk's occupancy.  out[3*i..] = {units/s, units per SM clock, mean SM MHz}
 * (units: row updates, or prime-row updates) for the mixes named by
 * pk_mix_names().  Returns the count.
 */
int pk_measure_mix_ceilings(int device, double* out, int max_out);
const char* pk_mix_names(void);

/* Dependent-chain latencies in SM cycles for the ops named by
 * pk_latency_names() (one warp, one chain).  Returns the count. */
int pk_measure_latencies(int device, double* out, int max_out);
const char* pk_latency_names(void);

#ifdef __cplusplus
}
#endif

#endif /* PERMKIT_GPU_H */
