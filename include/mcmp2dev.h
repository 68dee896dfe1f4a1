/* mcmp2dev.h — C ABI of the B200 MC-MP2 walker loop (libmcmp2dev.so).
 *
 * This is the drop-in boundary for the reference's hot path. The reference has no FFI;
 * its seam is the private Engine::advance (reference proj/core/src/driver.cpp:440-450),
 * whose public callees are metropolis_step (sampler.hpp:59-60), TauSampler::sample
 * (weights.hpp:58), mc_step_estimate (estimator.hpp:55-57) and BlockingAccumulator::add
 * (estimator.hpp:64). Each entry point below names the reference interface it replaces.
 * Plain C types only; the caller owns every host buffer, the handle deep-copies inputs at
 * create time and keeps no host pointers. No exceptions cross this ABI: each call returns
 * a status and mcmp2dev_last_error() carries the reference's message text.
 *
 * Threading: one handle per (device, worker) (driver.cpp:423-438 runs one std::thread per
 * worker). A handle is used by one host thread at a time; handles on different devices may
 * run concurrently. There is no global mutable state except the create-failure message.
 */
#ifndef MCMP2DEV_H
#define MCMP2DEV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCMP2DEV_ABI_VERSION 2

/* status codes (SURVEY.md section 8(b) "Errors") */
enum {
  MCMP2DEV_OK = 0,
  MCMP2DEV_INVALID_ARGUMENT = 1, /* reference throws std::invalid_argument */
  MCMP2DEV_RUNTIME = 2,          /* reference throws std::runtime_error    */
  MCMP2DEV_CUDA = 3              /* CUDA failure (no reference analogue)   */
};

/* pair-term convention (reference estimator.cpp:26-32 is LITERAL) */
enum { MCMP2DEV_ESTIMATOR_LITERAL = 0, MCMP2DEV_ESTIMATOR_PHYSICAL = 1 };

/* Immutable system: SpinorSet + WeightSpec + TauSampler (model.hpp:74-117,
 * weights.hpp:28-63). Basis functions of all channels are concatenated in channel order
 * (channel 0..ncomp-1, SPINOR-TEXT `basis` records, model.cpp:302-323). */
typedef struct mcmp2dev_system {
  int ncomp;                  /* 1, 2 or 4 (model.cpp:99-100)                               */
  int n_occ, n_vir;           /* spinor split (model.hpp:81-83)                              */
  const int* channel_count;   /* [ncomp] functions per channel                               */
  const double* fn_center;    /* [nfunc][3]                                                  */
  const int* fn_lm;           /* [nfunc][2] (l, m), l <= 3                                   */
  const int* fn_prim_offset;  /* [nfunc + 1] into prim arrays                                */
  const double* prim_zeta;    /* [nprim]                                                     */
  const double* prim_coeff;   /* [nprim] BasisFunction::evaluation_coeffs (model.hpp:49)     */
  const double* coeff;        /* [nfunc][n_occ + n_vir][2] complex C, row-major (re, im)     */
  const double* energies;     /* [n_occ + n_vir] ascending per block (model.cpp:122-129)     */
  int nsites;                 /* WeightSpec sites, one per nucleus (weights.cpp:57-82)       */
  const double* site_pos;     /* [nsites][3]                                                 */
  const double* site_prim;    /* [nsites][2][2] (coeff incl. s norm, zeta) (weights.cpp:74-79) */
  const double* site_zeta1;   /* [nsites] leading exponent for init spread (weights.hpp:44)  */
  double ng;                  /* N_g closed form (weights.cpp:84-89)                         */
  double lambda;              /* TauSampler rate = 2 (eps_LUMO - eps_HOMO) (weights.cpp:113) */
  double w_direct, w_exchange;/* mp2_pair_prefactors(ncomp) (model.cpp:86-88)                */
  int estimator;              /* MCMP2DEV_ESTIMATOR_*                                        */
} mcmp2dev_system;

/* Walker ensemble state, the WalkerEnsemble save/load record (sampler.cpp:95-120) with the
 * PhiloxRng text state (rng.hpp:36-40, rng.cpp:76-94). `walkers` is caller-owned
 * [m][9] = r1[3], r2[3], g1, g2, weight. */
typedef struct mcmp2dev_ensemble {
  int m;
  double sigma_step;
  long long proposed, accepted;
  uint32_t rng_key[2];
  uint32_t rng_counter[4];
  uint32_t rng_idx;
  double* walkers;
} mcmp2dev_ensemble;

typedef struct mcmp2dev_handle mcmp2dev_t;

/* Per-step replay result: StepEstimate (estimator.hpp:23-26) plus the pair sums of the
 * direct and exchange terms before division by C(m,2). */
typedef struct mcmp2dev_step {
  double value, imag;
  double direct_re, direct_im, exchange_re, exchange_im;
} mcmp2dev_step;

/* Per-step record with the INT8 V path's accuracy guard (mcmp2dev_advance_ex / _replay_ex).
 * est_err_*: the guard's estimate of the INT8 error of the direct / exchange pair sums (a
 * model of the slice remainders and dropped slice products propagated through the literal
 * contraction, csrc/pair_oz.cu); abs_*: sums of |pair term| (the condition-aware error of
 * SURVEY 7 is |error| / (abs / C(m,2))); int8_v: 1 when the V blocks of this step ran on the
 * INT8 path; fallback: 0 the main INT8 pass was kept, 1 the guard rejected it and the
 * refinement pass (one more slice diagonal) was kept, 2 the step was recomputed on the FP64
 * DMMA pair kernel (value and sums are then the DMMA ones). The guard fields are 0 on the DMMA
 * path. */
typedef struct mcmp2dev_step_ex {
  double value, imag;
  double direct_re, direct_im, exchange_re, exchange_im;
  double est_err_direct, est_err_exchange, abs_direct, abs_exchange;
  int int8_v, fallback;
} mcmp2dev_step_ex;

/* ---- lifetime ---------------------------------------------------------------------- */
/* Deep-copies `sys` to `device`, sized for up to max_walkers electron pairs.
 * Replaces Engine construction of the per-worker state (driver.cpp:338-374). */
int mcmp2dev_create(const mcmp2dev_system* sys, int device, int max_walkers, mcmp2dev_t** out);
int mcmp2dev_destroy(mcmp2dev_t* h);
/* message of the last failed call on h (or of the last failed create when h is NULL) */
const char* mcmp2dev_last_error(const mcmp2dev_t* h);
int mcmp2dev_abi_version(void);

/* ---- ensemble ---------------------------------------------------------------------- */
/* init_ensemble(m, molecule, spec, seed, stream) (sampler.cpp:21-47), on the device,
 * consuming the reference's Philox stream in the reference's order. */
int mcmp2dev_init_ensemble(mcmp2dev_t* h, int m, uint64_t seed, uint32_t stream);
/* burn_in(ens, spec, n_burn, adapt) (sampler.cpp:81-93); counters reset at the end. */
int mcmp2dev_burn_in(mcmp2dev_t* h, long n_burn, int adapt);
int mcmp2dev_set_sigma_step(mcmp2dev_t* h, double sigma);  /* WalkerEnsemble::set_sigma_step */
/* checkpoint I/O: WalkerEnsemble::load / save (sampler.cpp:95-120) */
int mcmp2dev_set_ensemble(mcmp2dev_t* h, const mcmp2dev_ensemble* e);
int mcmp2dev_get_ensemble(mcmp2dev_t* h, mcmp2dev_ensemble* e); /* e->walkers: [m][9] */

/* ---- batched ensembles ----------------------------------------------------------------
 * Several reference workers in ONE handle (the std::thread workers of driver.cpp:423-438, each
 * with its own ensemble and Philox stream, driver.cpp:354-356), so small systems fill the GPU:
 * ensemble e (0 <= e < nens) is init_ensemble(m, seed, stream0 + e); every step advances all
 * of them in the same launches. Needs m % 16 == 0 and m <= 480; the handle must
 * be created with max_walkers >= nens * m (and nens <= max_walkers / 16). advance() then writes
 * values/imags as [nsteps][nens]; burn_in and set_sigma_step apply to every ensemble;
 * get/set_ensemble_at address one ensemble (same m, the batch seed, stream stream0 + e).
 * init_ensemble / set_ensemble return the handle to a single ensemble. */
int mcmp2dev_init_batch(mcmp2dev_t* h, int nens, int m, uint64_t seed, uint32_t stream0);
int mcmp2dev_batch_size(const mcmp2dev_t* h);  /* ensembles advanced per step (1 unless batched) */
int mcmp2dev_get_ensemble_at(mcmp2dev_t* h, int ens, mcmp2dev_ensemble* e);
int mcmp2dev_set_ensemble_at(mcmp2dev_t* h, int ens, const mcmp2dev_ensemble* e);
/* every ensemble at once (two copies): es[nens], each with its own walkers buffer [m][9] */
int mcmp2dev_get_ensembles(mcmp2dev_t* h, mcmp2dev_ensemble* es);
int mcmp2dev_set_ensembles(mcmp2dev_t* h, const mcmp2dev_ensemble* es);
/* advance() of ensembles [0, nactive) only; the others keep walkers, RNG state and counters
 * (unequal step shares, driver.cpp:307-309: the extra steps go to the lowest worker indices).
 * values/imags are [nsteps][nens]; entries of inactive ensembles are not steps. */
int mcmp2dev_advance_batch(mcmp2dev_t* h, long nsteps, int nactive, double* values, double* imags);

/* ---- the hot loop ------------------------------------------------------------------ */
/* nsteps x { metropolis_step; tau = sample(rng.uniform()); mc_step_estimate } with the
 * per-step (value, imag) written to host arrays so the caller's BlockingAccumulator::add
 * runs in the reference order (driver.cpp:443-448). values/imags may be NULL (kept on
 * device; for kernel timing). */
int mcmp2dev_advance(mcmp2dev_t* h, long nsteps, double* values, double* imags);
/* Optional: capture the CUDA graphs advance() replays (32 steps each) for the current
 * ensemble now, so the first advance() does not pay the capture; executes nothing. */
int mcmp2dev_prepare(mcmp2dev_t* h);
/* Replay: mc_step_estimate at given walker positions and tau (estimator.cpp:35-63).
 * walkers [nsteps][m][8] = r1[3], r2[3], g1, g2; tau [nsteps]; out [nsteps]. The device
 * ensemble is not modified. m = 2 is sample_term (estimator.cpp:65-75). */
int mcmp2dev_replay(mcmp2dev_t* h, int m, long nsteps, const double* walkers, const double* tau,
                    mcmp2dev_step* out);
/* advance / replay with the full per-step record (guard fields); single ensembles */
int mcmp2dev_advance_ex(mcmp2dev_t* h, long nsteps, mcmp2dev_step_ex* out);
int mcmp2dev_replay_ex(mcmp2dev_t* h, int m, long nsteps, const double* walkers, const double* tau,
                       mcmp2dev_step_ex* out);

/* ---- instrumentation (not on the reference surface) -------------------------------- */
/* Accumulated device time (ms) and launch counts of the kernel classes since the last
 * reset, measured with CUDA events on the handle's stream:
 * out[0..3] = ms of {walk, spinor, pair, total}, out[4..7] = launches of the same. */
int mcmp2dev_profile(mcmp2dev_t* h, int enable, int reset, double* out);
/* The pair stage's kernels on the INT8 V path, accumulated like mcmp2dev_profile (same enable
 * and reset): out[0..2] = ms of {oz_slice_kernel, oz_vgemm_kernel, pair_kr_kernel}, out[3] =
 * profiled steps that took the path, out[4] = int8 tensor ops of the last V-GEMM launch,
 * out[5] = ms of the accuracy guard's refinement and DMMA launches (literal estimator). */
int mcmp2dev_profile_pair(mcmp2dev_t* h, double* out);
/* Algorithmic work of one step at the current m: FLOP of the pair stage
 * (C(m,2) * F_pair) and of the spinor stage (2m * 4 * R * n_p), bytes written to Phi. */
int mcmp2dev_work(mcmp2dev_t* h, double* pair_flop, double* spinor_flop, double* phi_bytes);
/* FP64 tensor work the pair kernel actually issues per step at the current m (DMMA count x
 * 512 FLOP, including tile/k padding): 3 real products per complex product, and half the
 * blocks on the Kramers path. pair_flop / executed is the algorithmic saving. */
int mcmp2dev_work_executed(mcmp2dev_t* h, double* pair_dmma_flop);
/* synchronise the handle's stream */
int mcmp2dev_synchronize(mcmp2dev_t* h);
/* the handle's cudaStream_t (as void*), for callers that time or order work around it */
void* mcmp2dev_stream(mcmp2dev_t* h);
/* Kramers-restricted pair kernel: used when the spinor columns are time-reversal pairs to
 * within 1e-12 (relative deviation of the pairing relations from max |C|, of the pair energies
 * from max |eps|; the kernel derives each odd column from its even partner, so results move by
 * O(deviation)). mode -1 queries, 0 disables, 1 enables if eligible; returns the active state
 * (1/0). Results agree with the general path to rounding (see csrc/pair_kr.cu). */
int mcmp2dev_kramers(mcmp2dev_t* h, int mode);
/* the deviation from exact time-reversal pairing measured at create (+inf: the basis lists or
 * column counts do not pair) */
int mcmp2dev_kramers_deviation(const mcmp2dev_t* h, double* deviation);
/* V blocks of the Kramers pair stage (K = n_vir, ~90% of the pair work) on the INT8 tensor
 * cores: FP64 operands split into six int8 slices of balanced radix-256 digits (Ozaki), exact
 * int8 products summed in int32/int64, one FP64 rounding (csrc/pair_oz.cu). Used for single ensembles on the Kramers
 * path with n_vir <= 512 and the 16 x 8 pair tiles (m >= 64 walkers, enough tiles for the
 * SMs); elsewhere the DMMA V phase runs. mode -1 queries, 0 selects DMMA, 1 selects INT8.
 * Default: INT8 for the literal estimator when n_vir > 16 (with a single 32-wide k-step of K'
 * the V-GEMM's per-tile epilogue, not its MMAs, sets the pace and the DMMA kernel is faster);
 * the physical estimator defaults to DMMA and runs INT8 unguarded when selected. Returns 1 when
 * the INT8 V path is selected and the system is eligible. Agreement with the FP64 path: see
 * mcmp2dev_guard. */
int mcmp2dev_pair_path(mcmp2dev_t* h, int mode);
/* Energy-ordered truncation of the INT8 V-GEMM's K loop (on by default; exact). The virtual
 * energies ascend (model.cpp:126-127) and Phi_v carries exp(-eps tau / 2), so at this step's tau
 * the high-energy spinors may fall below the last slice of every row they appear in: their
 * digits are all zero. oz_slice_kernel records, per point pair, the last 16-spinor k-step with
 * a nonzero digit, and oz_vgemm_kernel runs each tile's k-steps only up to the smaller of its
 * Q block's and P block's counts. The skipped slice products are exact zeros, so the step's sums
 * are bit-identical to the full loop (tests/test_gpu_oz.py). In the k-steps before those, the
 * leading slices (most significant digits) of every row may be zero as well: the slice kernel
 * also records, per point pair and k-step, the first slice with a nonzero digit, and a k-step
 * whose A rows have a and whose B rows have b leading zero slices issues only the products
 * (s, t) with s >= a, t >= b (none when a + b >= 6) and copies only those slices. mode -1
 * queries, 0 runs every k-step in full, 1 skips empty k-steps and leading zero slices
 * (default), 2 skips whole empty k-steps only; returns the active mode. */
int mcmp2dev_oz_truncation(mcmp2dev_t* h, int mode);
/* INT8 V path, literal estimator: oz_slice_kernel on a side stream of the handle, concurrent
 * with the O pass (both read Phi only; the V-GEMM waits for both). mode -1 queries, 0 runs them
 * in series on the handle's stream, 1 overlaps them (default; profiling passes always serialise
 * so each kernel is timed alone). Results do not depend on it. */
int mcmp2dev_oz_overlap(mcmp2dev_t* h, int mode);
/* out2 = {k-steps (32 of K' = 2 n_vir) issued by the main-pass V-GEMM launches since the INT8
 * buffers were allocated -- counted in slice products / 21, so a partly empty k-step counts the
 * share of its 21 products that ran --, k-steps of one untruncated launch at the last step's sizes}. */
int mcmp2dev_oz_ksteps(mcmp2dev_t* h, double* out2);
/* Accuracy guard of the INT8 V path (literal estimator). After each INT8 step the V-GEMM's
 * last CTA compares the estimated error of the direct sum, the exchange sum and the step value
 * with tol times their magnitude. A step that fails (or is not finite) gets a refinement pass
 * on the INT8 tensor cores (the 7th slices and the next slice diagonal, ~1/8 of the modelled error;
 * the main pass keeps every pair's f values for it), and if the refined step still fails it
 * is recomputed on the FP64 DMMA pair kernel. Both are launched every step and exit at once
 * unless needed, so the graphs stay fixed. tol <= 0 turns the guard off; default 2e-10; NaN
 * only queries. previous (may be NULL) receives the old tolerance. The estimate is a model
 * checked against the oracle (tests/test_oz_guard_model.py) and against the DMMA path on
 * chains of up to 2 x 10^4 steps (>= 2.5x the actual error, median 22x), not a rigorous bound
 * (that would reject every step). At cfg4 (m = 2048, 2 x 10^4 steps) 1.1% of the steps fail the
 * main pass and 0.2% the refinement, kept steps are within 3.8e-11 of FP64, while the unguarded
 * path exceeds the 1e-10 gate on 6-16 steps (tests/test_gpu_guard.py, tools/guard_chain.py). */
int mcmp2dev_guard(mcmp2dev_t* h, double tol, double* previous);
/* out5 = {INT8-path steps checked, steps refined, steps recomputed on DMMA, largest estimated
 * relative error of a step kept on INT8, tolerance} since the last call; resets the counters. */
int mcmp2dev_guard_stats(mcmp2dev_t* h, double* out5);

#ifdef __cplusplus
}
#endif
#endif /* MCMP2DEV_H */
