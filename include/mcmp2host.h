/* mcmp2host.h — C entry points of the host library libmcmp2host.so (the re-hosted
 * reference driver around libmcmp2dev.so). Used by the Python wrapper, bench.py and the
 * distributed runner; the CLI `mcmp2` is the C++ front end (reference tools/mcmp2_main.cpp).
 * Every call returns 0 on success, 1 for the reference's std::invalid_argument, 2 for
 * std::runtime_error; mcmp2h_last_error() holds the message. */
#ifndef MCMP2HOST_H
#define MCMP2HOST_H

#include <stdint.h>

#include "mcmp2dev.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* mcmp2h_last_error(void);

/* mcmp2 run / resume / merge (driver.hpp:74-88); report text as format_report */
int mcmp2h_run(const char* config_text, char* report, int cap);
int mcmp2h_run_hooked(const char* config_text, long abort_after_intervals, char* report, int cap);
int mcmp2h_resume(const char* checkpoint_path, char* report, int cap);
int mcmp2h_merge(const char* const* paths, int n, double* value, double* sigma_bar, long long* steps);
int mcmp2h_parse_config(const char* config_text, char* canonical, int cap);
uint64_t mcmp2h_fnv1a64(const char* bytes, long n);

/* a loaded system: SPINOR-TEXT + weight overrides from config text (model.cpp:275-351,
 * weights.cpp:57-90), flattened for mcmp2dev_create */
typedef struct mcmp2h_system mcmp2h_system;
mcmp2h_system* mcmp2h_system_load(const char* spinor_path, const char* config_text);
void mcmp2h_system_free(mcmp2h_system* s);
const mcmp2dev_system* mcmp2h_system_view(const mcmp2h_system* s);
/* ints: ncomp, n_occ, n_vir, rows; dbls: ng, lambda, orthonormality deviation */
int mcmp2h_system_info(const mcmp2h_system* s, int* ints, double* dbls);
int mcmp2h_system_g(const mcmp2h_system* s, const double* pts, int n, double* out);
int mcmp2h_save_spinor_set(const char* in_path, const char* out_path);

/* one worker on one device (init_ensemble + burn_in at create); the accumulator state is
 * returned as {steps, sum, imag_sum, mean, sigma_bar, in_block, partial, nblocks,
 * acceptance, imag_ratio} (10 doubles; WorkerSummary of driver.cpp:207-216). */
typedef struct mcmp2h_worker mcmp2h_worker;
mcmp2h_worker* mcmp2h_worker_create(const char* config_text, int worker_index, int device);
void mcmp2h_worker_free(mcmp2h_worker* w);
int mcmp2h_worker_advance(mcmp2h_worker* w, long nsteps, double* values, double* imags);
int mcmp2h_worker_stats(mcmp2h_worker* w, double* out8);
int mcmp2h_worker_block_means(mcmp2h_worker* w, double* out, int cap);
mcmp2dev_t* mcmp2h_worker_device(mcmp2h_worker* w);

/* Workers [first_index, first_index + count) of one process on one device (the multi-GPU
 * driver's rank): one batched handle when the walker count allows it (include/mcmp2dev.h,
 * batched ensembles), else one handle each; init + burn-in at create (driver.cpp:354-358).
 * advance: worker k takes nsteps[k] steps; stats: as mcmp2h_worker_stats for worker k. */
typedef struct mcmp2h_group mcmp2h_group;
mcmp2h_group* mcmp2h_group_create(const char* config_text, int first_index, int count, int device);
void mcmp2h_group_free(mcmp2h_group* g);
int mcmp2h_group_size(const mcmp2h_group* g);
int mcmp2h_group_advance(mcmp2h_group* g, const long long* nsteps);
int mcmp2h_group_stats(mcmp2h_group* g, int k, double* out10);

/* The checkpoint of a run whose workers live in several processes (one rank per GPU): the file
 * is mcmp2h_checkpoint_header (driver.cpp:222-230) followed by every worker's
 * mcmp2h_group_record in worker order (driver.cpp:232-247), byte-identical to what the
 * single-process Engine writes, so `mcmp2 resume` / `mcmp2 merge` read it; mcmp2h_group_trace
 * is a worker's trace lines (driver.cpp:311-321). Text calls copy when cap suffices and always
 * set *need to the size with the terminator. mcmp2h_checkpoint_config checks the stored hash
 * (driver.cpp:482-491) and returns the stored config; mcmp2h_group_resume builds workers
 * [first_index, first_index + count) from their records instead of init + burn-in, the cached
 * weights re-verified (driver.cpp:360-373). */
int mcmp2h_checkpoint_header(const char* config_text, int nworkers, char* buf, long cap, long* need);
int mcmp2h_group_record(mcmp2h_group* g, int k, char* buf, long cap, long* need);
int mcmp2h_group_trace(mcmp2h_group* g, int k, char* buf, long cap, long* need);
int mcmp2h_checkpoint_config(const char* checkpoint_path, char* canonical, int cap, int* nworkers);
mcmp2h_group* mcmp2h_group_resume(const char* checkpoint_path, int first_index, int count, int device);

/* writes <dir>/<name>.spinor and <dir>/<name>.conf for BASELINE configs cfg1..cfg4, cfg5-N */
int mcmp2h_generate(const char* name, const char* dir);

/* host-side pieces of the reference surface, for the CPU test suite */
int mcmp2h_blocking(const double* values, long n, long block_size, double* out4);
int mcmp2h_merge_estimates(const double* parts, int n, double* out3);
uint64_t mcmp2h_config_hash(const char* config_text, uint64_t spinor_hash);
int mcmp2h_philox_stream(uint64_t seed, uint32_t stream, uint64_t pos, int n, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
