/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot path.
 * See oracle.c for the file:line each function follows.  Indices are 1-based
 * like the reference API.  Return codes: 0 ok, 1 invalid_argument,
 * 2 logic_error, 3 runtime_error (message via orc_last_error()). */
#ifndef TSD_ORACLE_H
#define TSD_ORACLE_H
#include <stdint.h>

typedef struct {
    int64_t index;
    double nn_dist_sq;
    double nn_dist;
} orc_record;

const char* orc_last_error(void);
int orc_gen_randomwalk(int64_t n, uint64_t seed, double* out);
int orc_init_stats(const double* x, int64_t n, int64_t m, double* mu, double* sigma);
int orc_advance_stats(const double* x, int64_t n, int64_t m0, int64_t m1, double* mu,
                      double* sigma);
double orc_ref_sq_dist(const double* x, int64_t n, int64_t m, int64_t i, int64_t j);
int orc_brute_force_nn(const double* x, int64_t n, int64_t m, double* out);
int64_t orc_range_discords(const double* x, int64_t n, int64_t m, double r_sq, orc_record* recs,
                           int64_t cap);
int orc_compute_layout(int64_t n, int64_t m, int64_t seglen, int64_t out[4]);
int orc_next_threshold(const double* hist, int64_t hlen, int phase, int64_t min_len,
                       double last_r, int failed, double* out);
int orc_merlin(const double* x, int64_t n, int64_t min_len, int64_t max_len, int64_t top_k,
               int64_t seglen, int64_t workers, int64_t max_retries, int reuse_stats,
               int64_t* counts, orc_record* recs, double* final_r, int64_t* retries,
               uint8_t* failed);
#endif
