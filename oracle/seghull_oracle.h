/* oracle/seghull_oracle.h -- TEST INFRASTRUCTURE ONLY (see seghull_oracle.c). */
#ifndef SEGHULL_ORACLE_H
#define SEGHULL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 1 + seghull::Errc (error.hpp:8-19); 0 = OK */
enum {
  OR_OK = 0,
  OR_EMPTY_INPUT = 1,
  OR_NON_FINITE_INPUT = 2,
  OR_DEGENERATE_INPUT = 3,
  OR_INPUT_TOO_LARGE = 4,
  OR_INTERNAL_ERROR = 5
};

/* hull.hpp:35-40 SegmentStats */
typedef struct {
  uint64_t iteration, segments, points_remaining, points_removed;
} or_segment_stats;

void or_gen_uniform(uint64_t n, uint64_t seed, double* x, double* y);
void or_gen_circle(uint64_t n, uint64_t seed, double* x, double* y);
uint64_t or_gen_disk(uint64_t n, uint64_t seed, double* x, double* y);

void or_find_extremes(const double* x, const double* y, uint64_t n, uint64_t out[4]);
uint64_t or_preprocess(const double* x, const double* y, uint64_t n, double* out_x,
                       double* out_y, uint64_t* out_idx, uint64_t* out_kept);
int or_first_split(const double* x, const double* y, uint64_t n, double* out_x, double* out_y,
                   uint8_t* out_head);
int or_hull_run(const double* x, const double* y, uint64_t n, int mode, double* out_x,
                double* out_y, uint64_t* out_src, uint64_t* out_h, or_segment_stats* stats,
                uint64_t stats_cap, uint64_t* out_rounds, uint64_t* out_kept,
                uint64_t* bad_index);
int or_monotone_chain(const double* x, const double* y, uint64_t n, double* out_x,
                      double* out_y, uint64_t* out_h);
int or_canonical_index(const double* x, const double* y, uint64_t n, const double* vx,
                       const double* vy, uint64_t h, int64_t* out_idx);
uint64_t or_fnv1a_vertices(const double* vx, const double* vy, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif
