/* hg_oracle.h -- CPU restatement of the reference's stencil/dmp path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this; the
 * product never does.  Buffers use the reference's host layout: row-major, last dimension
 * fastest, halo included, logical lower bound `lb` (buffer.hpp:25-57, buffer.cpp:65-70).
 * Programs use the product's descriptor format (include/hg/hg.h), which is pinned to the
 * reference's own modules by tests/golden/ fixtures.
 */
#ifndef HG_ORACLE_H
#define HG_ORACLE_H
#include <stdint.h>
#include <stddef.h>
#include "../include/hg/hg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_buf {
  int rank;
  int elem; /* bytes: 4 (f32) or 8 (f64) */
  int64_t shape[3];
  int64_t lb[3];
  unsigned char *data;
} or_buf;

double or_init_value(int field, int rank, const int64_t *coord);
void or_fill_init(or_buf *b, int field, const int64_t *origin);
uint64_t or_fingerprint(const or_buf *b);
void or_binding_after(int ngroups, const int32_t *glen, const int32_t *groups, int nargs,
                      int64_t steps, int32_t *out);
/* One step function invocation over `binding` (bufs indexed by argument slot). */
int or_step(const hg_program *p, or_buf **slots, int nthreads);
/* runSerialStencil: T steps with rotation; perm_out[i] = initial buffer bound to slot i. */
int or_run(const hg_program *p, or_buf **bufs, int64_t T, int32_t *perm_out, int nthreads);
int64_t or_neighbor_rank(int n, int64_t rank, const int64_t *dir, const int64_t *grid);
void or_coord_from_rank(int n, int64_t rank, const int64_t *grid, int64_t *coord);
int64_t or_rank_from_coord(int n, const int64_t *coord, const int64_t *grid);
void or_local_interval(int64_t extent, int64_t parts, int64_t part, int64_t *lb, int64_t *ub);
int or_exchanges(int n, const int64_t *core, const int64_t *below, const int64_t *above,
                 const int64_t *grid, const int64_t *coord, hg_exchange *out, int cap);
int or_pack(const or_buf *b, const int64_t *at, const int64_t *size, unsigned char *out);
int or_unpack(or_buf *b, const int64_t *at, const int64_t *size, const unsigned char *in);
/* simulate(): local program + decomposition; global init buffers (reference bounds);
 * writes gathered final fields (final binding order) into `out` (same shapes as global). */
int or_simulate(const hg_program *local, const hg_decomp *dc, or_buf **global_init, int nfields,
                int64_t T, or_buf **out, int nthreads);
/* Per-rank local state after T steps of simulate (halos included), for halo parity. */
int or_simulate_rank_state(const hg_program *local, const hg_decomp *dc, or_buf **global_init,
                           int nfields, int64_t T, int64_t want_rank, or_buf **local_out,
                           int nthreads);
const char *or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
