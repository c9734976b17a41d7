/* hg_oracle.c -- CPU restatement of the reference's stencil time loop + dmp halo swap.
 *
 * TEST INFRASTRUCTURE ONLY (see hg_oracle.h).  Compiled with -O2 -ffp-contract=off, the
 * reference's own contract (proj/CMakeLists.txt:8-10): every f32/f64 op is one IEEE RN op in
 * program order, exactly like the interpreter (proj/core/src/exec/interpreter.cpp:495-506).
 * OpenMP only splits independent points (outermost dimension); it never reassociates.
 * Parity of this file is pinned against fixtures produced by the real reference
 * (tests/golden/, made by tests/golden/make_golden.py through oracle/_ref).
 */
#include "hg_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
const char *or_last_error(void) { return g_err; }
static int fail(const char *m) {
  snprintf(g_err, sizeof g_err, "%s", m);
  return -1;
}

/* mix64 + initValue: proj/core/src/exec/buffer.cpp:142-156 */
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

double or_init_value(int field, int rank, const int64_t *coord) {
  uint64_t h = mix64((uint64_t)field + 1);
  for (int d = 0; d < rank; ++d)
    h = mix64(h ^ (uint64_t)coord[d]);
  return (double)(h >> 11) * 0x1.0p-53;
}

static int64_t count_of(const or_buf *b) {
  int64_t n = 1;
  for (int d = 0; d < b->rank; ++d)
    n *= b->shape[d];
  return n;
}

/* fillInit: buffer.cpp:158-179 (f32 = static_cast<float>(double)).  `origin` shifts the
 * logical coordinate, which is what scatterRank of a global init amounts to
 * (simulator.cpp:995-1025). */
void or_fill_init(or_buf *b, int field, const int64_t *origin) {
  int64_t n = count_of(b);
  int r = b->rank;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t raw[3] = {0, 0, 0}, c[3];
    int64_t rem = i;
    for (int d = r - 1; d >= 0; --d) {
      raw[d] = rem % b->shape[d];
      rem /= b->shape[d];
    }
    for (int d = 0; d < r; ++d)
      c[d] = b->lb[d] + raw[d] + (origin ? origin[d] : 0);
    double v = or_init_value(field, r, c);
    if (b->elem == 4) {
      float f = (float)v;
      memcpy(b->data + i * 4, &f, 4);
    } else {
      memcpy(b->data + i * 8, &v, 8);
    }
  }
}

/* FNV-1a over the raw bytes: buffer.cpp:181-188 */
uint64_t or_fingerprint(const or_buf *b) {
  uint64_t h = 0xcbf29ce484222325ull;
  int64_t n = count_of(b) * b->elem;
  for (int64_t i = 0; i < n; ++i) {
    h ^= b->data[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* rotationSources (stencil_transforms.cpp:233-242) + bindingAfter (serial.cpp:42-55) */
static void rotation_sources(int ngroups, const int32_t *glen, const int32_t *groups, int nargs,
                             int *src) {
  for (int i = 0; i < nargs; ++i)
    src[i] = i;
  int at = 0;
  for (int g = 0; g < ngroups; ++g) {
    for (int j = 0; j < glen[g]; ++j)
      src[groups[at + j]] = groups[at + (j + 1) % glen[g]];
    at += glen[g];
  }
}

void or_binding_after(int ngroups, const int32_t *glen, const int32_t *groups, int nargs,
                      int64_t steps, int32_t *out) {
  int src[HG_MAX_FIELDS], cur[HG_MAX_FIELDS], nxt[HG_MAX_FIELDS];
  rotation_sources(ngroups, glen, groups, nargs, src);
  for (int i = 0; i < nargs; ++i)
    cur[i] = i;
  for (int64_t t = 0; t < steps; ++t) {
    for (int i = 0; i < nargs; ++i)
      nxt[i] = cur[src[i]];
    memcpy(cur, nxt, sizeof(int) * (size_t)nargs);
  }
  for (int i = 0; i < nargs; ++i)
    out[i] = cur[i];
}

/* One invocation of the step function: stencil.load clones (interpreter.cpp:676-682), the
 * apply evaluates its region once per point of its domain in row-major order into fresh
 * result buffers (:713-758) with bounds-checked accesses (:759-780), then each
 * stencil.store copies its region (:683-712).  Results are staged so an in-place store
 * sees the loaded (pre-step) values, as the clone does. */
static int or_step_multi(const hg_program *p, or_buf **slots, int nthreads);

int or_step(const hg_program *p, or_buf **slots, int nthreads) {
  if (p->napplies > 0)
    return or_step_multi(p, slots, nthreads);
  int r = p->rank;
  /* apply domain = hull of the store regions (propagate-bounds' result bounds) */
  int64_t ia[3] = {0, 0, 0}, ib[3] = {1, 1, 1};
  for (int k = 0; k < p->nresults; ++k)
    for (int d = 0; d < r; ++d) {
      if (k == 0 || p->store[k].lb[d] < ia[d])
        ia[d] = p->store[k].lb[d];
      if (k == 0 || p->store[k].ub[d] > ib[d])
        ib[d] = p->store[k].ub[d];
    }
  int64_t ext[3] = {1, 1, 1}, npts = 1;
  for (int d = 0; d < r; ++d) {
    ext[d] = ib[d] - ia[d];
    if (ext[d] <= 0)
      return 0;
    npts *= ext[d];
  }
  int es = p->dtype == HG_F32 ? 4 : 8;
  unsigned char *res[HG_MAX_RESULTS];
  for (int k = 0; k < p->nresults; ++k)
    res[k] = (unsigned char *)malloc((size_t)(npts * es));
  int trapped = 0;
  /* operand buffers: stencil.load of the bound field */
  const or_buf *opb[HG_MAX_FIELDS];
  for (int o = 0; o < p->noperands; ++o)
    opb[o] = slots[p->operand_field[o]];
  (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t outer = 0; outer < ext[0]; ++outer) {
    float *vf = (float *)malloc(sizeof(float) * (size_t)p->nops);
    double *vd = (double *)malloc(sizeof(double) * (size_t)p->nops);
    int64_t inner = npts / ext[0];
    for (int64_t q = 0; q < inner; ++q) {
      int64_t pt[3];
      pt[0] = ia[0] + outer;
      int64_t rem = q;
      for (int d = r - 1; d >= 1; --d) {
        pt[d] = ia[d] + rem % ext[d];
        rem /= ext[d];
      }
      for (int i = 0; i < p->nops; ++i) {
        const hg_op *op = &p->ops[i];
        switch (op->code) {
        case HG_OP_ACCESS: {
          const or_buf *b = opb[op->operand];
          int64_t idx = 0;
          for (int d = 0; d < r; ++d) {
            int64_t rr = pt[d] + op->off[d] - b->lb[d];
            if (rr < 0 || rr >= b->shape[d]) {
              trapped = 1;
              rr = 0;
            }
            idx = idx * b->shape[d] + rr;
          }
          if (es == 4)
            memcpy(&vf[i], b->data + idx * 4, 4);
          else
            memcpy(&vd[i], b->data + idx * 8, 8);
          break;
        }
        case HG_OP_CONST:
          if (es == 4) {
            uint32_t u = (uint32_t)op->bits;
            memcpy(&vf[i], &u, 4);
          } else {
            memcpy(&vd[i], &op->bits, 8);
          }
          break;
        case HG_OP_ADD:
          if (es == 4) vf[i] = vf[op->a] + vf[op->b]; else vd[i] = vd[op->a] + vd[op->b];
          break;
        case HG_OP_SUB:
          if (es == 4) vf[i] = vf[op->a] - vf[op->b]; else vd[i] = vd[op->a] - vd[op->b];
          break;
        case HG_OP_MUL:
          if (es == 4) vf[i] = vf[op->a] * vf[op->b]; else vd[i] = vd[op->a] * vd[op->b];
          break;
        case HG_OP_DIV:
          if (es == 4) vf[i] = vf[op->a] / vf[op->b]; else vd[i] = vd[op->a] / vd[op->b];
          break;
        default:
          trapped = 1;
        }
      }
      int64_t li = outer * inner + q;
      for (int k = 0; k < p->nresults; ++k) {
        if (es == 4)
          memcpy(res[k] + li * 4, &vf[p->result_op[k]], 4);
        else
          memcpy(res[k] + li * 8, &vd[p->result_op[k]], 8);
      }
    }
    free(vf);
    free(vd);
  }
  if (trapped) {
    for (int k = 0; k < p->nresults; ++k)
      free(res[k]);
    return fail("stencil access escapes the value bounds");
  }
  /* stores */
  for (int k = 0; k < p->nresults; ++k) {
    or_buf *dst = slots[p->store_field[k]];
    const hg_bounds *sb = &p->store[k];
    int64_t sn = 1, se[3] = {1, 1, 1};
    for (int d = 0; d < r; ++d) {
      se[d] = sb->ub[d] - sb->lb[d];
      sn *= se[d];
    }
    for (int64_t q = 0; q < sn; ++q) {
      int64_t rem = q, pt[3];
      for (int d = r - 1; d >= 0; --d) {
        pt[d] = sb->lb[d] + rem % se[d];
        rem /= se[d];
      }
      int64_t si = 0, di = 0;
      for (int d = 0; d < r; ++d) {
        int64_t sr = pt[d] - ia[d], dr = pt[d] - dst->lb[d];
        if (sr < 0 || sr >= ext[d] || dr < 0 || dr >= dst->shape[d]) {
          for (int kk = 0; kk < p->nresults; ++kk)
            free(res[kk]);
          return fail("store region escapes the field bounds");
        }
        si = si * ext[d] + sr;
        di = di * dst->shape[d] + dr;
      }
      memcpy(dst->data + di * es, res[k] + si * es, (size_t)es);
    }
  }
  for (int k = 0; k < p->nresults; ++k)
    free(res[k]);
  return 0;
}

/* runSerialStencil: serial.cpp:57-88 */
int or_run(const hg_program *p, or_buf **bufs, int64_t T, int32_t *perm_out, int nthreads) {
  int n = p->nfields;
  int src[HG_MAX_FIELDS];
  rotation_sources(p->ngroups, p->group_len, p->groups, n, src);
  int32_t bind[HG_MAX_FIELDS], nxt[HG_MAX_FIELDS];
  for (int i = 0; i < n; ++i)
    bind[i] = i;
  or_buf *slots[HG_MAX_FIELDS];
  for (int64_t t = 0; t < T; ++t) {
    for (int i = 0; i < n; ++i)
      slots[i] = bufs[bind[i]];
    if (or_step(p, slots, nthreads))
      return -1;
    for (int i = 0; i < n; ++i)
      nxt[i] = bind[src[i]];
    memcpy(bind, nxt, sizeof(int32_t) * (size_t)n);
  }
  if (perm_out)
    for (int i = 0; i < n; ++i)
      perm_out[i] = bind[i];
  return 0;
}

/* rankFromCoord / coordFromRank / neighborRank: dmp_ops.cpp:21-49 */
int64_t or_rank_from_coord(int n, const int64_t *coord, const int64_t *grid) {
  int64_t r = 0;
  for (int d = 0; d < n; ++d)
    r = r * grid[d] + coord[d];
  return r;
}

void or_coord_from_rank(int n, int64_t rank, const int64_t *grid, int64_t *coord) {
  for (int d = n - 1; d >= 0; --d) {
    coord[d] = rank % grid[d];
    rank /= grid[d];
  }
}

int64_t or_neighbor_rank(int n, int64_t rank, const int64_t *dir, const int64_t *grid) {
  int64_t c[3];
  or_coord_from_rank(n, rank, grid, c);
  for (int d = 0; d < n; ++d) {
    c[d] += dir[d];
    if (c[d] < 0 || c[d] >= grid[d])
      return -1;
  }
  return or_rank_from_coord(n, c, grid);
}

/* StandardSlicing::localInterval: dmp_ops.cpp:107-115 */
void or_local_interval(int64_t extent, int64_t parts, int64_t part, int64_t *lb, int64_t *ub) {
  int64_t base = extent / parts, rem = extent % parts;
  *lb = part * base + (part < rem ? part : rem);
  *ub = *lb + base + (part < rem ? 1 : 0);
}

/* DecompositionStrategy::exchanges: dmp_ops.cpp:63-105 */
int or_exchanges(int n, const int64_t *core, const int64_t *below, const int64_t *above,
                 const int64_t *grid, const int64_t *coord, hg_exchange *out, int cap) {
  int k = 0;
  for (int d = 0; d < n; ++d) {
    for (int s = 0; s < 2; ++s) {
      int sign = s == 0 ? -1 : 1;
      int64_t width = sign < 0 ? below[d] : above[d];
      if (width == 0)
        continue;
      if (coord) {
        int64_t dir[3] = {0, 0, 0};
        dir[d] = sign;
        if (or_neighbor_rank(n, or_rank_from_coord(n, coord, grid), dir, grid) < 0)
          continue;
      }
      hg_exchange e;
      memset(&e, 0, sizeof e);
      for (int j = 0; j < n; ++j) {
        e.at[j] = below[j];
        e.size[j] = core[j];
      }
      if (sign < 0) {
        e.at[d] = 0;
        e.size[d] = width;
        e.offset[d] = width;
      } else {
        e.at[d] = below[d] + core[d];
        e.size[d] = width;
        e.offset[d] = -width;
      }
      e.to[d] = sign;
      if (k < cap)
        out[k] = e;
      ++k;
    }
  }
  return k;
}

/* packRegion / unpackRegion: simulator.cpp:523-584 (row-major over the box). */
static int box_walk(or_buf *b, const int64_t *at, const int64_t *size, unsigned char *io,
                    int unpack) {
  int r = b->rank, w = b->elem;
  int64_t n = 1;
  for (int d = 0; d < r; ++d)
    n *= size[d];
  int64_t p[3] = {0, 0, 0};
  for (int64_t k = 0; k < n; ++k) {
    int64_t idx = 0;
    for (int d = 0; d < r; ++d) {
      int64_t raw = at[d] + p[d];
      if (raw < 0 || raw >= b->shape[d])
        return fail("exchange region escapes the buffer");
      idx = idx * b->shape[d] + raw;
    }
    if (unpack)
      memcpy(b->data + idx * w, io + k * w, (size_t)w);
    else
      memcpy(io + k * w, b->data + idx * w, (size_t)w);
    for (int d = r - 1; d >= 0; --d) {
      if (++p[d] < size[d])
        break;
      p[d] = 0;
    }
  }
  return 0;
}

int or_pack(const or_buf *b, const int64_t *at, const int64_t *size, unsigned char *out) {
  return box_walk((or_buf *)b, at, size, out, 0);
}

int or_unpack(or_buf *b, const int64_t *at, const int64_t *size, const unsigned char *in) {
  return box_walk(b, at, size, (unsigned char *)in, 1);
}

/* ---- simulate: simulator.cpp:1066-1203 with RankHooks::swap (:772-834) ---------------- */

static or_buf *alloc_like(const hg_bounds *bd, int rank, int elem) {
  or_buf *b = (or_buf *)calloc(1, sizeof(or_buf));
  b->rank = rank;
  b->elem = elem;
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) {
    b->lb[d] = bd->lb[d];
    b->shape[d] = bd->ub[d] - bd->lb[d];
    n *= b->shape[d];
  }
  b->data = (unsigned char *)calloc((size_t)n, (size_t)elem);
  return b;
}

static void free_buf(or_buf *b) {
  if (b) {
    free(b->data);
    free(b);
  }
}

/* scatterRank: local raw p <-> global logical lb_local + p + coord*core (simulator.cpp:995-1025) */
static int scatter(const or_buf *g, or_buf *l, const int64_t *shift) {
  int r = l->rank, w = l->elem;
  int64_t n = count_of(l);
  for (int64_t i = 0; i < n; ++i) {
    int64_t rem = i, raw[3], sidx = 0;
    for (int d = r - 1; d >= 0; --d) {
      raw[d] = rem % l->shape[d];
      rem /= l->shape[d];
    }
    for (int d = 0; d < r; ++d) {
      int64_t s = l->lb[d] + raw[d] + shift[d] - g->lb[d];
      if (s < 0 || s >= g->shape[d])
        return fail("local field escapes the global field");
      sidx = sidx * g->shape[d] + s;
    }
    memcpy(l->data + i * w, g->data + sidx * w, (size_t)w);
  }
  return 0;
}

/* gatherRank: core cells only (simulator.cpp:1027-1060) */
static void gather(const or_buf *l, or_buf *g, const int64_t *core_lb, const int64_t *core,
                   const int64_t *shift) {
  int r = l->rank, w = l->elem;
  int64_t n = 1;
  for (int d = 0; d < r; ++d)
    n *= core[d];
  for (int64_t i = 0; i < n; ++i) {
    int64_t rem = i, p[3], li = 0, gi = 0;
    for (int d = r - 1; d >= 0; --d) {
      p[d] = core_lb[d] + shift[d] + rem % core[d];
      rem /= core[d];
    }
    for (int d = 0; d < r; ++d) {
      li = li * l->shape[d] + (p[d] - shift[d] - l->lb[d]);
      gi = gi * g->shape[d] + (p[d] - g->lb[d]);
    }
    memcpy(g->data + gi * w, l->data + li * w, (size_t)w);
  }
}

static int sim_core(const hg_program *local, const hg_decomp *dc, or_buf **global_init,
                    int nfields, int64_t T, or_buf **out, int64_t want_rank, or_buf **local_out,
                    int nthreads) {
  int r = local->rank, es = local->dtype == HG_F32 ? 4 : 8;
  int64_t P = 1;
  for (int d = 0; d < dc->ndim; ++d)
    P *= dc->grid[d];
  if (dc->ndim != r)
    return fail("process grid rank does not match the domain");
  /* rank-0 core lower bound = the local store region's lb */
  int64_t core_lb[3] = {0, 0, 0};
  const hg_bounds *st0 = local->napplies > 0 ? &local->mstore[0] : &local->store[0];
  for (int d = 0; d < r; ++d)
    core_lb[d] = st0->lb[d];
  or_buf ***rb = (or_buf ***)calloc((size_t)P, sizeof(or_buf **));
  for (int64_t q = 0; q < P; ++q) {
    rb[q] = (or_buf **)calloc((size_t)nfields, sizeof(or_buf *));
    int64_t c[3], shift[3] = {0, 0, 0};
    or_coord_from_rank(r, q, dc->grid, c);
    for (int d = 0; d < r; ++d)
      shift[d] = c[d] * dc->core[d];
    for (int f = 0; f < nfields; ++f) {
      rb[q][f] = alloc_like(&local->fields[f], r, es);
      if (scatter(global_init[f], rb[q][f], shift))
        return -1;
    }
  }
  int src[HG_MAX_FIELDS];
  rotation_sources(local->ngroups, local->group_len, local->groups, nfields, src);
  int32_t bind[HG_MAX_FIELDS], nxt[HG_MAX_FIELDS];
  for (int i = 0; i < nfields; ++i)
    bind[i] = i;
  int rc = 0;
  for (int64_t t = 0; t < T && !rc; ++t) {
    /* every dmp.swap of the step body, in order; each is a set of disjoint copies, so
     * "all ranks send, then all ranks receive" is exactly the buffered-send protocol. */
    for (int s = 0; s < dc->nswaps && !rc; ++s) {
      const hg_swap *sw = &dc->swaps[s];
      int fbuf = bind[sw->field];
      unsigned char **msg =
          (unsigned char **)calloc((size_t)(P * sw->nexchanges), sizeof(unsigned char *));
      for (int64_t q = 0; q < P && !rc; ++q)
        for (int e = 0; e < sw->nexchanges; ++e) {
          const hg_exchange *x = &sw->ex[e];
          if (or_neighbor_rank(r, q, x->to, dc->grid) < 0)
            continue;
          int64_t sat[3], n = 1;
          for (int d = 0; d < r; ++d) {
            sat[d] = x->at[d] + x->offset[d];
            n *= x->size[d];
          }
          msg[q * sw->nexchanges + e] = (unsigned char *)malloc((size_t)(n * es));
          rc = or_pack(rb[q][fbuf], sat, x->size, msg[q * sw->nexchanges + e]);
        }
      for (int64_t q = 0; q < P && !rc; ++q)
        for (int e = 0; e < sw->nexchanges; ++e) {
          const hg_exchange *x = &sw->ex[e];
          int64_t nb = or_neighbor_rank(r, q, x->to, dc->grid);
          if (nb < 0)
            continue;
          /* the neighbour's message for us travels in its opposite direction */
          int mate = -1;
          for (int e2 = 0; e2 < sw->nexchanges; ++e2) {
            int opp = 1;
            for (int d = 0; d < r; ++d)
              if (sw->ex[e2].to[d] != -x->to[d])
                opp = 0;
            if (opp)
              mate = e2;
          }
          if (mate < 0 || !msg[nb * sw->nexchanges + mate]) {
            rc = fail("deadlock: no matching message");
            break;
          }
          rc = or_unpack(rb[q][fbuf], x->at, x->size, msg[nb * sw->nexchanges + mate]);
        }
      for (int64_t i = 0; i < P * sw->nexchanges; ++i)
        free(msg[i]);
      free(msg);
    }
    for (int64_t q = 0; q < P && !rc; ++q) {
      or_buf *slots[HG_MAX_FIELDS];
      for (int i = 0; i < nfields; ++i)
        slots[i] = rb[q][bind[i]];
      rc = or_step(local, slots, nthreads);
    }
    for (int i = 0; i < nfields; ++i)
      nxt[i] = bind[src[i]];
    memcpy(bind, nxt, sizeof(int32_t) * (size_t)nfields);
  }
  if (!rc && out) {
    /* gathered over a clone of globalInit[origin[i]] (simulator.cpp:1192-1200) */
    for (int i = 0; i < nfields; ++i) {
      memcpy(out[i]->data, global_init[bind[i]]->data,
             (size_t)(count_of(global_init[bind[i]]) * es));
      for (int64_t q = 0; q < P; ++q) {
        int64_t c[3], shift[3] = {0, 0, 0};
        or_coord_from_rank(r, q, dc->grid, c);
        for (int d = 0; d < r; ++d)
          shift[d] = c[d] * dc->core[d];
        gather(rb[q][bind[i]], out[i], core_lb, dc->core, shift);
      }
    }
  }
  if (!rc && local_out && want_rank >= 0 && want_rank < P)
    for (int i = 0; i < nfields; ++i) /* local buffers in final binding order */
      memcpy(local_out[i]->data, rb[want_rank][bind[i]]->data,
             (size_t)(count_of(rb[want_rank][bind[i]]) * es));
  for (int64_t q = 0; q < P; ++q) {
    for (int f = 0; f < nfields; ++f)
      free_buf(rb[q][f]);
    free(rb[q]);
  }
  free(rb);
  return rc;
}

int or_simulate(const hg_program *local, const hg_decomp *dc, or_buf **global_init, int nfields,
                int64_t T, or_buf **out, int nthreads) {
  return sim_core(local, dc, global_init, nfields, T, out, -1, NULL, nthreads);
}

int or_simulate_rank_state(const hg_program *local, const hg_decomp *dc, or_buf **global_init,
                           int nfields, int64_t T, int64_t want_rank, or_buf **local_out,
                           int nthreads) {
  return sim_core(local, dc, global_init, nfields, T, NULL, want_rank, local_out, nthreads);
}

/* Multi-apply step: applies run in program order; each evaluates its region over its whole
 * result bounds into fresh temps (materializeApply, stencil_transforms.cpp:334-379; the
 * interpreter does the same per apply, interpreter.cpp:713-758); field operands read the
 * loaded (pre-step) values; then every stencil.store copies its region (:683-712). */
static int or_step_multi(const hg_program *p, or_buf **slots, int nthreads) {
  const int r = p->rank, es = p->dtype == HG_F32 ? 4 : 8;
  or_buf tmp[HG_MAX_TEMPS];
  memset(tmp, 0, sizeof tmp);
  int rc = 0;
  (void)nthreads;
  for (int a = 0; a < p->napplies && !rc; ++a) {
    const hg_apply *A = &p->applies[a];
    const hg_op *ops = p->ops + A->op_begin;
    int64_t ext[3] = {1, 1, 1}, npts = 1;
    for (int d = 0; d < r; ++d) {
      ext[d] = A->domain.ub[d] - A->domain.lb[d];
      npts *= ext[d];
    }
    for (int k = 0; k < A->nresults; ++k) {
      or_buf *t = &tmp[A->result_temp[k]];
      t->rank = r;
      t->elem = es;
      for (int d = 0; d < r; ++d) {
        t->lb[d] = A->domain.lb[d];
        t->shape[d] = ext[d];
      }
      t->data = (unsigned char *)calloc((size_t)npts, (size_t)es);
    }
    const or_buf *opb[HG_MAX_FIELDS];
    for (int o = 0; o < A->noperands; ++o)
      opb[o] = A->operand[o] >= 0 ? slots[A->operand[o]] : &tmp[-A->operand[o] - 1];
    int trapped = 0;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < npts; ++q) {
      float vf[1024];
      double vd[1024];
      int64_t pt[3], rem = q;
      for (int d = r - 1; d >= 0; --d) {
        pt[d] = A->domain.lb[d] + rem % ext[d];
        rem /= ext[d];
      }
      for (int i = 0; i < A->nops && i < 1024; ++i) {
        const hg_op *op = &ops[i];
        switch (op->code) {
        case HG_OP_ACCESS: {
          const or_buf *b = opb[op->operand];
          int64_t idx = 0;
          for (int d = 0; d < r; ++d) {
            int64_t rr = pt[d] + op->off[d] - b->lb[d];
            if (rr < 0 || rr >= b->shape[d]) {
              trapped = 1;
              rr = 0;
            }
            idx = idx * b->shape[d] + rr;
          }
          if (es == 4) memcpy(&vf[i], b->data + idx * 4, 4); else memcpy(&vd[i], b->data + idx * 8, 8);
          break;
        }
        case HG_OP_CONST:
          if (es == 4) {
            uint32_t u = (uint32_t)op->bits;
            memcpy(&vf[i], &u, 4);
          } else {
            memcpy(&vd[i], &op->bits, 8);
          }
          break;
        case HG_OP_ADD: if (es == 4) vf[i] = vf[op->a] + vf[op->b]; else vd[i] = vd[op->a] + vd[op->b]; break;
        case HG_OP_SUB: if (es == 4) vf[i] = vf[op->a] - vf[op->b]; else vd[i] = vd[op->a] - vd[op->b]; break;
        case HG_OP_MUL: if (es == 4) vf[i] = vf[op->a] * vf[op->b]; else vd[i] = vd[op->a] * vd[op->b]; break;
        default: if (es == 4) vf[i] = vf[op->a] / vf[op->b]; else vd[i] = vd[op->a] / vd[op->b]; break;
        }
      }
      for (int k = 0; k < A->nresults; ++k) {
        or_buf *t = &tmp[A->result_temp[k]];
        if (es == 4) memcpy(t->data + q * 4, &vf[A->result_op[k]], 4);
        else memcpy(t->data + q * 8, &vd[A->result_op[k]], 8);
      }
    }
    if (trapped)
      rc = fail("stencil access escapes the value bounds");
  }
  for (int k = 0; k < p->nstores && !rc; ++k) {
    const or_buf *src = &tmp[p->mstore_temp[k]];
    or_buf *dst = slots[p->mstore_field[k]];
    const hg_bounds *sb = &p->mstore[k];
    int64_t se[3] = {1, 1, 1}, sn = 1;
    for (int d = 0; d < r; ++d) {
      se[d] = sb->ub[d] - sb->lb[d];
      sn *= se[d];
    }
    for (int64_t q = 0; q < sn && !rc; ++q) {
      int64_t rem = q, pt[3], si = 0, di = 0;
      for (int d = r - 1; d >= 0; --d) {
        pt[d] = sb->lb[d] + rem % se[d];
        rem /= se[d];
      }
      for (int d = 0; d < r; ++d) {
        int64_t sr = pt[d] - src->lb[d], dr = pt[d] - dst->lb[d];
        if (sr < 0 || sr >= src->shape[d] || dr < 0 || dr >= dst->shape[d]) {
          rc = fail("store region escapes the field bounds");
          break;
        }
        si = si * src->shape[d] + sr;
        di = di * dst->shape[d] + dr;
      }
      if (!rc)
        memcpy(dst->data + di * es, src->data + si * es, (size_t)es);
    }
  }
  for (int t = 0; t < HG_MAX_TEMPS; ++t)
    free(tmp[t].data);
  return rc;
}
