/* hg.h -- C-ABI of halogen-b200, the B200-native stencil time-stepping + dmp halo-swap path.
 *
 * Plain C: pointers, sizes and opaque handles only (no torch / C++ types).  Every function
 * returns an hg_status (0 = HG_OK); the message of the last failure on the calling thread is
 * hg_last_error().  CUDA streams are passed as `void*` (a cudaStream_t; NULL = legacy default).
 *
 * What each group replaces in the reference (paths under /root/reference/proj/core):
 *
 *   hg_program / hg_op ......... the stencil-level module a step function is built from:
 *                                func @step(fields...) { stencil.load; stencil.apply{access,
 *                                arith.constant, addf/subf/mulf/divf}; stencil.store }
 *                                (src/exec/kernels.cpp:139-243 builds it; src/exec/serial.cpp:22-40
 *                                finds it; src/exec/interpreter.cpp:676-780 interprets it).
 *   hg_build_kernel_program .... exec::buildKernel(KernelSpec)          kernels.cpp:139-243
 *   hg_plan_create/destroy ..... the Interpreter a runSerialStencil call constructs
 *                                (serial.cpp:76) + the caller's field Buffers (buffer.hpp:25-57),
 *                                but device-resident in HBM.
 *   hg_plan_init_fields ........ exec::initialFields / fillInit        kernels.cpp:245-272,
 *                                buffer.cpp:142-179 (bit-identical, computed on the GPU)
 *   hg_plan_upload/download .... moving a host exec::Buffer in/out (row-major, last dim fastest,
 *                                halo included, buffer.cpp:65-70)
 *   hg_plan_run ................ exec::runSerialStencil time loop        serial.cpp:57-88
 *   hg_plan_binding ............ the returned binding / exec::bindingAfter serial.cpp:42-55
 *   hg_binding_after ........... exec::bindingAfter                     serial.cpp:42-55
 *   hg_init_value .............. exec::initValue                        buffer.cpp:142-156
 *   hg_fingerprint ............. exec::fingerprint (FNV-1a)             buffer.cpp:181-188
 *   hg_rank_from_coord/... ..... ir::dmp::rankFromCoord/coordFromRank/neighborRank
 *                                                                        dmp_ops.cpp:21-49
 *   hg_local_interval .......... StandardSlicing::localInterval          dmp_ops.cpp:107-115
 *   hg_exchanges ............... DecompositionStrategy::exchanges        dmp_ops.cpp:63-105
 *   hg_decompose_program ....... the `decompose` pass on a step program  dmp_transforms.cpp:101-312
 *   hg_plan_pack/unpack ........ packRegion/unpackRegion                 simulator.cpp:523-584
 *   hg_dmp_* ................... RankHooks::swap + Endpoint/Transport    simulator.cpp:772-834,
 *                                201-260, 409-424; transport.cpp:13-40: a face-halo exchange of
 *                                device buffers, either NVLink stores fused into the stencil
 *                                kernel (CUDA IPC between processes, peer pointers inside one
 *                                process; x faces as packed slabs) or NCCL send/recv driven from
 *                                C++ (hg_dmp_opts.transport); bounded waits report a stuck peer
 *                                as HG_ETRAP like the reference's deadlock report
 *                                (simulator.cpp:143-173)
 *   hg_sim_run ................. exec::simulate's per-step loop          simulator.cpp:1066-1203
 *                                (all ranks of one process; one rank per GPU runs the fused
 *                                protocol, ranks sharing a GPU are event-ordered)
 *   hg_decompose_program_deep .. beyond the reference: deep (k-step) halos
 *   hg_gpts_per_sec ............ exec::gptsPerSec                        throughput.cpp:19-23
 */
#ifndef HG_HG_H
#define HG_HG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_MAX_RANK 3
#define HG_MAX_FIELDS 16
#define HG_MAX_RESULTS 8
#define HG_MAX_OPS 4096
#define HG_MAX_EXCHANGES 6
#define HG_MAX_APPLIES 32
#define HG_MAX_TEMPS 64
#define HG_MAX_STORES 16

typedef enum hg_status {
  HG_OK = 0,
  HG_EINVAL = 1,       /* malformed descriptor / argument */
  HG_EUNSUPPORTED = 2, /* well-formed, but no kernel family handles it (never a CPU fallback) */
  HG_ECUDA = 3,        /* CUDA runtime/driver failure (no GPU, launch error, ...) */
  HG_ETRAP = 4,        /* what the reference interpreter would trap on (ir::TrapError) */
  HG_ENOMEM = 5,
  HG_ESTATE = 6        /* call out of order (e.g. dmp peers not connected) */
} hg_status;

typedef enum hg_dtype { HG_F32 = 1, HG_F64 = 2 } hg_dtype;

typedef enum hg_opcode {
  HG_OP_ACCESS = 1, /* stencil.access %operand[off]          (stencil_ops.cpp, interpreter.cpp:759-780) */
  HG_OP_CONST = 2,  /* arith.constant : raw FloatAttr bits (attributes.hpp:32-41); f32 in low 32 bits */
  HG_OP_ADD = 3,    /* arith.addf a, b   (interpreter.cpp:495-506, IEEE RN, no FMA contraction) */
  HG_OP_SUB = 4,    /* arith.subf a, b */
  HG_OP_MUL = 5,    /* arith.mulf a, b */
  HG_OP_DIV = 6     /* arith.divf a, b */
} hg_opcode;

/* One SSA op of the apply region, in program order; operands refer to earlier op indices. */
typedef struct hg_op {
  int32_t code;    /* hg_opcode */
  int32_t a, b;    /* ADD/SUB/MUL/DIV operand op indices */
  int32_t operand; /* ACCESS: apply operand (region argument) index */
  int64_t off[HG_MAX_RANK]; /* ACCESS: offsets per dimension */
  uint64_t bits;   /* CONST: raw bits of the constant in the program dtype */
} hg_op;

/* Logical bounds of a field type !field<[lb,ub)x...> (types.hpp:43-64), halo included. */
typedef struct hg_bounds {
  int64_t lb[HG_MAX_RANK];
  int64_t ub[HG_MAX_RANK];
} hg_bounds;

/* One stencil.apply of a multi-apply step (an apply may consume earlier applies' results;
 * the reference evaluates such a producer over its whole result bounds into a temp,
 * stencil_transforms.cpp:334-379, interpreter.cpp:713-758). */
typedef struct hg_apply {
  int32_t noperands;
  int32_t operand[HG_MAX_FIELDS]; /* >= 0: field argument (stencil.load); < 0: temp (-t-1) */
  int32_t op_begin, nops;         /* region = ops[op_begin .. op_begin+nops); operand indices
                                     inside the region are region-relative */
  int32_t nresults;
  int32_t result_op[HG_MAX_RESULTS];   /* region-relative op index returned as result r */
  int32_t result_temp[HG_MAX_RESULTS]; /* temp defined by result r */
  hg_bounds domain;               /* evaluation domain = bounds of its result temps */
} hg_apply;

/* A stencil-level step function: fields (arguments), one apply, its stores, time slots. */
typedef struct hg_program {
  int32_t rank;    /* 1..3 */
  int32_t dtype;   /* hg_dtype; every field and op shares it */
  int32_t nfields; /* step-function arguments, all fields */
  hg_bounds fields[HG_MAX_FIELDS];
  int32_t noperands;                     /* apply operands (each a stencil.load of a field) */
  int32_t operand_field[HG_MAX_FIELDS];  /* field argument loaded for apply operand i */
  int32_t nops;
  const hg_op *ops;                      /* apply region body, nops entries (caller-owned) */
  int32_t nresults;                      /* stencil.return operands == stores */
  int32_t result_op[HG_MAX_RESULTS];     /* op index returned as result r */
  int32_t store_field[HG_MAX_RESULTS];   /* stencil.store of result r to this field argument */
  hg_bounds store[HG_MAX_RESULTS];       /* stored region [lb,ub) of result r */
  int32_t ngroups;                       /* stencil.time_slots (stencil_transforms.cpp:196-242) */
  int32_t group_len[HG_MAX_FIELDS];
  int32_t groups[HG_MAX_FIELDS];         /* groups flattened, group_len[i] entries each */
  /* Multi-apply steps (napplies > 0): nops/ops hold every apply's region back to back and
   * noperands/operand_field list the stencil.load fields in step order (decompose puts a swap
   * before each); result_op..store above are unused; the applies run in order and the stores
   * copy temps into fields. */
  int32_t napplies;
  const hg_apply *applies;               /* caller-owned, napplies entries */
  int32_t ntemps;
  int32_t nstores;
  int32_t mstore_temp[HG_MAX_STORES];    /* stencil.store of this temp ... */
  int32_t mstore_field[HG_MAX_STORES];   /* ... into this field argument ... */
  hg_bounds mstore[HG_MAX_STORES];       /* ... over this region */
} hg_program;

/* #dmp.exchange<at size source offset to> (attributes.hpp:69-75), buffer-local raw coords. */
typedef struct hg_exchange {
  int64_t at[HG_MAX_RANK];
  int64_t size[HG_MAX_RANK];
  int64_t offset[HG_MAX_RANK];
  int64_t to[HG_MAX_RANK];
} hg_exchange;

/* One dmp.swap(%field) {grid, exchanges} placed before the load of `field`. */
typedef struct hg_swap {
  int32_t field;
  int32_t nexchanges;
  hg_exchange ex[2 * HG_MAX_RANK];
} hg_swap;

/* The decomposition of a program: dmp.topology + the swaps in step order + this rank. */
typedef struct hg_decomp {
  int32_t ndim;
  int64_t grid[HG_MAX_RANK];
  int64_t core[HG_MAX_RANK]; /* per-rank core size (dmp.cores / geometryOf coreSize) */
  int32_t nswaps;
  hg_swap swaps[HG_MAX_FIELDS];
} hg_decomp;

typedef struct hg_plan hg_plan;
typedef struct hg_dmp hg_dmp;

/* Per-buffer device layout (for tools/tests; the product API never needs it). */
typedef struct hg_layout {
  int32_t rank;
  int32_t elem_bytes;
  int64_t shape[HG_MAX_RANK]; /* logical allocation shape, halo included */
  int64_t lb[HG_MAX_RANK];
  int64_t pitch;              /* elements between consecutive rows of the last dim */
  int64_t col0;               /* element column of raw index 0 of the last dim */
  int64_t rows;               /* prod(shape[0..rank-2]) */
  void *device_ptr;           /* base of the allocation */
} hg_layout;

/* ---- errors / info -------------------------------------------------------------------- */
const char *hg_last_error(void);
int hg_version(void);
int hg_device_count(int *n);

/* ---- host-side reference algorithms (no GPU needed) ---------------------------------- */
double hg_init_value(int field_idx, int rank, const int64_t *coord);
uint64_t hg_fingerprint(const void *bytes, size_t n);
int hg_binding_after(int ngroups, const int32_t *group_len, const int32_t *groups, int nargs,
                     int64_t steps, int32_t *out);
double hg_gpts_per_sec(int64_t core_points, int64_t steps, double seconds);
int64_t hg_rank_from_coord(int n, const int64_t *coord, const int64_t *grid);
void hg_coord_from_rank(int n, int64_t rank, const int64_t *grid, int64_t *coord);
int64_t hg_neighbor_rank(int n, int64_t rank, const int64_t *dir, const int64_t *grid);
void hg_local_interval(int64_t extent, int64_t parts, int64_t part, int64_t *lb, int64_t *ub);
/* Fills up to `cap` exchanges; returns the count (template form when grid/coord are NULL). */
int hg_exchanges(int n, const int64_t *core, const int64_t *below, const int64_t *above,
                 const int64_t *grid, const int64_t *coord, hg_exchange *out, int cap);

/* exec::buildKernel: kind "heat" | "wave" | "copy", rank 1..3, order 2|4|8, dtype f32/f64.
 * Writes the program into *prog and its ops into ops[cap_ops] (f32 constants are the f64
 * constants re-read from their shortest decimal, exactly as the printed module retyped to f32). */
int hg_build_kernel_program(const char *kind, int rank, int64_t extent, int order, int dtype,
                            hg_program *prog, hg_op *ops, int cap_ops);

/* Reads the stencil-level textual IR (the reference's `.xir` syntax, printer.cpp/parser.cpp):
 * one all-field func.func with stencil.load / dmp.swap / stencil.apply (one, or several that
 * may consume each other -> the multi-apply form, applies[cap_applies]) / stencil.store.
 * Writes the program (+ ops[cap_ops]); for a decomposed module also *decomp and
 * *decomposed = 1.  The module's dmp.reference text (the pre-decompose snapshot) is copied
 * into reference[ref_cap] when given.  Errors carry "<xir>:line:col: message". */
int hg_parse_program(const char *text, hg_program *prog, hg_op *ops, int cap_ops,
                     hg_apply *applies, int cap_applies, hg_decomp *decomp, int *decomposed,
                     char *reference, size_t ref_cap);

/* Validates a program; on HG_OK writes the kernel family that would run it
 * ("star3d_r2_heat", "generic", ...) into name[cap]. No GPU needed. */
int hg_program_match(const hg_program *prog, char *name, size_t cap);

/* Apply fusion: a multi-apply step as one single-apply program (temps inlined: each temp
 * access becomes the producer's DAG at the shifted point, memoised per (apply, shift)).
 * Bit-identical to materialising the temps.  HG_EUNSUPPORTED when the inlined DAG would
 * exceed the op budget or leave the field bounds. */
int hg_fuse_applies(const hg_program *prog, hg_program *out, hg_op *ops, int cap_ops);

/* The fused-apply family (generated straight-line code for any apply DAG): generate the
 * kernel source for `prog` and compile it with NVRTC for sm_100a, without a GPU.  Writes the
 * generated CUDA source into src[cap] (may be NULL) and the cubin size into *cubin_bytes. */
int hg_apply_compile(const hg_program *prog, char *src, size_t cap, size_t *cubin_bytes);

/* The decompose pass on a program (dmp_transforms.cpp:101-312): rewrites *local (field bounds
 * = rank-0 core widened by the halos, stores = rank-0 core) and fills *decomp (one swap per
 * stencil.load, template exchanges).  `local` may alias `global` for single-apply programs;
 * for a multi-apply program (no apply may read another's result, as in the reference) the
 * caller sets local->applies to a buffer of global->napplies entries, which receives the
 * applies with their domains rewritten to the local core. */
int hg_decompose_program(const hg_program *global, int ndim, const int64_t *grid,
                         hg_program *local, hg_decomp *decomp);
/* The same, with halos (and exchange boxes) `depth` times as wide in every split dimension
 * (grid > 1): the communication-avoiding form hg_dmp runs with hg_dmp_opts.depth = depth.
 * Beyond the reference (which swaps before every load, dmp_transforms.cpp:276-300); the
 * gathered cores stay bit-identical. */
int hg_decompose_program_deep(const hg_program *global, int ndim, const int64_t *grid,
                              int depth, hg_program *local, hg_decomp *decomp);

/* ---- plans: device-resident fields + the compiled step --------------------------------- */
int hg_plan_create(const hg_program *prog, int device, hg_plan **out);
int hg_plan_destroy(hg_plan *plan);
int hg_plan_kernel_name(const hg_plan *plan, char *name, size_t cap);
int hg_plan_layout(const hg_plan *plan, int buffer, hg_layout *out);
/* Fill every buffer i (halo included) with initValue(i, logical coord + origin[d]);
 * origin may be NULL (zeros).  The decomposed form passes the rank's core offset. */
int hg_plan_init_fields(hg_plan *plan, const int64_t *origin, void *stream);
/* Host <-> device copy of buffer `buffer` (initial argument index) in the reference's
 * row-major packed layout; bytes must equal the buffer's logical size.  Pinned (device-mapped)
 * host memory moves in one zero-copy kernel pass at the flat PCIe rate; pageable memory goes
 * through the copy engines.  Uploads are asynchronous on `stream`; downloads return when the
 * bytes are on the host. */
int hg_plan_upload(hg_plan *plan, int buffer, const void *host, size_t bytes, void *stream);
/* hg_plan_upload minus the region the next step overwrites before anything reads it: when the
 * slot `buffer` is bound to is stored into (one store) and not loaded by the step, its store
 * box is not moved (runSerialStencil's output slot: the core of u_out, the reference's fresh
 * apply result copied over it at step 1, interpreter.cpp:683-712).  The caller must run at
 * least one step before reading the buffer back. */
int hg_plan_upload_live(hg_plan *plan, int buffer, const void *host, size_t bytes, void *stream);
int hg_plan_download(hg_plan *plan, int buffer, void *host, size_t bytes, void *stream);
/* `steps` time steps, rotating the binding after each (runSerialStencil). */
int hg_plan_run(hg_plan *plan, int64_t steps, void *stream);
/* perm[i] = initial buffer index now bound to argument slot i; steps taken so far. */
int hg_plan_binding(const hg_plan *plan, int32_t *perm, int64_t *steps_done);
int hg_plan_reset_binding(hg_plan *plan);
/* packRegion / unpackRegion of a box of buffer `buffer` to/from a packed device array. */
int hg_plan_pack(hg_plan *plan, int buffer, const int64_t *at, const int64_t *size,
                 void *dst_device, void *stream);
int hg_plan_unpack(hg_plan *plan, int buffer, const int64_t *at, const int64_t *size,
                   const void *src_device, void *stream);
/* Tuning knobs of the star family: z-chunks per column tile (0 = auto) and whether the
 * z-boundary chunks run last (lets halo exchange overlap interior compute). */
int hg_plan_set_tuning(hg_plan *plan, int chunks, int boundary_last);
/* Debug builds of a run (HG_DEBUG_GUARDS=1 at plan creation): every device buffer of the plan
 * sits between 64 KB canary bands; HG_ETRAP if any kernel wrote into one (the memcheck-style
 * out-of-bounds-write check this pool allows: compute-sanitizer is closed here).  HG_OK
 * without guards. */
int hg_plan_check_guards(hg_plan *plan);
/* Caller-bound device memory: buffer `buffer` lives in the caller's allocation
 * from now on (the plan's own is freed; the caller's is never freed by the plan).  It must be
 * device memory of the plan's device, 128-byte aligned, at least hg_plan_layout()'s
 * pitch * rows * elem_bytes bytes, laid out as hg_plan_layout describes (pitched rows, core
 * on 128-byte lines).  The contents are the caller's: hg_plan_init_fields / upload fill it, or
 * the caller writes it.  Plans with bound buffers never use the opt-in two-step passes. */
int hg_plan_bind(hg_plan *plan, int buffer, void *device_ptr, size_t bytes);
/* Block until all work queued for the plan's device has finished. */
int hg_plan_synchronize(hg_plan *plan);
/* Kernel launches issued by this plan so far (for bench/gpu_launches accounting). */
int64_t hg_plan_launch_count(const hg_plan *plan);

/* ---- dmp: halo swap across ranks (NVLink peer memory or NCCL) -------------------------- */
#define HG_TRANSPORT_P2P 0  /* NVLink peer stores fused into the stencil kernel + flags */
#define HG_TRANSPORT_NCCL 1 /* packed boxes, NCCL send/recv on a side stream, overlapped */
#define HG_NCCL_ID_BYTES 128
typedef struct hg_dmp_opts {
  int transport;                            /* HG_TRANSPORT_P2P (default) | _NCCL */
  int nranks;                               /* NCCL: ranks in the communicator (= grid size) */
  unsigned char nccl_id[HG_NCCL_ID_BYTES];  /* NCCL: hg_nccl_unique_id() of one rank, shared */
  double timeout_s;                         /* bounded halo waits: 0 = default (30 s),
                                               < 0 = wait forever */
  int depth;                                /* deep halos: exchange depth*w-wide halos every
                                               `depth` steps, the ring recomputed redundantly
                                               (decomposition from hg_decompose_program_deep);
                                               0 or 1 = every step, as the reference */
} hg_dmp_opts;
/* One rank's endpoint of the decomposed program (RankHooks + Endpoint, simulator.cpp:201-260,
 * 772-834).  hg_dmp_create = hg_dmp_create_ex with default options (P2P). */
int hg_dmp_create(hg_plan *plan, const hg_decomp *decomp, int64_t rank, hg_dmp **out);
/* NCCL: every rank calls this concurrently (ncclCommInitRank) with the same id. */
int hg_dmp_create_ex(hg_plan *plan, const hg_decomp *decomp, int64_t rank,
                     const hg_dmp_opts *opts, hg_dmp **out);
int hg_nccl_unique_id(void *id /* HG_NCCL_ID_BYTES */);
int hg_dmp_destroy(hg_dmp *dmp);
/* P2P multi-process: export this rank's CUDA IPC handles (buffers, packed x-face receive
 * slabs, signal flags) as a blob, all-gather the blobs with any host transport, import every
 * neighbour's. */
int hg_dmp_ipc_export(hg_dmp *dmp, void *blob, size_t cap, size_t *len);
int hg_dmp_ipc_import(hg_dmp *dmp, int64_t peer_rank, const void *blob, size_t len);
/* Time steps of this rank: swap dirty fields, wait for the neighbours' halos, compute.
 * Collective over all ranks (every rank runs the same step counts).  Asynchronous on
 * `stream`.  A halo wait that exceeds the timeout (a stuck or dead peer) does not hang the
 * GPU: it is recorded, hg_dmp_status reports it, and later calls return HG_ETRAP. */
int hg_dmp_run(hg_dmp *dmp, int64_t steps, void *stream);
/* Waits for the dmp's queued work; HG_ETRAP ("rank r: halo round from neighbour rank n
 * (face ...) did not arrive for epoch e within X s") if a halo wait timed out. */
int hg_dmp_status(hg_dmp *dmp);
int hg_dmp_set_timeout(hg_dmp *dmp, double seconds /* <= 0: forever */);
/* Single process: connect the n ranks (peer pointers).  hg_sim_run runs all of them step by
 * step: with one rank per device, the multi-process protocol (fused NVLink swap, in-kernel
 * waits); ranks sharing a device are ordered by CUDA events (simulate's loop,
 * simulator.cpp:1066-1203).  Returns after the ranks finished (HG_ETRAP on a timed-out wait). */
int hg_sim_connect(hg_dmp **ranks, int n);
int hg_sim_run(hg_dmp **ranks, int n, int64_t steps, void **streams);
int64_t hg_dmp_bytes_exchanged(const hg_dmp *dmp); /* payload bytes put so far */
/* Host data was uploaded into the plan's buffers: every halo is stale, swap all on next use.
 * Collective in multi-process P2P mode: every rank calls it after its own uploads (on the
 * stream of its next hg_dmp_run, or fenced before it); the next run first performs a
 * receiver-ready handshake so no neighbour puts into a buffer still being uploaded. */
int hg_dmp_invalidate(hg_dmp *dmp);

#ifdef __cplusplus
}
#endif

#endif /* HG_HG_H */
