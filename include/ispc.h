/*
 * ispc.h — C-ABI of the B200 candidate-evaluation backend (libispc.so).
 *
 * This is the drop-in boundary for the reference's evaluation path
 * ("candidate -> kernel -> run -> time"). The reference evaluates a fully
 * specified candidate with
 *
 *   LoopNest    reconstruct(const Kernel&, const SpaceContext&, const Candidate&)
 *                                                    (proj/core/include/ispace/loop_nest.hpp:52)
 *   std::string emit_source(const Kernel&, const LoopNest&)      (loop_nest.hpp:62)
 *   CostReport  evaluate(const Kernel&, const LoopNest&, const MachineParams&)
 *                                                    (proj/core/include/ispace/simulate.hpp:33)
 *
 * reconstruct() stays on the reference side. Its result, together with the
 * Kernel backbone, crosses this boundary as a flat `ispc_nest` (plain structs,
 * indices and sizes, no C++ types). Behind the boundary the backend replaces
 * emit_source() with an sm_100a CUDA emitter (ispc_emit_cuda) and evaluate()
 * with NVRTC compilation, a CUDA-event-timed launch on a B200 and an
 * on-device output check (ispc_evaluate and the finer-grained calls below).
 *
 * Conventions: every entry point returns an int status (ISPC_OK == 0, < 0 is
 * an error class); no exception crosses the ABI; the text of the last error of
 * a device (or of the calling thread for device-less calls) is available from
 * ispc_last_error(). One ispc_dev per GPU, used by one host thread at a time.
 * ispc_emit_cuda and ispc_compile need no GPU and are thread-safe.
 */
#ifndef ISPC_H
#define ISPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISPC_ABI_VERSION 2u
#define ISPC_NONE 0xFFFFFFFFu

/* ---- status codes ------------------------------------------------------- */
enum {
  ISPC_OK = 0,
  ISPC_E_ARG = -1,      /* malformed nest / bad argument                      */
  ISPC_E_CUDA = -2,     /* CUDA driver/runtime failure (non-sticky)           */
  ISPC_E_NVRTC = -3,    /* NVRTC compilation failed                           */
  ISPC_E_LAUNCH = -4,   /* launch failed (resources, grid limits)             */
  ISPC_E_MISMATCH = -5, /* output differs from the expected values            */
  ISPC_E_TIMEOUT = -6,  /* device watchdog fired: time >= budget              */
  ISPC_E_ILLEGAL = -7,  /* statically rejected on B200 (see ispc_last_error)  */
  ISPC_E_NOMEM = -8,    /* device allocation failed                           */
  ISPC_E_STICKY = -9    /* context-killing fault; device must be reopened     */
};

/* ---- flat Kernel + LoopNest ---------------------------------------------
 * Mirrors, field by field, the reference structs:
 *   Op                  kernels.hpp:14      ispc_op
 *   AddrTerm            kernels.hpp:21-25   ispc_addr_term
 *   InductionVar        kernels.hpp:27-30   ispc_ivar
 *   Operand             kernels.hpp:32-43   ispc_operand
 *   Comm                kernels.hpp:49-58   ispc_comm
 *   InstInfo            kernels.hpp:60-66   ispc_inst
 *   DimInfo/LogicalInfo kernels.hpp:68-78   ispc_dim
 *   RegionInfo          kernels.hpp:80-84   ispc_region
 *   NestNode            loop_nest.hpp:25-35 ispc_node
 *   LoopNest            loop_nest.hpp:37-44 ispc_nest (shapes, sizes, mem_space, cache)
 * Object ids are the reference's ObjId values (backbone object indices).
 * Variable-length lists live in `pool` (uint32) and are addressed by
 * (begin, count). Children of a node are contiguous in `nodes`.
 */
enum ispc_op { ISPC_OP_ADD = 0, ISPC_OP_MUL, ISPC_OP_MAD, ISPC_OP_CAST, ISPC_OP_LOAD, ISPC_OP_STORE };
enum ispc_operand_kind {
  ISPC_OPND_CONST = 0, ISPC_OPND_INPUT, ISPC_OPND_INDVAR, ISPC_OPND_PRODUCED, ISPC_OPND_REDUCE, ISPC_OPND_MAPPED
};
enum ispc_dim_kind { ISPC_LOOP = 0, ISPC_BLOCK, ISPC_THREAD, ISPC_UNROLL, ISPC_VECTOR };
enum ispc_mem_space { ISPC_GLOBAL = 0, ISPC_SHARED };
enum ispc_cache {
  ISPC_CACHE_L1 = 0, ISPC_CACHE_L2, ISPC_CACHE_READ_ONLY, ISPC_CACHE_NONE,
  ISPC_CACHE_STREAM /* building blocks only: ld.global.nc.L1::no_allocate.L2::256B */
};
enum ispc_node_kind { ISPC_NODE_DIM = 0, ISPC_NODE_INST, ISPC_NODE_BARRIER };

typedef struct {
  uint32_t dim;              /* ObjId of the iteration dimension              */
  uint32_t size_dims_begin;  /* pool slice: dims whose sizes multiply `base`  */
  uint32_t size_dims_count;
  uint32_t _pad;
  int64_t base;
} ispc_addr_term;

typedef struct {
  int64_t offset;
  uint32_t terms_begin; /* slice of ispc_nest.terms */
  uint32_t terms_count;
} ispc_ivar;

typedef struct {
  uint32_t kind;         /* ispc_operand_kind                                    */
  uint32_t input;        /* INPUT: index into input_names                        */
  uint32_t ivar;         /* INDVAR: index into ivars                             */
  uint32_t producer;     /* PRODUCED / MAPPED: ObjId                             */
  uint32_t init;         /* REDUCE: ObjId of the initializer                     */
  uint32_t comm;         /* MAPPED / REDUCE: index into comms, or ISPC_NONE      */
  uint32_t pairs_begin;  /* pool slice of (producer dim, consumer dim) ObjIds    */
  uint32_t pairs_count;  /* number of pairs (pool holds 2*pairs_count ids)       */
  uint32_t reduce_begin; /* REDUCE: pool slice of reduction dims                 */
  uint32_t reduce_count;
  int64_t value;         /* CONST                                                */
} ispc_operand;

typedef struct {
  uint32_t obj;             /* ObjId                                        */
  uint32_t op;              /* ispc_op                                      */
  uint32_t region;          /* LOAD / STORE: region ObjId, else ISPC_NONE   */
  uint32_t ivar;            /* LOAD / STORE: index into ivars               */
  uint32_t operands_begin;  /* slice of ispc_nest.operands                  */
  uint32_t operands_count;
  uint32_t dims_begin;      /* pool slice: iteration dims, outermost first  */
  uint32_t dims_count;
  uint32_t live;            /* 1 when the instruction is in the nest        */
  uint32_t cache;           /* ispc_cache (LoopNest::cache), LOAD/STORE     */
} ispc_inst;

typedef struct {
  uint32_t obj;
  uint32_t input;      /* 1: kernel argument (x, y, z, a, b, c)          */
  uint32_t live;       /* 1: present in LoopNest::mem_space              */
  uint32_t mem_space;  /* ispc_mem_space                                 */
  int64_t elems;
  int64_t elem_bytes;
} ispc_region;

typedef struct {
  uint32_t obj;
  uint32_t logical;    /* ObjId of the logical axis                      */
  uint32_t is_static;
  uint32_t _pad;
  int64_t size;        /* LoopNest::sizes: concrete extent               */
} ispc_dim;

typedef struct {
  uint32_t producer, consumer, region, store, load; /* ObjIds              */
  uint32_t pairs_begin, pairs_count;                /* as in ispc_operand */
  uint32_t fired;                                   /* lowering fired     */
} ispc_comm;

typedef struct {
  uint32_t kind;         /* ispc_node_kind                                 */
  uint32_t dim_kind;     /* ispc_dim_kind (DIM nodes)                      */
  int32_t thread_level;  /* THREAD: 0 = outermost hardware level, else -1  */
  int32_t block_level;   /* BLOCK: 0 = outermost grid level, else -1       */
  uint32_t inst;         /* INST: ObjId                                    */
  uint32_t dims_begin;   /* DIM: pool slice, the fused class (smallest first) */
  uint32_t dims_count;
  uint32_t children_begin; /* index into nodes                             */
  uint32_t children_count;
  uint32_t _pad;
  int64_t size;          /* DIM: extent                                    */
} ispc_node;

typedef struct {
  uint32_t abi_version;  /* ISPC_ABI_VERSION                                */
  const char* kernel_name;
  uint32_t num_objects;
  const char* const* object_names; /* by ObjId                              */
  uint32_t num_insts;    const ispc_inst* insts;
  uint32_t num_regions;  const ispc_region* regions;
  uint32_t num_dims;     const ispc_dim* dims;
  uint32_t num_ivars;    const ispc_ivar* ivars;
  uint32_t num_terms;    const ispc_addr_term* terms;
  uint32_t num_operands; const ispc_operand* operands;
  uint32_t num_comms;    const ispc_comm* comms;
  uint32_t num_inputs;   const char* const* input_names; /* scalar inputs ("alpha") */
  uint32_t pool_size;    const uint32_t* pool;
  uint32_t num_nodes;    const ispc_node* nodes;
  uint32_t roots_begin, roots_count;
  uint32_t num_thread_levels; /* LoopNest::thread_shape, outermost first      */
  uint32_t num_block_levels;  /* LoopNest::block_shape, outermost first       */
  int64_t thread_shape[3];
  int64_t block_shape[3];
} ispc_nest;

/* ---- emission -------------------------------------------------------------- */

/* One kernel parameter of an emitted kernel, in declaration order. */
enum ispc_param_kind { ISPC_PARAM_REGION = 0, ISPC_PARAM_INPUT, ISPC_PARAM_DEADLINE, ISPC_PARAM_TMAP };
typedef struct {
  uint32_t kind;      /* ispc_param_kind                                       */
  uint32_t index;     /* REGION: region ObjId; INPUT: input index              */
  uint32_t is_input;  /* REGION: 1 problem region bound by name, 0 temporary   */
  uint32_t _pad;
  int64_t elems;      /* REGION: elements the kernel may touch                 */
  char name[24];      /* REGION: region name ("x", "tmp0"); INPUT: "alpha"     */
} ispc_param;

/* A TMA tensor map (CUtensorMap, passed by value as a __grid_constant__
 * parameter) the runtime encodes over a bound problem region at launch. */
typedef struct {
  uint32_t param;        /* index of the kernel parameter it fills          */
  uint32_t rank;         /* 2 or 3                                          */
  uint32_t swizzle;      /* 0 none, 1 32B, 2 64B, 3 128B, 4 128B with 32-B atoms */
  uint32_t _pad;
  char region[24];       /* problem region name                             */
  uint64_t dims[3];      /* elements, innermost first                       */
  uint64_t strides[2];   /* bytes between consecutive dims[1], dims[2]      */
  uint32_t box[3];       /* elements per copy, innermost first              */
  uint32_t _pad2;
} ispc_tmap;

#define ISPC_MAX_PARAMS 32
#define ISPC_MAX_TMAPS 4
typedef struct {
  char name[64];         /* extern "C" __global__ symbol                   */
  uint64_t grid_x;       /* linearized grid (block levels, mixed radix)    */
  uint32_t block[3];     /* blockDim.{x,y,z}; innermost level is x         */
  uint32_t static_smem;  /* bytes of SHARED tmp regions                    */
  uint32_t num_params;
  uint32_t pdl;          /* 1: launch with programmatic stream serialization
                            (the kernel's first statement is griddepcontrol.wait,
                            so it touches memory only after the previous grid of
                            the stream completed; its CTAs may be scheduled
                            while that grid drains)                        */
  ispc_param params[ISPC_MAX_PARAMS];
  uint32_t watchdog;     /* 1 when the kernel polls the deadline parameter */
  uint32_t reg_elems;    /* register-array elements per thread (static)    */
  uint64_t source_hash;  /* FNV-1a of the kernel body (dedupe key)         */
  uint32_t cluster[3];   /* thread-block cluster dims ({0,0,0}: no cluster) */
  uint32_t num_tmaps;
  ispc_tmap tmaps[ISPC_MAX_TMAPS];
} ispc_launch;

typedef struct {
  uint32_t watchdog;      /* 0 off, 1 on, 2 auto (on when the loop work is large) */
  uint32_t max_reg_elems; /* reject nests needing more register-array floats (0: 512) */
  uint32_t max_unrolled;  /* reject nests whose unrolled body exceeds this many insts (0: 16384) */
  uint32_t _pad;
} ispc_emit_opts;

/* Emits one sm_100a CUDA kernel (a self-contained NVRTC translation unit
 * fragment: the caller may concatenate several into one program after
 * ispc_cuda_prelude()). `fn_name` NULL picks "ispc_k<hash>". Writes at most
 * `cap` bytes (NUL-terminated) and the full length to *len. Returns
 * ISPC_E_ILLEGAL (with the reason in ispc_last_error) when the schedule cannot
 * run correctly on the device: cross-block value flow through a temporary,
 * register/unroll budgets, grid limits, out-of-range addresses. */
int ispc_emit_cuda(const ispc_nest* nest, const ispc_emit_opts* opts, const char* fn_name,
                   char* buf, size_t cap, size_t* len, ispc_launch* launch);

/* Device helpers every emitted kernel relies on (cache-hinted ld/st, timer). */
const char* ispc_cuda_prelude(void);

/* Pseudo-source rendering of the nest through this ABI, byte-compatible with
 * the reference's emit_source() (loop_nest.cpp:389-609). Used to prove the flat
 * description carries the whole schedule. */
int ispc_emit_pseudo(const ispc_nest* nest, char* buf, size_t cap, size_t* len);

/* ---- B200 building-block kernels -------------------------------------------
 * gemv, shared/cp.async-staged sgemm, batched sgemm and the tcgen05 sgemm of
 * BASELINE.json cannot be written in the reference's gpu.space (SURVEY.md
 * 0.4-0.5): their decisions live in a second space in the reference's own
 * language (host/tiles.space, built through build_space, candidate.hpp:37-49).
 * A fully specified candidate of that space crosses the boundary as this flat
 * struct, the counterpart of ispc_nest; ispc_emit_tiles turns it into one
 * sm_100a kernel assembled from hand-written building blocks. */
enum ispc_tile_kind { ISPC_TILE_GEMV = 0, ISPC_TILE_SGEMM, ISPC_TILE_BATCHED, ISPC_TILE_SGEMM_TC, ISPC_TILE_AXPY };
enum ispc_staging { ISPC_STAGE_DIRECT = 0, ISPC_STAGE_SHARED, ISPC_STAGE_CP_ASYNC, ISPC_STAGE_TMA };
enum ispc_engine { ISPC_ENGINE_FFMA = 0, ISPC_ENGINE_TF32, ISPC_ENGINE_TF32X3 };
enum ispc_xreduce { ISPC_XRED_SHUFFLE = 0, ISPC_XRED_SHARED };

typedef struct {
  uint32_t kind;                 /* ispc_tile_kind                                  */
  uint32_t staging, engine;      /* ispc_staging, ispc_engine                       */
  uint32_t xreduce, cache;       /* ispc_xreduce, ispc_cache (global operand loads) */
  uint32_t lds;                  /* FFMA2 sgemm: 1 = fragments by 32-bit ld.shared.v4,
                                    0 = by generic pointers                         */
  int64_t m, n, k, batch;        /* problem shape (column-major operands)           */
  /* decided tile parameters; 0 = not a parameter of this kind                    */
  int32_t thr_m, thr_n;          /* sgemm: CTA threads along m / n                  */
  int32_t tm, tn;                /* per-thread output tile (sgemm, batched)         */
  int32_t bk;                    /* k depth staged per step                         */
  int32_t bn;                    /* tcgen05: UMMA N (M is 128 per CTA)              */
  int32_t stages;                /* shared-memory ring depth                        */
  int32_t vec;                   /* global vector width (floats)                    */
  int32_t lanes_m, lanes_n;      /* gemv: warp lanes along rows / columns           */
  int32_t warps_m, warps_n;      /* gemv: warps along rows / columns                */
  int32_t split;                 /* gemv: cluster CTAs splitting the columns (DSMEM);
                                    sgemm: split-K cluster; tcgen05: 2 = cta_group::2 pair */
  int32_t unroll;                /* gemv: column loop unroll                        */
  int32_t per_cta;               /* batched: problems per CTA                       */
  int32_t threads;               /* axpy stream: threads per CTA                    */
  int32_t grid;                  /* axpy stream: CTAs (0: one vector group per thread);
                                    tcgen05 / gemv: persistent CTAs (0: one tile each) */
  int32_t pdl;                   /* 1: programmatic dependent launch (ispc_launch.pdl) */
} ispc_tile_config;

/* Emits the kernel of a tile configuration (same conventions as
 * ispc_emit_cuda). ISPC_E_ILLEGAL when the configuration cannot run on a B200
 * (shape not divisible, shared memory, threads, registers, cluster size). */
int ispc_emit_tiles(const ispc_tile_config* cfg, const char* fn_name, char* buf, size_t cap, size_t* len,
                    ispc_launch* launch);

/* ---- compilation (no GPU needed; thread-safe) ------------------------------ */
typedef struct ispc_module ispc_module;

/* Compiles `n` sources (each: prelude-less kernel fragments) into ONE NVRTC
 * program for `arch` (NULL: "sm_100a") and returns the cubin. */
int ispc_compile(const char* const* srcs, int n, const char* arch, ispc_module** out);
int ispc_module_cubin(const ispc_module* m, const void** data, size_t* size);
const char* ispc_module_log(const ispc_module* m);
void ispc_module_free(ispc_module* m);

/* ---- device, problem binding, timed launch, check ------------------------- */
typedef struct ispc_dev ispc_dev;

int ispc_dev_open(int ordinal, ispc_dev** out);
void ispc_dev_close(ispc_dev* d);
const char* ispc_last_error(const ispc_dev* d); /* NULL d: calling thread's last error */
/* Test hook: a store through an invalid address on the device's stream; returns
 * ISPC_E_STICKY (and poisons the context) when the fault happened. A faulted
 * process cannot open the device again (cudaErrorDevicesUnavailable, measured
 * on the B200 boxes); a new process can. */
int ispc_dev_inject_fault(ispc_dev* d);
int ispc_dev_info(const ispc_dev* d, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes,
                  int* sm_clock_khz);

/* Problem kinds: the reference builders (kernels.cpp:373-488) plus the B200
 * extensions named in BASELINE.json. Region names follow the builders. */
enum ispc_problem_kind {
  ISPC_PROB_AXPY = 0,        /* z = alpha*x + y;  regions x,y,z [n]           */
  ISPC_PROB_OUTER = 1,       /* c[i*n+j] = a[i]*b[j]; regions a[m],b[n],c[m*n] */
  ISPC_PROB_MATMUL = 2,      /* column-major C = A*B, A element stride a_stride */
  ISPC_PROB_GEMV = 3,        /* y = A*x, A column-major m x n                  */
  ISPC_PROB_BATCHED = 4      /* batch x (C = A*B), 32x32x64 column-major       */
};
typedef struct {
  uint32_t kind;
  uint32_t _pad;
  int64_t m, n, k, batch, a_stride;
  uint64_t seed;
  float alpha;
  float _pad2;
} ispc_problem;

/* Allocates and fills (on device, from `seed`) the inputs, allocates the
 * outputs and computes the expected outputs with the in-library golden
 * kernels. Rebinding frees the previous problem. */
int ispc_bind_problem(ispc_dev* d, const ispc_problem* p);
/* Region pointer / size of the bound problem by region name ("x", "c", ...). */
int ispc_problem_region(ispc_dev* d, const char* name, uint64_t* dev_ptr, int64_t* elems);

/* Loading and unloading may be called from any host thread (e.g. compile
 * threads loading the next module while the device thread launches). */
int ispc_module_load(ispc_dev* d, const ispc_module* m, int* handle);
int ispc_module_unload(ispc_dev* d, int handle);

/* Checking: bit_exact compares bits with the golden sequential kernels.
 * Otherwise an element fails when |out - exp| > rtol * scale, with scale the
 * golden sum of |products| (sum |a||x| for gemv, sum |a||b| for matmuls) for
 * reductions, |exp| elsewhere: the norm-wise test a reordered reduction
 * (shuffle, split, tensor core) is held to. */
typedef struct {
  uint32_t warmup;        /* untimed launches after the first (checked) one  */
  uint32_t reps;          /* timed launches; median reported                 */
  uint32_t flush_l2;      /* 1: write an L2-sized buffer before every launch */
  uint32_t check;         /* 1: verify outputs after the first launch        */
  uint32_t bit_exact;     /* 1: require identical bits, else rtol            */
  uint32_t rotate;        /* >= 2: timed launches run back to back over this
                             many copies of the inputs (inputs larger than L2
                             in aggregate), mean per launch; else one launch
                             per event pair                                   */
  double rtol;            /* relative tolerance when !bit_exact              */
  double budget_ns;       /* watchdog budget per launch (0: 2 s); armed on the
                             device when the launch starts (a rotation group of
                             R launches gets R budgets)                       */
} ispc_time_opts;

typedef struct {
  int status;             /* ISPC_OK, ISPC_E_MISMATCH, ISPC_E_TIMEOUT, ...   */
  int _pad;
  double median_ns;       /* median of the timed launches                    */
  double min_ns;
  double first_ns;        /* duration of the first (checked) launch          */
  double max_err;         /* max |out - expected| / max(|expected|, 1e-30)   */
  int64_t mismatches;     /* elements differing (bits or beyond rtol)        */
} ispc_time_result;

/* Launches kernel `name` of loaded module `handle` with the problem's buffers
 * (NaN-prefilled outputs, GLOBAL temporaries from a scratch pool). */
int ispc_launch_timed(ispc_dev* d, int handle, const ispc_launch* launch,
                      const ispc_time_opts* opts, ispc_time_result* res);

/* Batched evaluation of several kernels of one loaded module with two host
 * round trips in all (no per-launch synchronisation):
 *   screen: per item, NaN-filled outputs, one launch timed by CUDA events with
 *           its watchdog deadline armed on the device right before it, and the
 *           on-device check (skipped when the watchdog fired) - every item;
 *   refine: `warmup` + `reps` timed launches (median; rotation groups as in
 *           ispc_launch_timed) for the items that passed the check and whose
 *           screened time is <= refine_below_ns (INFINITY: all of them).
 * A failure to bind or launch one item is reported in its result's status;
 * the call fails only for errors of the device (ISPC_E_STICKY, ...). */
typedef struct {
  const ispc_launch* launch;
  ispc_time_opts opts;     /* per item: budget, check / bit_exact / rtol, reps */
} ispc_batch_item;
int ispc_launch_batch(ispc_dev* d, int handle, int n, const ispc_batch_item* items,
                      double refine_below_ns, ispc_time_result* res);

/* Compares the bound outputs with the expected outputs on the device. */
int ispc_check(ispc_dev* d, double rtol, int bit_exact, double* max_err, int64_t* mismatches,
               int* ok);

/* Copies a region of the bound problem to host memory. */
int ispc_read_region(ispc_dev* d, const char* name, void* host, size_t bytes);
/* Overwrites an input region of the bound problem from host memory (pinned
 * memory copies at full PCIe/C2C speed) and recomputes the expected outputs. */
int ispc_write_region(ispc_dev* d, const char* name, const void* host, size_t bytes);
/* Reads the expected output computed by the golden kernels. */
int ispc_read_expected(ispc_dev* d, const char* name, void* host, size_t bytes);

/* Device-timeline marks on the device's stream (CUDA events, 8 slots):
 * elapsed milliseconds between two recorded marks. */
int ispc_dev_mark(ispc_dev* d, int slot);
int ispc_dev_mark_elapsed(ispc_dev* d, int slot_a, int slot_b, double* ms);

/* Pins (page-locks, portable across devices) host memory the search shares
 * between GPU workers, e.g. the incumbent bound (cudaHostRegister). */
int ispc_host_register(void* p, size_t bytes);
int ispc_host_unregister(void* p);

/* One-shot replacement of evaluate(): emit + compile + load + timed launch +
 * check. The mirror of CostReport is ispc_time_result (time in ns). */
int ispc_evaluate(ispc_dev* d, const ispc_nest* nest, const ispc_emit_opts* eopts,
                  const ispc_time_opts* topts, ispc_time_result* res, ispc_launch* launch);

/* Same one-shot path for a building-block configuration (ispc_emit_tiles). */
int ispc_evaluate_tiles(ispc_dev* d, const ispc_tile_config* cfg, const ispc_time_opts* topts,
                        ispc_time_result* res, ispc_launch* launch);

#ifdef __cplusplus
}
#endif
#endif /* ISPC_H */
