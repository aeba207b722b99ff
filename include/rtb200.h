/*
 * rtb200 — B200 execution backend for recurrent-tensor / PDG programs.
 *
 * C ABI (plain pointers, sizes and POD descriptors; no torch types).  The
 * host side (paper_2501_05408_b200/) lowers a dependence graph into a
 * program of kernel launches over "boxes" (slab of a node's domain x its
 * payload) and loops over the dims the dependence structure serialises;
 * this library runs that program on one CUDA stream.
 *
 * Reference interfaces each entry replaces (paths relative to the
 * reference root, pkg/src/recten/):
 *   rt_run            runtime.py:460-475 reference_execute (the executor
 *                     loop _Oracle.value/read, runtime.py:344-425) — runs a
 *                     lowered program: loops + launches + memory ops
 *   rt_launch         runtime.py:37-44, 236-271 the KERNELS table ABI
 *                     fn(node, vals, env, rng): one kernel family per call
 *   rt_status_read    runtime.py:25-30, 176-177, 186-188 error reporting
 *                     (RuntimeError_/OracleError) via a device status word
 *   rt_memcpy_*       SPEC.md:558-561 Backend move-between-tiers (the
 *                     offload/fetch of polysched.py:936-1105, realised as
 *                     pinned cudaMemcpyAsync on a side stream)
 *   rt_rng_fill       runtime.py:50-55, 391-394 per-point
 *                     default_rng((seed, tag, *point)) draws, bit-exact
 *   rt_nccl_*, rt_set_collectives, rt_coll_exec
 *                     the gradient all-reduce of an env-sharded
 *                     run (no reference counterpart: the reference is
 *                     single-process), issued from the program itself
 *   rt_pool_*, rt_offload, rt_fetch, rt_block_update, rt_stack
 *                     SPEC.md:541-561 the runtime's Backend (allocate,
 *                     deallocate, move-between-tiers, dynamic-update, stack)
 *                     and MemorySim (device/host live+peak, transfer
 *                     counters, overflow = hard error) — specified by the
 *                     reference, implemented nowhere in it
 */
#ifndef RTB200_H
#define RTB200_H

#ifdef __CUDACC_RTC__   /* NVRTC: no libc headers */
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#else
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RT_MAXD 10    /* max rank of an iteration box (slab dims + payload dims) */
#define RT_MAXENV 8   /* max loop dims visible to a launch                        */
#define RT_MAXIN 8    /* max operand views of one elementwise launch             */
#define RT_MAXCHK 3   /* max range checks per view                               */
#define RT_CODE 256   /* program words per launch                                */
#define RT_KONST 32   /* float constants per launch                              */

enum rt_dtype { RT_F64 = 0, RT_F32 = 1, RT_I64 = 2, RT_BOOL = 3 };

enum rt_kernel {
  RT_K_EW = 1,       /* fused elementwise/layout/merge/gather program        */
  RT_K_REDUCE = 2,   /* sum / discounted sum over (possibly ragged) ranges   */
  RT_K_SCAN = 3,     /* linear recurrence y = x + g*y_prev along one dim      */
  RT_K_GEMM = 4,     /* strided/batched/contracting fp32|fp64 matmul          */
  RT_K_RNG = 5,      /* SeedSequence->PCG64->{normal,uniform} per point       */
  RT_K_UDF = 6,      /* synthetic environment (dsl.py:288-307) per point      */
  RT_K_SPLITK = 7,   /* split-K partial reduction for RT_K_GEMM               */
  RT_K_MEMCPY = 8,   /* stream-ordered tier move of a swapped buffer (rt_memcpy_params) */
  RT_K_LOOP = 9,     /* persistent kernel running a whole row-local loop      */
  RT_K_GEMM_TC = 10, /* RT_K_GEMM on tcgen05 (3xTF32, TMEM accumulators)      */
  RT_K_THIN = 11,    /* HBM-bound skinny GEMMs (narrow contraction / small K)  */
  RT_K_GEMM_TMA = 12 /* RT_K_GEMM on tcgen05 fed by TMA (plain 2-D operands)   */
};

enum rt_status_code {
  RT_OK = 0,
  RT_ERR_ROW_RANGE = 1,     /* index_select row outside 0..n-1 (runtime.py:186-188) */
  RT_ERR_SLICE_RANGE = 2,   /* index_select rows lo:hi outside (runtime.py:176-177) */
  RT_ERR_CUDA = 3,
  RT_ERR_BAD_ARG = 4,
  RT_ERR_UNKNOWN_KERNEL = 5,
  RT_ERR_DIV_ZERO = 6,      /* index expression // or % by zero (symexpr.py:491-506);
                               aux = (dividend, 0 for //, 1 for %) */
  RT_ERR_OVERFLOW = 7       /* device tier over capacity (SPEC.md:554-557 MemorySim) */
};

/* A flat index over a box, decomposed row-major. */
typedef struct {
  int32_t nd;
  int32_t _pad;
  int64_t ext[RT_MAXD];
} rt_box;

/* An operand's addressing over a box: element offset
 *   off + sum_e env[e]*off_env[e] + sum_d idx[d]*stride[d]
 * valid iff every check  0 <= c0 + sum_e env[e]*c_env[e] + sum_d idx[d]*a[d] < hi
 * (an invalid load yields 0; the planner guarantees invalid loads are never
 * selected where the reference would have read them). */
typedef struct {
  uint64_t ptr;
  int32_t dtype;
  int32_t nchk;
  int64_t off;
  int64_t off_env[RT_MAXENV];
  int64_t stride[RT_MAXD];
  int64_t chk_c0[RT_MAXCHK];
  int64_t chk_hi[RT_MAXCHK];
  int32_t chk_env[RT_MAXCHK][RT_MAXENV];
  int32_t chk_a[RT_MAXCHK][RT_MAXD];
} rt_view;

/* Every parameter block starts with this header; rt_run patches env[]
 * before each launch. */
typedef struct {
  int64_t env[RT_MAXENV];
  int32_t node;        /* graph node id, for error reports */
  int32_t status_slot; /* unused: status word is global   */
  uint64_t status;     /* device pointer to int32[4] status word */
} rt_hdr;

/* RT_K_EW: out[idx] = program(views)(idx) for idx over box. */
typedef struct {
  rt_hdr h;
  rt_box box;
  int64_t total;
  int32_t nin;
  int32_t f64;         /* compute in double (else float) */
  rt_view out;
  rt_view in[RT_MAXIN];
  int32_t code[RT_CODE];
  double konst[RT_KONST];
} rt_ew_params;

/* RT_K_REDUCE: out[p] = sum_{k in ranges(p)} w(k) * in[p, k]
 * box = output points (nd_out dims); red = reduced dims with extents given
 * as affine forms (lo fixed at the view, len per point) or int programs. */
typedef struct {
  rt_hdr h;
  rt_box box;          /* output box */
  int64_t total;
  int32_t nred;        /* number of reduced dims (<= 4) */
  int32_t op;          /* 0 = sum, 1 = discounted sum along red dim 0 */
  double gamma;
  int32_t reverse;     /* dsum weights reversed */
  int32_t f64;
  int32_t len_prog[4]; /* -1: len = len0 + sum a*idx + env; else program entry */
  int64_t len0[4];
  int64_t len_env[4][RT_MAXENV];
  int64_t len_a[4][RT_MAXD];
  int64_t red_stride[4];   /* input element stride per reduced dim */
  int32_t lo_prog[4];      /* -1 none; else program computing the start offset shift */
  int32_t threads_per_out; /* 1 or a power of two <= 1024 */
  int32_t splits;      /* column mode: reduce range split in `splits` partials */
  uint64_t part;       /* column mode: fp64 scratch [splits][total] (0: row mode) */
  rt_view in;          /* strides over the output box; lo folded in */
  rt_view out;
  int32_t code[RT_CODE];
  double konst[RT_KONST];
} rt_reduce_params;

/* RT_K_SCAN: along dim `sdim` of box: y[j] = x[j] + gamma*y[j-1] (or j+1). */
typedef struct {
  rt_hdr h;
  rt_box box;          /* full box including the scan dim */
  int64_t total_lines; /* prod of extents except the scan dim */
  int32_t sdim;
  int32_t reverse;
  double gamma;
  int32_t f64;
  int32_t chunk;       /* elements per chunk along the line (0 = whole line) */
  rt_view in;
  rt_view out;
  /* window form: y[j] = S[lo(j)] - gamma^(hi-lo) * S[hi(j)], unused if win=0 */
  int32_t win;
  int32_t tile;        /* 2: cp.async ring, line-major; 3: the same, step-major;
                        * 4: bulk-copy pipeline per line (chunk = elements per stage) */
  /* gae != 0: the scanned value is the TD residual computed on the fly,
   * x[j] = in[j] + gae_c * (j+1 < L ? in2[j+1] : gae_vb) - in2[j]
   * (GAE(lambda): delta = r + gamma V[t+1] - V, bootstrap gae_vb at T-1),
   * so delta never round-trips through HBM. */
  int32_t gae;
  int32_t stages;      /* tile 4: shared-memory stages per line */
  double gae_c, gae_vb;
  rt_view in2;
} rt_scan_params;

/* RT_K_MEMCPY: one stream-ordered copy of `bytes` from src to dst
 * (cudaMemcpyAsync, kind inferred from the addresses: device <-> pinned host).
 * The general swap (swap.py plan_gap_swap) offloads a swap-managed buffer
 * after its last touch before an idle gap and fetches it back before its next
 * touch; as a launch record it is ordered, profiled and graph-captured like a
 * kernel. */
typedef struct {
  rt_hdr h;
  uint64_t dst;
  uint64_t src;
  int64_t bytes;
  int32_t dir;         /* 0 offload (device -> host), 1 fetch (host -> device) */
  int32_t _pad;
} rt_memcpy_params;

/* RT_K_GEMM: for z in Z, C[z,m,n] (+)= sum_k A[z,m,k] * B[z,k,n].
 * Each of Z, M, N, K is a flat index decomposed over its own small box;
 * every operand carries strides for each decomposed coordinate. */
typedef struct {
  int32_t nd;
  int32_t _pad;
  int64_t ext[4];
} rt_gbox;

typedef struct {
  uint64_t ptr;
  int32_t dtype;
  int32_t _pad;
  int64_t off;
  int64_t off_env[RT_MAXENV];
  int64_t sz[4];   /* strides for the Z coordinates  */
  int64_t s1[4];   /* strides for the M (A,C) or K (B) coordinates */
  int64_t s2[4];   /* strides for the K (A) or N (B,C) coordinates */
} rt_gop;

typedef struct {
  rt_hdr h;
  rt_gbox Z, M, N, K;
  int64_t z, m, n, k;  /* flat sizes */
  int32_t f64;
  int32_t splits;      /* split-K factor (partials to `part` when > 1) */
  int32_t accumulate;  /* C += result */
  int32_t epilogue;    /* 0 none, 1 tanh */
  rt_gop A, B, C;
  uint64_t part;       /* device scratch [splits, z, m, n] when splits > 1 */
  rt_gop bias;         /* added when bias.ptr != 0 (strides over Z,M: s1 for M? uses s2 over N) */
} rt_gemm_params;

/* RT_K_SPLITK: C[z,m,n] = sum_s part[s,z,m,n] */
typedef struct {
  rt_hdr h;
  rt_gbox Z, M, N;
  int64_t z, m, n;
  int32_t splits;
  int32_t f64;
  int32_t accumulate;
  int32_t epilogue;
  uint64_t part;
  rt_gop C;
  rt_gop bias;
} rt_splitk_params;

/* RT_K_THIN: GEMMs with one narrow side, which are HBM-bound (the dW of a
 * narrow layer over all T*E points, or a K<=32 product).  Names: W is the
 * wide index (streamed, contiguous), R the narrow one, K the contraction.
 *   variant 1: C[w,r] = sum_k X[k,w] * Y[k,r]   (K split over blockIdx.y,
 *              fp32/fp64 partials part[s, w*part_w + r*part_r] -> RT_K_SPLITK)
 *   variant 2: C[w,r] = epi(sum_k X[w,k] * Y[k,r] + bias[r])   (K <= 32)
 *   variant 3: C[w,r] (+)= epi(sum_k X[w,k] * Y[k,r] + bias[r]) for R <= 8
 *              and 32 <= K <= 1024 (policy/value heads over all points):
 *              a warp per row group, Y held in registers, rows streamed
 *              with 16-byte loads; w decomposed over the box W (strides
 *              X.s2[0..], C.s1[0..]); vec != 0 when rows are 16-B aligned.
 * Strides: X.s1[0] along k, X.s2[0] along w; Y.s1[0] along k, Y.s2[0]
 * along r; C.s1[0] along w, C.s2[0] along r; bias.s2[0] along r. */
typedef struct {
  rt_hdr h;
  int32_t variant;
  int32_t f64;
  int64_t w, r, k;
  int32_t splits;
  int32_t accumulate;
  int32_t epilogue;
  int32_t vec;
  int64_t part_w, part_r;
  uint64_t part;
  rt_gop X, Y, C, bias;
  rt_gbox W;           /* variant 3: decomposition of w (nd == 0: flat) */
  /* variant 2 + gate with k2 > 0: a second narrow-K product over the same
   * rows added before the gate, C = (X Y + X2 Y2) * (1 - h*h) (the sum of
   * two heads' backward into one hidden layer, executor.find_gate_epilogues) */
  int64_t k2;
  rt_gop X2, Y2;
  /* variant 1 with ones != 0: a column of ones appended to Y -- the bias
   * gradient sum_k X[k,w] of the same contraction (executor.find_ones_bias),
   * per-split partials into part2[s, w] (reduced by a second RT_K_SPLITK) */
  int32_t ones;
  int32_t colsum;      /* variant 2 vectorised: fp64 column sums of C over the rows
                        * into part2[blockIdx, r] (a bias gradient of the output,
                        * executor.find_colsum_epilogues; RT_K_SPLITK finishes) */
  uint64_t part2;
  /* variant 2 vectorised + gate, dw != 0: also the weight gradient of the
   * product's first operand against the gate operand, sum_rows h[w,c] X[w,k]
   * (dW of the head whose backward this is: dW3 = h2^T dmu), fp64 partials
   * per CTA into part3[blockIdx, c, k]; dw2: the same for X2 into part4 */
  int32_t dw, dw2;
  uint64_t part3, part4;
  /* variant 3 with r2 > 0: a sibling head over the same rows, outputs
   * r - r2 .. r - 1 from the weights Y2 (+ bias2) into C2 (the policy and
   * value heads reading the trunk once, executor.find_sibling_rows) */
  int64_t r2;
  rt_gop C2, bias2;
} rt_thin_params;

/* Point coordinates for per-point entropy: coordinate j of the node's
 * domain point is box index coord_src[j] when >= 0, else env[-1-coord_src[j]]. */

/* RT_K_RNG: per point of box, draw `count` values from
 * default_rng((prefix words..., *coords)) in C order (runtime.py:50-55). */
typedef struct {
  rt_hdr h;
  rt_box box;            /* slab box (points) */
  int64_t total;
  int32_t nprefix;       /* entropy words before the point coordinates */
  int32_t ncoord;        /* number of point coordinates (full node domain) */
  uint32_t prefix[8];
  int32_t coord_src[RT_MAXD];
  int64_t coord_add[RT_MAXD];   /* added to coordinate j (global index of a sharded dim) */
  int32_t dist;          /* 0 normal, 1 uniform */
  int32_t count;         /* values per point */
  rt_view out;           /* strides over box; `count` contiguous values per point */
} rt_rng_params;

/* RT_K_UDF: synthetic env body of dsl.make_udf_fn per point (dsl.py:288-307):
 * base = salt + sum_k mean(in_k); out_j ~ tanh(base + 0.3 N) | bool | i64. */
typedef struct {
  rt_hdr h;
  rt_box box;
  int64_t total;
  int32_t nprefix;
  int32_t ncoord;
  uint32_t prefix[8];
  int32_t coord_src[RT_MAXD];
  int64_t coord_add[RT_MAXD];
  double salt;
  int32_t nin;
  int32_t nout;
  int32_t in_count[4];   /* payload elements per input (mean over them) */
  int32_t out_count[4];
  int32_t out_kind[4];   /* rt_dtype of each output */
  rt_view in[4];         /* strides over box; payload contiguous after */
  rt_view out[4];
} rt_udf_params;

/* RT_K_LOOP: one persistent launch for a whole loop whose body is row-local
 * (every dependence inside the body keeps the slab coordinates, e.g. the
 * acting recurrence over t with all envs b independent).  Each CTA owns a
 * block of rows and runs every body op on them, step after step, with
 * __syncthreads between ops; no grid-wide synchronisation is needed.
 * Sub-op descriptors live in HBM unfolded; env terms are folded per step. */
typedef struct {
  int32_t kernel;       /* RT_K_EW | RT_K_GEMM | RT_K_UDF | RT_K_RNG */
  int32_t f64;
  uint64_t params;      /* device pointer to the op's parameter block */
  int64_t row_elems;    /* flat box elements per row (EW/RNG/UDF: per point) */
  uint64_t noise;       /* UDF: pre-drawn normals [rows, ..., count] (0: draw in loop) */
  int64_t noise_off;    /* UDF: element offset of (row 0, loop index 0) in `noise` */
  int64_t noise_row;    /* UDF: elements between consecutive rows in `noise` */
  int64_t noise_step;   /* UDF: elements between consecutive loop indices */
  int32_t param_bytes;  /* size of the parameter block */
  int32_t smem_off;     /* byte offset of the CTA's shared-memory copy of it */
} rt_loop_op;

typedef struct {
  rt_hdr h;
  int32_t slot;         /* env slot of the loop dim */
  int32_t nops;
  int64_t start, stop, step;
  int64_t rows;         /* slab points shared by every op */
  int32_t rows_per_cta;
  int32_t smem_bytes;   /* dynamic shared memory: [A rows | TMA ring] */
  int32_t ring_off;     /* byte offset of the weight-panel ring */
  int32_t a_off;        /* byte offset of the GEMM A-row staging area */
  uint64_t ops;         /* device pointer to rt_loop_op[nops] */
  uint64_t prof;        /* optional int64[nops]: CTA 0's clock64 cycles per op */
  int32_t blk_slot;     /* blk_len > 0: run [env[blk_slot]*blk_len, +blk_len) */
  int32_t red_off;      /*   (one time block per launch); red_off: byte      */
  int64_t blk_len;      /*   offset of the K-split GEMM reduction area         */
} rt_loop_params;

/* Launch record: one kernel family + its parameter block. */
typedef struct {
  int32_t kernel;
  int32_t param_bytes;
  uint64_t params;     /* host pointer to the parameter block */
  int32_t grid[3];
  int32_t block[3];
  int32_t smem;
  int32_t cluster;     /* > 1: thread-block cluster size along x (JIT kernels) */
  uint64_t jit_fn;     /* CUfunction specialised for this record (0: library kernel) */
} rt_launch_rec;

/* Program instructions for rt_run. */
enum rt_op {
  RT_OP_LAUNCH = 1,    /* a = launch record index                          */
  RT_OP_FOR = 2,       /* a = env slot, b = start, c = end (exclusive for  */
                       /*     step +1; for step -1 runs b down to c+1),    */
                       /*     d = step, e = pc after matching END          */
  RT_OP_END = 3,       /* a = pc of matching FOR                           */
  RT_OP_EVENT = 4,     /* a = event slot: record on the stream             */
  RT_OP_COPY = 5,      /* device copy: a = rec idx of an rt_copy record    */
  RT_OP_HOOK = 6,      /* host hook a (e.g. an NCCL all-reduce of a slab,   */
                       /* a swap copy): rt_run_segment returns RT_HOOK      */
                       /* with the next pc                                  */
  RT_OP_ENVMOD = 7,    /* env[a] = env[b] mod c (ring slot of a time block) */
  RT_OP_COLL = 8,      /* in-program collective a (rt_set_collectives): sum
                          all-reduce of its slab on the program's stream;
                          captured into CUDA graphs like a launch */
  RT_OP_ENVADD = 9     /* env[a] += b (a skewed schedule's lag around the
                          lagged nodes of a band, planner.skew_steps)      */
};

/* A sum all-reduce of a slab of one buffer (a gradient summed over the
 * env-sharded dim): element offset off0 + sum_e env[e] *
 * off_env[e] from ptr, count elements.  flush = 0: joins a bucket that the
 * next flushing collective reduces as one NCCL group. */
typedef struct {
  uint64_t ptr;
  int64_t off0;
  int64_t off_env[RT_MAXENV];
  int64_t count;
  int32_t dtype;
  int32_t flush;
} rt_coll;

#define RT_HOOK 100

typedef struct {
  int32_t op;
  int32_t a;
  int64_t b, c, d;
  int32_t e;
  int32_t _pad;
} rt_instr;

/* ---- entry points ------------------------------------------------------ */
#ifndef __CUDACC_RTC__

int rt_version(void);
/* Launch one kernel family with `rec`, patching env[0..nenv) into its header. */
int rt_launch(const rt_launch_rec* rec, const int64_t* env, int32_t nenv, uint64_t stream);
/* Run a lowered program (loops + launches) on `stream`.  events: optional
 * cudaEvent_t handles for RT_OP_EVENT. */
int rt_run(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs, int32_t nrec,
           int64_t* env, int32_t nenv, uint64_t stream, const uint64_t* events, int32_t nevents);
/* Run from *pc_io until the end (returns 0) or until a RT_OP_HOOK (returns
 * RT_HOOK with *pc_io = pc after the hook and *hook_out = its id). */
int rt_run_segment(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs, int32_t nrec,
                   int64_t* env, int32_t nenv, uint64_t stream, int32_t* pc_io, int32_t* hook_out);
/* Capture a program into a CUDA graph (loops unrolled, env folded per
 * launch) and replay it; the graph-exec handle is returned in *out. */
int rt_graph_capture(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs, int32_t nrec,
                     int64_t* env, int32_t nenv, uint64_t stream, uint64_t* out);
int rt_graph_capture_ev(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs,
                        int32_t nrec, int64_t* env, int32_t nenv, uint64_t stream,
                        const uint64_t* events, int32_t nevents, uint64_t* out);
int rt_graph_launch(uint64_t graph_exec, uint64_t stream);
int rt_graph_destroy(uint64_t graph_exec);
/* Run a program with an event pair around every launch instance; per launch
 * record: total device ms and instance count.  Synchronises the stream. */
int rt_profile(const rt_instr* prog, int32_t nprog, const rt_launch_rec* recs, int32_t nrec,
               int64_t* env, int32_t nenv, uint64_t stream, double* rec_ms, int64_t* rec_count);
/* Compile CUDA source with NVRTC for sm_100a and load kernel `name`; the
 * CUfunction handle is returned in *fn_out (module kept for the process).
 * opts: NUL-separated option strings (count nopt).  On failure the NVRTC log
 * is available from rt_last_error(). */
int rt_jit_compile(const char* src, const char* name, const char* opts, int32_t nopt,
                   uint64_t* fn_out);
/* Load a previously compiled cubin image and fetch kernel `name`. */
int rt_jit_load(const void* image, const char* name, uint64_t* fn_out);
/* Compile to a cubin image (for an on-disk cache); *size in/out. */
int rt_jit_cubin(const char* src, const char* opts, int32_t nopt, void* out, uint64_t* size);
/* Device status word: int32[4] = {code, node, aux0, aux1}; allocate/clear/read. */
int rt_status_alloc(uint64_t* dev_ptr);
int rt_status_read(uint64_t dev_ptr, int32_t* host4, uint64_t stream);
int rt_status_clear(uint64_t dev_ptr, uint64_t stream);
int rt_status_free(uint64_t dev_ptr);
/* Pinned-host tier moves (offload / fetch) on a side stream with an event. */
int rt_memcpy_d2h_async(void* host_pinned, uint64_t dev, uint64_t bytes, uint64_t stream);
/* Strided tier moves (offload / fetch of one time block of a swap-managed
 * buffer: `height` rows of `width` bytes; polysched.py:936-1105 offload/fetch
 * realised as cudaMemcpy2DAsync on the copy stream). */
int rt_memcpy2d_d2h_async(void* host_pinned, uint64_t hpitch, uint64_t dev, uint64_t dpitch,
                          uint64_t width, uint64_t height, uint64_t stream);
int rt_memcpy2d_h2d_async(uint64_t dev, uint64_t dpitch, const void* host_pinned,
                          uint64_t hpitch, uint64_t width, uint64_t height, uint64_t stream);
int rt_memcpy_h2d_async(uint64_t dev, const void* host_pinned, uint64_t bytes, uint64_t stream);
/* Standalone bit-exact RNG fill (numpy default_rng((words..., *coords)) per
 * row): rows x count values of dist into dev (f64).  For tests/tools. */
int rt_rng_fill(uint64_t dev_out, const uint32_t* prefix, int32_t nprefix,
                const int64_t* coords, int32_t ncoord, int64_t rows, int32_t count,
                int32_t dist, uint64_t stream);
const char* rt_last_error(void);
/* ---- Backend + MemorySim ----------
 * A stream-ordered device pool with the MemorySim's accounting:
 * stats8 = {capacity, live, peak, host_live, host_peak, offloads, fetches,
 * bytes_moved}; capacity 0 = unbounded; rt_pool_alloc past capacity fails
 * with RT_ERR_OVERFLOW. */
int rt_pool_create(int32_t device, uint64_t capacity, uint64_t* pool_out);
int rt_pool_destroy(uint64_t pool);
int rt_pool_alloc(uint64_t pool, uint64_t bytes, uint64_t stream, uint64_t* dev_out);
int rt_pool_free(uint64_t pool, uint64_t dev, uint64_t stream);
int rt_pool_host(uint64_t pool, int64_t delta_bytes);    /* host tier live += delta */
int rt_pool_stats(uint64_t pool, uint64_t* stats8);
/* move-between-tiers: `height` rows of `width` bytes (height 1: one span) on
 * `stream` after `after_event` (0: none), recording `done_event` (0: none);
 * events are caller-owned cudaEvent_t handles. */
int rt_offload(uint64_t pool, void* host_pinned, uint64_t hpitch, uint64_t dev, uint64_t dpitch,
               uint64_t width, uint64_t height, uint64_t stream, uint64_t after_event,
               uint64_t done_event);
int rt_fetch(uint64_t pool, uint64_t dev, uint64_t dpitch, const void* host_pinned, uint64_t hpitch,
             uint64_t width, uint64_t height, uint64_t stream, uint64_t after_event,
             uint64_t done_event);
/* dynamic-update: block[slot * elem_bytes ..] = src[0 .. elem_bytes) */
int rt_block_update(uint64_t block, int64_t slot, uint64_t src, uint64_t elem_bytes,
                    uint64_t stream);
/* stack: dst[i * elem_bytes ..] = srcs[i][0 .. elem_bytes), i < n */
int rt_stack(uint64_t dst, const uint64_t* srcs, int32_t n, uint64_t elem_bytes, uint64_t stream);
int rt_set_error(int code, const char* what);
/* ---- NCCL (in-program collectives, csrc/coll.cu) -----------------------
 * The library's own communicator (NCCL resolved with dlopen): rank 0 makes
 * a unique id, every rank joins with it; rt_set_collectives registers the
 * RT_OP_COLL table of the program about to run (per calling thread). */
int rt_nccl_unique_id(unsigned char* out128);
int rt_nccl_comm_init(int32_t nranks, int32_t rank, const unsigned char* id128, uint64_t* comm_out);
int rt_nccl_comm_destroy(uint64_t comm);
int rt_nccl_allreduce(uint64_t comm, uint64_t ptr, uint64_t count, int32_t dtype, uint64_t stream);
int rt_set_collectives(uint64_t comm, const rt_coll* colls, int32_t ncoll);
int rt_coll_exec(int32_t idx, const int64_t* env, int32_t nenv, uint64_t stream);
#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif
#endif /* RTB200_H */
