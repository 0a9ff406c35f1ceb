/*
 * tess.h -- C-ABI of the B200-native Tesseract (2.5-D tensor parallel) path.
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (tesseract-sim, /root/reference/proj/include/tsim). Each entry point names
 * the reference interface it replaces as `ref: file:line`. All functions are
 * extern "C", exception-free and return a tess_status mirroring the
 * reference's exception taxonomy (error.hpp:11-48); the message of the last
 * failure on the calling thread is available from tess_last_error().
 *
 * Ownership: callers own every buffer they pass. A tess_ctx owns its
 * communicators, events and device workspace (SUMMA panels, partial sums,
 * layer caches). One tess_ctx per rank; a ctx is used by one host thread at
 * a time (ref: runtime.hpp:91-94, RankCtx is per-thread). Per-rank calls are
 * asynchronous on the given CUDA stream (cudaStream_t passed as void*; NULL
 * means the legacy default stream).
 *
 * Dtypes: TESS_F32 computes in fp32 on CUDA cores (the fp32 parity mode,
 * rel. error <= 1e-5 vs the fp64 reference); TESS_BF16 stores activations and
 * weights in bf16 and runs every contraction on tcgen05 tensor cores with fp32
 * accumulation (weight gradients, LayerNorm statistics, softmax and all
 * reductions are fp32).
 */
#ifndef TESS_H_
#define TESS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TESS_OK = 0,
  TESS_ERR_SHAPE = 1,          /* ref: error.hpp:16 ShapeError */
  TESS_ERR_DIVISIBILITY = 2,   /* ref: error.hpp:22 DivisibilityError */
  TESS_ERR_GRID = 3,           /* ref: error.hpp:28 GridError */
  TESS_ERR_SPMD = 4,           /* ref: error.hpp:34 SpmdError (rank failure, mismatched
                                  collective, deadlock, NCCL error) */
  TESS_ERR_IO = 5,             /* ref: error.hpp:39 IoError */
  TESS_ERR_CONFIG = 6,         /* ref: error.hpp:44 ConfigError */
  TESS_ERR_CUDA = 7,           /* CUDA runtime / launch failure */
  TESS_ERR_UNSUPPORTED = 8,    /* layout the sm_100a kernels cannot address */
  TESS_ERR_INVALID = 9         /* null handle / bad enum */
} tess_status;

typedef enum { TESS_F32 = 0, TESS_BF16 = 1, TESS_F64 = 2 } tess_dtype;

/* ref: grid.hpp:30 GroupKind {Row, Column, Depth} */
typedef enum { TESS_ROW = 0, TESS_COL = 1, TESS_DEPTH = 2 } tess_group;

/* ref: algorithms.hpp:15 MatmulVariant {NN, NT, TN} */
typedef enum { TESS_NN = 0, TESS_NT = 1, TESS_TN = 2 } tess_variant;

/* ref: shard.hpp:27 Scheme (the two Tesseract layouts) */
typedef enum { TESS_SCHEME_A = 0, TESS_SCHEME_B = 1 } tess_scheme;

/* ref: layers.hpp:187 LayerOp */
typedef enum {
  TESS_OP_FEEDFORWARD = 0,
  TESS_OP_ATTENTION = 1,
  TESS_OP_LAYERNORM = 2,
  TESS_OP_BIAS_ADD = 3,
  TESS_OP_BLOCK = 4
} tess_layer_op;

/* ref: runtime.hpp:20 CollectiveKind (meter index) */
typedef enum {
  TESS_KIND_BROADCAST = 0,
  TESS_KIND_REDUCE = 1,
  TESS_KIND_ALL_REDUCE = 2,
  TESS_KIND_SHIFT = 3,
  TESS_KIND_P2P = 4
} tess_kind;

/* tess_matmul flags */
#define TESS_ACCUMULATE 0x1u      /* C += result (fp32 C) instead of C = result */
#define TESS_SUM_OVER_DEPTH 0x2u  /* TN: all-reduce the layer partial over depth
                                     (ref: algorithms.cpp:72-74) */

typedef struct tess_ctx tess_ctx;

/* Transformer geometry, ref: layers.hpp:22-27 LayerDims */
typedef struct {
  int batch, seq, hidden, heads;
} tess_layer_dims;

/* Per-rank parameter shard, ref: layers.hpp:70-75 BlockShard. Device
 * pointers. Weights are TesseractB blocks in the compute dtype:
 * w_qkv [h/q, 3h/q] (per-head interleaved Q|K|V columns, layers.hpp:38-41),
 * w_proj [h/q, h/q], w_ff1 [h/q, 4h/q], w_ff2 [4h/q, h/q]. LayerNorm
 * vectors are the j-slice [h/q] in fp32. */
typedef struct {
  const void* w_qkv;
  const void* w_proj;
  const void* w_ff1;
  const void* w_ff2;
  const float* ln1_gain;
  const float* ln1_bias;
  const float* ln2_gain;
  const float* ln2_bias;
  double eps;
} tess_block_shard;

/* Per-rank gradient shard (fp32 device buffers, same shapes as the shard),
 * ref: layers.hpp:79-82 BlockShardGrads. Any pointer may be NULL. */
typedef struct {
  float* w_qkv;
  float* w_proj;
  float* w_ff1;
  float* w_ff2;
  float* ln1_gain;
  float* ln1_bias;
  float* ln2_gain;
  float* ln2_bias;
} tess_block_grads;

/* Flat communication meter, ref: runtime.hpp:24-69 CommStats (counted in
 * matrix elements, flat per-message counting) for ONE rank. by_kind holds
 * [messages, elements] charged on this rank's send side per tess_kind. */
typedef struct {
  uint64_t sent_messages, sent_elements, received_messages, received_elements;
  uint64_t by_kind[5][2];
} tess_comm_stats;

/* ------------------------------------------------------------------ grid
 * ref: grid.hpp:47-85 GridSpec; pure host functions. */
const char* tess_last_error(void);
const char* tess_version(void);
tess_status tess_grid_check(int q, int d, int allow_d_gt_q);           /* ref: grid.cpp:26-37 */
tess_status tess_grid_parse(const char* text, int allow_d_gt_q, int* q,
                            int* d);                                   /* ref: grid.cpp:133-169 */
tess_status tess_grid_rank_of(int q, int d, int i, int j, int k, int* rank); /* ref: grid.cpp:43-49 */
tess_status tess_grid_coord_of(int q, int d, int rank, int* i, int* j,
                               int* k);                                /* ref: grid.cpp:51-61 */
tess_status tess_grid_block_row(int q, int d, int i, int j, int k, int* h); /* ref: grid.cpp:63-69 */
tess_status tess_grid_group(int q, int d, int i, int j, int k, tess_group g,
                            int* group_index, int* slot, int* group_size); /* ref: grid.cpp:71-104 */
tess_status tess_grid_member_at(int q, int d, tess_group g, int group_index,
                                int slot, int* i, int* j, int* k);     /* ref: grid.cpp:106-131 */

/* ------------------------------------------------------- contexts / comms
 * ref: runtime.hpp:95-136 RankCtx, runtime.hpp:179-191 run_spmd. */

/* NCCL backend, one process per GPU: world communicator from a shared
 * ncclUniqueId (128 bytes, made by rank 0 with tess_nccl_unique_id and
 * distributed by the launcher), then ncclCommSplit into the row
 * (color k*q+i, key j), column (color k*q+j, key i) and depth
 * (color i*q+j, key k) communicators (ref: grid.cpp:79-95). */
tess_status tess_nccl_unique_id(void* out128);
tess_status tess_init_nccl(int q, int d, int allow_d_gt_q, int rank, int device,
                           const void* unique_id128, tess_ctx** out);

/* In-process backend: creates p = d*q*q contexts (one per rank, rank r on
 * devices[r], or all on the current device when devices is NULL). Each
 * context must be driven by its own host thread (as the reference's
 * SpmdRunner does); collectives rendezvous on the host and move data with
 * stream-ordered device copies / peer reads, summing in slot-ascending order
 * like the reference engine (ref: runtime.cpp:221-372). */
tess_status tess_init_local(int q, int d, int allow_d_gt_q, const int* devices,
                            tess_ctx** out_per_rank);
tess_status tess_destroy(tess_ctx* ctx);
tess_status tess_coord(const tess_ctx* ctx, int* rank, int* i, int* j, int* k);
tess_status tess_group_comm(tess_ctx* ctx, tess_group g, void** nccl_comm);
tess_status tess_get_comm_stats(const tess_ctx* ctx, tess_comm_stats* out);
tess_status tess_reset_comm_stats(tess_ctx* ctx);
/* Enables the reference trace format "<rank>:<step> <kind> <group> <root>
 * <bytes>" (ref: runtime.hpp:71-85, runtime.cpp:90-96); bytes are counted
 * as elements * 8 like the reference. */
tess_status tess_set_trace(tess_ctx* ctx, int enable);
tess_status tess_trace_text(const tess_ctx* ctx, char* buf, size_t cap, size_t* needed);

/* ------------------------------------------------------------ collectives
 * ref: runtime.hpp:105-121. Device buffers; fp32 sums. */
tess_status tess_broadcast(tess_ctx* ctx, tess_group g, int root_slot, void* buf,
                           size_t bytes, size_t elements, void* stream);
tess_status tess_reduce(tess_ctx* ctx, tess_group g, int root_slot, const float* send,
                        float* recv, size_t n, void* stream);
tess_status tess_all_reduce(tess_ctx* ctx, tess_group g, float* buf, size_t n, void* stream);
tess_status tess_barrier(tess_ctx* ctx);

/* ------------------------------------------------------------- partition
 * ref: shard.cpp:68-98 (partition) and 139-183 (combine). `global` is a
 * device (or host) row-major [rows, cols] matrix of dtype; `local` the
 * rank's device block. Bit-exact copies. */
tess_status tess_partition(tess_ctx* ctx, tess_scheme scheme, tess_dtype dtype,
                           const void* global, int64_t rows, int64_t cols, void* local,
                           void* stream);
tess_status tess_unpartition(tess_ctx* ctx, tess_scheme scheme, tess_dtype dtype,
                             const void* local, int64_t rows, int64_t cols, void* global,
                             void* stream);

/* --------------------------------------------------------------- products
 * ref: algorithms.hpp:91-96 nn/nt/tn_product_rank. Local block shapes:
 *   NN: a [ar, ak] (TesseractA), b [ak, bn] (TesseractB) -> c [ar, bn]
 *   NT: a [ar, an] (TesseractA), b [br, an] (TesseractB) -> c [ar, br]
 *   TN: a [ar, an] (TesseractA), b [ar, bn] (TesseractA) -> c [an, bn]
 *       (+ depth all-reduce with TESS_SUM_OVER_DEPTH)
 * `in` is the dtype of a and b; c_type F32 or the input dtype. */
tess_status tess_matmul(tess_ctx* ctx, tess_variant v, tess_dtype in, const void* a,
                        int64_t a_rows, int64_t a_cols, const void* b, int64_t b_rows,
                        int64_t b_cols, void* c, tess_dtype c_type, uint32_t flags,
                        void* stream);

/* Fused epilogue of a local product (north_star: bias / GeLU / dropout-scale
 * in the tcgen05 GEMM epilogue; the reference's blocks have no linear biases
 * and no dropout, layers.hpp:42-49, so this extends the path rather than
 * replacing a reference call). Order per output element:
 *   v = AB (+ bias[col]) ; GeLU: pre_activation = v, v = gelu(v) ;
 *   dropout: v = keep ? v / (1 - p) : 0 ; v += residual ; store (or += with
 *   TESS_ACCUMULATE).
 * keep = a counter hash of (seed, row0 + local row, col0 + local col) -- the
 * GLOBAL coordinate of the element, so every Tesseract block drops exactly
 * what the unsharded product drops (host reference: tess_dropout_keep).
 * bias: fp32 [local columns]; residual / pre_activation: the output's type
 * and shape. bf16 inputs only. NN products on any grid (the epilogue runs on
 * the one GEMM that owns the block); NT / TN only where no reduction follows
 * (q == 1, and no depth sum). */
typedef struct {
  const float* bias;
  int gelu;
  void* pre_activation;
  float dropout_p;
  uint64_t dropout_seed;
  int64_t row0, col0;
  const void* residual;
} tess_epilogue;

tess_status tess_matmul_ex(tess_ctx* ctx, tess_variant v, tess_dtype in, const void* a,
                           int64_t a_rows, int64_t a_cols, const void* b, int64_t b_rows,
                           int64_t b_cols, void* c, tess_dtype c_type, uint32_t flags,
                           const tess_epilogue* epilogue, void* stream);
/* The dropout mask of tess_epilogue: 1 = element (row, col) kept. */
int tess_dropout_keep(uint64_t seed, int64_t row, int64_t col, float p);

/* ----------------------------------------------------------------- layers
 * ref: layers.hpp:123-161 (rank-level fwd/bwd) and layers.cpp:604-692
 * (layer_run). x, dy, y, dx are the rank's TesseractA activation blocks
 * [batch*seq/(d*q), hidden/q] in the compute dtype (device or pinned/pageable
 * host memory; host buffers are staged through the context). The forward
 * cache lives in the context until the matching backward (one outstanding
 * forward per op per context). `x` must stay valid until the backward.
 * grads may be NULL (the collective sequence is unchanged, ref:
 * layers.cpp:372-377); with accumulate=0 gradients are overwritten, else
 * added (ref: layers.cpp:368-371 add()). dbias (BiasAdd) is fp32 [hidden/q],
 * valid on i == 0 ranks (ref: layers.cpp:507-517).
 * Host outputs (y, dx in host memory) leave on the context's copy stream so
 * they overlap the caller's next work; order a stream after them with
 * tess_stream_join before reading them (the global operators do). Pinned
 * host inputs are read asynchronously (cudaMemcpyAsync semantics): keep
 * them unchanged until the call's work has completed (tess_stream_join +
 * a stream synchronize); pageable ones are consumed before the call returns. */
tess_status tess_layer_forward(tess_ctx* ctx, tess_layer_op op, tess_dtype dtype,
                               const tess_layer_dims* dims, const tess_block_shard* shard,
                               const void* bias_row0, const void* x, void* y, void* stream);
tess_status tess_layer_backward(tess_ctx* ctx, tess_layer_op op, tess_dtype dtype,
                                const tess_layer_dims* dims, const tess_block_shard* shard,
                                const void* dy, void* dx, tess_block_grads* grads,
                                int accumulate, float* dbias, void* stream);

/* Forward + backward of one layer op in one call, both inputs given up front
 * (the reference's layer_run(op, x, dy, ...) at rank level, layers.cpp:
 * 604-692): identical results to tess_layer_forward + tess_layer_backward;
 * host x and dy go up on a context upload stream into staging buffers
 * double-buffered per call, each copy waiting only for its buffer's reader
 * two calls back: consecutive steps' copies overlap the previous step's
 * compute; x gates the forward, dy only the backward. */
tess_status tess_layer_step(tess_ctx* ctx, tess_layer_op op, tess_dtype dtype,
                            const tess_layer_dims* dims, const tess_block_shard* shard,
                            const void* bias_row0, const void* x, const void* dy, void* y,
                            void* dx, tess_block_grads* grads, int accumulate, float* dbias,
                            void* stream);

/* A stack of `layers` Transformer blocks, forward through every block then
 * backward in reverse, on this rank (the inner loops of the reference's
 * train_toy, layers.cpp:1006-1026, without its loss and update; BASELINE
 * config 5's 24-layer stack). shards / grads: one per layer (grads may be
 * NULL). Block l uses forward-cache slot base + l, base = the slot selected
 * by tess_set_cache_slot; activations between blocks stay on the device.
 * With tess_set_megatron the 1-D scheme's block runs. x / dy / y / dx as in
 * tess_layer_step (device or host). */
tess_status tess_stack_step(tess_ctx* ctx, tess_dtype dtype, const tess_layer_dims* dims,
                            int layers, const tess_block_shard* shards, const void* x,
                            const void* dy, void* y, void* dx, tess_block_grads* grads,
                            int accumulate, void* stream);

/* Makes `stream` wait for everything the context still has in flight on its
 * side streams: pending host copies of layer outputs and deferred
 * collectives (the reference's calls return completed values; this is the
 * completion point of the asynchronous C-ABI). */
tess_status tess_stream_join(tess_ctx* ctx, void* stream);

/* Selects the forward-cache slot used by subsequent tess_layer_forward /
 * tess_layer_backward calls on this context, so a stack of layers can keep
 * one outstanding forward each (the reference keeps caller-owned
 * BlockCacheRank objects, layers.hpp:114-119). Default 0. */
tess_status tess_set_cache_slot(tess_ctx* ctx, int slot);

/* Fault injection (the reference's verify inject_fault, verify.cpp:84-86,
 * carried into the runtime so its failure semantics can be tested):
 *   TESS_FAULT_PERTURB          global tesseract_matmul only: the combined
 *                               result's element (0,0) += 1e-3 (exactly the
 *                               reference's injected fault)
 *   TESS_FAULT_RANK_FAIL        the rank raises at its collective number `at`
 *                               (every partner aborts; the call fails with
 *                               TESS_ERR_SPMD naming the coordinate)
 *   TESS_FAULT_SKIP_COLLECTIVE  the rank silently skips collective `at`
 *                               (its partners block; the in-process backend
 *                               reports the deadlock naming every divergent
 *                               rank and what it waits on, runtime.cpp:433-471)
 * One-shot. tess_set_global_fault arms the next global call of this host
 * thread (rank `rank` of its grid; ignored by PERTURB). */
typedef enum {
  TESS_FAULT_NONE = 0,
  TESS_FAULT_PERTURB = 1,
  TESS_FAULT_RANK_FAIL = 2,
  TESS_FAULT_SKIP_COLLECTIVE = 3
} tess_fault;
tess_status tess_inject_fault(tess_ctx* ctx, tess_fault kind, int64_t at_collective);
tess_status tess_set_global_fault(tess_fault kind, int rank, int64_t at_collective);

/* Measurement switch (no reference counterpart): with enable != 0 every
 * collective of this context is metered and traced as usual but moves no
 * data, so a step timed this way is the step without communication; the
 * exposed-communication share of the step is (t - t_noop) / t.
 * Results computed while it is on are meaningless. */
tess_status tess_set_comm_noop(tess_ctx* ctx, int enable);

/* 1-D tensor-parallel (Megatron) layer scheme for this rank (BASELINE config
 * 5's comparator; the reference ships only its two-linear kernel,
 * algorithms.cpp:244-265). Needs a [1,1,p] line grid (q == 1): x, dy, y, dx
 * are the full [batch*seq, hidden] activations on every rank; the shard
 * holds W_qkv / W_ff1 column blocks k (heads [k n/p, (k+1) n/p)), W_proj /
 * W_ff2 row blocks k, and the full LayerNorm vectors; the proj / FF2 outputs
 * and the QKV / FF1 dgrads are all-reduced over the depth group, weight
 * gradients stay per shard. Applies to the layer calls that follow. */
tess_status tess_set_megatron(tess_ctx* ctx, int enable);

/* ---------------------------------------------------------- global level
 * Whole-matrix operators with host fp64 buffers, mirroring the reference's
 * value-semantics API: partition -> per-rank SPMD (one host thread per rank,
 * in-process backend) -> combine. `compute` selects TESS_F32 or TESS_BF16
 * (inputs are rounded once to it). devices: p device ordinals or NULL (all
 * ranks on the current device). stats_rank: p x 4 counters [sent msgs,
 * sent elems, recv msgs, recv elems] and stats_kind: 5 x 2, both optional,
 * with the reference's CommStats semantics. */
tess_status tess_tesseract_matmul(int q, int d, int allow_d_gt_q, tess_variant v,
                                  tess_dtype compute, const double* a, int64_t a_rows,
                                  int64_t a_cols, const double* b, int64_t b_rows,
                                  int64_t b_cols, double* c, const int* devices,
                                  uint64_t* stats_rank, uint64_t* stats_kind);
/* ref: algorithms.hpp:54-57 */
tess_status tess_tesseract_backward(int q, int d, int allow_d_gt_q, tess_dtype compute,
                                    const double* dc, const double* a, const double* b,
                                    int64_t m, int64_t k, int64_t n, double* da,
                                    double* db, const int* devices, uint64_t* stats_rank,
                                    uint64_t* stats_kind);
/* ref: algorithms.hpp:78-80 tesseract_backward_dense */

/* The last global call made by the calling host thread (tesseract_matmul,
 * tesseract_backward, layer_run, megatron_layer_run, train_toy): per-rank,
 * per-kind send counters sent_by_kind [p][5][2] (messages, elements per
 * CollectiveKind Broadcast, Reduce, AllReduce, Shift, PointToPoint) and
 * per-rank receive counters recv [p][2]; *ranks = p. These rebuild the
 * reference's CommStats exactly: add_send(r, kind, m, e) per (r, kind) and
 * add_recv(r, any kind, m, e) per r (runtime.hpp:56-59; receives carry no
 * kind, runtime.cpp:59-64). cap_ranks: rank capacity of the buffers. */
tess_status tess_global_last_stats(int* ranks, uint64_t* sent_by_kind, uint64_t* recv,
                                   size_t cap_ranks);
/* Record collective traces in the global calls of this host thread (the
 * reference's TesseractOptions::record_trace, algorithms.hpp:24-30), and read
 * the last call's trace: write_trace() text, ranks in order (runtime.cpp:90-96,
 * 149-156). */
tess_status tess_set_global_trace(int enable);
tess_status tess_global_last_trace(char* buf, size_t cap, size_t* needed);
tess_status tess_layer_run(tess_layer_op op, const tess_layer_dims* dims, int q, int d,
                           int allow_d_gt_q, tess_dtype compute, const double* x,
                           const double* dy, const double* const* params, double eps,
                           double* y, double* dx, double* const* grads, double* dbias,
                           const int* devices, uint64_t* stats_rank,
                           uint64_t* stats_kind);
/* ref: layers.hpp:195-197 layer_run; params/grads: 8 host fp64 arrays in
 * BlockParams order (w_qkv, w_proj, w_ff1, w_ff2, ln1_gain, ln1_bias,
 * ln2_gain, ln2_bias); grads may be NULL; dbias [hidden] for BiasAdd. */

/* Config 5's comparison schemes for tess_stack_run. */
typedef enum { TESS_STACK_TESSERACT = 0, TESS_STACK_MEGATRON = 1 } tess_stack_scheme;

/* Global-level layer stack: `layers` blocks forward then backward (see
 * tess_stack_step) on host fp64 buffers. TESS_STACK_TESSERACT runs the
 * [q,q,d] grid (SUMMA is d = 1, ref algorithms.cpp:105-118);
 * TESS_STACK_MEGATRON the 1-D scheme on a [1,1,d] line (q must be 1; the
 * megatron_1d_linear split of algorithms.cpp:244-265 applied to every
 * block). params / grads: layers*8 arrays in BlockParams order per layer
 * (grads or any entry may be NULL); y, dx [batch*seq, hidden]; grads are
 * overwritten. Same math as chaining ref transformer_block forward and
 * backward (layers.cpp:460-487) through the stack. */
tess_status tess_stack_run(tess_stack_scheme scheme, const tess_layer_dims* dims, int layers,
                           int q, int d, int allow_d_gt_q, tess_dtype compute, const double* x,
                           const double* dy, const double* const* params, double eps,
                           double* y, double* dx, double* const* grads, const int* devices,
                           uint64_t* stats_rank, uint64_t* stats_kind);

/* ref: layers.hpp:245-267 train_toy (the sharded half): `layers` Transformer
 * blocks trained with MSE loss against `target` and plain SGD (learning rate
 * lr) for `steps` steps on the [q,q,d] grid; the loss of every step (before
 * its update) is written to losses[steps]. params: layers*8 host fp64 arrays
 * (BlockParams order per layer). */
tess_status tess_train_toy(const tess_layer_dims* dims, int layers, int steps, double lr, int q,
                           int d, int allow_d_gt_q, tess_dtype compute, const double* x,
                           const double* target, const double* const* params, double eps,
                           double* losses, const int* devices, uint64_t* stats_rank,
                           uint64_t* stats_kind);

/* ref: algorithms.hpp:82-85 megatron_1d_linear -- the 1-D tensor-parallel
 * comparator (config 5): on a [1,1,p] line grid W1 [xc, w1c] is column-split,
 * W2 [w1c, w2c] row-split, every rank computes X W1_k W2_k and one all-reduce
 * sums the partials; out [xr, w2c] (fp32 result before any cast). */
tess_status tess_megatron_1d_linear(int p, tess_dtype compute, const double* x, int64_t xr,
                                    int64_t xc, const double* w1, int64_t w1r, int64_t w1c,
                                    const double* w2, int64_t w2r, int64_t w2c, double* out,
                                    const int* devices, uint64_t* stats_rank,
                                    uint64_t* stats_kind);

/* Global-level 1-D (Megatron) counterpart of tess_layer_run on p ranks (see
 * tess_set_megatron): same argument meaning, outputs combined from the
 * shards (column / row blocks of the weight gradients, the replicated y, dx
 * and LayerNorm gradients from rank 0). bias_add is not supported. */
tess_status tess_megatron_layer_run(tess_layer_op op, const tess_layer_dims* dims, int p,
                                    tess_dtype compute, const double* x, const double* dy,
                                    const double* const* params, double eps, double* y,
                                    double* dx, double* const* grads, const int* devices,
                                    uint64_t* stats_rank, uint64_t* stats_kind);

/* ref: matrix.cpp:352-370 checksum (FNV-1a over rows, cols and the
 * little-endian doubles; printed by the reference as "fnv1a:%x"). */
uint64_t tess_checksum(int64_t rows, int64_t cols, const double* values);
/* ref: matrix.cpp:244-350 save_matrix / load_matrix: ".csv" paths are CSV
 * (shortest round-trip text), anything else is the "TMX1" binary format.
 * tess_load_matrix with values == NULL returns only the shape. */
tess_status tess_save_matrix(const char* path, int64_t rows, int64_t cols, const double* values);
tess_status tess_load_matrix(const char* path, int64_t* rows, int64_t* cols, double* values);

/* Number of kernels launched by this library on the calling process since
 * load (for the bench's gpu_launches claim). */
uint64_t tess_kernel_launches(void);

/* GEMM launch profiling: when enabled, every local GEMM launch is bracketed
 * by CUDA events on its own stream; tess_profile_read synchronises them and
 * returns the summed device time (ms), algorithmic flops (2*M*N*K per
 * launch) and launch count since the last tess_profile_enable.
 * on: 0 off, 1 keyed per kernel instantiation, 2 keyed per instantiation
 * plus shape and epilogue ("... M= N= K= b= epi=<Epi>"). */
tess_status tess_profile_enable(int on);
tess_status tess_profile_read(double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches);
/* Per kernel instantiation since tess_profile_enable, as JSON text
 * {"<kernel>": [device_ms, algorithmic_flops, launches], ...}. */
tess_status tess_profile_json(char* buf, size_t cap, size_t* needed);

/* Debug: copies the last attention phase trace (clock64 stamps of CTA 0,
 * recorded with TESS_ATTN_TRACE set) into out (up to 512 values);
 * TESS_ERR_INVALID when none was recorded. Only the tool-only kernel
 * experiments (csrc/tools/attn_bwd_experiments.cuh) record one; the shipped
 * kernels carry no trace code. No reference counterpart. */
tess_status tess_debug_attn_trace(long long* out, int n);

/* Test hook of the peer-window transport behind the fused pair reduce of the
 * NCCL backend (CUDA IPC window + system-scope release/acquire sequence
 * words): two processes (rank 0 and 1, same or different GPUs) swap IPC
 * handles through files in `dir` and run `iters` acquire/fill/open/check/
 * close rounds of n floats (2n after half-way: the window grows). *bad =
 * elements that did not match the partner's pattern. Replaces nothing in the
 * reference (its reduce is runtime.cpp:485-513). */
tess_status tess_debug_peer_window(int rank, const char* dir, size_t n, int iters,
                                   unsigned long long* bad);

/* Test hooks of the SM-free SUMMA panel transport (csrc/summa.cpp,
 * csrc/peer.h PanelLink): the GEMM may be launched before a panel lands and
 * waits on the device per row chunk for a flag written with a stream memory
 * operation after the chunk's copy-engine transfer.
 * tess_debug_gemm_ready: one process; a two-segment NN GEMM [M,2K]x[2K,N]
 * is launched, then (delay_ms later) its second A panel arrives from pinned
 * host memory in `chunks` chunks; *bad = outputs differing (bitwise) from
 * the same GEMM over resident panels; *ms_wait = device time of the flagged
 * GEMM. tess_debug_panel_link: two processes (rank 0 root, rank 1 receiver,
 * handles swapped through files in `dir`), `iters` pushes of a [M,K] panel
 * (2M after half-way), each consumed by a GEMM the receiver launched before
 * the root started the push; *bad as above. Replace nothing in the
 * reference (its broadcasts are runtime.cpp:485-513). */
tess_status tess_debug_gemm_ready(int64_t M, int64_t K, int64_t N, int chunks, int delay_ms,
                                  unsigned long long* bad, float* ms_wait);
tess_status tess_debug_panel_link(int rank, const char* dir, int64_t M, int64_t K, int64_t N,
                                  int iters, int chunks, int delay_ms, unsigned long long* bad);

#ifdef __cplusplus
}
#endif

#endif /* TESS_H_ */
