/*
 * rcv.h — C ABI of librcv.so, the B200 (sm_100a) data plane of the ReCoVer
 * data-parallel gradient commit.
 *
 * The reference (`steadybatch`, /root/reference/pkg/src/steadybatch) is a pure
 * Python/numpy package; its "FFI" for this path is the Python module API.  Each
 * entry point below names the reference operation whose data movement it
 * replaces (file:line under pkg/src/steadybatch/).  The control plane
 * (membership, epoch, roles, quotas) stays in the host mirror of that API
 * (paper_2605_11215_b200/{comm,buckets,policy,trainer}.py), which calls these
 * functions through ctypes.
 *
 * Conventions
 *   - every function returns 0 on success, a negative RCV_E* code otherwise;
 *     rcv_last_error() returns a thread-local message for the last failure.
 *   - all buffers are caller-owned device pointers (UVA: a pointer may live on
 *     a peer GPU when peer access is enabled, see rcv_enable_peer_access).
 *   - every call is stream-ordered on the caller's cudaStream_t (`stream`,
 *     passed as void*); nothing synchronises the host.
 *   - dtypes: RCV_F32, RCV_F64 (accumulator / output types) and RCV_BF16
 *     (input-only: bf16 gradients accumulated in fp32).
 *   - floating-point folds are evaluated in the exact association order the
 *     function documents; no reassociation, no FMA contraction, the final
 *     scale is an IEEE true division (x / divisor), matching numpy.
 */
#ifndef RCV_H_
#define RCV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCV_F32 0
#define RCV_F64 1
#define RCV_BF16 2

#define RCV_OK 0
#define RCV_EINVAL (-1)
#define RCV_ECUDA (-2)
#define RCV_ERANGE (-3)

#define RCV_MAX_IN 64  /* max fold inputs (replicas / microbatch slots) */
#define RCV_MAX_OUT 64 /* max fold outputs (member views)               */

/* fold op byte (one per input, see rcv_fold): bits 0-5 = number of merges of
 * the two top stack entries after pushing this input; bit 6 = push +0.0 + v
 * instead of v (reproduces numpy's `zeros; +=`, which turns -0.0 into +0.0). */
#define RCV_OP_MERGES_MASK 0x3f
#define RCV_OP_CANON 0x40

/* kernel variant selector for rcv_fold / rcv_tree_commit */
#define RCV_VARIANT_AUTO 0
#define RCV_VARIANT_TMA 1    /* cp.async.bulk → smem ring → fold → STG.128 */
#define RCV_VARIANT_DIRECT 2 /* LDG.128 with prefetch, fold in registers  */
#define RCV_VARIANT_SCALAR 3 /* one element per thread (any alignment)    */

const char *rcv_last_error(void);
int rcv_version(void);
/* Number of kernels this library has launched in this process (the bench's
 * gpu_launches is the difference across its timed region). */
unsigned long long rcv_launch_count(void);

/* Number of CUDA devices visible (0 without a GPU; never fails on CPU). */
int rcv_device_count(int *n);

/* Enable peer access between every ordered pair of `devices` (single-process
 * multi-GPU mode).  Replaces nothing in the reference (its replicas share one
 * address space, comm.py:1-9); it is what makes views on different GPUs
 * addressable from one kernel. */
int rcv_enable_peer_access(int n_dev, const int *devices);

/* Generic ordered fold — the single data-plane primitive.
 *   For every element e in [0, numel): run the stack program
 *     for i in 0..n_in-1: push(in[i][e]) (as +0.0+v when ops[i] & CANON);
 *                         repeat (ops[i] & MERGES) times: b=pop, a=pop, push(a+b)
 *   the single remaining value v becomes v / divisor when divisor != 0, and is
 *   written to out[0..n_out-1][e].
 *   in_dtypes[i] is acc_dtype or (acc_dtype == F32 only) RCV_BF16.
 *   Outputs may alias inputs (each element is read completely before it is
 *   written).  n_in == 0 writes +0.0 (np.zeros_like, comm.py:197-198). */
int rcv_fold(int n_in, const void *const *in, const uint8_t *ops,
             const int *in_dtypes, int n_out, void *const *out, int acc_dtype,
             size_t numel, double divisor, int variant, void *stream);

/* Communicator.ulfm_allreduce data phase (comm.py:191-200): the views of the
 * `n` members in ascending replica id; bit i of contrib_mask set ⇔ member i
 * contributes (non-spare, or any member while boundary_latch, comm.py:193).
 * total = left fold over contributors in ascending order, starting from the
 * first contributor's value (comm.py:196 `vec.copy()`, so -0.0 survives);
 * every member's view (spares included) receives total (comm.py:199-200), or
 * +0.0 when nobody contributes.  divisor != 0 additionally scales (used by the
 * fused commit, trainer.py:446). In place. */
int rcv_masked_allreduce(void *const *views, int n, uint64_t contrib_mask,
                         int dtype, size_t numel, double divisor,
                         void *stream);

/* Same, with the members' views spread over several GPUs of this process
 * (peer access enabled).  Device d folds the d-th contiguous 16-byte-aligned
 * slice of the bucket, reading every contributor's slice over NVLink and
 * writing every member's slice (a fused reduce-scatter + all-gather in one
 * launch per device).  streams[d] is the stream for devices[d]; the call
 * orders all streams before and after with events. */
int rcv_masked_allreduce_multidev(void *const *views, int n,
                                  uint64_t contrib_mask, int dtype,
                                  size_t numel, double divisor, int n_dev,
                                  const int *devices, void *const *streams);

/* ReplicaState.execute_microbatch accumulation `self.flat += grad`
 * (trainer.py:212, 225): acc = acc + grad, or +0.0 + grad when `first`
 * (folds the `flat[:] = 0.0` of begin_iteration, trainer.py:192, into the
 * first push).  grad_dtype may be RCV_BF16 when acc_dtype is RCV_F32. */
int rcv_accumulate(void *acc, const void *grad, int acc_dtype, int grad_dtype,
                   size_t numel, int first, void *stream);

/* K-ACC: one push of the canonical dyadic accumulator (SURVEY §7.3 R1,
 * §8(b)), the B200 replacement of the per-microbatch `flat += grad`
 * (trainer.py:202-229).  A replica's microbatch gradients enter a
 * binary-counter stack of canonical-tree nodes; pushing microbatch m merges
 * it with the c stack entries it completes, in one pass:
 *     out = stack[0] + (stack[1] + (... + (stack[c-1] + grad)))
 * where stack[c-1] is the top (the left sibling of m's leaf) and stack[0]
 * the deepest merged node; `out` may alias stack[0] (elementwise, in place)
 * or be a fresh slot when c == 0.  The gradient arrives as it leaves
 * backward, one segment per parameter tensor (seg_ptr[i] holds seg_len[i]
 * elements of flat positions [seg_off[i], seg_off[i] + seg_len[i])), so
 * nothing is copied into a flat buffer first.  Segments must be ascending,
 * contiguous from 0, each a multiple of 4 elements and 16-byte aligned
 * (8-byte for bf16); n_seg <= 256, c <= 8.  Every add is round-to-nearest
 * fp32, so a node's value is bitwise the canonical subtree's. */
int rcv_kacc_push(const void *const *seg_ptr, const uint64_t *seg_off,
                  const uint64_t *seg_len, int n_seg, int grad_dtype,
                  const float *const *stack, int c, float *out, size_t numel,
                  void *stream);

/* Canonical-order commit (the B200 design): `blocks` are
 * partial sums of aligned dyadic microbatch-index blocks [lo, lo+2^level)
 * over a canonical binary tree of next_pow2(n_leaves) leaves, empty leaves
 * skipped (not added as zeros).  The kernel evaluates that tree in
 * post-order, divides by divisor (trainer.py:446 `flat / B`), and writes
 * every out[j].  The result is a function of the leaf values only, never of
 * which replica computed which block. */
typedef struct {
  const void *ptr;
  uint32_t lo;
  uint32_t level;
  int dtype;
} rcv_block;
int rcv_tree_commit(const rcv_block *blocks, int n_blocks, uint32_t n_leaves,
                    int n_out, void *const *out, int acc_dtype, size_t numel,
                    double divisor, int variant, void *stream);

/* rcv_tree_commit on sub-ranges: every block pointer is advanced by
 * in_offset elements (of its own dtype) and every output by out_offset
 * elements, so a caller can prebuild the pointer arrays once per plan and
 * commit bucket after bucket (or owner slice after owner slice) with two
 * integers — the per-bucket host cost is one call. */
int rcv_tree_commit_at(const rcv_block *blocks, int n_blocks,
                       uint32_t n_leaves, int n_out, void *const *out,
                       int acc_dtype, size_t in_offset, size_t out_offset,
                       size_t numel, double divisor, int variant,
                       void *stream);

/* Host-side helper: the post-order fold program for rcv_tree_commit, exposed
 * so tests can check it without a GPU.  ops_out must hold n_blocks bytes;
 * blocks are taken in ascending `lo` order (the caller sorts). Returns the
 * maximum stack depth in *max_depth. */
int rcv_tree_program(const uint32_t *lo, const uint32_t *level, int n_blocks,
                     uint32_t n_leaves, uint8_t *ops_out, int *max_depth);

/* snapshot_and_tag deep copy (buckets.py:68) and rewinds (buckets.py:136,
 * 162): device-to-device copy. */
int rcv_copy(void *dst, const void *src, size_t bytes, void *stream);

/* begin_iteration `flat[:] = 0.0` (trainer.py:192) and the spare discard
 * `b.data[:] = 0.0` (buckets.py:147-148). */
int rcv_zero(void *dst, size_t bytes, void *stream);

/* np.array_equal between replica buffers (trainer.py:441-444, 451-453):
 * adds the number of differing 32-bit words of a and b to *d_count (a device
 * uint64).  Bitwise, so -0.0 != +0.0 and NaN payloads compare by bits. */
int rcv_compare(const void *a, const void *b, size_t bytes,
                unsigned long long *d_count, void *stream);

/* The optimizer commit `params -= lr * (flat / float(b))` (trainer.py:450),
 * evaluated as three IEEE roundings in numpy's order. */
int rcv_sgd_commit(void *params, const void *flat, int dtype, size_t numel,
                   double b, double lr, void *stream);

/* Deterministic example synthesis (trainer.py:64-87), a bit-exact device port
 * of _unit_lanes:  out[l] = ((mix64(base + l*C1) >> 11) * 2^-53) * scale +
 * shift for l in [0, n), all in float64; then, when floor7 != 0, out[l] =
 * floor(out[l] * 7.0) - 3.0 (the constant stream's g0, trainer.py:152).
 * base = seed*C1 + index*C2 + salt*C3 mod 2^64 is computed by the caller. */
int rcv_unit_lanes(double *out, uint64_t base, size_t n, double scale,
                   double shift, int floor7, void *stream);

/* Toy-model gradient and loss (trainer.py:103-131) for one example:
 *   linear:   r = params.x - y ; grad = r * x ; loss = r * r
 *   constant: grad = x         ; loss = params.x
 * where x = lanes[0:dim], and for linear y = wstar.x + 0.1*lanes[dim]
 * (trainer.py:165-168).  Dot products are a fixed-order multi-block fold
 * (deterministic for a given dim). scal must hold 2 + 1024 doubles (the
 * block partials follow the two results).
 * grad (dim doubles; may be NULL to compute the loss only) and scal (two
 * doubles: scal[0] = r for linear / 1.0 for constant, scal[1] = loss) are
 * device outputs. */
int rcv_toy_grad(int kind_linear, const double *params, const double *lanes,
                 const double *wstar, size_t dim, double *grad, double *scal,
                 void *stream);

/* ---- multi-process (one process per GPU) -------------------------------
 * The reference has no processes (comm.py:1-9: collectives are atomic rounds
 * of one interpreter); these entry points are what a ProcessGroupULFM-style
 * backend binds instead: buffers shared between the rank
 * processes of one node over NVLink, and a stream-ordered flag barrier whose
 * spin is bounded, so a peer that stopped responding is reported as a status
 * bit instead of hanging the GPU (the crash-stop detection of comm.py:129). */

/* Export the allocation containing `ptr` (cudaIpcGetMemHandle); handle_out
 * receives 64 bytes, *offset_out the offset of ptr inside the allocation. */
int rcv_ipc_export(const void *ptr, void *handle_out, size_t *offset_out);

/* Map a peer's exported allocation (cached per handle) and return the device
 * pointer to base + offset in this process. */
int rcv_ipc_import(const void *handle, size_t offset, void **ptr_out);

/* cuMem VMM shareable allocation (real-kill mode): `bytes` of device memory
 * on the current GPU, mapped for every GPU that can reach it, exported as a
 * POSIX file descriptor.  Importers hold a reference to the physical memory,
 * so a peer's buffers stay valid after the peer process dies. */
int rcv_vmm_alloc(size_t bytes, void **ptr_out, size_t *size_out, int *fd_out);
/* Map a peer's exported allocation (fd already duplicated into this process,
 * e.g. with pidfd_getfd); owner_device is the GPU holding the memory. */
int rcv_vmm_import(int fd, size_t size, int owner_device, void **ptr_out);

/* ---- NVLink SHARP multicast objects (NVLS) --------------------------------
 * The all-gather half of the combine writes every owner slice into the
 * landing buffer of every live rank (ref:comm.py:199-200, "write the total to
 * every member").  Through a multicast object that is one store per vector:
 * the NVSwitch replicates it to every GPU of the team, so a rank's NVLink
 * egress for the all-gather is its slice once instead of once per peer.
 * Only stores are multicast; the reduction stays on the SMs in canonical
 * order (an in-switch reduction has no defined order).
 *
 * Setup, every rank of the team: one rank creates the object and exports it
 * (rcv_mc_create), the others import the descriptor (rcv_mc_import); every
 * rank adds its GPU (rcv_mc_add_device); after ALL ranks have added theirs,
 * each binds its landing buffer -- a VMM allocation, rcv_vmm_alloc -- at
 * offset 0 (rcv_mc_bind) and maps the object (rcv_mc_map).  Sizes and the
 * bound address are multiples of rcv_mc_granularity.  *handle is an opaque
 * CUmemGenericAllocationHandle. */
int rcv_mc_supported(int *ok);
int rcv_mc_granularity(int n_dev, size_t *gran);
int rcv_mc_create(size_t bytes, int n_dev, uint64_t *handle, size_t *size_out, int *fd_out);
int rcv_mc_import(int fd, uint64_t *handle);
int rcv_mc_add_device(uint64_t handle);
int rcv_mc_bind(uint64_t handle, void *local_ptr, size_t bytes);
int rcv_mc_map(uint64_t handle, size_t size, void **mc_ptr);
int rcv_mc_release(uint64_t handle, void *mc_ptr, size_t size);

/* Cross-GPU barrier among the ranks in live_mask: rank `me` stores `value`
 * into slot `me` of every live peer's flag array (peer_flags[r], mapped
 * pointers), then waits until its own local_flags[r] >= value for every live
 * peer r, each wait bounded by timeout_ns of %globaltimer.  A peer that times
 * out sets bit r in *status (device uint32) instead of blocking forever;
 * a peer whose bit is already set is neither signalled nor awaited again. 
 * Launched on `stream`, ordered after the caller's prior work. */
int rcv_barrier(uint64_t *local_flags, void *const *peer_flags, int n, int me,
                uint64_t live_mask, uint64_t value, uint64_t timeout_ns,
                uint32_t *status, void *stream);

/* ---- native per-bucket runtime for the multi-process commit --------------
 * One context per rank (flags, status, side / barrier / broadcast streams,
 * the barrier sequence, the pending local broadcasts); one plan per leaf
 * cover (prepared fold requests: validated once, relaunched per bucket).  A
 * bucket call j then costs the host one call: rcv_plan_bucket enqueues, with
 * barrier lag L (RCV_BARRIER_LAG, default 2)
 *   [membership shrank since the previous call: barrier over the previous
 *    live mask behind this rank's last combine, departing ranks included]
 *   side stream:  wait(barrier j-S+L: pool set j%S free, its stamp 0) ->
 *                 [broadcasts, fragmented covers] -> pre-reduce nodes into
 *                 pool set j%S -> record(ready)
 *   bar stream:   wait(ready) -> wait(combine j-L) -> barrier (before its
 *                 signal re-checks the stamps combine j-L read and stamps
 *                 its own set j%S = j+1; after its wait checks every
 *                 producer's stamp of set j%S == j+1 and stamps its own set
 *                 (j+S-L)%S = 0, the next one to be overwritten)
 *                 -> record(arrived)
 *   main stream:  wait(arrived) -> combine(owner slice) -> record(combined)
 *   bcast stream: wait(arrived) -> broadcasts of the buckets combined at
 *                 calls <= j-L (perfect covers: one node per live rank)
 * With L = 2 barrier j overlaps combine j-1, so the combines run back to
 * back; L = 1 is the serial barrier -> combine order.
 * rcv_ctx_finish closes the step (barrier behind every combine + last
 * broadcasts).
 * rcv_ctx_create loads every kernel of the library up front (CUDA lazy
 * loading could otherwise need a context sync while a kernel waits on a
 * peer's flag).
 * S = rcv_pool_sets() partial-pool sets, allocated by the caller
 * (plan set_stride apart).
 * local_flags / peer_flags: 128 uint64 per rank ([0,64) barrier sequence per
 * peer, [64,64+S) pool-set stamps).
 * status: two uint32 words: [0] peers that timed out (bit per rank),
 * [1] stamp mismatches seen by this rank's combines (bit 0: a partial was
 * not ready, bit 1: it was overwritten while being read).  Nonzero word 1
 * means the committed bits of that step are not trustworthy. */
typedef struct rcv_ctx rcv_ctx;
typedef struct rcv_plan rcv_plan;

/* Number S of partial-pool sets a context rotates through (4; the
 * RCV_POOL_SETS measurement switch takes 3..8). */
int rcv_pool_sets(void);

int rcv_ctx_create(int n_ranks, int me, uint64_t *local_flags,
                   void *const *peer_flags, uint32_t *status,
                   uint64_t timeout_ns, rcv_ctx **out);
int rcv_ctx_destroy(rcv_ctx *ctx);
int rcv_ctx_finish(rcv_ctx *ctx, uint64_t live_mask, int participate,
                   void *main_stream);
int rcv_ctx_set_timing(rcv_ctx *ctx, int on);
/* A barrier over live_mask behind everything this context enqueued (side
 * and broadcast streams joined; main_stream waits for it), outside the
 * bucket sequence:
 * the real-kill protocol's synchronisation point before it decides a step
 * (a departed rank of the previous mask joins it, as for a bucket call). */
int rcv_ctx_poll(rcv_ctx *ctx, uint64_t live_mask, int participate, void *main_stream);
/* Real-kill mode: the node's liveness dead word (rcv_liveness_dead_word,
 * device pointer) that barrier kernels consult while they wait: a peer
 * declared dead is neither waited for nor signalled (status word 0 gets its
 * bit, guarded combines skip). NULL detaches. */
int rcv_ctx_set_liveness(rcv_ctx *ctx, const uint32_t *device_dead_word);
/* Drain recorded launch timings (call after synchronising): up to `max`
 * entries of kind (0 pre-reduce, 1 barrier, 2 broadcast, 3 combine),
 * milliseconds, algorithmic HBM bytes, NVLink in / out bytes. */
int rcv_ctx_timing(rcv_ctx *ctx, int max, int *kind, float *ms, double *bytes,
                   double *nvl_in, double *nvl_out, int *count);

typedef struct {
  int n_pre;                     /* local pre-reduce nodes */
  const rcv_block *pre_blocks;   /* their leaves, concatenated */
  const int *pre_counts;         /* leaves per node */
  const uint32_t *pre_leaves;    /* canonical subtree size (2^level) per node */
  void *const *pre_out;          /* pool slot of each node in set 0 */
  size_t set_stride;             /* elements from pool set 0 to set 1 */
  int n_comb;                    /* cover nodes (0: this rank takes no part) */
  const rcv_block *comb_blocks;  /* every node's pool slot in set 0, ascending lo */
  const int *comb_rank;          /* rank producing each cover node (stamps) */
  uint32_t n_leaves;             /* B */
  int n_comb_out;
  void *const *comb_out;         /* primary replica of every live rank */
  int slice_q, slice_nr;         /* this rank's owner slice among the live ranks */
  int n_bcast;
  const void *bcast_src;         /* this rank's primary */
  void *const *bcast_out;        /* this rank's other live replicas */
  int acc_dtype;
  double divisor;
  int variant, comb_variant;
  uint64_t live_mask;
  int participate;
  int remote_in, remote_out;     /* NVLink accounting of the combine */
  int guarded;                   /* real-kill mode: skip the combine once a
                                    live peer timed out (status word 0) */
  uint32_t comb_out_mc;          /* bit j: comb_out[j] is a multicast address
                                    (rcv_mc_map) bound to every live rank's
                                    landing buffer; stored with multimem.st */
} rcv_plan_desc;

int rcv_plan_create(rcv_ctx *ctx, const rcv_plan_desc *desc, rcv_plan **out);
int rcv_plan_destroy(rcv_plan *plan);
int rcv_plan_bucket(rcv_plan *plan, size_t lo, size_t n, void *main_stream);

/* ---- node-local liveness (real-kill mode; live.cpp) ----------------------
 * Replaces a barrier-timeout detection with a heartbeat: every rank's native
 * thread stamps its slot of the POSIX shared-memory segment `name` every
 * period_ns (CLOCK_MONOTONIC); a peer whose stamp is older than deadline_ns,
 * or whose process is gone, gets its bit OR-ed into the segment's dead word.
 * The segment is registered as mapped host memory, so every GPU's barrier
 * kernel reads the word while it waits (rcv_ctx_set_liveness).  Agreement:
 * poll point `seq` (1, 2, ... in the replicated control flow) is decided by
 * the first rank reaching it, which compare-and-swaps the current dead word
 * into the segment's decision ring; every rank gets the same mask back for
 * the same seq (the survivors' common view of comm.py:129-172's failed set). */
typedef struct rcv_liveness rcv_liveness;
int rcv_liveness_create(const char *name, int rank, int world, uint64_t period_ns,
                        uint64_t deadline_ns, rcv_liveness **out);
int rcv_liveness_dead_word(rcv_liveness *lv, const uint32_t **device_ptr, uint32_t *now);
int rcv_liveness_decide(rcv_liveness *lv, uint64_t seq, uint32_t *mask_out,
                        uint64_t *decided_ns);
/* Per-rank timestamps (CLOCK_MONOTONIC ns): last heartbeat, first declared
 * dead (0: alive), self-reported kill (benchmarks), and the clock now. */
int rcv_liveness_stats(rcv_liveness *lv, int rank, uint64_t *beat_ns, uint64_t *dead_ns,
                       uint64_t *kill_ns, uint64_t *now);
int rcv_liveness_note_kill(rcv_liveness *lv);
int rcv_liveness_destroy(rcv_liveness *lv, int unlink_name);

#ifdef __cplusplus
}
#endif
#endif /* RCV_H_ */
