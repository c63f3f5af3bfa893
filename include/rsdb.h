/*
 * rsdb.h -- C ABI of the RaggedShard / DBuffer collective step (veScale-FSDP,
 * arxiv 2602.22437), B200-native (sm_100a CUDA + NCCL over NVLink 5).
 *
 * Citation keys: P:<n> = /root/reference/PAPER.md line n; SURVEY §8 = the
 * hot-path scope table this library implements (rows a1..a8).
 *
 * The four calls of the method (BASELINE.json north_star):
 *     plan(tensors, block_sizes, world) -> layout        rsdb_plan
 *     all_gather(unit)                                    rsdb_all_gather
 *     reduce_scatter(unit)                                rsdb_reduce_scatter
 *     step_8bit_adam(shard)                               rsdb_step_8bit_adam
 * plus the DBuffer batched allocation (rsdb_arena_sizes / rsdb_dbuffer_*),
 * the communicator bootstrap, and the copy-in/copy-out kernel used by the
 * row-wise (FSDP2 Shard(0)) measurement baseline.
 *
 * Conventions (all entry points):
 *  - Every call returns rsdb_status; 0 = OK.  On error a message is kept in
 *    thread-local storage, readable with rsdb_last_error() until the next
 *    rsdb_* call on the same thread.
 *  - Element counts and offsets are int64 ELEMENTS unless a name says bytes.
 *  - Host objects (layout, comm, unit, dbuffer) are created and freed by the
 *    library.  DEVICE MEMORY FOR DATA IS OWNED BY THE CALLER (e.g. torch
 *    tensors' data_ptr()); the library never frees it.  The library allocates
 *    only its own small metadata tables (block / padding tables, < 0.02 B per
 *    element) at unit / dbuffer creation and frees them in *_free; every
 *    *_free accepts NULL (no-op).
 *  - Device calls take a cudaStream_t (passed as void*; NULL = legacy default
 *    stream), are stream-ordered and asynchronous, and return after enqueue.
 *    CUDA launch errors and synchronous NCCL errors come back as status;
 *    asynchronous NCCL errors surface at the next call on that comm.
 *  - No CPU fallback exists: a call that needs a GPU and finds none fails
 *    with RSDB_ECUDA.
 *  - Thread safety: planning functions are pure and thread-safe; calls on one
 *    unit / dbuffer / comm must be serialised by the caller.
 */
#ifndef RSDB_H_
#define RSDB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t rsdb_status;
#define RSDB_OK 0
#define RSDB_EINVAL 1      /* bad argument (block < 1, world < 1, unknown dtype ...)   */
#define RSDB_EMISMATCH 2   /* buffer / layout / world / rank / dtype mismatch, or a     */
                           /* quantization block that would straddle a shard boundary   */
#define RSDB_ECUDA 3       /* CUDA runtime / launch error (incl. no device)             */
#define RSDB_ENCCL 4       /* NCCL error                                                */
#define RSDB_EINTERNAL 5   /* planner inconsistency: must never happen                  */

/* element types */
#define RSDB_BF16 0
#define RSDB_F32 1

/* granularity declarations (P:156-159, P:419 orig_param_policy) */
#define RSDB_GRAN_FLAT 0   /* param = q: blocks of q contiguous elements; g = min(q, e)  */
#define RSDB_GRAN_ROWS 1   /* param = r: r rows of the last dim; g = min(r*shape[-1], e) */
#define RSDB_GRAN_WHOLE 2  /* whole tensor is one block (Muon); g = e            */
#define RSDB_GRAN_ELEM 3   /* element granularity (paper default); g = 1         */

const char* rsdb_last_error(void);
int32_t rsdb_abi_version(void); /* 1 */

/* ======================================================================== */
/* a1 -- granularity.  Pure host.                         */
/* ======================================================================== */
/* Block size g_t (elements) for a tensor of `ndim` dims `shape`.  Tail blocks
 * are allowed when g does not divide e (the tensor's last block is shorter).
 * EINVAL: ndim < 1, any shape[i] < 1, param < 1 for FLAT/ROWS, unknown kind. */
rsdb_status rsdb_block_elems(int32_t ndim, const int64_t* shape, int32_t kind,
                             int64_t param, int64_t* g_out);

/* ======================================================================== */
/* a2/a3 -- planning (PAPER §5: problem P:212-232, Algorithm 1,    */
/* case analysis P:287).  Pure host, deterministic, thread-safe, no CUDA.    */
/* ======================================================================== */
typedef struct rsdb_layout rsdb_layout; /* opaque, library-owned */

/* Plan one FSDP unit: n tensors in the given (default) order with
 * numel[t] = e_t >= 1 and block[t] = g_t >= 1 elements; `world` = m >= 1
 * devices; elem_bytes in {1,2,4} (one dtype per unit); gcoll_bytes (16 =
 * NCCL's alignment) gives g_coll = max(1, gcoll_bytes/elem_bytes).
 * Computes S* (per-device shard size, a multiple of g_coll) and starts l_t so
 * that tensor t occupies [l_t, l_t+e_t) of the m*S global buffer and device k
 * owns [k*S, (k+1)*S), with every block of every tensor wholly on
 * one device.  Never fails for valid input (S = ceil(E/g)*g is always
 * feasible); n = 0 gives S = 0.  *out must be freed with rsdb_layout_free. */
rsdb_status rsdb_plan(int32_t n, const int64_t* numel, const int64_t* block,
                      int32_t world, int32_t elem_bytes, int32_t gcoll_bytes,
                      rsdb_layout** out);

/* The same with one of the tensor orders of P:279 (the paper
 * adopts the default order): 0 default, 1 sorted by sharding block size
 * (descending, stable), 2 sorted by the caller's shape keys (descending,
 * stable; identical shapes adjacent; keys may be NULL otherwise), 3 the best
 * of these (smallest S, ties to the earlier order).  Tensors are placed in the
 * chosen order; starts are still reported in input order. */
#define RSDB_ORDER_DEFAULT 0
#define RSDB_ORDER_BLOCK 1
#define RSDB_ORDER_SHAPE 2
#define RSDB_ORDER_BEST 3
rsdb_status rsdb_plan_ordered(int32_t n, const int64_t* numel, const int64_t* block,
                              int32_t world, int32_t elem_bytes, int32_t gcoll_bytes,
                              int32_t ordering, const int64_t* shape_keys, rsdb_layout** out);

/* A layout with caller-chosen S and starts (e.g. the even-split / FSDP1 flat
 * baseline of BASELINE config 5).  Validated against P:226-229; if
 * require_gcoll != 0 S must also be a multiple of g_coll.  EINVAL if invalid. */
rsdb_status rsdb_layout_from_starts(int32_t n, const int64_t* numel, const int64_t* block,
                                    int32_t world, int32_t elem_bytes, int32_t gcoll_bytes,
                                    int64_t S, const int64_t* starts, int32_t require_gcoll,
                                    rsdb_layout** out);

int64_t rsdb_layout_shard_numel(const rsdb_layout*); /* S            */
int64_t rsdb_layout_padding(const rsdb_layout*);     /* m*S - E      */
int64_t rsdb_layout_total_numel(const rsdb_layout*); /* E            */
int32_t rsdb_layout_world(const rsdb_layout*);       /* m            */
int32_t rsdb_layout_ntensors(const rsdb_layout*);    /* n            */
int32_t rsdb_layout_elem_bytes(const rsdb_layout*);
/* l_t for t in input order into l_out[n]. */
rsdb_status rsdb_layout_starts(const rsdb_layout*, int64_t* l_out);
/* Number of violated constraints of P:226-229 (+ S % g_coll); 0 for plans. */
rsdb_status rsdb_layout_validate(const rsdb_layout*, int64_t* n_violations);
/* Padding intervals [lo, hi) of the global buffer, ascending.  Call with
 * lo = hi = NULL to get *n; then with arrays of >= *n entries. */
rsdb_status rsdb_layout_padding_intervals(const rsdb_layout*, int64_t* n, int64_t* lo, int64_t* hi);
/* a3: pieces of tensors in `rank`'s shard: tensor index, offset inside the
 * shard, length, offset inside the tensor.  Two-call protocol as above. */
rsdb_status rsdb_layout_rank_segments(const rsdb_layout*, int32_t rank, int64_t* n,
                                      int32_t* tensor, int64_t* local_off, int64_t* len,
                                      int64_t* tensor_off);
/* a3: quantization blocks of `rank`: block j of tensor t covers tensor
 * elements [j*qblock, min((j+1)*qblock, e_t)).  Emits (offset inside the
 * shard, length) in ascending order.  EMISMATCH if a block straddles a shard
 * boundary (only possible when g_t is not a multiple of qblock). */
rsdb_status rsdb_layout_rank_blocks(const rsdb_layout*, int32_t rank, int64_t qblock,
                                    int64_t* n, int64_t* off, int32_t* len);
/* Quantization block spec per tensor (the paper's 8-bit Adam uses
 * 32x32 tiles with 32-row sharding granularity):
 *   tile_rows == 0: contiguous blocks of tile_cols elements of the flattened
 *                   tensor (row_len ignored) -- the qblock form;
 *   tile_rows  > 0: the tensor viewed as [e_t / row_len, row_len] is cut into
 *                   tile_rows x tile_cols tiles, row-major, edge tiles smaller. */
typedef struct {
  int64_t row_len;
  int32_t tile_rows;
  int32_t tile_cols;
} rsdb_qspec;
/* a3 with tiles: blocks of `rank` as (offset of the first element inside the
 * shard, rows, cols, pitch = elements between rows), tensors in order, tiles
 * row-major.  specs[n_tensors].  EMISMATCH if a tile straddles a shard
 * boundary (granularity not a multiple of tile_rows rows); EINVAL if
 * row_len does not divide e_t or a size is < 1.  Two-call protocol. */
rsdb_status rsdb_layout_rank_tiles(const rsdb_layout*, int32_t rank, const rsdb_qspec* specs,
                                   int64_t* n, int64_t* off, int32_t* rows, int32_t* cols,
                                   int64_t* pitch);
/* Plan JSON {"m","g_coll","S","E","padding","numel","block","starts"} into buf
 * (NUL-terminated if cap suffices); *needed = bytes incl. NUL. */
rsdb_status rsdb_layout_to_json(const rsdb_layout*, char* buf, int64_t cap, int64_t* needed);
void rsdb_layout_free(rsdb_layout*);

/* ======================================================================== */
/* Communicator: NCCL over NVLink 5 / NVSwitch (P:341 standard runtimes).    */
/* ======================================================================== */
typedef struct rsdb_comm rsdb_comm;
/* Rank 0 creates the id; the caller broadcasts its 128 bytes (e.g. with
 * torch.distributed.broadcast_object_list) -- bootstrap only. */
rsdb_status rsdb_unique_id(uint8_t out[128]);
/* Collective over all `world` ranks; binds the comm to CUDA device `device`
 * (which becomes current on the calling thread). */
rsdb_status rsdb_comm_init(const uint8_t id[128], int32_t world, int32_t rank,
                           int32_t device, rsdb_comm** out);
int32_t rsdb_comm_rank(const rsdb_comm*);
int32_t rsdb_comm_world(const rsdb_comm*);
void rsdb_comm_free(rsdb_comm*);
/* Single-device multi-rank mode (testing / debugging the p2p path on one
 * GPU): a communicator for logical rank `rank` of `world` <= 8 ranks that all
 * live in THIS process, rank `rank` on the CURRENT device (the ranks may
 * share one device or be spread over several) -- one comm per logical rank.
 * It has no NCCL communicator: the NCCL entry points (rsdb_all_gather,
 * rsdb_reduce_scatter, rsdb_unit_reduce_scatter_f32) return EINVAL on its
 * units; every p2p / fused / FP8 / Muon / ring call works, through a p2p
 * object from rsdb_p2p_create_local.  The caller issues each logical rank's
 * calls on its own CUDA stream (the ranks' kernels must run concurrently;
 * the library splits the device's SMs among them).  EINVAL on bad world /
 * rank, ECUDA without a device. */
rsdb_status rsdb_comm_create_local(int32_t world, int32_t rank, rsdb_comm** out);

/* ======================================================================== */
/* Unit: one planned FSDP unit bound to caller-owned device buffers.         */
/* ======================================================================== */
typedef struct {
  void* param_full; /* m*S elements of the unit dtype (bf16 | f32).  AllGather
                       is in place: rank k's shard is param_full+k*S,
                       tensor views live at param_full+l_t (a5).               */
  void* grad_full;  /* m*S elements of the unit dtype: gradients written
                       through the views (autograd).  For f32 units this may
                       equal grad_f32 (the group op then scales in place).     */
  void* grad_f32;   /* m*S fp32: ReduceScatter buffer, in place; after
                       rsdb_reduce_scatter rank k's reduced shard is
                       grad_f32 + k*S.                                          */
} rsdb_unit_bufs;
typedef struct rsdb_unit rsdb_unit;

/* Binds a layout, an optional comm (NULL: collectives unavailable, local
 * group op and optimizer still usable -- used by single-GPU tests), the rank
 * this process holds, buffers (16-byte aligned: EMISMATCH otherwise) and the
 * 8-bit Adam block size qblock (block table via rsdb_layout_rank_blocks;
 * EMISMATCH if a block would straddle; qblock = 0: a collectives-only unit
 * with no optimizer block table -- the 8-bit Adam calls then have nothing to
 * update).  EINVAL if qblock < 0.  The layout is copied. */
rsdb_status rsdb_unit_create(const rsdb_layout*, rsdb_comm* comm_or_null, int32_t rank,
                             const rsdb_unit_bufs* bufs, int64_t qblock, rsdb_unit** out);
/* The same with per-tensor quantization specs (2-D tiles, N2): specs[n]. */
rsdb_status rsdb_unit_create_q(const rsdb_layout*, rsdb_comm* comm_or_null, int32_t rank,
                               const rsdb_unit_bufs* bufs, const rsdb_qspec* specs, rsdb_unit** out);
int64_t rsdb_unit_num_blocks(const rsdb_unit*); /* blocks on this rank */
void rsdb_unit_free(rsdb_unit*);

/* a4: in-place AllGather of the unit buffer (ncclAllGather of S elements from
 * param_full + rank*S into param_full).  Views need no Copy-Out. */
rsdb_status rsdb_all_gather(rsdb_unit*, void* stream);

/* a6 alone: the fused DBuffer group op: grad_f32[i] =
 * fp32(grad_full[i]) * fl(1/m) over the whole m*S buffer in one pass,
 * padding positions written 0. */
rsdb_status rsdb_unit_cast_scale(rsdb_unit*, void* stream);

/* a6 + a7: the group op, then the in-place fp32 ReduceScatter (sum) of
 * grad_f32; rank k's result is grad_f32 + k*S = (1/m) sum_r G_r[kS:(k+1)S]. */
rsdb_status rsdb_reduce_scatter(rsdb_unit*, void* stream);

/* a7 alone: the in-place fp32 ReduceScatter (sum) of grad_f32 as it stands
 * (rsdb_reduce_scatter == rsdb_unit_cast_scale + this; split so that the two
 * can be timed separately). */
rsdb_status rsdb_unit_reduce_scatter_f32(rsdb_unit*, void* stream);

/* a8: block-wise 8-bit Adam on the local ragged shard, no
 * communication.  The per-step scalars (1 - lr*wd, lr/(1-b1^t),
 * sqrt(1-b2^t)) are formed in fp64 on the host and rounded to fp32; the
 * element arithmetic is fp32 (P:344 FP32 master weights). */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
} rsdb_adam_cfg;
typedef struct {
  void* master_f32; /* S fp32 master weights of this rank            */
  void* m_q;        /* S int8   first-moment codes (signed, absmax/127)        */
  void* v_q;        /* S uint8  second-moment codes (unsigned, absmax/255)     */
  void* m_absmax;   /* nblocks fp32, block i of rsdb_layout_rank_blocks order  */
  void* v_absmax;   /* nblocks fp32                                            */
} rsdb_adam_state;
/* Reads the gradient shard grad_f32 + rank*S, updates master / codes /
 * absmax, writes the unit-dtype parameter shard param_full + rank*S (the next
 * AllGather's send buffer).  Elements outside blocks (padding) untouched.
 * step >= 1 (EINVAL otherwise). */
rsdb_status rsdb_step_8bit_adam(rsdb_unit*, const rsdb_adam_state*, const rsdb_adam_cfg*,
                                int64_t step, void* stream);
/* The same step with the dynamic code map (see
 * rsdb_dbuffer_step_8bit_adam_dynamic); m_q is read and written as uint8. */
rsdb_status rsdb_step_8bit_adam_dynamic(rsdb_unit*, const rsdb_adam_state*, const rsdb_adam_cfg*,
                                        int64_t step, void* stream);
/* Host only: the two 256-value maps (ascending fp32) the dynamic codec uses. */
rsdb_status rsdb_dynamic_code_maps(float* m_map, float* v_map);
/* Host only: the lookup tables the dynamic codec's kernels decide codes with
 * (the nearest-map-value rule above, tabulated; exported so tests can replay
 * the kernels' decision).  For y = fl(x / A) in [-1, 1], with bits b of y,
 * mag = b & 0x7fffffff, MB = 6 (m, signed map) or 7 (v, unsigned map),
 * SH = 23 - MB, LOW = 2^SH - 1:
 *   idx = max((mag >> SH) - (100 << MB), 0)   (+ (28 << MB) if y's sign bit is set, m only)
 *   e   = table[idx]
 *   yl  = mag & LOW, or LOW - (mag & LOW) if the sign bit is set (m only)
 *   code = (e >> 24) + (yl >= (e & 0xffffff))
 * m_table holds RSDB_DYN_TABLE_M_LEN entries, v_table RSDB_DYN_TABLE_V_LEN
 * (caller-owned).  EINVAL on NULL. */
#define RSDB_DYN_TABLE_M_LEN 3584
#define RSDB_DYN_TABLE_V_LEN 3584
rsdb_status rsdb_dynamic_code_tables(uint32_t* m_table, uint32_t* v_table);

/* ======================================================================== */
/* Fused collectives over NVLink peer memory.              */
/* Each rank maps the other ranks' buffers (CUDA IPC over NVLink 5 /         */
/* NVSwitch) and the collective runs inside ONE sm_100a kernel per call:     */
/*  - rsdb_reduce_scatter_p2p: a6+a7 fused -- rank k reads G_r[kS:(k+1)S]    */
/*    (bf16) from every rank r, sums fp32(G_r)*fl(1/m) in rank order 0..m-1  */
/*    in fp32 (bit-identical to the oracle), zeroes padding, writes          */
/*    grad_f32 + k*S.  Wire bytes (m-1)*S*2 per rank (half of fp32 RS).      */
/*  - rsdb_all_gather_p2p: a4 -- rank k's copy engine writes its own shard  */
/*    into every peer's param_full (same offsets; pushes over NVLink).       */
/* Ordering: a start barrier (every rank has issued the call, so all prior  */
/* stream work -- grads / optimizer writes -- is complete) and a done        */
/* barrier (every rank finished reading its peers) through a signal buffer;  */
/* the kernel returns only after the done barrier, so later stream work may  */
/* overwrite the buffers.  All ranks must issue the same p2p calls in the    */
/* same order (SPMD).  World <= 8 (one NVLink domain).                       */
/* ======================================================================== */
#define RSDB_IPC_BYTES 72          /* cudaIpcMemHandle_t (64) + offset (8)   */
#define RSDB_P2P_SIGNAL_BYTES 4096 /* signal buffer size per rank            */
typedef struct rsdb_p2p rsdb_p2p;
/* IPC handle + offset of the device allocation containing dev_ptr. */
rsdb_status rsdb_ipc_handle(const void* dev_ptr, uint8_t out[RSDB_IPC_BYTES]);
/* Maps n_bufs buffers of every rank.  local_bufs[0] MUST be a zero-filled
 * device buffer of >= RSDB_P2P_SIGNAL_BYTES (the signal buffer, caller
 * owned); local_bufs[i] / sizes[i] are this rank's buffers (e.g. the
 * GRAD_FULL and PARAM_FULL arenas); all_handles holds world * n_bufs
 * handles from rsdb_ipc_handle, rank-major (the caller all-gathers them,
 * e.g. with torch.distributed.all_gather_object).  EINVAL on bad sizes,
 * ECUDA if a handle cannot be opened (no P2P path). */
rsdb_status rsdb_p2p_create(rsdb_comm* comm, int32_t n_bufs, void* const* local_bufs,
                            const int64_t* sizes, const uint8_t* all_handles, rsdb_p2p** out);
/* Local mode (comm from rsdb_comm_create_local): all_bufs holds world *
 * n_bufs device pointers, rank-major (all_bufs[r * n_bufs + i] = logical
 * rank r's buffer i, on rank r's device; i = 0 the zero-filled signal
 * buffers, one per rank); sizes[i] as above, equal for every rank.  Each
 * logical rank creates its own p2p object over the same table.  Ranks on the
 * same device share its SMs (grids divided by their number); peer access to
 * the other devices is enabled (ECUDA if there is no P2P path).  EMISMATCH
 * if comm is not local. */
rsdb_status rsdb_p2p_create_local(rsdb_comm* comm, int32_t n_bufs, void* const* all_bufs,
                                  const int64_t* sizes, rsdb_p2p** out);
/* Barrier spin limit of the p2p kernels (default 60 s): a kernel whose peer
 * never arrives stops waiting after `seconds`, sets an error flag in its
 * rank's signal buffer and returns (its results are then invalid) instead of
 * hanging the device.  EINVAL if seconds <= 0. */
rsdb_status rsdb_p2p_set_timeout(rsdb_p2p*, double seconds);
/* CTA budget of the SM-driven p2p kernels issued through this object
 * (collectives, fused RS + Adam (+ AG), FP8 AllGather, Muon redistribution):
 * at most max_ctas CTAs, so a collective overlapping compute on another
 * stream leaves the rest of the SMs to it (overlapping; cf. NCCL's CTA
 * budget).  0 (default) = the whole device.  Applies to the object it is set
 * on (a channel from rsdb_p2p_channel has its own).  EINVAL if < 0. */
rsdb_status rsdb_p2p_set_max_ctas(rsdb_p2p*, int32_t max_ctas);
/* Synchronises the device, reads and clears this rank's error flag into
 * *flags (0 = every barrier completed); ECUDA if a barrier timed out. */
rsdb_status rsdb_p2p_check(rsdb_p2p*, int64_t* flags);
/* A device-side barrier of every rank on `stream`: when the stream passes
 * it, every rank's stream has reached its own call (the start / done
 * barriers of the p2p kernels, with no data).  Same SPMD rule as the
 * collectives.  EINVAL on a null p2p; world 1: no-op. */
rsdb_status rsdb_p2p_barrier(rsdb_p2p*, void* stream);
/* An independent collective channel over p's mappings, for collectives that
 * run concurrently on different streams (e.g. an AllGather prefetched on a
 * copy stream while the compute stream runs a ReduceScatter, "optimized
 * communication overlapping").  Same buffers and peers, its own epoch and its
 * own signal words: channel c uses bytes [256c, 256c + 256) of every rank's
 * signal buffer, so c in [1, RSDB_P2P_SIGNAL_BYTES / 256).  Within a channel
 * the SPMD rule holds (same calls in the same order on every rank); two calls
 * on different channels may overlap.  The channel borrows p's mappings: free
 * it before p.  EINVAL (null, c out of range, p itself a channel). */
rsdb_status rsdb_p2p_channel(const rsdb_p2p* p, int32_t channel, rsdb_p2p** out);
void rsdb_p2p_free(rsdb_p2p*);
/* The unit's grad_full (bf16 units) / param_full must lie inside one of the
 * registered buffers at the same offset on every rank (true for DBuffer
 * arenas: offsets are rank-independent for PARAM_FULL / GRAD_FULL).
 * EMISMATCH otherwise.  The p2p object may be NULL at world 1 (AllGather is
 * then the identity, ReduceScatter the group op alone). */
rsdb_status rsdb_reduce_scatter_p2p(rsdb_unit*, rsdb_p2p*, void* stream);
rsdb_status rsdb_all_gather_p2p(rsdb_unit*, rsdb_p2p*, void* stream);
/* a6 + a7 + a8 in ONE kernel: the ReduceScatter of the unit's bf16 gradients
 * over NVLink (rank-order fp32 sum x 1/m, as rsdb_reduce_scatter_p2p) feeds
 * the block-wise 8-bit Adam update of this rank's shard directly (as
 * rsdb_step_8bit_adam); the fp32 reduced gradient is not written (grad_f32 is
 * left untouched).  p2p may be NULL when world == 1.  Results are identical
 * to rsdb_reduce_scatter_p2p followed by rsdb_step_8bit_adam.  The state
 * pointers: `st`, or NULL for a unit of a DBuffer (its arenas). */
rsdb_status rsdb_reduce_scatter_adam_p2p(rsdb_unit*, rsdb_p2p* p2p_or_null, const rsdb_adam_state* st,
                                         const rsdb_adam_cfg*, int64_t step, void* stream);
/* The same step with the NEXT AllGather (a4) fused in: every updated bf16
 * parameter of this rank's shard is also stored over NVLink into every peer's
 * param_full at the same offset, so on return (stream order) every rank holds
 * the full updated parameters -- the result of rsdb_reduce_scatter_adam_p2p
 * followed by rsdb_all_gather_p2p.  p2p must also map param_full.  Peers must
 * not read their param_full while the call runs (its start barrier orders it
 * after every rank's prior work).  world 1: identical to the call above. */
rsdb_status rsdb_reduce_scatter_adam_gather_p2p(rsdb_unit*, rsdb_p2p* p2p_or_null,
                                                const rsdb_adam_state* st, const rsdb_adam_cfg*,
                                                int64_t step, void* stream);

/* ======================================================================== */
/* DBuffer batched allocation: one allocation per    */
/* buffer kind for all units, persistent offsets, one optimizer launch.      */
/* ======================================================================== */
#define RSDB_KIND_PARAM_FULL 0 /* m*S * eb   */
#define RSDB_KIND_GRAD_FULL 1  /* m*S * eb (0 for f32 units: grads live in GRAD_F32) */
#define RSDB_KIND_GRAD_F32 2   /* m*S * 4    */
#define RSDB_KIND_MASTER 3     /* S * 4      */
#define RSDB_KIND_MQ 4         /* S          */
#define RSDB_KIND_VQ 5         /* S          */
#define RSDB_KIND_MABS 6       /* nblocks(rank) * 4 */
#define RSDB_KIND_VABS 7       /* nblocks(rank) * 4 */
#define RSDB_NKINDS 8
/* Byte size of each kind's arena for `rank` and each unit's byte offset in it
 * (unit_offsets[u*RSDB_NKINDS + kind]); every offset is a multiple of
 * align_bytes (>= 16, power of two).  MASTER/MQ/VQ share element offsets.
 * All units belong to one FSDP group: EMISMATCH if their worlds m differ;
 * EINVAL for a null layout, rank outside [0, m) or a bad align_bytes. */
rsdb_status rsdb_arena_sizes(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                             int64_t qblock, int64_t align_bytes, int64_t* bytes_per_kind,
                             int64_t* unit_offsets);
typedef struct rsdb_dbuffer rsdb_dbuffer;
/* Creates every unit inside caller-allocated arenas arena_base[RSDB_NKINDS]
 * (sizes from rsdb_arena_sizes with the same align_bytes), plus one combined
 * block table so that the optimizer runs as ONE launch over all units. */
rsdb_status rsdb_dbuffer_create(const rsdb_layout* const* units, int32_t n_units,
                                rsdb_comm* comm_or_null, int32_t rank, int64_t qblock,
                                int64_t align_bytes, void* const* arena_base,
                                rsdb_dbuffer** out);
/* The same two calls with per-unit, per-tensor quantization specs
 * (specs[u] points to rsdb_qspec[n_tensors(u)]; N2 tiles). */
rsdb_status rsdb_arena_sizes_q(const rsdb_layout* const* units, int32_t n_units, int32_t rank,
                               const rsdb_qspec* const* specs, int64_t align_bytes,
                               int64_t* bytes_per_kind, int64_t* unit_offsets);
rsdb_status rsdb_dbuffer_create_q(const rsdb_layout* const* units, int32_t n_units,
                                  rsdb_comm* comm_or_null, int32_t rank,
                                  const rsdb_qspec* const* specs, int64_t align_bytes,
                                  void* const* arena_base, rsdb_dbuffer** out);
rsdb_unit* rsdb_dbuffer_unit(rsdb_dbuffer*, int32_t i); /* borrowed; NULL if out of range */
int64_t rsdb_dbuffer_num_blocks(const rsdb_dbuffer*);
/* a8 over every unit's shard in one kernel launch. */
rsdb_status rsdb_dbuffer_step_8bit_adam(rsdb_dbuffer*, const rsdb_adam_cfg*, int64_t step,
                                        void* stream);
/* a6 + a7 + a8 for EVERY unit of the DBuffer in ONE kernel launch (the fused
 * ReduceScatter + 8-bit Adam of rsdb_reduce_scatter_adam_p2p over all units'
 * blocks; at world 1 the cast + Adam over the whole model).  Requires bf16
 * units; p2p (NULL iff world 1) must map this DBuffer's GRAD_FULL arena. */
rsdb_status rsdb_dbuffer_reduce_scatter_adam(rsdb_dbuffer*, rsdb_p2p* p2p_or_null,
                                             const rsdb_adam_cfg*, int64_t step, void* stream);
/* rsdb_dbuffer_reduce_scatter_adam with the AllGather fused in (as
 * rsdb_reduce_scatter_adam_gather_p2p): the whole step a6+a7+a8+a4 over every
 * unit in ONE kernel launch.  p2p must map GRAD_FULL and PARAM_FULL arenas
 * from their bases. */
rsdb_status rsdb_dbuffer_reduce_scatter_adam_gather(rsdb_dbuffer*, rsdb_p2p* p2p_or_null,
                                                    const rsdb_adam_cfg*, int64_t step, void* stream);
/* N2: the same one-launch 8-bit Adam with the DYNAMIC (tree) code map of
 * Dettmers et al. (P:419 [dettmers8]; reading R25 in DESIGN.md) instead of
 * the linear absmax code: m_q / v_q hold uint8 indices into the 256-value
 * signed / unsigned maps (the code of 0 is 127 / 0), dequantisation
 * map[code] * absmax, requantisation to the nearest map value of x / absmax
 * (fp32, ties to the lower code). */
rsdb_status rsdb_dbuffer_step_8bit_adam_dynamic(rsdb_dbuffer*, const rsdb_adam_cfg*, int64_t step,
                                                void* stream);
/* End-to-end step from HOST memory (the path a user without device-resident
 * gradients takes; P:93-94's Copy-In/RS/Adam/Copy-Out chain with the copies
 * pipelined).  For every unit in FSDP backward order (last unit first, the
 * same order on every rank):
 *   1. H2D: host_grads[u] -> the unit's GRAD_FULL (bf16, m*S elements, in the
 *      planned layout: padding included) on a library-owned copy stream;
 *   2. the fused ReduceScatter + 8-bit Adam kernel of the unit on `stream`
 *      (rsdb_reduce_scatter_adam_gather_p2p at world > 1, so every rank's
 *      gathered buffer receives the update; rsdb_reduce_scatter_adam_p2p at
 *      world 1), with the unit's DBuffer-bound optimizer state;
 *   3. D2H: this rank's updated bf16 shard (S elements at param_full + rank*S)
 *      -> host_shards[u] on a second library-owned copy stream.
 * Unit u's copy-in overlaps unit u+1's kernel and copy-out; a unit whose
 * shard exceeds 16 M elements runs as ceil(S / 16 M) block-range launches
 * (a count that depends only on S, so it is the same on every rank) whose
 * copy-outs overlap the next launch.  Ordering across
 * calls is kept with per-unit events (a unit's gradients are overwritten only
 * after its previous kernel, its shard only after its previous copy-out).
 * Stream-ordered: the copies start after the work already on `stream`, and
 * `stream` reaches the end of the call only when every copy is done, so a
 * cudaStreamSynchronize(stream) makes host_shards valid.
 *   host_grads[n_units], host_shards[n_units]: host pointers, caller-owned;
 *     pinned (cudaHostAlloc / torch pin_memory) for asynchronous copies.
 *   p2p_or_null: required at world > 1 (maps GRAD_FULL and PARAM_FULL).
 * Errors: EINVAL (null pointer, step < 1), EMISMATCH (f32 units), ECUDA. */
rsdb_status rsdb_dbuffer_step_host(rsdb_dbuffer*, rsdb_p2p* p2p_or_null, const rsdb_adam_cfg*,
                                   int64_t step, const void* const* host_grads, void* const* host_shards,
                                   void* stream);
/* Grouped zero of every unit's gradient buffer ("zero"). */
rsdb_status rsdb_dbuffer_zero_grads(rsdb_dbuffer*, void* stream);
void rsdb_dbuffer_free(rsdb_dbuffer*);

/* ======================================================================== */
/* Batched ragged copy (FSDP2 interleaved Copy-In/Copy-Out baseline,  */
/* P:107, Table 1): one launch copies n segments, optional cast and scale.   */
/* ======================================================================== */
typedef struct {
  const void* src; /* device */
  void* dst;       /* device */
  int64_t numel;
} rsdb_segment;
typedef struct rsdb_copy_plan rsdb_copy_plan;
/* Persistent copy plan (addresses are persistent across steps, like the
 * DBuffer map): segs_host is a HOST array copied into a library-owned device
 * table here (synchronously).  Run: dst[i] = cast(src[i] * scale) for every
 * segment; dtypes RSDB_BF16 / RSDB_F32; segments must not overlap. */
rsdb_status rsdb_copy_plan_create(const rsdb_segment* segs_host, int64_t n, int32_t src_dtype,
                                  int32_t dst_dtype, float scale, rsdb_copy_plan** out);
rsdb_status rsdb_copy_run(const rsdb_copy_plan*, void* stream);
void rsdb_copy_plan_free(rsdb_copy_plan*);

/* ======================================================================== */
/* N2: FP8 (E4M3) 128x128 block quantization of the parameters fused with   */
/* the AllGather ("Block-wise Quantization", "DeepSeek's 128x128 */
/* tiling"; readings R18-R20 in DESIGN.md): 1 byte per element on the wire. */
/* ======================================================================== */
typedef struct rsdb_fp8_unit rsdb_fp8_unit;
/* layout: a unit of 2-D weights planned with elem_bytes 1 (g_coll = 16
 * elements) at 128-row granularity (block = 128 * row_len), so every tile lies
 * on one rank.  specs[n_tensors]: the tile cut of each tensor (row_len,
 * tile_rows, tile_cols; normally 128 x 128), as for rsdb_layout_rank_tiles.
 * Device buffers (caller-owned): master_shard = this rank's S fp32 master
 * weights (16-B aligned); codes_full = m*S bytes (the gathered E4M3 codes at
 * the layout's offsets; padding is never written); scales_full =
 * rsdb_fp8_unit_num_tiles() floats, one per tile in buffer order (tensors in
 * order, tiles row-major): the dequantization factor fl(A / 448), A = tile
 * absmax (0 for an all-zero tile, whose codes are 0).  A tile straddling a
 * shard boundary is EMISMATCH; EINVAL on null pointers or bad specs. */
rsdb_status rsdb_fp8_unit_create(const rsdb_layout*, const rsdb_qspec* specs, rsdb_comm* comm_or_null,
                                 int32_t rank, const float* master_shard, uint8_t* codes_full,
                                 float* scales_full, rsdb_fp8_unit** out);
int64_t rsdb_fp8_unit_num_tiles(const rsdb_fp8_unit*);   /* all ranks */
int64_t rsdb_fp8_unit_first_slot(const rsdb_fp8_unit*);  /* this rank's first tile slot */
/* ONE kernel: quantize every tile of this rank's shard (cvt.rn.satfinite
 * E4M3 of fl(x * fl(448 / A))) and store the codes and the tile scales into
 * every rank's codes_full / scales_full (NVLink stores; p2p must map both
 * buffers of every rank at the same offsets, NULL iff world 1).  On return
 * (stream order) every rank holds the full gathered codes and scales. */
rsdb_status rsdb_fp8_quantize_all_gather(rsdb_fp8_unit*, rsdb_p2p* p2p_or_null, void* stream);
void rsdb_fp8_unit_free(rsdb_fp8_unit*);

/* ======================================================================== */
/* N3: distributed Muon over RaggedShard (Algorithm 2;  */
/* readings R21-R24 in DESIGN.md).                                          */
/* ======================================================================== */
typedef struct rsdb_muon rsdb_muon;
typedef struct {
  double lr;         /* eta (default 0.02) */
  double momentum;   /* mu (0.95), Nesterov form: buf = mu buf + g; u = g + mu buf */
  double eps;        /* Newton-Schulz normalisation X = U / (||U||_F + eps) (1e-7) */
  int32_t ns_steps;  /* quintic iterations (5), coefficients (3.4445, -4.7750, 2.0315) */
} rsdb_muon_cfg;
typedef struct {
  float* master;       /* S fp32: this rank's master shard (updated in place) */
  float* momentum;     /* S fp32: momentum buffer shard (updated in place) */
  const float* grad;   /* S fp32: the reduced gradient shard (e.g. GRAD_F32 + rank*S) */
  float* u;            /* S fp32 scratch: the momentum output, read by the roots (p2p-registered) */
  void* param_bf16;    /* S bf16 shard written with the update, or NULL */
  void* workspace;     /* rsdb_muon_workspace_bytes(): the root matrices + NS scratch (p2p-registered) */
} rsdb_muon_bufs;
/* rows[t], cols[t]: the matrix shape of tensor t (rows*cols == numel), or
 * 0, 0 for tensors Muon skips (norms, biases: left untouched).  SelectRoot
 * (R24): matrices by decreasing rows*cols*min(rows,cols), each to the least
 * loaded rank (ties: the rank owning most of it, then the lowest rank) --
 * identical on every rank.  precision RSDB_F32: Newton-Schulz in fp32
 * (cuBLAS SGEMM); RSDB_BF16: bf16 operands, fp32 accumulation (tensor cores,
 * Muon's reference precision).  comm NULL iff world 1. */
rsdb_status rsdb_muon_create(const rsdb_layout*, const int64_t* rows, const int64_t* cols,
                             rsdb_comm* comm_or_null, int32_t rank, int32_t precision,
                             rsdb_muon** out);
/* Host only (no CUDA): SelectRoot (R24) for every tensor -> roots[n] (-1 for
 * non-matrices); the assignment rsdb_muon_create uses.  EINVAL on bad shapes. */
rsdb_status rsdb_muon_select_roots(const rsdb_layout*, const int64_t* rows, const int64_t* cols,
                                   int32_t* roots);
int32_t rsdb_muon_root(const rsdb_muon*, int32_t tensor);    /* -1: not a matrix */
int64_t rsdb_muon_workspace_bytes(const rsdb_muon*);         /* this rank's */
rsdb_status rsdb_muon_bind(rsdb_muon*, const rsdb_muon_bufs*);
/* One Muon step of every matrix of the unit (Algorithm 2): momentum on the
 * shard; ONE kernel gathers every matrix onto its root over NVLink
 * (Redistribute(u, RaggedShard(r))); Newton-Schulz on the root; ONE kernel
 * returns each owner its piece and applies w -= eta sqrt(max(1,rows/cols)) o
 * (Redistribute(o, p) + update, bf16 shard written).  p2p (NULL iff world 1)
 * must map every rank's `u` and `workspace`. */
rsdb_status rsdb_muon_step(rsdb_muon*, rsdb_p2p* p2p_or_null, const rsdb_muon_cfg*, void* stream);
void rsdb_muon_free(rsdb_muon*);
/* The Newton-Schulz GEMM of the bf16 mode (Alg. 2 l.10, reading R22), a
 * hand-written tcgen05 kernel (TMA 128-B swizzled tiles -> tcgen05.mma, fp32
 * accumulators in TMEM, fused epilogue):
 *   C = alpha * A . B^T + beta * D     (and, if CT != NULL, CT = C^T)
 * A: M x K, B: N x K, D / C: M x N, CT: N x M -- all row-major bf16 device
 * matrices with leading dimensions (elements) lda, ldb, ldd, ldc, ldct that
 * are multiples of 8 and 16-B aligned base pointers (D unused when beta = 0).
 * fp32 accumulation, one bf16 rounding of alpha*acc + beta*D.  C must not
 * overlap A, B or D.  rsdb_muon_step's bf16 mode issues three per iteration
 * (A = W W^T; B = cA A + bA; W' = B W + aW with W'^T).  EINVAL on bad
 * dimensions / alignment, ECUDA on launch errors. */
rsdb_status rsdb_ns_gemm_bf16(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, const void* B,
                              int64_t ldb, float alpha, float beta, const void* D, int64_t ldd, void* C,
                              int64_t ldc, void* CT, int64_t ldct, void* stream);
/* The same for a product the caller knows is SYMMETRIC (M = N, e.g. W W^T,
 * or c A A + b A with A symmetric -- the first two GEMMs of every
 * Newton-Schulz iteration): only the output tiles reaching the upper triangle
 * are computed (~half the flops); the upper triangle (diagonal included) is
 * stored directly and the lower triangle as its mirror image, so C is exactly
 * symmetric.  Same arguments and errors as rsdb_ns_gemm_bf16 (C is M x M). */
rsdb_status rsdb_ns_gemm_bf16_sym(int32_t M, int32_t K, const void* A, int64_t lda, const void* B, int64_t ldb,
                                  float alpha, float beta, const void* D, int64_t ldd, void* C, int64_t ldc,
                                  void* stream);

/* ======================================================================== */
/* K-slot unsharded ring: only K units' gathered         */
/* parameters / gradients are resident; each unit keeps a persistent        */
/* parameter shard, slots are reused in stream (event) order.               */
/* ======================================================================== */
/* Ring mode for a (non-DBuffer) unit: the persistent S-element parameter
 * shard (caller-owned, 16-B aligned, same element type as the unit).  The
 * 8-bit Adam calls then write the updated shard there instead of into
 * param_full + rank*S; NULL turns ring mode off.  EMISMATCH for DBuffer units. */
rsdb_status rsdb_unit_set_shard(rsdb_unit*, void* param_shard);
/* Points the unit at other gathered buffers (a ring slot): the same rules as
 * rsdb_unit_create (non-null, 16-B aligned, grad_full != grad_f32 for bf16). */
rsdb_status rsdb_unit_rebind(rsdb_unit*, const rsdb_unit_bufs*);
/* AllGather from the persistent shards: param_full[r*S ...] = shard of rank r
 * for every r.  Each rank's copy engine pushes its own shard into region
 * `rank` of every rank's param_full (its own by a local copy, the peers' over
 * NVLink), between the p2p start/done barriers.  p2p (NULL iff world 1) must
 * map every rank's param_full (the ring slot) at the same offset (EINVAL
 * otherwise); the shard itself need not be mapped. */
rsdb_status rsdb_all_gather_shards_p2p(rsdb_unit*, rsdb_p2p* p2p_or_null, void* stream);
typedef struct rsdb_ring rsdb_ring;
/* A ring of k slots handed out round robin: acquisition i gets slot i mod k
 * on every rank (so peers agree on slot addresses); the stream waits until
 * the slot's previous holder released it. */
rsdb_status rsdb_ring_create(int32_t k_slots, rsdb_ring** out);
rsdb_status rsdb_ring_acquire(rsdb_ring*, void* stream, int32_t* slot);
rsdb_status rsdb_ring_release(rsdb_ring*, int32_t slot, void* stream);  /* records the slot's event */
void rsdb_ring_free(rsdb_ring*);

#ifdef __cplusplus
}
#endif
#endif /* RSDB_H_ */
