/*
 * hdp.h -- C-ABI of libhdp.so: the synchronous data-parallel mixed-precision
 * LSTM training step of arXiv 1912.00286, B200 (sm_100a) native.
 *
 * The calls follow the paper's problem statement, PAPER.md:89-97:
 *   1. initialise the parameters randomly           -> caller; hdp_load_params
 *   2. broadcast them to every worker                -> hdp_load_params (ncclBroadcast)
 *   3. fprop + bprop on each worker's mini-batch     -> hdp_lstm_forward / hdp_lstm_backward
 *   4. aggregate the gradients and average them      -> hdp_grad_average_update
 *   5. update optimizer state and global weights     -> hdp_grad_average_update (fused, K11)
 *   6. broadcast the updated parameters              -> hdp_grad_average_update (allgather)
 * with the learning-rate schedule of PAPER.md:106-121 (hdp_set_lr_schedule)
 * and the loss scale alpha of PAPER.md:177-180 (hdp_set_loss_scale).
 *
 * Conventions
 *  - Every function returns 0 (HDP_OK) or a negative HDP_ERR_* code; nothing
 *    aborts or throws across the ABI.  hdp_last_error() returns a
 *    thread-local message for the most recent failure.
 *  - Argument and shape errors are detected on the host before anything is
 *    enqueued (HDP_ERR_ARG; no state changed).
 *  - `stream` arguments are cudaStream_t handles passed as void*; all compute
 *    calls are asynchronous and stream-ordered on it.
 *  - Device memory is owned by the caller: hdp_configure reports the arena
 *    size, the caller allocates it (256-byte aligned) and hdp_bind()s it.
 *    The library owns (and hdp_destroy frees) its NCCL communicator, its
 *    internal streams (capture, exchange, the fused head's side stream, one
 *    per layer for the layer-diagonal forward), events and captured CUDA
 *    graphs; at world > 1 with the NVLink exchange the IPC-shared gradient /
 *    weight / flag windows it allocates (peers map them, so they cannot live
 *    in the caller's arena); the phase-trace buffer when that debug option is
 *    used; plus transient staging buffers inside hdp_load_params /
 *    hdp_gather_master.
 *  - One context per process = one rank = one GPU.  A context is not
 *    thread-safe.  Every rank must make the same sequence of calls with the
 *    same B, T and epoch (NCCL's rule, and the paper's lock-step, :104).
 */
#ifndef HDP_H_
#define HDP_H_

#ifdef __cplusplus
extern "C" {
#endif

#define HDP_UID_BYTES 128

enum {
  HDP_OK = 0,
  HDP_ERR_ARG = -1,         /* invalid argument / shape; nothing was enqueued        */
  HDP_ERR_CUDA = -2,        /* CUDA runtime / driver failure                          */
  HDP_ERR_NCCL = -3,        /* NCCL failure (incl. asynchronous communicator errors) */
  HDP_ERR_NONFINITE = -4,   /* Inf/NaN gradients seen (PAPER.md:134 overflow hazard) */
  HDP_ERR_STATE = -5,       /* call-order violation, or context poisoned             */
  HDP_ERR_UNSUPPORTED = -6
};

/* Precision modes: math / synchronisation / update.    */
enum { HDP_MATH_FP32 = 0,     /* the paper's baseline: everything fp32 (:147)      */
       HDP_MATH_MIXED16 = 1,  /* fp16 math + fp16 wire + fp32 master/update         */
       HDP_MATH_BF16 = 2      /* NEXT-3 variant (not in the paper): bfloat16 at every
                                 16-bit rounding point of MIXED16 (weights, inputs,
                                 h, gates, dA, gradients, wire), fp32 accumulation,
                                 fp32 master/update (reading Q29); dense
                                 inputs are bf16; runs the per-step GEMM path (the
                                 fused recurrences are fp16-only); no recurrent dropout */
};
/* Wire format of the gradient exchange.              */
enum { HDP_WIRE_FP16_A2A = 0,     /* fp16 all-to-all, fp32 rank-ordered sum in K11 (default) */
       HDP_WIRE_FP16_NCCLSUM = 1, /* ncclReduceScatter(ncclHalf, sum): NCCL-native fp16 sum  */
       HDP_WIRE_FP32 = 2          /* fp32 gradients, ncclReduceScatter(ncclFloat, sum)       */
};
enum { HDP_OPT_SGDM = 0,  /* Eqs. 1-2                              */
       HDP_OPT_ADAM = 1   /* "any optimizer" (:98), Kingma & Ba with bias correction  */
};
/* How steps 4-6 move the data (hdp_model_desc.exchange).       */
enum { HDP_EXCH_AUTO = 0,  /* world >= 2: HDP_EXCH_P2P where it applies, else NCCL;
                              world == 1: K11 over the local gradient slots             */
       HDP_EXCH_NCCL = 1,  /* NCCL collectives per bucket (all-to-all / reduce-scatter,
                              K11, all-gather), or K11 alone at world == 1              */
       HDP_EXCH_P2P = 2,   /* NEXT-2: one kernel reads every rank's fp16 gradient shard
                              over NVLink peer memory (CUDA IPC), does the K11 arithmetic
                              and stores the fp16 weights into every rank's copy.  Needs
                              mixed math, the fp16 all-to-all wire and world <= 8.  At
                              world == 1 with 2 <= sim_workers <= 8 it runs as a LOOPBACK:
                              the contributions are the simulated workers' gradient slots
                              and the kernel writes sim_workers weight copies (copy 0 is the
                              working copy, the others are readable as debug buffer
                              "Wcopy"), so the kernel's arithmetic and protocol are tested
                              on one GPU.  HDP_ERR_UNSUPPORTED where it does not apply.   */
       HDP_EXCH_TASK0 = 3  /* ablation, the paper's steps 4-6 literally:
                              every worker's gradients go to task 0 (NCCL grouped sends),
                              task 0 sums them in fp32 rank order and updates the WHOLE
                              model (K11, master and optimizer state on rank 0 only), then
                              broadcasts the weights.  Same per-element arithmetic as the
                              owner-sharded paths (bit-identical results), N times the
                              update work and memory on rank 0.  fp16 all-to-all or fp32
                              wire; world == 1 behaves as HDP_EXCH_NCCL.                */
};

typedef struct hdp_ctx hdp_ctx;

/* Model description (Fig. 2, :64-80; readings Q1-Q4, Q21-Q24).
 * n_layers == 0 describes a flat parameter vector of `flat_params`
 * elements with no forward/backward (the C5 update sweep).            */
typedef struct {
  int n_layers;        /* stacked LSTM layers L >= 0                              */
  int input_dim;       /* I of layer 0 (dense input); ignored if vocab > 0       */
  int hidden;          /* h                                                       */
  int fc_hidden;       /* per-step FC(ReLU) width before the 1-unit output; 0 = none */
  int head_last_step;  /* 1: one output per sequence at t = T-1 (IMDB-style)      */
  int vocab;           /* > 0: int32 token input through an embedding             */
  int embed_dim;       /* embedding width when vocab > 0                          */
  int max_batch;       /* per-rank batch upper bound                              */
  int max_seq;         /* sequence length upper bound                             */
  int math;            /* HDP_MATH_*                                              */
  int wire;            /* HDP_WIRE_*                                              */
  int optimizer;       /* HDP_OPT_*                                               */
  int sim_workers;     /* >= 1; > 1 only when world == 1 (simulated workers)      */
  long long flat_params; /* n_layers == 0 only                                    */
  int exchange;        /* HDP_EXCH_*                                              */
} hdp_model_desc;

typedef struct {
  long long n_params;        /* canonical (unpadded) parameter count                */
  long long n_params_padded; /* device layout length (padded, bucketed)             */
  long long n_buckets;
  long long arena_bytes;     /* device bytes the caller must allocate and bind      */
} hdp_sizes;

/* One parameter block.  Canonical host layout (hdp_load_params):
 *   [E (vocab x embed)]?  then per layer l: W_l [4h][I_l], U_l [4h][h],
 *   b_l [4h] with gate blocks i, f, g, o (row = gate*h + unit);
 *   then [F [fc][h], fb [fc]]?, wo [fc or h], bo [1].                    */
typedef struct {
  char name[16];
  long long canon_offset; /* offset in the canonical host vector                 */
  long long rows, cols;   /* canonical shape (cols = 1 for vectors)              */
  long long dev_offset;   /* offset in the device parameter vector               */
  long long dev_rows, dev_cols; /* padded device shape                           */
  int bucket;             /* exchange bucket (readiness order: head first)       */
} hdp_block;

/* NCCL unique id, generated on rank 0 and shipped to the others by the
 * caller (e.g. torch.distributed.broadcast_object_list).              */
int hdp_nccl_unique_id(unsigned char uid[HDP_UID_BYTES]);

/* init(world, rank) of north_star.  world == 1 needs no uid (may be NULL).
 * Selects `device` for the calling thread and creates the communicator.
 * device == -1 creates a host-only context (no CUDA, no NCCL) that can
 * configure and answer layout / schedule queries (hdp_param_block, hdp_lr)
 * but not bind or compute -- used by CPU tests of the host logic.        */
int hdp_init(int world, int rank, const unsigned char* uid, int device, hdp_ctx** out);
int hdp_destroy(hdp_ctx* ctx);
const char* hdp_last_error(void);

/* Validate the model and compute the device layout and arena size.
 * All ranks must pass identical descriptions: at world > 1 a 64-bit hash of
 * the description is all-reduced (min and max over the ranks) and a
 * mismatch returns HDP_ERR_ARG on every rank (collective call).          */
int hdp_configure(hdp_ctx* ctx, const hdp_model_desc* desc, hdp_sizes* out);
/* Bind the caller-owned device arena (>= arena_bytes, 256-B aligned).
 * Zero-fills it, sets up kernels and streams.                         */
int hdp_bind(hdp_ctx* ctx, void* arena, long long arena_bytes);

/* The exchange path configure resolved desc.exchange to:
 * 0 = K11 over the local gradient slots (world 1), 1 = NCCL collectives + K11,
 * 2 = the one-kernel NVLink exchange across ranks, 3 = its world-1 loopback,
 * 4 = the task-0 ablation; negative if not configured.                 */
int hdp_exchange_kind(const hdp_ctx* ctx);

int hdp_num_blocks(const hdp_ctx* ctx);
int hdp_param_block(const hdp_ctx* ctx, int i, hdp_block* out);

/* PAPER.md:91-92 steps 1-2.  `params` = canonical fp32 host vector
 * (n_params), read on `root` only (others may pass NULL); broadcast to
 * all ranks; fp32 master shards and optimizer state (zero) initialised;
 * the working copy (fp16 in mixed mode) set.  Synchronous; collective.  */
int hdp_load_params(hdp_ctx* ctx, const float* params, int root);
/* Read back the fp32 master weights into a canonical host vector.
 * Synchronous; collective (allgather of the shards).                  */
int hdp_gather_master(hdp_ctx* ctx, float* params_out);
/* Local, synchronous read-backs in the canonical layout (as fp32):
 * the working copy used by fprop, and slot `slot`'s gradients (they carry
 * the loss scale alpha).                              */
int hdp_read_weights(hdp_ctx* ctx, float* out);
int hdp_read_grads(hdp_ctx* ctx, int slot, float* out);

/* set_lr_schedule of north_star, PAPER.md:106-121:
 *   lambda_e = min(lambda0/(1 + N/n_half), max_eff_lr/N) * gamma^epoch
 * N = world * sim_workers.  momentum m of Eq. 1; Adam b1, b2, eps.
 * Errors: lambda0 <= 0, gamma not in (0,1], n_half <= 0 -> HDP_ERR_ARG. */
int hdp_set_lr_schedule(hdp_ctx* ctx, double lambda0, double gamma, double n_half, double max_eff_lr,
                        double momentum, double adam_b1, double adam_b2, double adam_eps);
/* The scheduled rate (fp64) for `epoch`; negative if not configured.  */
double hdp_lr(const hdp_ctx* ctx, int epoch);
/* Loss scale alpha > 0 (PAPER.md:177; default 10, :127).              */
int hdp_set_loss_scale(hdp_ctx* ctx, float alpha);
/* L2 regularisation coefficient l2 >= 0 ("application of L2
 * regularization"; SPEC.md:171 loss = alpha*mean hinge + alpha*l2*||W||^2;
 * DESIGN.md reading Q16).  Applies to every parameter w of the working
 * weights (fp16 copy in mixed mode, R1):
 *   - hdp_lstm_forward's loss_out gains l2 * sum(w^2) (fp64 partial sums,
 *     deterministic order);
 *   - hdp_grad_average_update adds fp32(2*l2) * w to the descaled average
 *     gradient before the optimizer step (K11; the alpha the term would carry
 *     inside the scaled loss cancels in the descale).
 * Default 0 (off).  Errors: l2 < 0 or not finite -> HDP_ERR_ARG, nothing
 * changed.  Changing it drops the captured forward graphs.               */
int hdp_set_l2(hdp_ctx* ctx, double l2);
/* Variational recurrent dropout (NEXT-3; "recurrent dropout";
 * DESIGN.md reading Q16b; oracle/dropout.py).  keep in (0, 1]; keep = 1 turns
 * it off (the default).  One Bernoulli(keep) mask per (update count, layer,
 * sequence, unit), fixed over the time steps: the recurrent GEMM of layer l
 * reads h~_{t-1} = fp16(fp32(h_{t-1}) * fp32(1/keep)) on kept units and 0
 * elsewhere; the next layer and the head see the unmasked h; BPTT multiplies
 * the recurrent gradient by the same mask and scale and dU accumulates
 * dA_t^T h~_{t-1}.  The mask is the counter-based hash of dropout.cuh keyed by
 * `seed`, the number of completed hdp_grad_average_update calls since this
 * call, the layer, the sequence's global index ((rank * slots + slot) * B + b)
 * and the unit.  Mixed mode only.  The two-layer wavefront kernels apply it in
 * their epilogues (masked recurrent operand pushed to the peers, masked dh_rec,
 * dU from h~); other shapes run the per-step GEMM path with the fused cell
 * epilogues (the per-layer persistent kernels have no dropout and are bypassed).
 * The library allocates (cudaMalloc)
 * the masked-input buffers, slots * L * (T+1) * B * h_p fp16, freed by
 * hdp_destroy.  Synchronises the device; drops the captured graphs.
 * Errors: keep outside (0, 1] -> HDP_ERR_ARG; FP32 mode -> HDP_ERR_UNSUPPORTED;
 * unbound -> HDP_ERR_STATE.                                                 */
int hdp_set_recurrent_dropout(hdp_ctx* ctx, double keep, unsigned int seed);
/* Dynamic loss scaling (NEXT-3; PAPER.md:134 names fp16 overflow as the hazard
 * of the static alpha of :177; reading Q14b).  growth_interval > 0
 * switches it on (0 = static alpha, the default): alpha moves to the device,
 * starting at the current hdp_set_loss_scale value, and every
 * hdp_grad_average_update first counts the non-finite values of all ranks'
 * fp16 gradients (all-reduced across ranks), then
 *   - count > 0: the update is skipped (fp32 master, optimizer state and fp16
 *     weights unchanged on every rank), alpha /= 2 (not below 1); the call does
 *     NOT return HDP_ERR_NONFINITE and the context is not poisoned;
 *   - count = 0: the update runs with inv_scale = fp32(1/(N*alpha)); after
 *     growth_interval consecutive finite steps alpha *= 2.
 * alpha stays on the device (no host synchronisation per step).  Requires a
 * bound context; toggling drops the captured forward graphs.
 * Errors: growth_interval < 0 -> HDP_ERR_ARG; unbound -> HDP_ERR_STATE;
 * the Adam optimizer -> HDP_ERR_UNSUPPORTED (its bias-correction step count
 * is kept on the host and would also count skipped steps).                  */
int hdp_set_dynamic_loss_scale(hdp_ctx* ctx, int growth_interval);
/* Current alpha and the number of skipped steps since dynamic scaling was
 * enabled (synchronises the device).  With static alpha: the set value, 0.   */
int hdp_loss_scale_state(hdp_ctx* ctx, float* alpha, int* skipped_steps);

/* fprop of slot `slot`'s mini-batch and the scaled hinge
 * loss Eq. 6 (:179).
 *   x       : dense input [B][T][input_dim], fp16 (mixed) or fp32 (FP32
 *             mode), or int32 tokens [B][T] when vocab > 0; host or device.
 *             Token ids must lie in [0, vocab): an id outside it is read as
 *             id 0 (no out-of-bounds access) and counted on the device; the
 *             next hdp_grad_average_update returns HDP_ERR_ARG for that step
 *             (its update has run) and poisons the context.
 *   targets : int8 in {-1,+1}, [B][T] (per-step heads) or [B] (last-step).
 *   y_out   : device fp32 [T][B] (or [B]); nullable.
 *   loss_out: device fp32 scalar = mean hinge WITHOUT alpha; nullable.
 * Slots 0..sim_workers-1; 1 <= B <= max_batch, 1 <= T <= max_seq.       */
int hdp_lstm_forward(hdp_ctx* ctx, const void* x, const void* targets, int B, int T, int slot, float* y_out,
                     float* loss_out, void* stream);
/* bprop / BPTT of the last forward of `slot`; writes that
 * slot's gradients (alpha-scaled; fp16 in mixed mode, one RNE of the fp32
 * accumulation) and marks each exchange bucket ready as it completes.
 * HDP_ERR_STATE if `slot` has no forward.                               */
int hdp_lstm_backward(hdp_ctx* ctx, int slot, void* stream);
/* PAPER.md:94-96 steps 4-6 for every bucket: exchange (NCCL, per
 * `wire`), fused fp32 average / alpha removal / overflow count /
 * SGD-m or Adam at lambda_epoch / fp16 recast (K11) on the owner shard,
 * allgather of the updated weights.  Overlaps the still-running backward
 * of lower layers.  If nonfinite_host != NULL the call synchronises and
 * stores the global count of non-finite gradient values there; a
 * non-zero count returns HDP_ERR_NONFINITE (also reported by the next
 * call when not synchronised) and poisons the context (HDP_ERR_STATE
 * until hdp_load_params).  HDP_ERR_STATE if a slot has no backward.      */
int hdp_grad_average_update(hdp_ctx* ctx, int epoch, void* stream, int* nonfinite_host);

/* Runtime options by name.
 * Context-scoped (ctx required, bound):
 *   "partial_fraction" f in (0, 1] -- NEXT-2 partial collection ("collecting
 *        a fraction of gradients (normally at 90-95%) before proceeding to averaging";
 *        SPEC.md:320-328): the exchange proceeds once q = ceil(f*N) of the N contributors'
 *        gradients are ready (rank 0 decides and publishes the set), averages exactly
 *        those -- fp32 rank-ordered sum times fp32(1/(count*alpha)) -- and discards the
 *        late ones for that step.  f = 1 (default) is the lock-step of :94.  Needs the
 *        one-kernel exchange (hdp_exchange_kind 2 or 3) and a static alpha, else
 *        HDP_ERR_UNSUPPORTED.  hdp_partial_state reads the last decision.
 *   "straggler_mask" (bits of contributor ids), "straggler_us" -- test injection: those
 *        contributors publish their readiness that much later (exercises the above).
 * Process-wide kernel selection (ctx may be NULL; kernels of graphs captured before the
 * call are kept -- a ctx passed here has its graphs dropped): "persistent",
 *   "wavefront", "wavefront_fusex", "wavefront_wgrad", "wavefront_tmem", "recur_nbg",
 *   "gemm_cta_group", "gemm_cluster_n", "pdl", "k7_bn", "k7_splits",
 *   "recur_trace", "layer_pipe", "head_fused", "k7_cluster", "fwd_pdl" (integers; see csrc/options.h;
 *   "head_fused" applies to contexts configured after the change).  They choose between implementations
 *   of the same arithmetic (ablations, tuning); the defaults are the measured best.
 * Errors: unknown name, value out of range -> HDP_ERR_ARG.                      */
int hdp_set_option(hdp_ctx* ctx, const char* name, double value);
/* Current value of a process-wide kernel switch (names as above).
 * Errors: unknown name, null pointer -> HDP_ERR_ARG.                            */
int hdp_get_option(const char* name, double* value);
/* The last partial-collection decision (synchronises): bit r of *mask set if
 * contributor r's gradients were averaged; *count = their number.             */
int hdp_partial_state(hdp_ctx* ctx, unsigned* mask, int* count);

/* Live profiler.  Kernel classes: */
enum { HDP_K_INPUT = 0,     /* input packing / embedding gather (A1 prologue, K10) */
       HDP_K_GEMM_X = 1,    /* K1  input projection X W^T + b (A1)                 */
       HDP_K_GEMM_H = 2,    /* K2  recurrent gate GEMM h U^T per step (A2)         */
       HDP_K_CELL_FWD = 3,  /* K3  fused cell forward (A3)                         */
       HDP_K_HEAD_FWD = 4,  /* K4  head + scaled hinge loss (A4)                   */
       HDP_K_HEAD_BWD = 5,  /* K5  head backward (A5)                              */
       HDP_K_CELL_BWD = 6,  /* K6  fused cell backward (A6)                        */
       HDP_K_GEMM_DH = 7,   /* K7  recurrent backward GEMM dA U per step (A7)      */
       HDP_K_GEMM_DW = 8,   /* K8  weight / bias gradients (A8)                    */
       HDP_K_GEMM_DX = 9,   /* K9  input gradient dA W (A8)                        */
       HDP_K_EMBED_BWD = 10,/* K10 embedding scatter-add (A8)                      */
       HDP_K_UPDATE = 11,   /* K11 fused average + update (A10)                    */
       HDP_K_COMM = 12,     /* NCCL exchange / allgather (A9, A11)                 */
       HDP_K_RECUR_FWD = 13,/* persistent fused K2+K3 over all t (A2+A3)           */
       HDP_K_RECUR_BWD = 14,/* persistent fused K6+K7 over all t (A6+A7)           */
       HDP_K_NTAGS = 15 };
/* enable != 0: subsequent forward / backward run eagerly (no CUDA graphs)
 * with a CUDA event pair around every launch on its stream.              */
int hdp_profile(hdp_ctx* ctx, int enable);
/* Synchronises; accumulated milliseconds and event-pair counts per class
 * (arrays of HDP_K_NTAGS, nullable); reset != 0 clears the totals.        */
int hdp_profile_read(hdp_ctx* ctx, double* ms, long long* launches, int reset);
/* Synchronises; the event-pair records collected since the last hdp_profile_read
 * as a timeline (the substitute for an nsys trace, which this image lacks): for
 * record i < min(*n, cap) its class tags[i], stream lanes[i] (0 the caller's,
 * 1 exchange / update, 2 the fused head's side stream, 3 + l the layer pipeline's
 * stream of layer l) and start / end t0_ms[i] / t1_ms[i] relative to the first
 * record's start.  *n = number of records.  Does not clear them.
 * Errors: null n, cap > 0 with a null array -> HDP_ERR_ARG.               */
int hdp_profile_timeline(hdp_ctx* ctx, int* tags, int* lanes, double* t0_ms, double* t1_ms, int cap, int* n);
/* Number of this library's kernels enqueued so far (graph launches count
 * their captured kernels; NCCL's and cub's kernels are not counted).     */
long long hdp_kernel_launches(const hdp_ctx* ctx);

/* Device pointers into the bound arena (for benches and tests). */
void* hdp_weights_ptr(hdp_ctx* ctx);           /* working copy, device layout          */
void* hdp_grads_ptr(hdp_ctx* ctx, int slot);   /* gradient slot, device layout        */
void* hdp_master_ptr(hdp_ctx* ctx);            /* this rank's fp32 master shards      */
/* Internal activation buffers of slot `slot` (diagnostics): name is one of
 * "Hs" (fp16 [L][T+1][B][hp]), "C" (fp32 [L][T][B][hp]), "gates"
 * (fp16 [L][T][B][4hp]), "X0" (fp16 [T][B][Ip0]), "dA" (fp16 [T][B][4hp]; the
 * top layer's in the 2-layer wavefront), "dA2" (layer 0's in the wavefront),
 * "Z" (the FC head's ReLU output, fp16 [T][B][Fp]),
 * "dH0"/"dH1" (fp32), "Hst" (recurrent dropout's masked inputs h~, fp16
 * [L][T_max+1][B_max][hp] with rows [t][B][hp] of the actual B inside),
 * "Wcopy" (HDP_EXCH_P2P loopback: weight copies 1..sim_workers-1, each a
 * device-layout fp16 vector of n_params_padded elements; slot argument
 * ignored).  Returns NULL for an unknown name or unbound context.  */
void* hdp_debug_buffer(hdp_ctx* ctx, int slot, const char* name);

/* ---------------------------------------------------------------------
 * Kernel-level entries (stateless; used by the C5 sweep and unit tests).
 * --------------------------------------------------------------------- */

/* K11 on caller buffers: contribution r is grads + r*src_stride elements
 * (fp16 if !grads_f32), r = 0..nsrc-1 summed in rank order; W/S1/S2 fp32
 * master / momentum (or Adam m, v); w16 or w32 receives the new working
 * copy (either may be NULL).  count % 8 == 0 and 16-byte aligned pointers
 * use 128-bit accesses (any count is accepted).  nonfinite_dev (device
 * int, nullable) is incremented by the number of Inf/NaN contributions.
 * adam = {b1, b2, eps, step k >= 1} (ignored for SGD-m).  l2x2 = fp32(2*l2)
 * adds the L2 gradient l2x2 * w_work after the descale (w_work = fp16(W) if
 * w16 is given, else W; 0 = off; hdp_set_l2).                             */
int hdp_fused_avg_update(const void* grads, long long src_stride, int nsrc, int grads_f32, long long count,
                         float* W, float* S1, float* S2, void* w16, float* w32, float inv_scale, float lr,
                         float momentum, int optimizer, const double* adam, int* nonfinite_dev, float l2x2, void* stream);

/* Gate-contraction GEMM, C[m][n] = sum_k A(m,k) B(n,k) (+bias, ReLU),
 * fp16 operands on the tcgen05 tensor cores, fp32 accumulate.
 *   a_mn = 0: A stored [M][K] (row stride lda); 1: A stored [K][M].
 *   b_mn = 0: B stored [N][K];                  1: B stored [K][N].
 *   c_mode 0: fp32 C[m*ldc+n]; 1: fp32 C[n*ldc+m]; 2: fp16 C[m*ldc+n].
 *   bias (fp32, nullable) indexed by n, or by m if bias_on_m.
 *   ws: fp32 split-K workspace (nullable), ws_floats its size.
 *   bn, splits: 0 = automatic.                                           */
int hdp_gemm_f16(const void* A, long long lda, int a_mn, const void* B, long long ldb, int b_mn, int M, int N,
                 int K, void* C, long long ldc, int c_mode, const float* bias, int bias_on_m, int relu,
                 int accumulate, float* ws, long long ws_floats, int bn, int splits, void* stream);
/* Same contract on fp32 operands with the FP32-mode SIMT kernel (c_mode 0/1). */
int hdp_gemm_f32(const float* A, long long lda, int a_mn, const float* B, long long ldb, int b_mn, int M, int N,
                 int K, float* C, long long ldc, int c_mode, const float* bias, int bias_on_m, int relu,
                 int accumulate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HDP_H_ */
