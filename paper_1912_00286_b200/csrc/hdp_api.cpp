// libhdp.so host runtime: the C-ABI of include/hdp.h.
//
// Owns the device layout (padded, gate-interleaved, bucketed), carves the
// caller's arena, captures the per-slot forward / per-bucket backward
// sequences into CUDA graphs, and drives the bucketed NCCL exchange with the
// fused average+update kernel (K11) on a side stream so that the update of
// bucket b overlaps the BPTT of the layers below it.
#include "../../include/hdp.h"

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"
#include "head.cuh"
#include "recur.cuh"
#include "p2p_exchange.cuh"
#include "options.h"
#include "recur_trace.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK_CUDA(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(HDP_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CK_NCCL(x)                                                                              \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) return fail(HDP_ERR_NCCL, "%s: %s", #x, ncclGetErrorString(r_));    \
  } while (0)
#define CK(x)                    \
  do {                           \
    int rc_ = (x);               \
    if (rc_ != HDP_OK) return rc_; \
  } while (0)

inline long r16(long v) { return (v + 15) / 16 * 16; }
inline long rup(long v, long a) { return (v + a - 1) / a * a; }

enum Kind { K_EMBED, K_W, K_U, K_B, K_F, K_FB, K_WO, K_BO, K_FLAT };

struct Block {
  std::string name;
  Kind kind;
  int layer;
  long canon_off, rows, cols;
  long dev_off, dev_rows, dev_cols;
  int bucket;
};

struct Bucket {
  long off = 0, len = 0;  // in the device parameter vector (elements)
  long shard = 0;         // len / world
  long moff = 0;          // offset of this rank's shard in the master buffers
};

struct SlotState {
  bool fwd = false, bwd = false;
  int B = 0, T = 0;
};

struct GraphKey {
  int slot, B, T, seg;
  bool operator<(const GraphKey& o) const {
    return std::tie(slot, B, T, seg) < std::tie(o.slot, o.B, o.T, o.seg);
  }
};

}  // namespace

struct hdp_ctx {
  int world = 1, rank = 0, device = 0;
  bool host_only = false;
  ncclComm_t comm = nullptr;
  // model
  bool configured = false, bound = false, loaded = false, poisoned = false;
  hdp_model_desc d{};
  bool f32 = false;       // FP32 math mode
  bool bf = false;        // bf16 math mode (NEXT-3): bfloat16 in place of fp16 at every rounding point
  bool gf32 = false;      // fp32 gradients / wire
  bool head_fused = false;  // FC head as one fused kernel (hdp::launch_head_fused), fixed at configure
  int nslots = 1;
  long hp = 0, Ip0 = 0, Fp = 0, esz = 2, gsz = 2;
  std::vector<long> Ip;   // per layer padded input width
  std::vector<Block> blocks;
  std::vector<Bucket> buckets;  // index = bucket id; exchange order = id order
  long n_params = 0, P = 0, M_own = 0, max_bucket = 0;
  size_t arena_bytes = 0;
  // arena carve
  char* arena = nullptr;
  char* w = nullptr;      // working weights [P] (fp16 or fp32)
  float* master = nullptr;
  float* s1 = nullptr;
  float* s2 = nullptr;
  char* grads = nullptr;  // [nslots][P]
  char* recv = nullptr;
  struct Slot {
    char* stage_x;
    int8_t* stage_t;
    char* X0;
    char* Hs;
    float* C;
    char* gates;
    char* Z;
    char* dz;
    float* y;
    float* dy;
    float* loss;
    float* partials;
    float* dHh;        // fused head: dH_top = dz F [rows][hp] fp32 (written by the forward)
    unsigned* ticket;  // fused head: last-CTA counter
  };
  std::vector<Slot> slot;
  float *Gx = nullptr, *Gh = nullptr, *dH[2] = {nullptr, nullptr}, *dhrec = nullptr, *dc = nullptr;
  char *dA = nullptr, *dz = nullptr;
  char* dA2 = nullptr;  // layer-0 dA of the 2-layer backward wavefront (layer 1 keeps dA)
  bool wave_bwd = false;  // the backward ran as one wavefront launch: layer buckets are ready together
  // NEXT-2 NVLink exchange: library-owned, IPC-shared windows (gradients, fp16 weights, flags)
  bool want_p2p = false;  // desc.exchange resolved at configure time
  bool task0 = false;     // HDP_EXCH_TASK0 at world > 1: the paper-literal reduce-to-task-0 ablation
  bool loopback = false;  // HDP_EXCH_P2P at world 1: simulated workers' slots as the peers
  char* wcopies = nullptr;  // loopback: weight copies 1..nslots-1 [nslots-1][P]
  bool p2p = false;
  char *gwin = nullptr, *wwin = nullptr;
  unsigned* fwin = nullptr;
  std::vector<void*> peer_open;       // IPC mappings to close
  hdp::P2PArgs p2pa;                  // peer tables + bucket table (step / scalars filled per call)
  unsigned p2p_step = 0;              // updates so far (status slot)
  unsigned p2p_seq = 0;               // exchange launches so far (flag values)
  unsigned p2p_ctr = 0;               // CTAs of those launches (completion counter target)
  int quorum = 0;                     // NEXT-2 partial collection: contributors to wait for (0 = all)
  double partial_fraction = 1.0;
  unsigned straggler_mask = 0;        // test injection (hdp_set_option)
  unsigned long long straggler_ns = 0;
  float* Gx1 = nullptr;  // layer-1 G_x of the split forward wavefront
  float* crp = nullptr;
  size_t crp_floats = 0;
  float* ws = nullptr;
  size_t ws_floats = 0;
  int32_t *keys_in = nullptr, *keys_out = nullptr, *vals_in = nullptr, *vals_out = nullptr;
  void* sort_temp = nullptr;
  float* emb_part = nullptr;
  int32_t* emb_range = nullptr;  // [2][vocab]: first / last sorted position of each token
  size_t sort_bytes = 0;
  int* status = nullptr;  // [0] nonfinite count
  float* loadbuf = nullptr;
  // runtime
  cudaStream_t cap = nullptr, comm_stream = nullptr;
  cudaEvent_t ev_done = nullptr, ev_count = nullptr;
  std::vector<cudaEvent_t> ev_bucket;
  // layer-diagonal forward schedule (option layer_pipe): one stream + one chunk event per layer
  std::vector<cudaStream_t> lstr;
  std::vector<cudaEvent_t> ev_layer;
  cudaEvent_t ev_fork = nullptr;
  // fused head: its backward segment (column sums + dF GEMM) runs on hstr next to the layers'
  cudaStream_t hstr = nullptr;
  cudaEvent_t ev_hfork = nullptr;
  float* ws_head = nullptr;  // split-K scratch of the head's dF GEMM (concurrent with the layers' GEMMs)
  int* count_host = nullptr;  // pinned [0] non-finite count, [1] out-of-range token ids
  bool count_pending = false;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, long long> graph_kernels;  // kernels per captured graph
  long long kernels = 0;                        // library kernels enqueued so far
  // live profiler: CUDA events around every launch (eager mode, no graphs)
  bool prof = false;
  struct ProfRec {
    int tag;
    cudaEvent_t a, b;
    int nk;
    int lane = 0;  // stream: 0 caller's, 1 exchange / update, 2 head side stream, 3 + l layer pipeline
  };
  std::vector<ProfRec> precs;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  double prof_ms[HDP_K_NTAGS] = {};
  long long prof_n[HDP_K_NTAGS] = {};
  std::vector<SlotState> st;
  // schedule
  bool lr_set = false;
  double lam0 = 0, gamma = 1, n_half = 1, max_eff = 0.1, mom = 0.9, b1 = 0.9, b2 = 0.999, eps = 1e-8;
  float alpha = 10.f;
  int dyn_interval = 0;       // dynamic loss scaling: growth interval (0 = static alpha)
  float* alpha_dev() const { return reinterpret_cast<float*>(status + 11); }  // device alpha
  const float* dyn_alpha() const { return dyn_interval > 0 ? alpha_dev() : nullptr; }
  int* dyn_state() const { return status + 8; }  // [0] step count, [1] good run, [2] skipped
  double l2 = 0.0;            // L2 coefficient (reading Q16), 0 = off
  // recurrent dropout (NEXT-3; reading Q16b): keep < 1 switches it on
  double keep = 1.0;
  uint32_t drop_seed = 0, drop_thr = 0;
  float drop_scale = 1.f;
  char* hst = nullptr;        // library-owned: per slot [L][T+1][B][hp] fp16 masked recurrent inputs
  bool drop_on() const { return keep < 1.0; }
  // the per-layer persistent recurrences have no dropout; the two-layer wavefronts do
  // (the fused recurrences are fp16-only: the bf16 mode runs the per-step path)
  bool recur_ok() const { return hdp::opt(hdp::OPT_PERSISTENT) != 0 && !drop_on() && !bf; }
  bool wave_ok() const { return hdp::opt(hdp::OPT_PERSISTENT) != 0 && !bf; }
  int* drop_step() const { return status + 14; }  // completed updates (mask counter)
  char* Hst(int slot, int l) const {
    return hst + ((size_t)slot * d.n_layers + l) * (size_t)(d.max_seq + 1) * d.max_batch * hp * 2;
  }
  double* l2part = nullptr;   // partial sums of the L2 loss term
  unsigned long long* trace = nullptr;  // recurrence phase trace (option recur_trace, profile mode)
  long adam_k = 0;

  int L() const { return d.n_layers; }
  // element types (kernels.cuh ET_*) of the working copy / activations and of the gradients
  int et() const { return f32 ? hdp::ET_F32 : bf ? hdp::ET_BF16 : hdp::ET_F16; }
  int gt() const { return gf32 ? hdp::ET_F32 : bf ? hdp::ET_BF16 : hdp::ET_F16; }
  int owner_index() const { return task0 ? 0 : rank; }  // which shard of each bucket this rank owns
  int Nw() const { return world * nslots; }
  void* W(int bi) const { return w + blocks[bi].dev_off * esz; }
  void* G(int s, int bi) const { return grads + ((long)s * P + blocks[bi].dev_off) * gsz; }
  int find(const char* n) const {
    for (size_t i = 0; i < blocks.size(); ++i)
      if (blocks[i].name == n) return (int)i;
    return -1;
  }
};

// ====================================================================== layout
namespace {

void build_layout(hdp_ctx* c) {
  const hdp_model_desc& d = c->d;
  c->blocks.clear();
  c->buckets.clear();
  const long h = d.hidden;
  c->hp = r16(h);
  c->Ip0 = d.vocab > 0 ? r16(d.embed_dim) : r16(d.input_dim);
  c->Fp = d.fc_hidden > 0 ? r16(d.fc_hidden) : 0;
  c->Ip.assign(d.n_layers, c->hp);
  if (d.n_layers > 0) c->Ip[0] = c->Ip0;
  long canon = 0;
  auto add = [&](const char* name, Kind k, int layer, long rows, long cols, long drows, long dcols) {
    Block b;
    b.name = name;
    b.kind = k;
    b.layer = layer;
    b.canon_off = canon;
    b.rows = rows;
    b.cols = cols;
    b.dev_rows = drows;
    b.dev_cols = dcols;
    b.dev_off = 0;
    b.bucket = -1;
    canon += rows * cols;
    c->blocks.push_back(b);
  };
  if (d.n_layers == 0) {
    add("flat", K_FLAT, -1, d.flat_params, 1, d.flat_params, 1);
  } else {
    const long i0 = d.vocab > 0 ? d.embed_dim : d.input_dim;
    if (d.vocab > 0) add("E", K_EMBED, -1, d.vocab, d.embed_dim, d.vocab, c->Ip0);
    char nm[16];
    for (int l = 0; l < d.n_layers; ++l) {
      const long il = l == 0 ? i0 : h;
      snprintf(nm, sizeof nm, "W%d", l);
      add(nm, K_W, l, 4 * h, il, 4 * c->hp, c->Ip[l]);
      snprintf(nm, sizeof nm, "U%d", l);
      add(nm, K_U, l, 4 * h, h, 4 * c->hp, c->hp);
      snprintf(nm, sizeof nm, "b%d", l);
      add(nm, K_B, l, 4 * h, 1, 4 * c->hp, 1);
    }
    if (d.fc_hidden > 0) {
      add("F", K_F, -1, d.fc_hidden, h, c->Fp, c->hp);
      add("fb", K_FB, -1, d.fc_hidden, 1, c->Fp, 1);
      add("wo", K_WO, -1, d.fc_hidden, 1, c->Fp, 1);
    } else {
      add("wo", K_WO, -1, h, 1, c->hp, 1);
    }
    add("bo", K_BO, -1, 1, 1, 1, 1);
  }
  c->n_params = canon;
  // buckets in readiness order: head, layer L-1 .. 0, embedding
  std::vector<std::vector<int>> groups;
  if (d.n_layers == 0) {
    groups.push_back({0});
  } else {
    std::vector<int> head, emb;
    std::vector<std::vector<int>> lay(d.n_layers);
    for (size_t i = 0; i < c->blocks.size(); ++i) {
      const Block& b = c->blocks[i];
      if (b.kind == K_EMBED) emb.push_back((int)i);
      else if (b.layer >= 0) lay[b.layer].push_back((int)i);
      else head.push_back((int)i);
    }
    groups.push_back(head);
    for (int l = d.n_layers - 1; l >= 0; --l) groups.push_back(lay[l]);
    if (!emb.empty()) groups.push_back(emb);
  }
  // owner-sharded: every bucket split into `world` shards; task 0 (the paper-literal
  // ablation) owns whole buckets
  const int nshard = c->task0 ? 1 : c->world;
  const long align_bucket = 64L * nshard;
  long off = 0, moff = 0;
  c->max_bucket = 0;
  for (size_t g = 0; g < groups.size(); ++g) {
    Bucket bk;
    bk.off = off;
    long p = off;
    for (int bi : groups[g]) {
      Block& b = c->blocks[bi];
      p = rup(p, 64);
      b.dev_off = p;
      b.bucket = (int)g;
      p += b.dev_rows * b.dev_cols;
    }
    bk.len = rup(p - off, align_bucket);
    bk.shard = bk.len / nshard;
    bk.moff = moff;
    moff += bk.shard;
    off += bk.len;
    c->max_bucket = std::max(c->max_bucket, bk.len);
    c->buckets.push_back(bk);
  }
  c->P = off;
  c->M_own = moff;
}

// canonical (r, col) -> device element offset within the block
inline long dev_index(const hdp_ctx* c, const Block& b, long r, long col) {
  if (b.kind == K_W || b.kind == K_U || b.kind == K_B) {
    const long h = c->d.hidden;
    const long g = r / h, j = r % h;
    return (4 * j + g) * b.dev_cols + col;  // gate rows interleaved per unit
  }
  return r * b.dev_cols + col;
}

struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(char* b) : base(b) {}
  char* take(size_t bytes) {
    off = rup(off, 256);
    char* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

size_t gemm_need(int M, int N, int K) {
  // mirror of the automatic split heuristic's worst case: splits <= 16
  (void)K;
  return (size_t)16 * M * N;
}

void carve(hdp_ctx* c, char* base) {
  const hdp_model_desc& d = c->d;
  Carver cv(base);
  const long P = c->P;
  c->w = cv.take(P * c->esz);
  c->master = (float*)cv.take(c->M_own * 4);
  c->s1 = (float*)cv.take(c->M_own * 4);
  c->s2 = d.optimizer == HDP_OPT_ADAM ? (float*)cv.take(c->M_own * 4) : nullptr;  // Adam's v only
  c->grads = cv.take((size_t)c->nslots * P * c->gsz);
  // bucket bi received at its own offset (task 0: every rank's whole vector, [world][P] on rank 0)
  c->recv = cv.take(c->world > 1 ? (c->task0 ? (c->rank == 0 ? (size_t)c->world : 0) : 1) * c->P * c->gsz : 0);
  c->status = (int*)cv.take(32768);  // [0] non-finite count, [16] out-of-range token ids;
                                       // +1024 B: recurrence barrier counters;
                                       // +4096 B: backward-wavefront hand-off counters
  c->wcopies = cv.take(c->loopback ? (size_t)(c->nslots - 1) * P * c->esz : 0);
  c->l2part = (double*)cv.take(hdp::l2_partials_doubles() * sizeof(double));
  c->slot.assign(c->nslots, hdp_ctx::Slot{});
  if (d.n_layers > 0) {
    const long B = d.max_batch, T = d.max_seq, L = d.n_layers, hp = c->hp, e = c->esz;
    const long rows = B * T;
    const long in_bytes = d.vocab > 0 ? 4 : (long)d.input_dim * e;
    for (int s = 0; s < c->nslots; ++s) {
      hdp_ctx::Slot& S = c->slot[s];
      S.stage_x = cv.take(rows * in_bytes);
      S.stage_t = (int8_t*)cv.take(rows);
      S.X0 = cv.take(rows * c->Ip0 * e);
      S.Hs = cv.take(L * (T + 1) * B * hp * e);
      S.C = (float*)cv.take(L * T * B * hp * 4);
      S.gates = cv.take(L * T * B * 4 * hp * e);
      // (the fused head keeps its per-CTA column partials here: grid x (2 Fp + 1) doubles)
      S.Z = cv.take(c->Fp ? std::max(rows * c->Fp * e,
                                     c->head_fused ? (long)hdp::head_fused_grid((int)rows) * (2 * c->Fp + 1) * 8 : 0L)
                          : 0);
      S.dz = cv.take(c->Fp ? rows * c->Fp * e : 0);  // A5's ReLU' output, written by the forward's head_out
      S.y = (float*)cv.take(rows * 4);
      S.dy = (float*)cv.take(rows * 4);
      S.loss = (float*)cv.take(4);
      S.partials = (float*)cv.take(hdp::head_partials_count((int)rows) * 4);
      // fused head: dH_top per slot (the backward of this slot reads it)
      S.dHh = (float*)cv.take(c->head_fused ? rows * hp * 4 : 0);
      S.ticket = (unsigned*)cv.take(c->head_fused ? 4 : 0);
    }
    c->Gx = (float*)cv.take(rows * 4 * hp * 4);
    c->Gh = (float*)cv.take(B * 4 * hp * 4);
    c->dA = cv.take(rows * 4 * hp * e);
    c->dA2 = cv.take(L == 2 && !c->f32 ? rows * 4 * hp * e : 0);
    c->Gx1 = (float*)cv.take(L == 2 && !c->f32 ? rows * 4 * hp * 4 : 0);
    const long dw = std::max(hp, c->Ip0);
    c->dH[0] = (float*)cv.take(rows * dw * 4);
    c->dH[1] = (float*)cv.take(rows * dw * 4);
    c->dhrec = (float*)cv.take(B * hp * 4);
    c->dc = (float*)cv.take(B * hp * 4);
    c->dz = nullptr;  // (per slot: S.dz)
    const long maxcols = std::max(std::max(4 * hp, 2 * c->Fp + 1), std::max(hp, 1L));
    c->crp_floats = hdp::colreduce_partials_floats((int)rows, (int)maxcols);
    c->crp = (float*)cv.take(c->crp_floats * 4);
    // split-K workspace for the weight-gradient GEMMs (K = B*T)
    size_t ws = 0;
    for (int l = 0; l < L; ++l) {
      ws = std::max(ws, gemm_need((int)(4 * hp), (int)c->Ip[l], (int)rows));
      ws = std::max(ws, gemm_need((int)(4 * hp), (int)hp, (int)rows));
    }
    if (c->Fp) ws = std::max(ws, gemm_need((int)c->Fp, (int)hp, (int)rows));
    ws = std::max(ws, (size_t)16 * B * hp);  // K7 partials of the fused cell backward
    if (c->f32) ws = 0;
    c->ws_floats = ws;
    c->ws = (float*)cv.take(ws * 4);
    c->ws_head = (float*)cv.take(c->head_fused ? gemm_need((int)c->Fp, (int)hp, (int)rows) * 4 : 0);
    if (d.vocab > 0) {
      c->keys_in = (int32_t*)cv.take(rows * 4);
      c->keys_out = (int32_t*)cv.take(rows * 4);
      c->vals_in = (int32_t*)cv.take(rows * 4);
      c->vals_out = (int32_t*)cv.take(rows * 4);
      c->sort_bytes = hdp::embed_sort_temp_bytes((int)rows);
      c->sort_temp = cv.take(c->sort_bytes);
      c->emb_part = (float*)cv.take(hdp::embed_part_floats((int)rows, (int)c->Ip0) * 4);
      c->emb_range = (int32_t*)cv.take((size_t)2 * d.vocab * 4);
    }
  }
  c->arena_bytes = rup(cv.off, 256);
}

// ---------------------------------------------------------------- profiler
cudaEvent_t prof_event(hdp_ctx* c) {
  if (c->evused == c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->evused++];
}
// Counts the kernels a launch site enqueues and, when profiling, brackets
// them with CUDA events on the launching stream.
struct KScope {
  hdp_ctx* c;
  int tag, nk;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  KScope(hdp_ctx* c_, int tag_, int nk_, cudaStream_t s_) : c(c_), tag(tag_), nk(nk_), s(s_) {
    if (c->prof) {
      a = prof_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~KScope() {
    c->kernels += nk;
    if (c->prof) {
      cudaEvent_t b = prof_event(c);
      cudaEventRecord(b, s);
      int lane = 0;
      if (s == c->comm_stream) lane = 1;
      else if (s == c->hstr) lane = 2;
      else
        for (size_t l = 0; l < c->lstr.size(); ++l)
          if (s == c->lstr[l]) lane = 3 + (int)l;
      c->precs.push_back({tag, a, b, nk, lane});
    }
  }
};

// ---------------------------------------------------------------- recurrence phase trace
// Option recur_trace = 1 in profile (eager) mode: the persistent / wavefront kernels stamp
// %globaltimer per phase; trace_report (recur_trace.cpp) prints the per-step means.
unsigned long long* trace_buffer(hdp_ctx* c, size_t words) {
  if (!c->prof || !hdp::opt(hdp::OPT_RECUR_TRACE)) return nullptr;
  if (!c->trace && cudaMalloc(&c->trace, ((size_t)6 * 8192 * 5 + 6 * 148 + 16) * sizeof(unsigned long long)) != cudaSuccess) {
    c->trace = nullptr;
    return nullptr;
  }
  (void)words;
  cudaMemset(c->trace, 0, ((size_t)6 * 8192 * 5 + 6 * 148 + 16) * sizeof(unsigned long long));
  return c->trace;
}
int trace_report(hdp_ctx* c, hdp::TraceKind kind, const unsigned long long* dev, int T, int layer, cudaStream_t s) {
  (void)c;
  if (T > 8192) return HDP_OK;
  std::vector<unsigned long long> h((size_t)6 * T * 5 + 6 * 148 + 16);  // + per-CTA entry / exit / role stamps, W-role stamps
  CK_CUDA(cudaStreamSynchronize(s));
  CK_CUDA(cudaMemcpy(h.data(), dev, h.size() * 8, cudaMemcpyDeviceToHost));
  hdp::print_trace(kind, h.data(), T, layer);
  return HDP_OK;
}

// ---------------------------------------------------------------- GEMM helper
int gemm(hdp_ctx* c, int tag, const void* A, long lda, int amn, const void* B, long ldb, int bmn, long M, long N,
         long K, const hdp::Epilogue& epi, cudaStream_t s, int force_bn = 0, int force_splits = 0,
         float* ws = nullptr /* split-K scratch; nullptr = the context's */) {
  hdp::GemmPlan p;
  int r;
  hdp::Epilogue ebf = epi;
  ebf.bf16 = c->bf ? 1 : 0;  // bf16 math mode: bfloat16 operands (idesc format bits) and 16-bit outputs
  if (c->f32)
    r = hdp::gemm_plan_f32(&p, (const float*)A, lda, amn, (const float*)B, ldb, bmn, (int)M, (int)N, (int)K, epi);
  else
    r = hdp::gemm_plan_tc(&p, (const __half*)A, lda, amn, (const __half*)B, ldb, bmn, (int)M, (int)N, (int)K, ebf,
                          ws ? ws : c->ws, c->ws_floats, force_bn, force_splits);
  if (r) return fail(HDP_ERR_ARG, "gemm plan %ldx%ldx%ld: %s", M, N, K, hdp::gemm_last_error());
  KScope ks(c, tag, p.tc && p.cr == 1 && (p.splits > 1 || epi.mode == hdp::EPI_LSTM_BWD) ? 2 : 1, s);
  CK_CUDA(hdp::gemm_run(p, s));
  return HDP_OK;
}

hdp::Epilogue epi_f32(void* out, long ldo, const void* bias = nullptr, int bias_f16 = 0) {
  hdp::Epilogue e;
  e.mode = hdp::EPI_F32;
  e.out = out;
  e.ldo = ldo;
  e.bias = bias;
  e.bias_f16 = bias_f16;
  return e;
}
// activation / gradient output in the working element type
hdp::Epilogue epi_elem(bool f32, void* out, long ldo) {
  hdp::Epilogue e;
  e.mode = f32 ? hdp::EPI_F32 : hdp::EPI_F16;
  e.out = out;
  e.ldo = ldo;
  return e;
}

// ---------------------------------------------------------------- forward
// A2 + A3 of layer l for t in [t0, t1): K2 with the cell in its epilogue (K3 alone at t = 0
// and in FP32 mode), reading the input projection from Gxb; split-K scratch wsb (nullable:
// the context's).  The per-step path of hdp_lstm_forward, whole or one time chunk at a time.
int fwd_steps(hdp_ctx* c, int si, int B, int T, int l, int t0, int t1, float* Gxb, cudaStream_t s, float* wsb) {
  const hdp_model_desc& d = c->d;
  hdp_ctx::Slot& S = c->slot[si];
  const long hp = c->hp, e = c->esz;
  const int f32 = c->f32;
  const int et = c->et();
  const long hs_layer = (long)(T + 1) * B * hp, c_layer = (long)T * B * hp, g_layer = (long)T * B * 4 * hp;
  (void)d;
  char nm[16];
  snprintf(nm, sizeof nm, "U%d", l);
  const int iU = c->find(nm);
  char* Hs = S.Hs + l * hs_layer * e;
  float* Cl = S.C + l * c_layer;
  char* Gl = S.gates + l * g_layer * e;
for (int t = t0; t < t1; ++t) {
    if (t > 0 && !f32) {
      // K2 with A3 in its epilogue: gates = h_{t-1} U^T + G_x[t] -> cell -> gates, c_t, h_t
      // (recurrent dropout: the GEMM reads h~_{t-1}, the epilogue also writes h~_t)
      hdp::Epilogue ef;
      const char* hin = c->drop_on() ? c->Hst(si, l) : Hs;
      if (c->drop_on()) {
        ef.htout = c->Hst(si, l) + (long)(t + 1) * B * hp * e;
        ef.drop_step = c->drop_step();
        ef.drop_seed = c->drop_seed;
        ef.drop_thr = c->drop_thr;
        ef.drop_layer = (uint32_t)l;
        ef.drop_seq0 = (uint32_t)((c->rank * c->nslots + si) * B);
        ef.drop_scale = c->drop_scale;
      }
      ef.mode = hdp::EPI_LSTM_FWD;
      ef.hp = (int)hp;
      ef.gx = Gxb + (long)t * B * 4 * hp;
      ef.cprev = Cl + (long)(t - 1) * B * hp;
      ef.cout = Cl + (long)t * B * hp;
      ef.gates = Gl + (long)t * B * 4 * hp * e;
      ef.hout = Hs + (long)(t + 1) * B * hp * e;
      CK(gemm(c, HDP_K_GEMM_H, hin + (long)t * B * hp * e, hp, 0, c->W(iU), hp, 0, B, 4 * hp, hp, ef, s, 0, 0, wsb));
      continue;
    }
    if (t > 0)  // K2: G_h = h_{t-1} U^T (A2)
      CK(gemm(c, HDP_K_GEMM_H, Hs + (long)t * B * hp * e, hp, 0, c->W(iU), hp, 0, B, 4 * hp, hp, epi_f32(c->Gh, 4 * hp), s, 0, 0, wsb));
    // K3 (A3)
    {
      KScope ks_(c, HDP_K_CELL_FWD, 1, s);
      CK_CUDA(hdp::launch_cell_fwd(et, Gxb + (long)t * B * 4 * hp, t > 0 ? c->Gh : nullptr,
                                   t > 0 ? Cl + (long)(t - 1) * B * hp : nullptr, Gl + (long)t * B * 4 * hp * e,
                                   Cl + (long)t * B * hp, Hs + (long)(t + 1) * B * hp * e, B, (int)hp, s));
    }
    if (c->drop_on()) {  // h~_0 (the fused epilogues write the later ones)
      KScope ks_(c, HDP_K_CELL_FWD, 1, s);
      CK_CUDA(hdp::launch_drop_mask(Hs + (long)(t + 1) * B * hp * e, c->Hst(si, l) + (long)(t + 1) * B * hp * e, B,
                                    (int)hp, c->drop_step(), c->drop_seed, (uint32_t)l,
                                    (uint32_t)((c->rank * c->nslots + si) * B), c->drop_thr, c->drop_scale, s));
    }
  }
  return HDP_OK;
}

int enqueue_forward(hdp_ctx* c, int si, int B, int T, cudaStream_t s) {
  const hdp_model_desc& d = c->d;
  hdp_ctx::Slot& S = c->slot[si];
  const long hp = c->hp, e = c->esz, L = d.n_layers;
  const long rows = (long)B * T;
  const int f32 = c->f32;
  const int et = c->et();  // element type passed to the non-GEMM launchers
  const long hs_layer = (long)(T + 1) * B * hp;  // elements per layer in Hs (actual B, T)
  const long c_layer = (long)T * B * hp;
  const long g_layer = (long)T * B * 4 * hp;
  // h_{-1} = 0 of every layer (row 0 of its Hs block): zeroed by the input-packing launch
  // (row bytes B h_p e and the layer stride are multiples of 16 B: h_p is a multiple of 16)
  hdp::ZeroRows zr;
  zr.base = reinterpret_cast<uint4*>(S.Hs);
  zr.stride = hs_layer * e / 16;
  zr.nvec = (long)B * hp * e / 16;
  zr.count = (int)L;
  if (d.vocab > 0)
    for (int l = 0; l < L; ++l) CK_CUDA(cudaMemsetAsync(S.Hs + l * hs_layer * e, 0, B * hp * e, s));
  if (d.vocab > 0)
    {
      KScope ks_(c, HDP_K_INPUT, 1, s);
      CK_CUDA(hdp::launch_embed_gather((const int32_t*)S.stage_x, B, T, c->W(c->find("E")), (int)c->Ip0, S.X0, et,
                                       d.vocab, c->status + 16, s));
    }
  else
    {
      KScope ks_(c, HDP_K_INPUT, 1, s);
      CK_CUDA(hdp::launch_pack_input(S.stage_x, et, B, T, d.input_dim, (int)c->Ip0, S.X0, et, s, zr));
    }
  char nm[16];
  // Layer-diagonal schedule of the per-step path (NEXT-1 at C4 scale; PAPER.md:82 BPTT over a
  // stacked LSTM): layer l's chunk of Tc steps needs only layer l-1's h over the same chunk,
  // so the L layers run as a pipeline on L streams -- layer l's K1 over the chunk's rows, then
  // its K2 + A3 steps -- and up to L per-step GEMMs (one per layer, different U) are in
  // flight at once instead of one (measured: two concurrent K2 chains 15.8 -> 12.6 us per GEMM,
  // tools/concurrent_gemm.py).  Same kernels, same per-element arithmetic as the sequential
  // loop.  G_x is shared: rows of chunk c are rewritten by layer l+1's K1 only after layer l
  // finished chunk c (its event), so one T x B x 4h_p buffer serves every layer.
  const int tc = hdp::opt(hdp::OPT_LAYER_PIPE);
  const bool any_fused = (L == 2 && !f32 && c->wave_ok() && hdp::recur2_fwd_supported(B, (int)hp)) ||
                         (!f32 && c->recur_ok() && hdp::recur_fwd_supported(B, (int)hp));
  if (tc > 0 && L >= 2 && !f32 && !any_fused && (int)c->lstr.size() >= L) {
    CK_CUDA(cudaEventRecord(c->ev_fork, s));
    for (int l = 0; l < L; ++l) CK_CUDA(cudaStreamWaitEvent(c->lstr[l], c->ev_fork, 0));
    for (int t0 = 0; t0 < T; t0 += tc) {
      const int t1 = t0 + tc < T ? t0 + tc : T;
      for (int l = 0; l < L; ++l) {
        cudaStream_t ls = c->lstr[l];
        if (l > 0) CK_CUDA(cudaStreamWaitEvent(ls, c->ev_layer[l - 1], 0));
        snprintf(nm, sizeof nm, "W%d", l);
        const int iW = c->find(nm);
        snprintf(nm, sizeof nm, "b%d", l);
        const int ib = c->find(nm);
        const long Ipl = c->Ip[l];
        const char* X = l == 0 ? S.X0 : S.Hs + ((l - 1) * hs_layer + (long)B * hp) * e;
        CK(gemm(c, HDP_K_GEMM_X, X + (long)t0 * B * Ipl * e, Ipl, 0, c->W(iW), Ipl, 0, (long)(t1 - t0) * B, 4 * hp,
                Ipl, epi_f32(c->Gx + (long)t0 * B * 4 * hp, 4 * hp, c->W(ib), 1), ls));
        CK(fwd_steps(c, si, B, T, l, t0, t1, c->Gx, ls, nullptr));
        CK_CUDA(cudaEventRecord(c->ev_layer[l], ls));
      }
    }
    for (int l = 0; l < L; ++l) CK_CUDA(cudaStreamWaitEvent(s, c->ev_layer[l], 0));
  }
  for (int l = 0; l < L; ++l) {
    if (tc > 0 && L >= 2 && !f32 && !any_fused && (int)c->lstr.size() >= L) break;  // done above
    snprintf(nm, sizeof nm, "W%d", l);
    const int iW = c->find(nm);
    snprintf(nm, sizeof nm, "U%d", l);
    const int iU = c->find(nm);
    snprintf(nm, sizeof nm, "b%d", l);
    const int ib = c->find(nm);
    const long Ipl = c->Ip[l];
    const char* X = l == 0 ? S.X0 : S.Hs + ((l - 1) * hs_layer + (long)B * hp) * e;
    char* Hs = S.Hs + l * hs_layer * e;
    float* Cl = S.C + l * c_layer;
    char* Gl = S.gates + l * g_layer * e;
    const bool wave = l == 0 && L == 2 && !f32 && c->wave_ok() && hdp::recur2_fwd_supported(B, (int)hp);
    const bool fusex = wave && hdp::recur2_fwd_fuses_x(B, (int)hp, (int)Ipl);
    // K1: G_x = X W^T + b for all t (A1); inside the wavefront's layer-0 role when fused
    if (!fusex)
      CK(gemm(c, HDP_K_GEMM_X, X, Ipl, 0, c->W(iW), Ipl, 0, rows, 4 * hp, Ipl, epi_f32(c->Gx, 4 * hp, c->W(ib), !f32), s));
    if (wave) {
      // both layers' recurrences as one wavefront; layer 1's input projection runs inside
      hdp::Recur2FwdArgs ra;
      ra.U0 = (const __half*)c->W(iU);
      ra.W1 = (const __half*)c->W(c->find("W1"));
      ra.U1 = (const __half*)c->W(c->find("U1"));
      ra.b1 = (const __half*)c->W(c->find("b1"));
      ra.Gx0 = c->Gx;
      if (fusex) {
        ra.X0 = (const __half*)X;
        ra.W0 = (const __half*)c->W(iW);
        ra.b0 = (const __half*)c->W(ib);
        ra.Ip0 = (int)Ipl;
      }
      ra.a1x = c->Gx1;
      ra.flags = (unsigned*)((char*)c->status + 4096);
      ra.Hs0 = (__half*)Hs;
      ra.C0 = Cl;
      ra.gates0 = (__half*)Gl;
      ra.Hs1 = (__half*)(S.Hs + hs_layer * e);
      ra.C1 = S.C + c_layer;
      ra.gates1 = (__half*)(S.gates + g_layer * e);
      ra.T = T;
      ra.B = B;
      ra.hp = (int)hp;
      if (c->drop_on()) {  // recurrent dropout inside the wavefront (NEXT-3)
        ra.Ht0 = (__half*)c->Hst(si, 0);
        ra.Ht1 = (__half*)c->Hst(si, 1);
        ra.drop_step = c->drop_step();
        ra.drop_seed = c->drop_seed;
        ra.drop_thr = c->drop_thr;
        ra.drop_seq0 = (uint32_t)((c->rank * c->nslots + si) * B);
        ra.drop_scale = c->drop_scale;
      }
      ra.trace = trace_buffer(c, 4 * 8192 * 5);
      {
        KScope ks_(c, HDP_K_RECUR_FWD, 1, s);
        CK_CUDA(hdp::launch_recur2_fwd(ra, s));
      }
      if (ra.trace) CK(trace_report(c, hdp::TRACE_FWD_WAVEFRONT, ra.trace, T, l, s));
      break;
    }
    if (!f32 && c->recur_ok() && hdp::recur_fwd_supported(B, (int)hp)) {
      // A2 + A3 for all t in one persistent kernel (U resident in SMEM)
      hdp::RecurFwdArgs ra;
      ra.U = (const __half*)c->W(iU);
      ra.Gx = c->Gx;
      ra.Hs = (__half*)Hs;
      ra.C = Cl;
      ra.gates = (__half*)Gl;
      ra.T = T;
      ra.B = B;
      ra.hp = (int)hp;
      ra.trace = trace_buffer(c, 8192 * 5);
      {
        KScope ks_(c, HDP_K_RECUR_FWD, 1, s);
        CK_CUDA(hdp::launch_recur_fwd(ra, s));
      }
      if (ra.trace) CK(trace_report(c, hdp::TRACE_FWD_LAYER, ra.trace, T, l, s));
      continue;
    }
    CK(fwd_steps(c, si, B, T, l, 0, T, c->Gx, s, nullptr));
  }
  // head (A4)
  const char* Htop = S.Hs + ((L - 1) * hs_layer + (long)B * hp) * e;
  const int iwo = c->find("wo"), ibo = c->find("bo");
  if (d.fc_hidden > 0 && c->head_fused) {
    // A4 + A5 (but dF) in one launch: z, y, loss, dy, dz, dH_top and the head's column partials
    hdp::HeadFusedArgs ha;
    ha.H = Htop;
    ha.F = c->W(c->find("F"));
    ha.fb = c->W(c->find("fb"));
    ha.wo = c->W(iwo);
    ha.bo = c->W(ibo);
    ha.tgt = S.stage_t;
    ha.dz = S.dz;
    ha.y = S.y;
    ha.dy = S.dy;
    ha.hinge = S.partials;
    ha.colpart = reinterpret_cast<double*>(S.Z);
    ha.loss = S.loss;
    ha.ticket = S.ticket;
    ha.dH = S.dHh;
    ha.rows = (int)rows;
    ha.B = B;
    ha.T = T;
    ha.hp = (int)hp;
    ha.Fp = (int)c->Fp;
    ha.alpha = c->alpha;
    ha.inv_terms = 1.f / (float)rows;
    ha.alpha_dev = c->dyn_alpha();
    ha.trace = trace_buffer(c, (size_t)hdp::head_fused_grid((int)rows) * 8);
    ha.pdl = hdp::opt(hdp::OPT_FWD_PDL) == 1;
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_head_fused(ha, s));
    }
    if (ha.trace && hdp::head_fused_grid((int)rows) <= 8192) CK(trace_report(c, hdp::TRACE_HEAD, ha.trace, hdp::head_fused_grid((int)rows), 0, s));
  } else if (d.fc_hidden > 0) {
    const int iF = c->find("F"), ifb = c->find("fb");
    hdp::Epilogue ez = epi_elem(f32, S.Z, c->Fp);
    ez.bias = c->W(ifb);
    ez.bias_f16 = !f32;
    ez.relu = 1;  // R7
    CK(gemm(c, HDP_K_HEAD_FWD, Htop, hp, 0, c->W(iF), hp, 0, rows, c->Fp, hp, ez, s));
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_head_out(et, S.Z, (int)rows, (int)c->Fp, c->Fp, c->W(iwo), c->W(ibo), S.stage_t, 0, B, T,
                                   c->alpha, 1.f / (float)rows, S.y, S.dy, S.partials, s, S.dz, c->dyn_alpha()));
    }
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_loss_final(S.partials, hdp::head_partials_count((int)rows), 1.f / (float)rows, S.loss, s));
    }
  } else if (d.head_last_step) {
    const char* Hlast = S.Hs + ((L - 1) * hs_layer + (long)T * B * hp) * e;
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_head_out(et, Hlast, B, (int)hp, hp, c->W(iwo), c->W(ibo), S.stage_t, 1, B, T, c->alpha,
                                   1.f / (float)B, S.y, S.dy, S.partials, s, nullptr, c->dyn_alpha()));
    }
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_loss_final(S.partials, hdp::head_partials_count(B), 1.f / (float)B, S.loss, s));
    }
  } else {
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_head_out(et, Htop, (int)rows, (int)hp, hp, c->W(iwo), c->W(ibo), S.stage_t, 0, B, T,
                                   c->alpha, 1.f / (float)rows, S.y, S.dy, S.partials, s, nullptr, c->dyn_alpha()));
    }
    {
      KScope ks_(c, HDP_K_HEAD_FWD, 1, s);
      CK_CUDA(hdp::launch_loss_final(S.partials, hdp::head_partials_count((int)rows), 1.f / (float)rows, S.loss, s));
    }
  }
  if (c->l2 > 0) {  // reported loss += l2 * ||w||^2 over the working weights
    KScope ks_(c, HDP_K_HEAD_FWD, 2, s);
    CK_CUDA(hdp::launch_l2_loss(et, c->w, c->P, c->l2part, c->l2, S.loss, s));
  }
  return HDP_OK;
}

// ---------------------------------------------------------------- backward
// seg 0 = head; seg 1 + k = layer L-1-k
int enqueue_backward_seg(hdp_ctx* c, int si, int B, int T, int seg, cudaStream_t s) {
  const hdp_model_desc& d = c->d;
  hdp_ctx::Slot& S = c->slot[si];
  const long hp = c->hp, e = c->esz, L = d.n_layers;
  const long rows = (long)B * T;
  const int f32 = c->f32, gf = c->gf32;
  const int et = c->et(), gt = c->gt();  // element types passed to the non-GEMM launchers
  const long hs_layer = (long)(T + 1) * B * hp;
  const long c_layer = (long)T * B * hp;
  const long g_layer = (long)T * B * 4 * hp;
  const char* Htop = S.Hs + ((L - 1) * hs_layer + (long)B * hp) * e;
  const int iwo = c->find("wo"), ibo = c->find("bo");
  if (seg == 0) {
    if (d.fc_hidden > 0 && c->head_fused) {
      const int iF = c->find("F"), ifb = c->find("fb");
      const long Fp = c->Fp;
      // the forward's fused head left dz, dH_top and per-CTA column partials: dwo, dfb, dbo
      // by the fixed-order fp64 pass 2, dF = dz^T H by the GEMM
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 1, s);
        CK_CUDA(hdp::launch_colreduce3_final(reinterpret_cast<const double*>(S.Z), hdp::head_fused_grid((int)rows),
                                             (int)Fp, gt, c->G(si, iwo), c->G(si, ifb), c->G(si, ibo), s));
      }
      CK(gemm(c, HDP_K_HEAD_BWD, S.dz, Fp, 1, Htop, hp, 1, Fp, hp, rows, epi_elem(gf, c->G(si, iF), hp), s, 0, 0,
              c->ws_head));
    } else if (d.fc_hidden > 0) {
      const int iF = c->find("F"), ifb = c->find("fb");
      const long Fp = c->Fp;
      // dz (R9) was written by the forward's head_out; dwo, dfb, dbo in one fused column pass
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 2, s);
        CK_CUDA(hdp::launch_colreduce3(et, S.Z, S.dz, Fp, (int)rows, (int)Fp, S.dy, c->crp, gt, c->G(si, iwo),
                                       c->G(si, ifb), c->G(si, ibo), s));
      }
      // dF = dz^T H   (M = Fp, N = hp, K = B*T; both operands MN-major)
      CK(gemm(c, HDP_K_HEAD_BWD, S.dz, Fp, 1, Htop, hp, 1, Fp, hp, rows, epi_elem(gf, c->G(si, iF), hp), s));
      // dH_top = dz F (M = B*T, N = hp, K = Fp; F read MN-major)
      CK(gemm(c, HDP_K_HEAD_BWD, S.dz, Fp, 0, c->W(iF), hp, 1, rows, hp, Fp, epi_f32(c->dH[0], hp), s));
    } else if (d.head_last_step) {
      const char* Hlast = S.Hs + ((L - 1) * hs_layer + (long)T * B * hp) * e;
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 1, s);
        CK_CUDA(hdp::launch_outer(et, S.dy, c->W(iwo), c->dH[0], B, (int)hp, s));
      }
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 2, s);
        CK_CUDA(hdp::launch_colreduce(et, Hlast, hp, B, (int)hp, S.dy, c->crp, gt, c->G(si, iwo), s));
      }
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 2, s);
        CK_CUDA(hdp::launch_colreduce(1, S.dy, 1, B, 1, nullptr, c->crp, gt, c->G(si, ibo), s));
      }
    } else {
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 1, s);
        CK_CUDA(hdp::launch_outer(et, S.dy, c->W(iwo), c->dH[0], (int)rows, (int)hp, s));
      }
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 2, s);
        CK_CUDA(hdp::launch_colreduce(et, Htop, hp, (int)rows, (int)hp, S.dy, c->crp, gt, c->G(si, iwo), s));
      }
      {
        KScope ks_(c, HDP_K_HEAD_BWD, 2, s);
        CK_CUDA(hdp::launch_colreduce(1, S.dy, 1, (int)rows, 1, nullptr, c->crp, gt, c->G(si, ibo), s));
      }
    }
    return HDP_OK;
  }
  const int l = (int)(L - seg);
  // dH_above of this layer lives in dH[(L-1-l) & 1]
  float* dHa = l == L - 1 && c->head_fused ? S.dHh : c->dH[(L - 1 - l) & 1];
  float* dHnext = c->dH[(L - l) & 1];
  char nm[16];
  snprintf(nm, sizeof nm, "W%d", l);
  const int iW = c->find(nm);
  snprintf(nm, sizeof nm, "U%d", l);
  const int iU = c->find(nm);
  snprintf(nm, sizeof nm, "b%d", l);
  const int ib = c->find(nm);
  const long Ipl = c->Ip[l];
  const char* X = l == 0 ? S.X0 : S.Hs + ((l - 1) * hs_layer + (long)B * hp) * e;
  const char* Hs = S.Hs + l * hs_layer * e;
  float* Cl = S.C + l * c_layer;
  const char* Gl = S.gates + l * g_layer * e;
  const bool last_only = d.head_last_step && l == L - 1;
  // 2 layers, mixed mode: both layers' BPTT and the dX1 projection in one wavefront
  // launch (segment for layer 1); layer 0's segment then only has its K8 / K9 work
  const bool wave = L == 2 && !f32 && c->wave_ok() && hdp::recur2_bwd_supported(B, (int)hp);
  // ... and, on the SMs the recurrences leave idle, the A8 weight gradients of both layers
  const bool wgrad = wave && !gf && hdp::recur2_bwd_wgrad(B, (int)hp, (int)c->Ip0);
  if (wave) c->wave_bwd = true;
  char* dAl = wave && l == 0 ? c->dA2 : c->dA;
  if (wave && l == 1) {
    hdp::Recur2BwdArgs wa;
    wa.U0 = (const __half*)c->W(c->find("U0"));
    wa.U1 = (const __half*)c->W(iU);
    wa.W1 = (const __half*)c->W(iW);
    wa.dHtop = dHa;
    wa.dHtop_last_only = last_only ? 1 : 0;
    wa.gates0 = (const __half*)S.gates;
    wa.gates1 = (const __half*)Gl;
    wa.C0 = S.C;
    wa.C1 = Cl;
    wa.dA0 = (__half*)c->dA2;
    wa.dA1 = (__half*)c->dA;
    wa.dX1 = dHnext;
    wa.flags = (unsigned*)((char*)c->status + 4096);
    wa.T = T;
    wa.B = B;
    wa.hp = (int)hp;
    if (c->drop_on()) {  // recurrent dropout inside the wavefront (NEXT-3)
      wa.Ht0 = (const __half*)c->Hst(si, 0);
      wa.Ht1 = (const __half*)c->Hst(si, 1);
      wa.drop_step = c->drop_step();
      wa.drop_seed = c->drop_seed;
      wa.drop_thr = c->drop_thr;
      wa.drop_seq0 = (uint32_t)((c->rank * c->nslots + si) * B);
      wa.drop_scale = c->drop_scale;
    }
    if (wgrad) {
      wa.Hs0 = (const __half*)S.Hs;
      wa.Hs1 = (const __half*)Hs;
      wa.X0 = (const __half*)S.X0;
      wa.Ip0 = (int)c->Ip0;
      const char* nms[4] = {"U1", "W1", "U0", "W0"};
      for (int i = 0; i < 4; ++i) wa.gW[i] = (__half*)c->G(si, c->find(nms[i]));
      wa.gb[0] = (__half*)c->G(si, c->find("b1"));
      wa.gb[1] = (__half*)c->G(si, c->find("b0"));
    }
    wa.trace = trace_buffer(c, 6 * 8192 * 5);
    {
      KScope ks_(c, HDP_K_RECUR_BWD, 1, s);
      CK_CUDA(hdp::launch_recur2_bwd(wa, s));
    }
    if (wa.trace) CK(trace_report(c, hdp::TRACE_BWD_WAVEFRONT, wa.trace, T, l, s));
  } else if (wave) {
    // layer 0: already done by the wavefront launch of the layer-1 segment
  } else if (!f32 && c->recur_ok() && hdp::recur_bwd_supported(B, (int)hp)) {
    // A6 + A7 for all t in one persistent kernel (U^T slice resident in SMEM)
    hdp::RecurBwdArgs ra;
    ra.U = (const __half*)c->W(iU);
    ra.dHa = dHa;
    ra.dHa_last_only = last_only ? 1 : 0;
    ra.gates = (const __half*)Gl;
    ra.C = Cl;
    ra.dA = (__half*)c->dA;
    ra.T = T;
    ra.B = B;
    ra.hp = (int)hp;
    ra.trace = trace_buffer(c, 8192 * 5);
    {
      KScope ks_(c, HDP_K_RECUR_BWD, 1, s);
      CK_CUDA(hdp::launch_recur_bwd(ra, s));
    }
    if (ra.trace) CK(trace_report(c, hdp::TRACE_BWD_LAYER, ra.trace, T, l, s));
  } else
  for (int t = T - 1; t >= 0; --t) {
    const float* dHa_t = last_only ? (t == T - 1 ? dHa : nullptr) : dHa + (long)t * B * hp;
    if (!f32) {
      // mixed mode: K6 of step T-1 alone, then K7(t) with K6(t-1) fused into its split-K reduction
      if (t == T - 1) {
        KScope ks_(c, HDP_K_CELL_BWD, 1, s);
        CK_CUDA(hdp::launch_cell_bwd(et, dHa_t, nullptr, Gl + (long)t * B * 4 * hp * e, Cl + (long)t * B * hp,
                                     t > 0 ? Cl + (long)(t - 1) * B * hp : nullptr, c->dc,
                                     c->dA + (long)t * B * 4 * hp * e, B, (int)hp, 1, s));
      }
      if (t > 0) {
        const int u = t - 1;
        hdp::Epilogue eb;
        eb.mode = hdp::EPI_LSTM_BWD;
        eb.hp = (int)hp;
        eb.dha = last_only ? nullptr : dHa + (long)u * B * hp;
        eb.gates = const_cast<char*>(Gl) + (long)u * B * 4 * hp * e;
        eb.ct = Cl + (long)u * B * hp;
        eb.cprev = u > 0 ? Cl + (long)(u - 1) * B * hp : nullptr;
        eb.dc = c->dc;
        eb.dA = c->dA + (long)u * B * 4 * hp * e;
        if (c->drop_on()) {
          eb.drop_step = c->drop_step();
          eb.drop_seed = c->drop_seed;
          eb.drop_thr = c->drop_thr;
          eb.drop_layer = (uint32_t)l;
          eb.drop_seq0 = (uint32_t)((c->rank * c->nslots + si) * B);
          eb.drop_scale = c->drop_scale;
        }
        // K = 4 hp is long and M = B small: 256-wide tiles, split K over ~120 CTAs
        int fbn = 0, fsp = 0;
        if (hp >= 1024) {  // C4 sweep (tools/c4_gemm_sweep.py): 256-wide tiles, ~128 CTAs
          const int tiles = (int)(((B + 127) / 128) * ((hp + 255) / 256));
          fbn = 256;
          fsp = std::max(1, std::min(128 / tiles, (int)(4 * hp / 64 / 4)));
          fsp = std::min(fsp, 16);
        }
        if (hdp::opt(hdp::OPT_K7_BN)) fbn = hdp::opt(hdp::OPT_K7_BN);  // tuning overrides
        if (hdp::opt(hdp::OPT_K7_SPLITS)) fsp = hdp::opt(hdp::OPT_K7_SPLITS);
        CK(gemm(c, HDP_K_GEMM_DH, c->dA + (long)t * B * 4 * hp * e, 4 * hp, 0, c->W(iU), hp, 1, B, hp, 4 * hp, eb, s,
                fbn, fsp));
      }
      continue;
    }
    // K6 (A6)
    {
      KScope ks_(c, HDP_K_CELL_BWD, 1, s);
      CK_CUDA(hdp::launch_cell_bwd(et, dHa_t, t < T - 1 ? c->dhrec : nullptr, Gl + (long)t * B * 4 * hp * e,
                                   Cl + (long)t * B * hp, t > 0 ? Cl + (long)(t - 1) * B * hp : nullptr, c->dc,
                                   c->dA + (long)t * B * 4 * hp * e, B, (int)hp, t == T - 1, s));
    }
    if (t > 0)  // K7: dh_rec = dA_t U (A7); U read MN-major as [K = 4hp][N = hp]
      CK(gemm(c, HDP_K_GEMM_DH, c->dA + (long)t * B * 4 * hp * e, 4 * hp, 0, c->W(iU), hp, 1, B, hp, 4 * hp,
              epi_f32(c->dhrec, hp), s));
  }
  if (!wgrad) {  // (else A8 was done inside the wavefront launch)
    // K8 (A8): dW = dA^T X, dU = dA^T H_{-1}, db = sum dA
    CK(gemm(c, HDP_K_GEMM_DW, dAl, 4 * hp, 1, X, Ipl, 1, 4 * hp, Ipl, rows, epi_elem(gf, c->G(si, iW), Ipl), s));
    CK(gemm(c, HDP_K_GEMM_DW, dAl, 4 * hp, 1, c->drop_on() ? c->Hst(si, l) : Hs, hp, 1, 4 * hp, hp, rows,
            epi_elem(gf, c->G(si, iU), hp), s));  // dU = sum_t dA_t^T h~_{t-1}
    KScope ks_(c, HDP_K_GEMM_DW, 2, s);
    CK_CUDA(hdp::launch_colreduce(et, dAl, 4 * hp, (int)rows, (int)(4 * hp), nullptr, c->crp, gt, c->G(si, ib), s));
  }
  if (l > 0 && !wave) {  // (the wavefront computed dX1 itself)
    // K9: dX = dA W  ->  dH_above of layer l-1 (W read MN-major as [K = 4hp][N = Ip])
    CK(gemm(c, HDP_K_GEMM_DX, dAl, 4 * hp, 0, c->W(iW), Ipl, 1, rows, Ipl, 4 * hp, epi_f32(dHnext, Ipl), s));
  } else if (d.vocab > 0) {
    CK(gemm(c, HDP_K_GEMM_DX, dAl, 4 * hp, 0, c->W(iW), Ipl, 1, rows, Ipl, 4 * hp, epi_f32(dHnext, Ipl), s));
    const int iE = c->find("E");
    {
      KScope ks_(c, HDP_K_EMBED_BWD, 2, s);
      CK_CUDA(hdp::launch_embed_backward((const int32_t*)S.stage_x, B, T, d.vocab, dHnext, (int)c->Ip0, c->keys_in,
                                         c->keys_out, c->vals_in, c->vals_out, c->sort_temp, c->sort_bytes,
                                         c->emb_part, c->G(si, iE), gt, c->emb_range, s));
    }
  }
  return HDP_OK;
}

int nsegs(const hdp_ctx* c) { return c->d.n_layers + 1; }

// capture (once) and launch; eager (no graph) while profiling
int run_graph(hdp_ctx* c, int si, int B, int T, int seg, cudaStream_t s) {
  if (c->prof) return seg < 0 ? enqueue_forward(c, si, B, T, s) : enqueue_backward_seg(c, si, B, T, seg, s);
  GraphKey k{si, B, T, seg};
  auto it = c->graphs.find(k);
  if (it == c->graphs.end()) {
    const long long before = c->kernels;
    CK_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
    int rc = seg < 0 ? enqueue_forward(c, si, B, T, c->cap) : enqueue_backward_seg(c, si, B, T, seg, c->cap);
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(c->cap, &g);
    const long long nk = c->kernels - before;
    c->kernels = before;
    if (rc != HDP_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(HDP_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t ex = nullptr;
    ce = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(HDP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    it = c->graphs.emplace(k, ex).first;
    c->graph_kernels[k] = nk;
  }
  CK_CUDA(cudaGraphLaunch(it->second, s));
  c->kernels += c->graph_kernels[k];
  return HDP_OK;
}

int check_ready(const hdp_ctx* c) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (!c->configured || !c->bound) return fail(HDP_ERR_STATE, "context not configured/bound");
  return HDP_OK;
}

double sched(const hdp_ctx* c, int epoch) {
  const double N = c->Nw();
  double lam = c->lam0 / (1.0 + N / c->n_half);  // Eq. 4
  if (lam * N > c->max_eff) lam = c->max_eff / N; // clip
  return lam * std::pow(c->gamma, (double)epoch); // Eq. 3
}

int nccl_async_check(hdp_ctx* c) {
  if (!c->comm) return HDP_OK;
  ncclResult_t ar;
  CK_NCCL(ncclCommGetAsyncError(c->comm, &ar));
  if (ar != ncclSuccess) return fail(HDP_ERR_NCCL, "NCCL async error: %s", ncclGetErrorString(ar));
  return HDP_OK;
}

ncclDataType_t gtype(const hdp_ctx* c) { return c->gf32 ? ncclFloat : c->bf ? ncclBfloat16 : ncclHalf; }
ncclDataType_t wtype(const hdp_ctx* c) { return c->f32 ? ncclFloat : c->bf ? ncclBfloat16 : ncclHalf; }

void p2p_bucket_table(hdp_ctx* c) {
  hdp::P2PArgs& a = c->p2pa;
  a.nb = (int)c->buckets.size();
  long vtot = 0;
  for (int bi = 0; bi < a.nb; ++bi) {
    const Bucket& bk = c->buckets[bi];
    a.off[bi] = bk.off;
    a.shard[bi] = bk.shard;
    a.moff[bi] = bk.moff;
    a.vpre[bi] = vtot;
    vtot += bk.shard / 8;
  }
  a.vpre[a.nb] = vtot;
  a.W = c->master;
  a.S1 = c->s1;
  a.S2 = c->s2;
}

// NEXT-2 loopback (world 1, HDP_EXCH_P2P): the exchange kernel's peers are the simulated
// workers' gradient slots and nslots weight copies in the arena; the flag protocol runs
// with one rank (its own flag block, library-owned).
int setup_loopback(hdp_ctx* c) {
  CK_CUDA(cudaMalloc(&c->fwin, hdp::P2P_FLAG_WORDS * sizeof(unsigned)));
  CK_CUDA(cudaMemset(c->fwin, 0, hdp::P2P_FLAG_WORDS * sizeof(unsigned)));
  hdp::P2PArgs& a = c->p2pa;
  a.N = c->nslots;
  a.NR = 1;
  a.rank = 0;
  a.loopback = 1;
  for (int r = 0; r < c->nslots; ++r) {
    a.g_peer[r] = c->grads + (size_t)r * c->P * c->gsz;
    a.w_peer[r] = (__half*)(r == 0 ? c->w : c->wcopies + (size_t)(r - 1) * c->P * c->esz);
  }
  a.flag_peer[0] = c->fwin;
  a.status_peer[0] = (int*)(c->fwin + hdp::P2P_STATUS);
  a.flag_local = c->fwin;
  p2p_bucket_table(c);
  c->p2p = true;
  return HDP_OK;
}

// NEXT-2: gradients and fp16 working weights move into library-owned cudaMalloc windows
// whose CUDA IPC handles are exchanged over the NCCL communicator; every rank maps every
// peer's windows, so one kernel can read the N contributions and write the N weight
// copies over NVLink (desc.exchange = HDP_EXCH_NCCL keeps the NCCL collectives).
int setup_p2p(hdp_ctx* c) {
  if (!c->want_p2p) return HDP_OK;
  if (c->loopback) return setup_loopback(c);
  const size_t gbytes = (size_t)c->P * c->gsz, wbytes = (size_t)c->P * c->esz;
  CK_CUDA(cudaMalloc(&c->gwin, gbytes));
  CK_CUDA(cudaMalloc(&c->wwin, wbytes));
  CK_CUDA(cudaMalloc(&c->fwin, hdp::P2P_FLAG_WORDS * sizeof(unsigned)));
  CK_CUDA(cudaMemset(c->gwin, 0, gbytes));
  CK_CUDA(cudaMemcpy(c->wwin, c->w, wbytes, cudaMemcpyDeviceToDevice));
  CK_CUDA(cudaMemset(c->fwin, 0, hdp::P2P_FLAG_WORDS * sizeof(unsigned)));
  cudaIpcMemHandle_t h[3];
  CK_CUDA(cudaIpcGetMemHandle(&h[0], c->gwin));
  CK_CUDA(cudaIpcGetMemHandle(&h[1], c->wwin));
  CK_CUDA(cudaIpcGetMemHandle(&h[2], c->fwin));
  const size_t hb = sizeof(h);
  char* dh = nullptr;
  CK_CUDA(cudaMalloc(&dh, hb * c->world));
  CK_CUDA(cudaMemcpy(dh + hb * c->rank, h, hb, cudaMemcpyHostToDevice));
  CK_NCCL(ncclAllGather(dh + hb * c->rank, dh, hb, ncclChar, c->comm, 0));  // also the setup barrier
  CK_CUDA(cudaStreamSynchronize(0));
  std::vector<cudaIpcMemHandle_t> all((size_t)3 * c->world);
  CK_CUDA(cudaMemcpy(all.data(), dh, hb * c->world, cudaMemcpyDeviceToHost));
  CK_CUDA(cudaFree(dh));
  hdp::P2PArgs& a = c->p2pa;
  a.N = c->world;
  a.NR = c->world;
  a.rank = c->rank;
  for (int r = 0; r < c->world; ++r) {
    void* ptr[3];
    for (int k = 0; k < 3; ++k) {
      if (r == c->rank) {
        ptr[k] = k == 0 ? (void*)c->gwin : k == 1 ? (void*)c->wwin : (void*)c->fwin;
      } else {
        CK_CUDA(cudaIpcOpenMemHandle(&ptr[k], all[(size_t)3 * r + k], cudaIpcMemLazyEnablePeerAccess));
        c->peer_open.push_back(ptr[k]);
      }
    }
    a.g_peer[r] = ptr[0];
    a.w_peer[r] = (__half*)ptr[1];
    a.flag_peer[r] = (unsigned*)ptr[2];
    a.status_peer[r] = (int*)((unsigned*)ptr[2] + hdp::P2P_STATUS);
  }
  a.flag_local = c->fwin;
  p2p_bucket_table(c);
  // the arena's gradient and weight regions are replaced by the shared windows
  c->grads = c->gwin;
  c->w = c->wwin;
  c->p2p = true;
  // all peers mapped (and their flags zeroed) before anyone's first exchange
  int* one = nullptr;
  CK_CUDA(cudaMalloc(&one, sizeof(int)));
  CK_NCCL(ncclAllReduce(one, one, 1, ncclInt32, ncclSum, c->comm, 0));
  CK_CUDA(cudaStreamSynchronize(0));
  CK_CUDA(cudaFree(one));
  return HDP_OK;
}

// Every rank must configure the same model (hdp.h): a 64-bit FNV-1a hash of the
// description's fields, all-reduced with min and max, must agree.
int check_desc_across_ranks(hdp_ctx* c, const hdp_model_desc& d) {
  if (c->world < 2 || c->host_only || !c->comm) return HDP_OK;
  const long long f[] = {d.n_layers, d.input_dim, d.hidden, d.fc_hidden, d.head_last_step, d.vocab, d.embed_dim,
                         d.max_batch, d.max_seq, d.math, d.wire, d.optimizer, d.sim_workers, d.flat_params,
                         d.exchange};
  unsigned long long h = 1469598103934665603ull;
  for (long long v : f)
    for (int b = 0; b < 8; ++b) {
      h ^= (unsigned long long)((v >> (8 * b)) & 0xff);
      h *= 1099511628211ull;
    }
  CK_CUDA(cudaSetDevice(c->device));
  unsigned long long* buf = nullptr;
  CK_CUDA(cudaMalloc(&buf, 2 * sizeof h));
  std::unique_ptr<unsigned long long, void (*)(unsigned long long*)> guard(buf, [](unsigned long long* p) { cudaFree(p); });
  const unsigned long long hh[2] = {h, h};
  CK_CUDA(cudaMemcpy(buf, hh, sizeof hh, cudaMemcpyHostToDevice));
  CK_NCCL(ncclGroupStart());
  CK_NCCL(ncclAllReduce(buf, buf, 1, ncclUint64, ncclMin, c->comm, 0));
  CK_NCCL(ncclAllReduce(buf + 1, buf + 1, 1, ncclUint64, ncclMax, c->comm, 0));
  CK_NCCL(ncclGroupEnd());
  unsigned long long mm[2];
  CK_CUDA(cudaMemcpy(mm, buf, sizeof mm, cudaMemcpyDeviceToHost));
  if (mm[0] != mm[1]) return fail(HDP_ERR_ARG, "hdp_configure: the ranks passed different model descriptions");
  return HDP_OK;
}

}  // namespace

// ====================================================================== options
namespace hdp {
int g_opt[OPT_COUNT] = {1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 16, 1, 0, 0};
namespace {
const char* const kOptNames[OPT_COUNT] = {"persistent",     "wavefront", "wavefront_fusex", "wavefront_wgrad",
                                          "wavefront_tmem", "recur_nbg", "gemm_cta_group",  "gemm_cluster_n",
                                          "pdl",            "k7_bn",     "k7_splits",       "recur_trace",
                                          "layer_pipe",     "head_fused",      "k7_cluster",
                                          "fwd_pdl"};
}
int opt_find(const char* name) {
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!strcmp(name, kOptNames[i])) return i;
  return -1;
}
}  // namespace hdp

// ====================================================================== C-ABI
extern "C" {

const char* hdp_last_error(void) { return g_err.c_str(); }

int hdp_nccl_unique_id(unsigned char uid[HDP_UID_BYTES]) {
  if (!uid) return fail(HDP_ERR_ARG, "null uid");
  static_assert(sizeof(ncclUniqueId) == HDP_UID_BYTES, "uid size");
  ncclUniqueId id;
  CK_NCCL(ncclGetUniqueId(&id));
  memcpy(uid, &id, HDP_UID_BYTES);
  return HDP_OK;
}

int hdp_init(int world, int rank, const unsigned char* uid, int device, hdp_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || device < -1)
    return fail(HDP_ERR_ARG, "hdp_init: bad arguments (world %d rank %d device %d)", world, rank, device);
  std::unique_ptr<hdp_ctx> c(new hdp_ctx());
  c->world = world;
  c->rank = rank;
  c->device = device;
  if (device == -1) {  // host-only context: layout / schedule queries, no CUDA, no NCCL
    c->host_only = true;
    *out = c.release();
    return HDP_OK;
  }
  if (world > 1 && !uid) return fail(HDP_ERR_ARG, "hdp_init: world > 1 needs a NCCL unique id");
  CK_CUDA(cudaSetDevice(device));
  if (world > 1) {
    ncclUniqueId id;
    memcpy(&id, uid, HDP_UID_BYTES);
    CK_NCCL(ncclCommInitRank(&c->comm, world, id, rank));
  }
  *out = c.release();
  return HDP_OK;
}

int hdp_destroy(hdp_ctx* c) {
  if (!c) return HDP_OK;
  if (c->host_only) {
    delete c;
    return HDP_OK;
  }
  cudaSetDevice(c->device);
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  for (auto ev : c->ev_bucket) cudaEventDestroy(ev);
  for (auto ev : c->ev_layer) cudaEventDestroy(ev);
  for (auto st : c->lstr) cudaStreamDestroy(st);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_hfork) cudaEventDestroy(c->ev_hfork);
  if (c->hstr) cudaStreamDestroy(c->hstr);
  for (auto ev : c->evpool) cudaEventDestroy(ev);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->ev_count) cudaEventDestroy(c->ev_count);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->count_host) cudaFreeHost(c->count_host);
  for (void* ptr : c->peer_open) cudaIpcCloseMemHandle(ptr);
  if (c->gwin) cudaFree(c->gwin);  // (loopback: gwin / wwin stay null, the arena holds them)
  if (c->wwin) cudaFree(c->wwin);
  if (c->fwin) cudaFree(c->fwin);
  if (c->hst) cudaFree(c->hst);
  if (c->trace) cudaFree(c->trace);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return HDP_OK;
}

int hdp_configure(hdp_ctx* c, const hdp_model_desc* desc, hdp_sizes* out) {
  if (!c || !desc) return fail(HDP_ERR_ARG, "null argument");
  if (c->bound) return fail(HDP_ERR_STATE, "already bound");
  const hdp_model_desc& d = *desc;
  if (d.n_layers < 0 || d.math < 0 || d.math > HDP_MATH_BF16 || d.wire < 0 || d.wire > 2 || d.optimizer < 0 ||
      d.optimizer > 1 || d.sim_workers < 1)
    return fail(HDP_ERR_ARG, "bad enum / layer count");
  if (d.sim_workers > 1 && c->world > 1) return fail(HDP_ERR_ARG, "sim_workers > 1 requires world == 1");
  if (d.sim_workers > 16) return fail(HDP_ERR_ARG, "sim_workers > 16");
  if (d.n_layers == 0) {
    if (d.flat_params <= 0) return fail(HDP_ERR_ARG, "flat model needs flat_params > 0");
  } else {
    if (d.hidden <= 0 || d.max_batch <= 0 || d.max_seq <= 0 || d.fc_hidden < 0)
      return fail(HDP_ERR_ARG, "hidden / max_batch / max_seq must be positive");
    if (d.vocab > 0 ? d.embed_dim <= 0 : d.input_dim <= 0) return fail(HDP_ERR_ARG, "input width must be positive");
    if (d.head_last_step && d.fc_hidden > 0) return fail(HDP_ERR_UNSUPPORTED, "last-step head with FC layer");
    if ((long)d.max_batch * d.max_seq > (1L << 30)) return fail(HDP_ERR_ARG, "batch*seq too large");
  }
  if (d.math == HDP_MATH_FP32 && d.wire == HDP_WIRE_FP16_NCCLSUM)
    return fail(HDP_ERR_ARG, "FP32 math cannot use the fp16 NCCL-sum wire");
  if (d.exchange < HDP_EXCH_AUTO || d.exchange > HDP_EXCH_TASK0) return fail(HDP_ERR_ARG, "bad exchange mode");
  if (d.exchange == HDP_EXCH_TASK0 && d.wire == HDP_WIRE_FP16_NCCLSUM)
    return fail(HDP_ERR_UNSUPPORTED, "task-0 ablation gathers the gradients unreduced (fp16 all-to-all or fp32 wire)");
  CK(check_desc_across_ranks(c, d));
  c->d = d;
  c->f32 = d.math == HDP_MATH_FP32;
  c->bf = d.math == HDP_MATH_BF16;
  c->gf32 = c->f32 || d.wire == HDP_WIRE_FP32;
  c->head_fused = !c->f32 && !c->bf && d.fc_hidden > 0 && !d.head_last_step && d.n_layers > 0 &&
                  hdp::head_fused_supported((int)r16(d.hidden), (int)r16(d.fc_hidden)) &&
                  hdp::opt(hdp::OPT_HEAD_FUSED) != 0;
  c->esz = c->f32 ? 4 : 2;
  c->gsz = c->gf32 ? 4 : 2;
  c->nslots = d.sim_workers;
  c->task0 = d.exchange == HDP_EXCH_TASK0 && c->world > 1;
  build_layout(c);
  {
    // NEXT-2 one-kernel exchange: fp16 gradients on the all-to-all wire, fp16 weights
    const bool fits = !c->f32 && (d.wire == HDP_WIRE_FP16_A2A || d.wire == HDP_WIRE_FP32) &&
                      (int)c->buckets.size() <= hdp::P2P_MAX_BUCKETS &&
                      ((c->world >= 2 && c->world <= hdp::P2P_MAX_RANKS) ||
                       (c->world == 1 && c->nslots >= 2 && c->nslots <= hdp::P2P_MAX_RANKS));
    if (d.exchange == HDP_EXCH_P2P && !fits)
      return fail(HDP_ERR_UNSUPPORTED, "HDP_EXCH_P2P needs mixed math, the fp16 all-to-all or fp32 wire and 2..%d ranks "
                  "(or simulated workers at world 1)", hdp::P2P_MAX_RANKS);
    c->want_p2p = fits && (d.exchange == HDP_EXCH_P2P || (d.exchange == HDP_EXCH_AUTO && c->world >= 2));
    c->loopback = c->want_p2p && c->world == 1;
  }
  carve(c, nullptr);
  c->configured = true;
  if (out) {
    out->n_params = c->n_params;
    out->n_params_padded = c->P;
    out->n_buckets = (long long)c->buckets.size();
    out->arena_bytes = (long long)c->arena_bytes;
  }
  return HDP_OK;
}

int hdp_bind(hdp_ctx* c, void* arena, long long bytes) {
  if (!c || !arena) return fail(HDP_ERR_ARG, "null argument");
  if (!c->configured) return fail(HDP_ERR_STATE, "configure first");
  if (c->bound) return fail(HDP_ERR_STATE, "already bound");
  if (c->host_only) return fail(HDP_ERR_STATE, "host-only context (device -1) cannot bind device memory");
  if ((size_t)bytes < c->arena_bytes) return fail(HDP_ERR_ARG, "arena too small: %lld < %zu", bytes, c->arena_bytes);
  if (reinterpret_cast<uintptr_t>(arena) & 255) return fail(HDP_ERR_ARG, "arena must be 256-byte aligned");
  CK_CUDA(cudaSetDevice(c->device));
  c->arena = (char*)arena;
  carve(c, c->arena);
  CK_CUDA(cudaMemset(c->arena, 0, c->arena_bytes));
  CK_CUDA(hdp::gemm_init());
  CK_CUDA(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
  CK_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  CK_CUDA(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  CK_CUDA(cudaEventCreateWithFlags(&c->ev_count, cudaEventDisableTiming));
  c->ev_bucket.resize(c->buckets.size());
  for (auto& ev : c->ev_bucket) CK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  c->lstr.resize(c->d.n_layers);
  c->ev_layer.resize(c->d.n_layers);
  for (auto& st : c->lstr) CK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (auto& ev : c->ev_layer) CK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK_CUDA(cudaStreamCreateWithFlags(&c->hstr, cudaStreamNonBlocking));
  CK_CUDA(cudaEventCreateWithFlags(&c->ev_hfork, cudaEventDisableTiming));
  CK_CUDA(cudaMallocHost(&c->count_host, 2 * sizeof(int)));
  c->count_host[0] = c->count_host[1] = 0;
  c->st.assign(c->nslots, SlotState{});
  CK(setup_p2p(c));
  CK_CUDA(cudaDeviceSynchronize());
  c->bound = true;
  return HDP_OK;
}

int hdp_num_blocks(const hdp_ctx* c) { return c ? (int)c->blocks.size() : 0; }

int hdp_exchange_kind(const hdp_ctx* c) {
  if (!c || !c->configured) return -1;
  if (c->task0) return 4;
  if (c->want_p2p) return c->loopback ? 3 : 2;
  return c->world > 1 ? 1 : 0;
}

int hdp_param_block(const hdp_ctx* c, int i, hdp_block* out) {
  if (!c || !out || !c->configured || i < 0 || i >= (int)c->blocks.size()) return fail(HDP_ERR_ARG, "bad block index");
  const Block& b = c->blocks[i];
  memset(out, 0, sizeof *out);
  snprintf(out->name, sizeof out->name, "%s", b.name.c_str());
  out->canon_offset = b.canon_off;
  out->rows = b.rows;
  out->cols = b.cols;
  out->dev_offset = b.dev_off;
  out->dev_rows = b.dev_rows;
  out->dev_cols = b.dev_cols;
  out->bucket = b.bucket;
  return HDP_OK;
}

namespace {
void canon_to_dev(const hdp_ctx* c, const float* in, std::vector<float>& out) {
  out.assign(c->P, 0.f);
  for (const Block& b : c->blocks)
    for (long r = 0; r < b.rows; ++r)
      for (long k = 0; k < b.cols; ++k) out[b.dev_off + dev_index(c, b, r, k)] = in[b.canon_off + r * b.cols + k];
}
void dev_to_canon(const hdp_ctx* c, const std::vector<float>& in, float* out) {
  for (const Block& b : c->blocks)
    for (long r = 0; r < b.rows; ++r)
      for (long k = 0; k < b.cols; ++k) out[b.canon_off + r * b.cols + k] = in[b.dev_off + dev_index(c, b, r, k)];
}
}  // namespace

int hdp_load_params(hdp_ctx* c, const float* params, int root) {
  CK(check_ready(c));
  if (root < 0 || root >= c->world) return fail(HDP_ERR_ARG, "bad root");
  if (c->rank == root && !params) return fail(HDP_ERR_ARG, "root needs params");
  CK_CUDA(cudaSetDevice(c->device));
  std::vector<float> host;
  if (c->rank == root) canon_to_dev(c, params, host);
  float* buf = nullptr;
  CK_CUDA(cudaMalloc(&buf, c->P * sizeof(float)));
  std::unique_ptr<float, void (*)(float*)> guard(buf, [](float* p) { cudaFree(p); });
  if (c->rank == root) CK_CUDA(cudaMemcpy(buf, host.data(), c->P * sizeof(float), cudaMemcpyHostToDevice));
  cudaStream_t s = c->comm_stream;
  if (c->world > 1) {
    CK_NCCL(ncclBroadcast(buf, buf, c->P, ncclFloat, root, c->comm, s));  // PAPER.md:92 step 2
  }
  // master shard <- owned slices; optimizer state <- 0; working copy <- params
  for (const Bucket& bk : c->buckets)
    CK_CUDA(cudaMemcpyAsync(c->master + bk.moff, buf + bk.off + (long)c->owner_index() * bk.shard, bk.shard * 4,
                            cudaMemcpyDeviceToDevice, s));
  CK_CUDA(cudaMemsetAsync(c->s1, 0, c->M_own * 4, s));
  if (c->s2) CK_CUDA(cudaMemsetAsync(c->s2, 0, c->M_own * 4, s));
  // working copy (R1): fp32 -> fp16 RNE in mixed mode (not on the hot path)
  if (c->f32) {
    CK_CUDA(cudaMemcpyAsync(c->w, buf, c->P * 4, cudaMemcpyDeviceToDevice, s));
  } else {
    std::vector<__half> h16(c->P);
    std::vector<float> full(c->P);
    CK_CUDA(cudaMemcpyAsync(full.data(), buf, c->P * 4, cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    if (c->bf) {
      for (long i = 0; i < c->P; ++i) {
        const __nv_bfloat16 b = __float2bfloat16_rn(full[i]);
        memcpy(&h16[i], &b, 2);
      }
    } else {
      for (long i = 0; i < c->P; ++i) h16[i] = __float2half_rn(full[i]);
    }
    CK_CUDA(cudaMemcpyAsync(c->w, h16.data(), c->P * 2, cudaMemcpyHostToDevice, s));
  }
  CK_CUDA(cudaStreamSynchronize(s));
  c->loaded = true;
  c->poisoned = false;
  c->count_pending = false;
  c->adam_k = 0;
  for (auto& st : c->st) st = SlotState{};
  return HDP_OK;
}

int hdp_gather_master(hdp_ctx* c, float* out) {
  CK(check_ready(c));
  if (!out) return fail(HDP_ERR_ARG, "null output");
  CK_CUDA(cudaSetDevice(c->device));
  float* buf = nullptr;
  CK_CUDA(cudaMalloc(&buf, c->P * sizeof(float)));
  std::unique_ptr<float, void (*)(float*)> guard(buf, [](float* p) { cudaFree(p); });
  cudaStream_t s = c->comm_stream;
  for (const Bucket& bk : c->buckets) {
    if (c->task0)  // task 0 holds the whole master
      CK_NCCL(ncclBroadcast(c->master + bk.moff, buf + bk.off, bk.shard, ncclFloat, 0, c->comm, s));
    else if (c->world > 1)
      CK_NCCL(ncclAllGather(c->master + bk.moff, buf + bk.off, bk.shard, ncclFloat, c->comm, s));
    else
      CK_CUDA(cudaMemcpyAsync(buf + bk.off, c->master + bk.moff, bk.shard * 4, cudaMemcpyDeviceToDevice, s));
  }
  std::vector<float> host(c->P);
  CK_CUDA(cudaMemcpyAsync(host.data(), buf, c->P * 4, cudaMemcpyDeviceToHost, s));
  CK_CUDA(cudaStreamSynchronize(s));
  dev_to_canon(c, host, out);
  return HDP_OK;
}

namespace {
int read_vec(hdp_ctx* c, const char* src, bool is_f32, float* out) {
  const bool is_bf = !is_f32 && c->bf;  // 16-bit vectors of the bf16 mode
  CK_CUDA(cudaSetDevice(c->device));
  CK_CUDA(cudaDeviceSynchronize());
  std::vector<float> host(c->P);
  if (is_f32) {
    CK_CUDA(cudaMemcpy(host.data(), src, c->P * 4, cudaMemcpyDeviceToHost));
  } else {
    std::vector<__half> h(c->P);
    CK_CUDA(cudaMemcpy(h.data(), src, c->P * 2, cudaMemcpyDeviceToHost));
    if (is_bf) {
      for (long i = 0; i < c->P; ++i) {
        uint16_t b;
        memcpy(&b, &h[i], 2);
        const uint32_t u = (uint32_t)b << 16;
        memcpy(&host[i], &u, 4);
      }
    } else {
      for (long i = 0; i < c->P; ++i) host[i] = __half2float(h[i]);
    }
  }
  dev_to_canon(c, host, out);
  return HDP_OK;
}
}  // namespace

int hdp_read_weights(hdp_ctx* c, float* out) {
  CK(check_ready(c));
  if (!out) return fail(HDP_ERR_ARG, "null output");
  return read_vec(c, c->w, c->f32, out);
}

int hdp_read_grads(hdp_ctx* c, int slot, float* out) {
  CK(check_ready(c));
  if (!out || slot < 0 || slot >= c->nslots) return fail(HDP_ERR_ARG, "bad slot / output");
  return read_vec(c, c->grads + (long)slot * c->P * c->gsz, c->gf32, out);
}

int hdp_set_lr_schedule(hdp_ctx* c, double lambda0, double gamma, double n_half, double max_eff_lr,
                        double momentum, double b1, double b2, double eps) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (!(lambda0 > 0) || !(gamma > 0 && gamma <= 1) || !(n_half > 0) || !(max_eff_lr > 0) ||
      !(momentum >= 0 && momentum < 1) || !(b1 >= 0 && b1 < 1) || !(b2 >= 0 && b2 < 1) || !(eps > 0))
    return fail(HDP_ERR_ARG, "bad schedule / optimizer constants");
  c->lam0 = lambda0;
  c->gamma = gamma;
  c->n_half = n_half;
  c->max_eff = max_eff_lr;
  c->mom = momentum;
  c->b1 = b1;
  c->b2 = b2;
  c->eps = eps;
  c->lr_set = true;
  return HDP_OK;
}

double hdp_lr(const hdp_ctx* c, int epoch) {
  if (!c || !c->lr_set || !c->configured || epoch < 0) return -1.0;
  return sched(c, epoch);
}

int hdp_set_recurrent_dropout(hdp_ctx* c, double keep, unsigned int seed) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (!(keep > 0.0 && keep <= 1.0)) return fail(HDP_ERR_ARG, "keep must be in (0, 1]");
  if (!c->bound) return fail(HDP_ERR_STATE, "context not bound");
  if (keep < 1.0 && (c->f32 || c->bf))
    return fail(HDP_ERR_UNSUPPORTED, "recurrent dropout is implemented for the fp16 mixed mode only");
  if (keep < 1.0 && c->d.n_layers == 0) return fail(HDP_ERR_ARG, "no LSTM layers");
  CK_CUDA(cudaSetDevice(c->device));
  CK_CUDA(cudaDeviceSynchronize());
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);  // kernel choice and operands change
  c->graphs.clear();
  if (keep < 1.0 && !c->hst) {
    const size_t bytes = (size_t)c->nslots * c->d.n_layers * (c->d.max_seq + 1) * c->d.max_batch * c->hp * 2;
    CK_CUDA(cudaMalloc(&c->hst, bytes));
    CK_CUDA(cudaMemset(c->hst, 0, bytes));  // slot t = 0 of every layer stays h~_{-1} = 0
  }
  CK_CUDA(cudaMemset(c->drop_step(), 0, sizeof(int)));
  c->keep = keep;
  c->drop_seed = seed;
  c->drop_thr = keep < 1.0 ? (uint32_t)std::floor(keep * 4294967296.0) : 0u;
  c->drop_scale = (float)(1.0 / keep);
  return HDP_OK;
}

int hdp_set_l2(hdp_ctx* c, double l2) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (!(l2 >= 0) || !std::isfinite(l2)) return fail(HDP_ERR_ARG, "l2 must be a finite number >= 0");
  if (c->l2 != l2) {  // the loss term is part of captured forward graphs
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  c->l2 = l2;
  return HDP_OK;
}

int hdp_set_dynamic_loss_scale(hdp_ctx* c, int growth_interval) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (growth_interval < 0) return fail(HDP_ERR_ARG, "growth_interval must be >= 0");
  if (!c->bound) return fail(HDP_ERR_STATE, "context not bound");
  if (growth_interval > 0 && c->quorum > 0)
    return fail(HDP_ERR_UNSUPPORTED, "dynamic loss scaling with partial collection");
  if (growth_interval > 0 && c->d.optimizer == HDP_OPT_ADAM)
    return fail(HDP_ERR_UNSUPPORTED, "dynamic loss scaling with Adam: the host-side bias-correction step count "
                "would also count skipped steps");
  CK_CUDA(cudaSetDevice(c->device));
  if ((c->dyn_interval > 0) != (growth_interval > 0)) {  // alpha source is baked into captured graphs
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  if (growth_interval > 0) {
    const int zero[3] = {0, 0, 0};
    CK_CUDA(cudaMemcpy(c->dyn_state(), zero, sizeof zero, cudaMemcpyHostToDevice));
    CK_CUDA(cudaMemcpy(c->alpha_dev(), &c->alpha, sizeof(float), cudaMemcpyHostToDevice));
  }
  c->dyn_interval = growth_interval;
  return HDP_OK;
}

int hdp_loss_scale_state(hdp_ctx* c, float* alpha, int* skipped_steps) {
  if (!c || !alpha || !skipped_steps) return fail(HDP_ERR_ARG, "null argument");
  if (c->dyn_interval > 0) {
    CK_CUDA(cudaSetDevice(c->device));
    CK_CUDA(cudaDeviceSynchronize());
    int st[3];
    CK_CUDA(cudaMemcpy(st, c->dyn_state(), sizeof st, cudaMemcpyDeviceToHost));
    CK_CUDA(cudaMemcpy(alpha, c->alpha_dev(), sizeof(float), cudaMemcpyDeviceToHost));
    *skipped_steps = st[2];
  } else {
    *alpha = c->alpha;
    *skipped_steps = 0;
  }
  return HDP_OK;
}

int hdp_set_loss_scale(hdp_ctx* c, float alpha) {
  if (!c) return fail(HDP_ERR_ARG, "null context");
  if (!(alpha > 0) || !std::isfinite(alpha)) return fail(HDP_ERR_ARG, "alpha must be a positive finite number");
  if (c->alpha != alpha) {  // alpha is baked into captured forward graphs
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  c->alpha = alpha;
  if (c->dyn_interval > 0) {
    CK_CUDA(cudaSetDevice(c->device));
    CK_CUDA(cudaMemcpy(c->alpha_dev(), &alpha, sizeof(float), cudaMemcpyHostToDevice));
  }
  return HDP_OK;
}

int hdp_lstm_forward(hdp_ctx* c, const void* x, const void* targets, int B, int T, int slot, float* y_out,
                     float* loss_out, void* stream) {
  CK(check_ready(c));
  if (c->d.n_layers == 0) return fail(HDP_ERR_UNSUPPORTED, "flat model has no forward");
  if (!x || !targets) return fail(HDP_ERR_ARG, "null input");
  if (slot < 0 || slot >= c->nslots) return fail(HDP_ERR_ARG, "slot %d out of range", slot);
  if (B < 1 || B > c->d.max_batch || T < 1 || T > c->d.max_seq)
    return fail(HDP_ERR_ARG, "B=%d T=%d outside [1,%d]x[1,%d]", B, T, c->d.max_batch, c->d.max_seq);
  if (!c->loaded) return fail(HDP_ERR_STATE, "parameters not loaded");
  if (c->poisoned) return fail(HDP_ERR_STATE, "context poisoned by non-finite gradients; reload parameters");
  cudaStream_t s = (cudaStream_t)stream;
  hdp_ctx::Slot& S = c->slot[slot];
  const long in_bytes = c->d.vocab > 0 ? 4 : (long)c->d.input_dim * c->esz;
  CK_CUDA(cudaMemcpyAsync(S.stage_x, x, (long)B * T * in_bytes, cudaMemcpyDefault, s));
  const long nt = c->d.head_last_step ? B : (long)B * T;
  CK_CUDA(cudaMemcpyAsync(S.stage_t, targets, nt, cudaMemcpyDefault, s));
  CK(run_graph(c, slot, B, T, -1, s));
  if (loss_out) CK_CUDA(cudaMemcpyAsync(loss_out, S.loss, 4, cudaMemcpyDefault, s));
  if (y_out) CK_CUDA(cudaMemcpyAsync(y_out, S.y, nt * 4, cudaMemcpyDefault, s));
  c->st[slot].fwd = true;
  c->st[slot].bwd = false;
  c->st[slot].B = B;
  c->st[slot].T = T;
  return HDP_OK;
}

int hdp_lstm_backward(hdp_ctx* c, int slot, void* stream) {
  CK(check_ready(c));
  if (slot < 0 || slot >= c->nslots) return fail(HDP_ERR_ARG, "slot %d out of range", slot);
  if (!c->st[slot].fwd) return fail(HDP_ERR_STATE, "backward without forward on slot %d", slot);
  if (c->poisoned) return fail(HDP_ERR_STATE, "context poisoned");
  cudaStream_t s = (cudaStream_t)stream;
  const int B = c->st[slot].B, T = c->st[slot].T;
  // fused head: the forward already produced dH_top, so the head's own gradient work (column
  // sums, dF GEMM) is off the layers' path -- it runs on a side stream, launched after the
  // first layer segment so the recurrence launch is dispatched first and the GEMM fills the
  // SMs it leaves idle
  const bool head_side = c->head_fused && c->hstr && nsegs(c) > 1;
  if (head_side) {
    CK_CUDA(cudaEventRecord(c->ev_hfork, s));
    CK_CUDA(cudaStreamWaitEvent(c->hstr, c->ev_hfork, 0));
  }
  for (int seg = 0; seg < nsegs(c); ++seg) {
    if (seg == 0 && head_side) continue;
    CK(run_graph(c, slot, B, T, seg, s));
    // bucket `seg` (head, then layers top-down) is complete: the exchange may start
    CK_CUDA(cudaEventRecord(c->ev_bucket[seg], s));
    if (seg == 1 && head_side) {
      CK(run_graph(c, slot, B, T, 0, c->hstr));
      CK_CUDA(cudaEventRecord(c->ev_bucket[0], c->hstr));
    }
  }
  if (head_side) CK_CUDA(cudaStreamWaitEvent(s, c->ev_bucket[0], 0));  // the caller's stream sees it all
  if (c->d.vocab > 0) CK_CUDA(cudaEventRecord(c->ev_bucket[nsegs(c)], s));  // embedding (after layer 0)
  c->st[slot].bwd = true;
  return HDP_OK;
}

int hdp_grad_average_update(hdp_ctx* c, int epoch, void* stream, int* nonfinite_host) {
  CK(check_ready(c));
  if (!c->lr_set) return fail(HDP_ERR_STATE, "learning-rate schedule not set");
  if (epoch < 0) return fail(HDP_ERR_ARG, "epoch < 0");
  if (!c->loaded) return fail(HDP_ERR_STATE, "parameters not loaded");
  if (c->poisoned) return fail(HDP_ERR_STATE, "context poisoned");
  if (c->d.n_layers > 0)
    for (int sl = 0; sl < c->nslots; ++sl)
      if (!c->st[sl].bwd) return fail(HDP_ERR_STATE, "slot %d has no backward", sl);
  CK_CUDA(cudaSetDevice(c->device));
  CK(nccl_async_check(c));
  // deferred report of the previous step's count (not synchronised then)
  if (c->count_pending) {
    CK_CUDA(cudaEventSynchronize(c->ev_count));
    c->count_pending = false;
    if (c->count_host[1] > 0) {
      c->poisoned = true;
      return fail(HDP_ERR_ARG, "%d token ids outside [0, %d) in the previous step", c->count_host[1], c->d.vocab);
    }
    if (*c->count_host > 0 && c->dyn_interval == 0) {
      c->poisoned = true;
      return fail(HDP_ERR_NONFINITE, "%d non-finite gradient values in the previous step (loss scale %g)",
                  *c->count_host, (double)c->alpha);
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int N = c->Nw();
  const double lam = sched(c, epoch);
  hdp::UpdateArgs a;
  a.inv_scale = (float)(1.0 / ((double)N * (double)c->alpha));  // R14
  a.lam = (float)lam;                                            // R15a
  a.mom = (float)c->mom;
  const int opt = c->d.optimizer;
  if (opt == HDP_OPT_ADAM) {
    const long k = ++c->adam_k;
    a.b1 = (float)c->b1;
    a.omb1 = (float)(1.0 - c->b1);
    a.b2 = (float)c->b2;
    a.omb2 = (float)(1.0 - c->b2);
    a.c1 = (float)(1.0 / (1.0 - std::pow(c->b1, (double)k)));
    a.c2 = (float)(1.0 / (1.0 - std::pow(c->b2, (double)k)));
    a.eps = (float)c->eps;
  }
  a.nonfinite = c->status;
  a.l2x2 = (float)(2.0 * c->l2);
  // Steps 4-6 run on the comm stream, each bucket group gated by the event its backward
  // segment recorded, so the update of the top layers overlaps the BPTT of the lower ones
  // (north_star "overlapped with BPTT on a side stream").  A flat model (C5: the caller wrote
  // the gradients) or a dynamic loss scale (the skip decision needs every gradient first)
  // makes the comm stream wait for everything enqueued on `s` instead.
  cudaStream_t cs = c->comm_stream;
  const bool dyn = c->dyn_interval > 0;
  if (c->d.n_layers == 0 || dyn) {
    CK_CUDA(cudaEventRecord(c->ev_done, s));
    CK_CUDA(cudaStreamWaitEvent(cs, c->ev_done, 0));
  }
  if (dyn) {
    // NEXT-3 dynamic loss scaling: the step's global non-finite count (all ranks' fp16
    // gradients) decides before any update whether the step is applied; alpha, kept on
    // the device, then follows the scale rule (oracle/optim.py dynamic_loss_scale)
    int* st = c->dyn_state();
    CK_CUDA(cudaMemsetAsync(st, 0, sizeof(int), cs));
    {
      KScope ks_(c, HDP_K_UPDATE, 1, cs);
      CK_CUDA(hdp::launch_count_nonfinite(c->grads, (long)c->nslots * c->P, c->gt(), st, cs));
    }
    if (c->world > 1) {
      KScope ks_(c, HDP_K_COMM, 0, cs);
      CK_NCCL(ncclAllReduce(st, st, 1, ncclInt32, ncclSum, c->comm, cs));
    }
    a.skip = st;
    a.alpha_dev = c->alpha_dev();
    a.n_workers = (double)N;
  }
  // Exchange groups: buckets become ready in order (head, layer L-1 .. 0, embedding); with the
  // backward wavefront every layer bucket is ready at once, so buckets 1.. form one group (one
  // launch / one NCCL group each instead of one per bucket).
  const size_t nb = c->buckets.size();
  std::vector<std::pair<size_t, size_t>> groups;
  if (c->wave_bwd && nb > 2) {
    groups.push_back({0, 1});
    groups.push_back({1, nb});
  } else {
    for (size_t bi = 0; bi < nb; ++bi) groups.push_back({bi, bi + 1});
  }
  const int* count_src = c->status;
  if (c->p2p) {
    // NEXT-2: one kernel per group does the exchange, the fused average + update and the
    // all-gather over NVLink peer memory (p2p_exchange.cu)
    const unsigned step = ++c->p2p_step;
    hdp::P2PArgs& p = c->p2pa;
    p.step = step;
    p.inv_scale = a.inv_scale;
    p.lam = a.lam;
    p.mom = a.mom;
    p.b1 = a.b1;
    p.omb1 = a.omb1;
    p.b2 = a.b2;
    p.omb2 = a.omb2;
    p.c1 = a.c1;
    p.c2 = a.c2;
    p.eps = a.eps;
    p.l2x2 = a.l2x2;
    p.w_bf16 = c->bf ? 1 : 0;
    p.skip = a.skip;
    p.alpha_dev = a.alpha_dev;
    p.n_workers = a.n_workers;
    p.alpha = (double)c->alpha;
    p.quorum = c->quorum;
    p.straggler_mask = c->straggler_mask;
    p.straggler_ns = c->straggler_ns;
    // the other status slot is next step's: zero it now (peers add to it only after my next "ready")
    CK_CUDA(cudaMemsetAsync(c->fwin + hdp::P2P_STATUS + ((step + 1) & 1), 0, sizeof(int), cs));
    for (const auto& gr : groups) {
      if (c->d.n_layers > 0)
        for (size_t bi = gr.first; bi < gr.second; ++bi) CK_CUDA(cudaStreamWaitEvent(cs, c->ev_bucket[bi], 0));
      p.bk0 = (int)gr.first;
      p.bk1 = (int)gr.second;
      p.seq = ++c->p2p_seq;
      const long vec = p.vpre[p.bk1] - p.vpre[p.bk0];
      // one wave of co-resident CTAs (register-limited occupancy), grid-striding over the vectors
      const int grid = (int)std::max(1L, std::min((vec + 255) / 256, (long)hdp::exch_resident_ctas(p, opt, c->gt())));
      c->p2p_ctr += (unsigned)grid;
      p.ctr_target = c->p2p_ctr;
      KScope ks_(c, HDP_K_UPDATE, 1, cs);
      CK_CUDA(hdp::launch_exch_update(p, opt, c->gt(), grid, cs));
    }
    count_src = (const int*)(c->fwin + hdp::P2P_STATUS + (step & 1));
  } else {
    CK_CUDA(cudaMemsetAsync(c->status, 0, sizeof(int), cs));
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const size_t b0 = groups[gi].first, b1 = groups[gi].second;
      const bool last = gi + 1 == groups.size();
      if (c->d.n_layers > 0)
        for (size_t bi = b0; bi < b1; ++bi) CK_CUDA(cudaStreamWaitEvent(cs, c->ev_bucket[bi], 0));
      if (c->task0) {
        // the paper's step 4 literally: every worker's gradients of the group
        // go to task 0 (grouped sends / receives, rank order kept by position)
        KScope ks_(c, HDP_K_COMM, 0, cs);
        CK_NCCL(ncclGroupStart());
        for (size_t bi = b0; bi < b1; ++bi) {
          const Bucket& bk = c->buckets[bi];
          if (c->rank == 0)
            for (int r = 0; r < c->world; ++r)
              CK_NCCL(ncclRecv(c->recv + ((size_t)r * c->P + bk.off) * c->gsz, bk.len, gtype(c), r, c->comm, cs));
          CK_NCCL(ncclSend(c->grads + bk.off * c->gsz, bk.len, gtype(c), 0, c->comm, cs));
        }
        CK_NCCL(ncclGroupEnd());
      } else if (c->world > 1) {
        KScope ks_(c, HDP_K_COMM, 0, cs);
        CK_NCCL(ncclGroupStart());
        for (size_t bi = b0; bi < b1; ++bi) {
          const Bucket& bk = c->buckets[bi];
          if (c->d.wire == HDP_WIRE_FP16_A2A)  // A9: owner j receives every rank's shard j, rank-ordered
            CK_NCCL(ncclAlltoAll(c->grads + bk.off * c->gsz, c->recv + bk.off * c->gsz, bk.shard, gtype(c), c->comm, cs));
          else  // NCCL-native reduction (fp16 sum, or fp32 wire)
            CK_NCCL(ncclReduceScatter(c->grads + bk.off * c->gsz, c->recv + bk.off * c->gsz, bk.shard, gtype(c), ncclSum,
                                      c->comm, cs));
        }
        CK_NCCL(ncclGroupEnd());
      }
      // world 1: a group's buckets are contiguous in every buffer (one shard each, master
      // offset = gradient offset), so the group is one K11 launch over their union
      const bool merge = c->world == 1;
      for (size_t bi = b0; bi < b1; ++bi) {
        if (c->task0 && c->rank != 0) break;  // step 5 runs on task 0 only
        const Bucket& bk = c->buckets[bi];
        a.count = bk.shard;
        if (merge) {
          const Bucket& bl = c->buckets[b1 - 1];
          a.count = bl.off + bl.len - bk.off;
          bi = b1 - 1;
        }
        a.W = c->master + bk.moff;
        a.S1 = c->s1 + bk.moff;
        a.S2 = c->s2 ? c->s2 + bk.moff : nullptr;
        a.w16 = c->f32 ? nullptr : (__half*)(c->w + (bk.off + (long)c->owner_index() * bk.shard) * 2);
        a.w32 = c->f32 ? (float*)(c->w + (bk.off + (long)c->owner_index() * bk.shard) * 4) : nullptr;
        const int grad_f32 = c->gt();
        a.w_bf16 = c->bf ? 1 : 0;
        if (c->world == 1) {
          a.g = c->grads + bk.off * c->gsz;  // slot r at + r*P
          a.g_stride = c->P;
          a.nsrc = c->nslots;
        } else if (c->task0) {
          a.g = c->recv + bk.off * c->gsz;   // worker r's gradients at + r*P
          a.g_stride = c->P;
          a.nsrc = c->world;
        } else {
          a.g = c->recv + bk.off * c->gsz;
          a.g_stride = bk.shard;
          a.nsrc = c->d.wire == HDP_WIRE_FP16_A2A ? c->world : 1;
        }
        KScope ks_(c, HDP_K_UPDATE, 1, cs);
        CK_CUDA(hdp::launch_avg_update(a, grad_f32, opt, cs));  // A10 / K11
      }
      if (c->world > 1) {  // A11: step 6 "broadcast" (+ the non-finite count, with the last group)
        KScope ks_(c, HDP_K_COMM, 0, cs);
        CK_NCCL(ncclGroupStart());
        for (size_t bi = b0; bi < b1; ++bi) {
          const Bucket& bk = c->buckets[bi];
          if (c->task0) {  // task 0 broadcasts the updated parameters
            CK_NCCL(ncclBroadcast(c->w + bk.off * c->esz, c->w + bk.off * c->esz, bk.len, wtype(c), 0, c->comm, cs));
            continue;
          }
          char* mine = c->w + (bk.off + (long)c->rank * bk.shard) * c->esz;
          CK_NCCL(ncclAllGather(mine, c->w + bk.off * c->esz, bk.shard, wtype(c), c->comm, cs));
        }
        if (last) CK_NCCL(ncclAllReduce(c->status, c->status, 1, ncclInt32, ncclSum, c->comm, cs));
        CK_NCCL(ncclGroupEnd());
      }
    }
  }
  if (dyn) {
    KScope ks_(c, HDP_K_UPDATE, 1, cs);
    CK_CUDA(hdp::launch_loss_scale_update(c->dyn_state(), c->alpha_dev(), c->dyn_interval, 2.f, 1.f, cs));
    count_src = c->dyn_state();
  }
  if (c->drop_on()) {  // next step's dropout masks
    KScope ks_(c, HDP_K_UPDATE, 1, cs);
    CK_CUDA(hdp::launch_increment(c->drop_step(), cs));
  }
  if (c->d.vocab > 0) {  // out-of-range token ids counted by this step's forward passes (the
    // next forward counts into the same word: read and cleared before it may start)
    CK_CUDA(cudaMemcpyAsync(c->count_host + 1, c->status + 16, sizeof(int), cudaMemcpyDeviceToHost, cs));
    CK_CUDA(cudaMemsetAsync(c->status + 16, 0, sizeof(int), cs));
  }
  CK_CUDA(cudaEventRecord(c->ev_done, cs));
  CK_CUDA(cudaStreamWaitEvent(s, c->ev_done, 0));  // next forward sees the new weights
  // the non-finite count's read-back stays off the caller's path (its source is written only
  // by the update / exchange kernels, i.e. after the next call's reset on this stream)
  CK_CUDA(cudaMemcpyAsync(c->count_host, count_src, sizeof(int), cudaMemcpyDeviceToHost, cs));
  CK_CUDA(cudaEventRecord(c->ev_count, cs));
  for (auto& st : c->st) st.bwd = false;
  if (nonfinite_host) {
    CK_CUDA(cudaEventSynchronize(c->ev_count));
    CK(nccl_async_check(c));
    *nonfinite_host = *c->count_host;
    if (c->count_host[1] > 0) {
      c->poisoned = true;
      return fail(HDP_ERR_ARG, "%d token ids outside [0, %d)", c->count_host[1], c->d.vocab);
    }
    if (*c->count_host > 0 && !dyn) {
      c->poisoned = true;
      return fail(HDP_ERR_NONFINITE, "%d non-finite gradient values (loss scale %g)", *c->count_host,
                  (double)c->alpha);
    }
  } else {
    c->count_pending = true;
  }
  return HDP_OK;
}

int hdp_set_option(hdp_ctx* c, const char* name, double value) {
  if (!name) return fail(HDP_ERR_ARG, "null option name");
  const std::string n(name);
  if (n == "partial_fraction" || n == "straggler_mask" || n == "straggler_us") {
    if (!c || !c->bound) return fail(HDP_ERR_STATE, "option %s needs a bound context", name);
    if (n == "partial_fraction") {
      if (!(value > 0.0 && value <= 1.0)) return fail(HDP_ERR_ARG, "partial_fraction must be in (0, 1]");
      const int N = c->Nw();
      const int q = (int)std::ceil(value * N - 1e-9);  // SPEC.md:322 ceil(f*N)
      if (q < N) {
        if (!c->p2p) return fail(HDP_ERR_UNSUPPORTED, "partial collection needs the one-kernel exchange");
        if (c->dyn_interval > 0) return fail(HDP_ERR_UNSUPPORTED, "partial collection with dynamic loss scaling");
      }
      c->partial_fraction = value;
      c->quorum = q < N ? std::max(q, 1) : 0;
    } else if (n == "straggler_mask") {
      if (!(value >= 0 && value < 4294967296.0)) return fail(HDP_ERR_ARG, "straggler_mask out of range");
      c->straggler_mask = (unsigned)value;
    } else {
      if (!(value >= 0 && value <= 10e6)) return fail(HDP_ERR_ARG, "straggler_us must be in [0, 1e7]");
      c->straggler_ns = (unsigned long long)(value * 1000.0);
    }
    return HDP_OK;
  }
  const int id = hdp::opt_find(name);
  if (id < 0) return fail(HDP_ERR_ARG, "unknown option %s", name);
  if (!(value >= -1 && value <= 1 << 20) || value != std::floor(value))
    return fail(HDP_ERR_ARG, "option %s takes an integer value", name);
  hdp::g_opt[id] = (int)value;
  if (c && !c->host_only) {
    CK_CUDA(cudaSetDevice(c->device));
    CK_CUDA(cudaDeviceSynchronize());
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  return HDP_OK;
}

int hdp_get_option(const char* name, double* value) {
  if (!name || !value) return fail(HDP_ERR_ARG, "null argument");
  const int id = hdp::opt_find(name);
  if (id < 0) return fail(HDP_ERR_ARG, "unknown option %s", name);
  *value = hdp::g_opt[id];
  return HDP_OK;
}

int hdp_partial_state(hdp_ctx* c, unsigned* mask, int* count) {
  CK(check_ready(c));
  if (!mask || !count) return fail(HDP_ERR_ARG, "null argument");
  if (!c->p2p || c->quorum == 0) {
    *mask = c->Nw() >= 32 ? 0xffffffffu : (1u << c->Nw()) - 1u;
    *count = c->Nw();
    return HDP_OK;
  }
  CK_CUDA(cudaSetDevice(c->device));
  CK_CUDA(cudaDeviceSynchronize());
  unsigned w[2];
  CK_CUDA(cudaMemcpy(w, c->fwin + hdp::P2P_DECISION, sizeof w, cudaMemcpyDeviceToHost));
  *mask = w[0];  // little-endian low word of (seq << 32) | mask
  *count = __builtin_popcount(w[0]);
  return HDP_OK;
}

int hdp_profile(hdp_ctx* c, int enable) {
  CK(check_ready(c));
  c->prof = enable != 0;
  return HDP_OK;
}

int hdp_profile_read(hdp_ctx* c, double* ms, long long* launches, int reset) {
  CK(check_ready(c));
  CK_CUDA(cudaDeviceSynchronize());
  for (const auto& r : c->precs) {
    float t = 0.f;
    CK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    c->prof_ms[r.tag] += t;
    c->prof_n[r.tag] += 1;
  }
  c->precs.clear();
  c->evused = 0;
  for (int i = 0; i < HDP_K_NTAGS; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_n[i];
    if (reset) {
      c->prof_ms[i] = 0;
      c->prof_n[i] = 0;
    }
  }
  return HDP_OK;
}

int hdp_profile_timeline(hdp_ctx* c, int* tags, int* lanes, double* t0_ms, double* t1_ms, int cap, int* n) {
  CK(check_ready(c));
  if (!n || cap < 0 || (cap > 0 && (!tags || !lanes || !t0_ms || !t1_ms))) return fail(HDP_ERR_ARG, "bad arguments");
  CK_CUDA(cudaDeviceSynchronize());
  *n = (int)c->precs.size();
  if (c->precs.empty()) return HDP_OK;
  const cudaEvent_t ref = c->precs[0].a;
  for (int i = 0; i < *n && i < cap; ++i) {
    const auto& r = c->precs[i];
    float a = 0.f, b = 0.f;
    CK_CUDA(cudaEventElapsedTime(&a, ref, r.a));
    CK_CUDA(cudaEventElapsedTime(&b, ref, r.b));
    tags[i] = r.tag;
    lanes[i] = r.lane;
    t0_ms[i] = a;
    t1_ms[i] = b;
  }
  return HDP_OK;
}

long long hdp_kernel_launches(const hdp_ctx* c) { return c ? c->kernels : -1; }

void* hdp_weights_ptr(hdp_ctx* c) { return c && c->bound ? c->w : nullptr; }
void* hdp_grads_ptr(hdp_ctx* c, int slot) {
  return c && c->bound && slot >= 0 && slot < c->nslots ? c->grads + (long)slot * c->P * c->gsz : nullptr;
}
void* hdp_master_ptr(hdp_ctx* c) { return c && c->bound ? c->master : nullptr; }

void* hdp_debug_buffer(hdp_ctx* c, int slot, const char* name) {
  if (!c || !c->bound || !name || slot < 0 || slot >= c->nslots || c->d.n_layers <= 0) return nullptr;
  hdp_ctx::Slot& S = c->slot[slot];
  const std::string n(name);
  if (n == "Hs") return S.Hs;
  if (n == "C") return S.C;
  if (n == "gates") return S.gates;
  if (n == "X0") return S.X0;
  if (n == "Z") return S.Z;  // (unfused head only: the fused head keeps its column partials there)
  if (n == "dz") return S.dz;
  if (n == "dA") return c->dA;
  if (n == "dA2") return c->dA2;
  if (n == "dH0") return c->dH[0];
  if (n == "dH1") return c->dH[1];
  if (n == "Hst") return c->hst ? c->Hst(slot, 0) : nullptr;  // recurrent dropout: h~ [L][T+1][B][hp]
  if (n == "Wcopy") return c->wcopies;                        // P2P loopback: weight copies 1..nslots-1
  return nullptr;
}

int hdp_fused_avg_update(const void* grads, long long src_stride, int nsrc, int grads_f32, long long count, float* W,
                         float* S1, float* S2, void* w16, float* w32, float inv_scale, float lr, float momentum,
                         int optimizer, const double* adam, int* nonfinite_dev, float l2x2, void* stream) {
  if (!grads || !W || !S1 || nsrc < 1 || count < 0 || (optimizer == HDP_OPT_ADAM && (!S2 || !adam)) ||
      optimizer < 0 || optimizer > 1)
    return fail(HDP_ERR_ARG, "hdp_fused_avg_update: bad arguments");
  hdp::UpdateArgs a;
  a.g = grads;
  a.g_stride = src_stride;
  a.nsrc = nsrc;
  a.count = count;
  a.W = W;
  a.S1 = S1;
  a.S2 = S2;
  a.w16 = (__half*)w16;
  a.w32 = w32;
  a.inv_scale = inv_scale;
  a.lam = lr;
  a.mom = momentum;
  a.nonfinite = nonfinite_dev;
  a.l2x2 = l2x2;
  if (optimizer == HDP_OPT_ADAM) {
    const double b1 = adam[0], b2 = adam[1], eps = adam[2], k = adam[3];
    a.b1 = (float)b1;
    a.omb1 = (float)(1.0 - b1);
    a.b2 = (float)b2;
    a.omb2 = (float)(1.0 - b2);
    a.c1 = (float)(1.0 / (1.0 - std::pow(b1, k)));
    a.c2 = (float)(1.0 / (1.0 - std::pow(b2, k)));
    a.eps = (float)eps;
  }
  const bool vec_ok = (count % 8 == 0) && (src_stride % 8 == 0) &&
                      !((uintptr_t)grads & 15) && !((uintptr_t)W & 15) && !((uintptr_t)S1 & 15) &&
                      !((uintptr_t)S2 & 15) && !((uintptr_t)w16 & 15) && !((uintptr_t)w32 & 15);
  if (!vec_ok) return fail(HDP_ERR_ARG, "hdp_fused_avg_update: needs count %% 8 == 0 and 16-byte aligned buffers");
  CK_CUDA(hdp::launch_avg_update(a, grads_f32, optimizer, (cudaStream_t)stream));
  return HDP_OK;
}

int hdp_gemm_f16(const void* A, long long lda, int a_mn, const void* B, long long ldb, int b_mn, int M, int N, int K,
                 void* C, long long ldc, int c_mode, const float* bias, int bias_on_m, int relu, int accumulate,
                 float* ws, long long ws_floats, int bn, int splits, void* stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0 || c_mode < 0 || c_mode > 2)
    return fail(HDP_ERR_ARG, "hdp_gemm_f16: bad arguments");
  hdp::Epilogue e;
  e.mode = c_mode;
  e.out = C;
  e.ldo = ldc;
  e.bias = bias;
  e.bias_on_m = bias_on_m;
  e.relu = relu;
  e.accumulate = accumulate;
  hdp::GemmPlan p;
  if (hdp::gemm_plan_tc(&p, (const __half*)A, lda, a_mn, (const __half*)B, ldb, b_mn, M, N, K, e, ws,
                        ws ? (size_t)ws_floats : 0, bn, splits))
    return fail(HDP_ERR_ARG, "hdp_gemm_f16: %s", hdp::gemm_last_error());
  static bool inited = false;
  if (!inited) {
    CK_CUDA(hdp::gemm_init());
    inited = true;
  }
  CK_CUDA(hdp::gemm_run(p, (cudaStream_t)stream));
  return HDP_OK;
}

int hdp_gemm_f32(const float* A, long long lda, int a_mn, const float* B, long long ldb, int b_mn, int M, int N, int K,
                 float* C, long long ldc, int c_mode, const float* bias, int bias_on_m, int relu, int accumulate,
                 void* stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0 || c_mode < 0 || c_mode > 1)
    return fail(HDP_ERR_ARG, "hdp_gemm_f32: bad arguments");
  hdp::Epilogue e;
  e.mode = c_mode;
  e.out = C;
  e.ldo = ldc;
  e.bias = bias;
  e.bias_on_m = bias_on_m;
  e.relu = relu;
  e.accumulate = accumulate;
  hdp::GemmPlan p;
  if (hdp::gemm_plan_f32(&p, A, lda, a_mn, B, ldb, b_mn, M, N, K, e))
    return fail(HDP_ERR_ARG, "hdp_gemm_f32: %s", hdp::gemm_last_error());
  CK_CUDA(hdp::gemm_run(p, (cudaStream_t)stream));
  return HDP_OK;
}

}  // extern "C"
