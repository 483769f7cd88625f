// spt_ffn_abi.cu -- the C ABI of include/spt_ffn.h: validation, workspace
// carving and dispatch to the sm_100a kernels.  Host code only.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cstdlib>

#include "internal.h"

namespace spt {

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPT_FFN_PDL");  // measured neutral on B200 (round 2): opt-in
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ---- per-kernel profiling: a pair of CUDA events around every launch, on the
// launch stream; aggregated on read.  Off by default (zero overhead).
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;

static cudaEvent_t ev_get() {
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void prof_begin(const char* name, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> l(g_prof_mu);
  ProfRec r{name, ev_get(), ev_get()};
  cudaEventRecord(r.a, s);
  g_prof.push_back(r);
}
void prof_end(cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> l(g_prof_mu);
  if (!g_prof.empty()) cudaEventRecord(g_prof.back().b, s);
}

static inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

static spt_status make_geom(const spt_ffn_desc* d, Geom* g) {
  if (!d) return SPT_ERR_INVALID_ARGUMENT;
  if (d->n_tokens < 0 || d->d_model <= 0 || d->d_ff <= 0 || d->n_blocks <= 0)
    return SPT_ERR_INVALID_ARGUMENT;
  if (d->top_k < 1 || d->top_k > d->n_blocks) return SPT_ERR_INVALID_ARGUMENT;
  if (d->d_ff % d->n_blocks) return SPT_ERR_INVALID_ARGUMENT;
  if (d->dtype != SPT_F32 && d->dtype != SPT_BF16) return SPT_ERR_INVALID_ARGUMENT;
  if (d->act < SPT_ACT_RELU || d->act > SPT_ACT_SWIGLU) return SPT_ERR_INVALID_ARGUMENT;
  if (d->gate != SPT_GATE_SIGMOID && d->gate != SPT_GATE_NONE) return SPT_ERR_INVALID_ARGUMENT;
  if (!(d->balance_weight >= 0.f) || d->balance_weight > 3.0e38f)  // NaN, < 0, Inf
    return SPT_ERR_INVALID_ARGUMENT;
  if (d->flags & ~SPT_FFN_DETERMINISTIC) return SPT_ERR_INVALID_ARGUMENT;
  g->T = d->n_tokens;
  g->d = d->d_model;
  g->D = d->d_ff;
  g->G = d->n_blocks;
  g->k = d->top_k;
  g->bw = g->D / g->G;
  g->mp = d->act == SPT_ACT_SWIGLU ? 2 : 1;
  g->dtype = d->dtype;
  g->act = d->act;
  g->gate = d->gate;
  g->pairs = g->T * g->k;
  g->rows_cap = g->pairs + (int64_t)g->G * kTileM;
  g->n_chunks = ceil_div(g->T, kRouteChunk);
  g->n_sub = ceil_div(g->T, kTopkChunk);
  g->gpad = (int)ceil_div(g->G, 16) * 16;
  g->esize = d->dtype == SPT_BF16 ? 2 : 4;
  g->lbw = d->balance_weight;
  if (g->G > kMaxBlocks) return SPT_ERR_UNSUPPORTED;
  if (g->d % 64) return SPT_ERR_UNSUPPORTED;
  if (g->bw % 16) return SPT_ERR_UNSUPPORTED;
  if (g->pairs + (int64_t)g->G * kTileM > INT32_MAX) return SPT_ERR_UNSUPPORTED;
  if (g->dtype == SPT_BF16 && !tc_supported(*g)) return SPT_ERR_UNSUPPORTED;
  // fp32: the split tensor-core path wherever the tcgen05 kernels support the
  // shape; the SIMT kernels otherwise (G > 128) and for the load-balancing
  // gradient (its dense dX term has no split kernel)
  g->split = g->dtype == SPT_F32 && tc_supported(*g) && g->lbw == 0.f && !simt_forced();
  return SPT_OK;
}

static int dwr_splits(const Geom& g) { return dense_tn_splits(g); }

struct Sizes {
  size_t z, h, stash;
  size_t part, dz, da, dlogit, dgate, dlg, dwr, counts, base, nb, ctr, tl, uo, tb, lbp, lbx, xs, ws_w, ws;
};

static Sizes compute_sizes(const Geom& g) {
  Sizes s{};
  const size_t e = (size_t)g.esize;
  s.z = align256((size_t)g.rows_cap * g.mp * g.bw * e);
  s.h = align256((size_t)g.rows_cap * g.bw * e);
  // the device tile schedules live in the stash: the forward builds them, the
  // backward reuses them (same routing)
  s.tl = align256((size_t)(ceil_div(g.pairs, kTileM) + g.G) * 4);
  s.uo = align256((size_t)(g.G + 2) * 4);
  s.tb = s.tl;
  s.stash = s.z + s.h + s.tl + s.uo + s.tb;
  s.part = align256((size_t)g.rows_cap * g.d * e);
  s.dz = align256((size_t)g.rows_cap * g.mp * g.bw * e);
  s.da = align256((size_t)g.rows_cap * g.bw * 4);  // fp32 dA rows (both paths)
  s.dlogit = align256((size_t)g.rows_cap * 4);
  s.dgate = align256((size_t)g.rows_cap * 4);
  s.dlg = g.tc() ? align256((size_t)2 * g.T * g.gpad * 2) : 0;
  s.dwr = g.tc() ? align256((size_t)dwr_splits(g) * g.G * g.d * 4) : 0;
  // split: bf16 hi | lo copies of x, dy and the weights (4 bytes per element)
  s.xs = g.split ? align256((size_t)g.T * g.d * 4) : 0;
  s.ws_w = g.split ? align256((size_t)g.mp * g.D * g.d * 4) + align256((size_t)g.D * g.d * 4) +
                         align256((size_t)g.G * g.d * 4)
                   : 0;
  s.counts = align256((size_t)g.n_sub * g.G * 4);
  s.base = s.counts;
  s.nb = align256((size_t)g.G * 4);
  s.ctr = 256;  // work counters (the dW kernels' grad-input combine side work)
  s.lbp = align256((size_t)g.n_chunks * g.G * 4);  // balance loss: per-chunk softmax sums
  s.lbx = g.lbw == 0.f ? 0                         // balance gradient: dense router term
          : align256(g.dtype == SPT_BF16 ? (size_t)g.T * g.d * 2 : (size_t)g.T * g.G * 4);
  s.ws = s.part + s.dz + s.da + s.dlogit + s.dgate + s.dlg + s.dwr + s.counts + s.base + s.nb + s.ctr +
         s.lbp + s.lbx + 2 * s.xs + s.ws_w;
  return s;
}

static Bufs carve(const Geom& g, void* stash, void* ws) {
  Sizes s = compute_sizes(g);
  Bufs b{};
  uint8_t* p = (uint8_t*)stash;
  if (p) {
    b.z = p;
    b.h = p + s.z;
    uint8_t* q = p + s.z + s.h;
    b.tile_list = (int32_t*)q; q += s.tl;
    b.unit_offsets = (int32_t*)q; q += s.uo;
    b.tile_block = (int32_t*)q;
  }
  uint8_t* w = (uint8_t*)ws;
  b.part = w; w += s.part;
  b.dz = w; w += s.dz;
  b.da = s.da ? (float*)w : nullptr; w += s.da;
  b.dlogit = (float*)w; w += s.dlogit;
  b.dgate = (float*)w; w += s.dgate;
  b.dlg = s.dlg ? (void*)w : nullptr; w += s.dlg;
  b.dwr_part = s.dwr ? (float*)w : nullptr; w += s.dwr;
  b.n_split = g.tc() ? dwr_splits(g) : 0;
  b.chunk_counts = (int32_t*)w; w += s.counts;
  b.chunk_base = (int32_t*)w; w += s.base;
  b.n_b = (int32_t*)w; w += s.nb;
  b.side_ctr = (int32_t*)w; w += s.ctr;
  b.lb_part = (float*)w; w += s.lbp;
  b.lb_x = s.lbx ? (void*)w : nullptr; w += s.lbx;
  if (g.split) {
    b.xs = w; w += s.xs;
    b.dys = w; w += s.xs;
    b.w1s = w; w += align256((size_t)g.mp * g.D * g.d * 4);
    b.w2s = w; w += align256((size_t)g.D * g.d * 4);
    b.wrs = w; w += align256((size_t)g.G * g.d * 4);
  }
  return b;
}

// LoRA-wrapped calls (ABI 3): the plain stash / workspace followed by the LoRA
// buffers (LoraArgs in internal.h).
struct LoraSizes {
  size_t ust, qhl, stash;                              // stash extras
  size_t xaug, waug, uv, rowp, gpart, spart, dhl, ws;  // workspace extras
  int n_split_u, n_split_v;
};

static spt_status lora_geom(const spt_ffn_desc* d, int32_t rank, Geom* g) {
  spt_status st = make_geom(d, g);
  if (st != SPT_OK) return st;
  if (rank < 1) return SPT_ERR_INVALID_ARGUMENT;
  if (g->dtype != SPT_BF16) return SPT_ERR_UNSUPPORTED;  // tcgen05 path only
  if ((int64_t)g->mp * rank > kLoraK) return SPT_ERR_UNSUPPORTED;
  return SPT_OK;
}

static Geom skinny_geom(const Geom& g, int n) {
  Geom h = g;
  h.G = n;
  h.gpad = (int)ceil_div(n, 16) * 16;
  return h;
}

static LoraSizes lora_sizes(const Geom& g, int r) {
  LoraSizes s{};
  const int64_t tiles = ceil_div(g.pairs, kTileM) + g.G;
  s.ust = align256((size_t)g.T * g.mp * r * 4);
  s.qhl = align256((size_t)2 * g.T * lora_qpad(r) * 2);
  s.stash = s.ust + s.qhl;
  const int ka = lora_ka(g.mp, r);
  s.xaug = align256((size_t)g.T * (g.d + ka) * 2);
  s.waug = align256((size_t)g.mp * g.D * (g.d + ka) * 2);
  s.uv = align256((size_t)g.T * g.mp * r * 4);
  s.rowp = align256((size_t)lora_chunks(g) * g.rows_cap * kLoraK * 4);
  s.gpart = align256((size_t)tiles * (g.mp + 1) * g.bw * r * 4);
  s.n_split_u = dense_tn_splits(skinny_geom(g, g.mp * r));
  s.n_split_v = dense_tn_splits(skinny_geom(g, r));
  s.spart = align256((size_t)std::max(s.n_split_u * g.mp * r, s.n_split_v * r) * g.d * 4);
  s.dhl = align256((size_t)2 * g.T * lora_upad(g, r) * 2);
  s.ws = s.xaug + s.waug + s.uv + s.rowp + s.gpart + s.spart + s.dhl;
  return s;
}

static LoraArgs lora_carve(const Geom& g, const spt_lora* lr, void* stash, void* ws) {
  const Sizes ps = compute_sizes(g);
  const LoraSizes s = lora_sizes(g, lr->rank);
  LoraArgs a{};
  a.r = lr->rank;
  a.ka = lora_ka(g.mp, lr->rank);
  a.b1 = lr->b1;
  a.c1 = lr->c1;
  a.b2 = lr->b2;
  a.c2 = lr->c2;
  uint8_t* p = (uint8_t*)stash + ps.stash;
  a.ust = (float*)p; p += s.ust;
  a.qhl = p;
  uint8_t* w = (uint8_t*)ws + ps.ws;
  a.xaug = w; w += s.xaug;
  a.waug = w; w += s.waug;
  a.uv = (float*)w; w += s.uv;
  a.rowp = (float*)w; w += s.rowp;
  a.gpart = (float*)w; w += s.gpart;
  a.spart = (float*)w; w += s.spart;
  a.dhl = w;
  a.n_split_u = s.n_split_u;
  a.n_split_v = s.n_split_v;
  return a;
}

static bool lora_complete(const spt_lora* l) { return l && l->b1 && l->c1 && l->b2 && l->c2; }

static RouteView view(const spt_route_buf* r) {
  return RouteView{r->logits,       r->topk_idx,   r->topk_gate, r->block_offsets,
                   r->bucket_token, r->bucket_gate, r->pair_slot, r->tile_offsets};
}

// Token-sized buffers may be NULL when T == 0 (empty allocations); the [G+1]
// offset arrays are always required.
static bool route_complete(const spt_route_buf* r, int64_t T) {
  if (!r || !r->block_offsets || !r->tile_offsets) return false;
  if (T == 0) return true;
  return r->logits && r->topk_idx && r->topk_gate && r->bucket_token && r->bucket_gate &&
         r->pair_slot;
}
static inline bool tok_ok(const void* p, int64_t T) { return p || T == 0; }

static spt_status device_ok() {
  // per device (a process may drive several GPUs); 0 = unknown, 1 = sm_100, 2 = other
  static std::atomic<int> cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return SPT_ERR_CUDA;
  }
  std::atomic<int>& c = cached[dev >= 0 && dev < 64 ? dev : 0];
  int v = c.load(std::memory_order_relaxed);
  if (!v) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    v = (major == 10 && minor == 0) ? 1 : 2;
    c.store(v, std::memory_order_relaxed);
  }
  return v == 1 ? SPT_OK : SPT_ERR_UNSUPPORTED;
}

static spt_status to_status(cudaError_t e) { return e == cudaSuccess ? SPT_OK : SPT_ERR_CUDA; }

}  // namespace spt

using namespace spt;

extern "C" {
#pragma GCC visibility push(default)

int spt_ffn_abi_version(void) { return SPT_FFN_ABI_VERSION; }

uint64_t spt_ffn_launch_count(void) { return g_launches.load(); }

spt_status spt_ffn_profile_enable(int on) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  g_prof_on = on != 0;
  for (auto& r : g_prof) {
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof.clear();
  return SPT_OK;
}

int64_t spt_ffn_profile_read(char* buf, size_t len) {
  std::lock_guard<std::mutex> l(g_prof_mu);
  std::map<std::string, std::pair<long, double>> agg;
  std::vector<std::string> order;
  for (auto& r : g_prof) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return -1;
    auto it = agg.find(r.name);
    if (it == agg.end()) {
      order.push_back(r.name);
      agg[r.name] = {1, ms};
    } else {
      it->second.first += 1;
      it->second.second += ms;
    }
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof.clear();
  std::string out;
  char line[256];
  for (auto& n : order) {
    snprintf(line, sizeof line, "%s %ld %.6f\n", n.c_str(), agg[n].first, agg[n].second);
    out += line;
  }
  if (buf && len) {
    size_t n = out.size() < len - 1 ? out.size() : len - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
}

const char* spt_status_string(spt_status s) {
  switch (s) {
    case SPT_OK: return "SPT_OK";
    case SPT_ERR_INVALID_ARGUMENT: return "SPT_ERR_INVALID_ARGUMENT";
    case SPT_ERR_UNSUPPORTED: return "SPT_ERR_UNSUPPORTED";
    case SPT_ERR_WORKSPACE_TOO_SMALL: return "SPT_ERR_WORKSPACE_TOO_SMALL";
    case SPT_ERR_CUDA: return "SPT_ERR_CUDA";
  }
  return "SPT_ERR_UNKNOWN";
}

spt_status spt_ffn_sizes(const spt_ffn_desc* desc, size_t* stash_bytes, size_t* workspace_bytes) {
  if (!stash_bytes || !workspace_bytes) return SPT_ERR_INVALID_ARGUMENT;
  Geom g;
  spt_status st = make_geom(desc, &g);
  if (st != SPT_OK) return st;
  Sizes s = compute_sizes(g);
  *stash_bytes = s.stash;
  *workspace_bytes = s.ws;
  return SPT_OK;
}

spt_status spt_ffn_route(const spt_ffn_desc* desc, const void* x, const void* w_r, unsigned flags,
                         const spt_route_buf* r, void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  spt_status st = make_geom(desc, &g);
  if (st != SPT_OK) return st;
  const bool logits_in = flags & SPT_ROUTE_LOGITS_IN;
  if (!route_complete(r, g.T) || !ws || (!logits_in && (!tok_ok(x, g.T) || !w_r)))
    return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws) return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  Bufs b = carve(g, nullptr, ws);
  RouteView rv = view(r);
  if (g.T == 0) {
    if (cudaMemsetAsync(r->block_offsets, 0, (g.G + 1) * 4, s) != cudaSuccess ||
        cudaMemsetAsync(r->tile_offsets, 0, (g.G + 1) * 4, s) != cudaSuccess)
      return SPT_ERR_CUDA;
    return SPT_OK;
  }
  cudaError_t e = cudaSuccess;
  if (!logits_in) {
    e = g.tc() ? tc_router(g, x, w_r, r->logits, s, &b)
               : launch_router_simt(g, x, w_r, r->logits, s);
    if (e != cudaSuccess) return SPT_ERR_CUDA;
  }
  return to_status(launch_topk_bucket(g, rv, b, s));
}

spt_status spt_ffn_balance_loss(const spt_ffn_desc* desc, const spt_route_buf* r, float* loss,
                                void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  spt_status st = make_geom(desc, &g);
  if (st != SPT_OK) return st;
  if (!route_complete(r, g.T) || !loss || !ws) return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws) return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  Bufs b = carve(g, nullptr, ws);
  return to_status(launch_balance_loss(g, view(r), b, loss, (cudaStream_t)stream));
}

spt_status spt_ffn_forward(const spt_ffn_desc* desc, const void* x, const void* w1, const void* w2,
                           const spt_route_buf* r, void* y, void* stash, void* ws, size_t ws_bytes,
                           void* stream) {
  Geom g;
  spt_status st = make_geom(desc, &g);
  if (st != SPT_OK) return st;
  if (!tok_ok(x, g.T) || !w1 || !w2 || !route_complete(r, g.T) || !tok_ok(y, g.T) || !stash || !ws)
    return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws) return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  if (g.T == 0) return SPT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  Bufs b = carve(g, stash, ws);
  RouteView rv = view(r);
  cudaError_t e = g.tc() ? tc_forward(g, x, w1, w2, rv, y, b, s)
                         : simt_forward(g, x, w1, w2, rv, y, b, s);
  return to_status(e);
}

spt_status spt_ffn_backward(const spt_ffn_desc* desc, const void* x, const void* w1, const void* w2,
                            const void* w_r, const spt_route_buf* r, const void* stash,
                            const void* dy, void* dx, float* dw1, float* dw2, float* dw_r,
                            float* dgate, unsigned flags, void* ws, size_t ws_bytes,
                            void* dw_event, void* stream) {
  Geom g;
  spt_status st = make_geom(desc, &g);
  if (st != SPT_OK) return st;
  if (!tok_ok(x, g.T) || !w1 || !w2 || !w_r || !route_complete(r, g.T) || !stash ||
      !tok_ok(dy, g.T) || !tok_ok(dx, g.T) || !dw1 || !dw2 || !dw_r || !ws)
    return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws) return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const bool acc = flags & SPT_BWD_ACCUMULATE_DW;
  if (g.T == 0) {
    if (acc) {
      if (dw_event && cudaEventRecord((cudaEvent_t)dw_event, s) != cudaSuccess) return SPT_ERR_CUDA;
      return SPT_OK;
    }
    const size_t w1b = (size_t)g.mp * g.D * g.d * 4, w2b = (size_t)g.D * g.d * 4,
                 wrb = (size_t)g.G * g.d * 4;
    if (cudaMemsetAsync(dw1, 0, w1b, s) != cudaSuccess || cudaMemsetAsync(dw2, 0, w2b, s) ||
        cudaMemsetAsync(dw_r, 0, wrb, s))
      return SPT_ERR_CUDA;
    if (dw_event && cudaEventRecord((cudaEvent_t)dw_event, s) != cudaSuccess) return SPT_ERR_CUDA;
    return SPT_OK;
  }
  Bufs b = carve(g, const_cast<void*>(stash), ws);
  RouteView rv = view(r);
  cudaEvent_t ev = (cudaEvent_t)dw_event;
  cudaError_t e = g.tc()
                      ? tc_backward(g, x, w1, w2, w_r, rv, dy, dx, dw1, dw2, dw_r, dgate, acc, b, ev, s)
                      : simt_backward(g, x, w1, w2, w_r, rv, dy, dx, dw1, dw2, dw_r, dgate, acc, b,
                                      ev, s);
  return to_status(e);
}

spt_status spt_ffn_lora_sizes(const spt_ffn_desc* desc, int32_t rank, size_t* stash_bytes,
                              size_t* workspace_bytes) {
  if (!stash_bytes || !workspace_bytes) return SPT_ERR_INVALID_ARGUMENT;
  Geom g;
  spt_status st = lora_geom(desc, rank, &g);
  if (st != SPT_OK) return st;
  const Sizes s = compute_sizes(g);
  const LoraSizes l = lora_sizes(g, rank);
  *stash_bytes = s.stash + l.stash;
  *workspace_bytes = s.ws + l.ws;
  return SPT_OK;
}

spt_status spt_ffn_lora_forward(const spt_ffn_desc* desc, const void* x, const void* w1,
                                const void* w2, const spt_lora* lora, const spt_route_buf* r,
                                void* y, void* stash, void* ws, size_t ws_bytes, void* stream) {
  if (!lora) return SPT_ERR_INVALID_ARGUMENT;
  Geom g;
  spt_status st = lora_geom(desc, lora->rank, &g);
  if (st != SPT_OK) return st;
  if (!tok_ok(x, g.T) || !w1 || !w2 || !lora_complete(lora) || !route_complete(r, g.T) ||
      !tok_ok(y, g.T) || !stash || !ws)
    return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws + lora_sizes(g, lora->rank).ws)
    return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  if (g.T == 0) return SPT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  Bufs b = carve(g, stash, ws);
  LoraArgs la = lora_carve(g, lora, stash, ws);
  return to_status(tc_forward(g, x, w1, w2, view(r), y, b, s, &la));
}

spt_status spt_ffn_lora_backward(const spt_ffn_desc* desc, const void* x, const void* w1,
                                 const void* w2, const void* w_r, const spt_lora* lora,
                                 const spt_route_buf* r, const void* stash, const void* dy,
                                 void* dx, const spt_lora_grads* grads, float* dw_r, float* dgate,
                                 unsigned flags, void* ws, size_t ws_bytes, void* grad_event,
                                 void* stream) {
  if (!lora || !grads) return SPT_ERR_INVALID_ARGUMENT;
  Geom g;
  spt_status st = lora_geom(desc, lora->rank, &g);
  if (st != SPT_OK) return st;
  if (!tok_ok(x, g.T) || !w1 || !w2 || !w_r || !lora_complete(lora) || !route_complete(r, g.T) ||
      !stash || !tok_ok(dy, g.T) || !tok_ok(dx, g.T) || !grads->db1 || !grads->dc1 ||
      !grads->db2 || !grads->dc2 || !dw_r || !ws)
    return SPT_ERR_INVALID_ARGUMENT;
  if (ws_bytes < compute_sizes(g).ws + lora_sizes(g, lora->rank).ws)
    return SPT_ERR_WORKSPACE_TOO_SMALL;
  if ((st = device_ok()) != SPT_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const bool acc = flags & SPT_BWD_ACCUMULATE_DW;
  const int rk = lora->rank;
  if (g.T == 0) {  // no tokens: zero gradients (unless accumulating)
    if (!acc) {
      const size_t n1 = (size_t)g.mp * rk * g.d * 4, n2 = (size_t)g.mp * g.D * rk * 4,
                   n3 = (size_t)g.D * rk * 4, n4 = (size_t)rk * g.d * 4,
                   n5 = (size_t)g.G * g.d * 4;
      if (cudaMemsetAsync(grads->db1, 0, n1, s) != cudaSuccess ||
          cudaMemsetAsync(grads->dc1, 0, n2, s) != cudaSuccess ||
          cudaMemsetAsync(grads->db2, 0, n3, s) != cudaSuccess ||
          cudaMemsetAsync(grads->dc2, 0, n4, s) != cudaSuccess ||
          cudaMemsetAsync(dw_r, 0, n5, s) != cudaSuccess)
        return SPT_ERR_CUDA;
    }
    if (grad_event && cudaEventRecord((cudaEvent_t)grad_event, s) != cudaSuccess)
      return SPT_ERR_CUDA;
    return SPT_OK;
  }
  Bufs b = carve(g, const_cast<void*>(stash), ws);
  LoraArgs la = lora_carve(g, lora, const_cast<void*>(stash), ws);
  la.db1 = grads->db1;
  la.dc1 = grads->dc1;
  la.db2 = grads->db2;
  la.dc2 = grads->dc2;
  la.accumulate = acc;
  return to_status(tc_backward(g, x, w1, w2, w_r, view(r), dy, dx, nullptr, nullptr, dw_r, dgate,
                               acc, b, (cudaEvent_t)grad_event, s, &la));
}

spt_status spt_mha_topl(const spt_topl_desc* desc, const uint8_t* codes_q, const uint8_t* codes_k,
                        int32_t* indices, void* stream) {
  if (!desc) return SPT_ERR_INVALID_ARGUMENT;
  const spt_topl_desc& d = *desc;
  if (d.n_heads < 0 || d.n_q < 0 || d.n_k < 0 || d.top_l < 1 || d.n_codebooks < 1 ||
      d.n_codebooks > topl_max_score() || d.n_codewords < 1 || d.n_codewords > 256 ||
      (d.causal != 0 && d.causal != 1))
    return SPT_ERR_INVALID_ARGUMENT;
  const int64_t nout = (int64_t)d.n_heads * d.n_q;
  if (nout == 0) return SPT_OK;
  if (!indices || !codes_q || (d.n_k > 0 && !codes_k)) return SPT_ERR_INVALID_ARGUMENT;
  // the kernel's static smem counts against the same 227 KB opt-in limit
  if (topl_smem_bytes(d.n_k, d.n_codebooks, d.n_codewords) + topl_static_smem_bytes() > 227 * 1024)
    return SPT_ERR_UNSUPPORTED;
  spt_status st = device_ok();
  if (st != SPT_OK) return st;
  return to_status(launch_topl(d.n_heads, d.n_q, d.n_k, d.n_codebooks, d.n_codewords, d.top_l,
                               d.causal, codes_q, codes_k, indices, (cudaStream_t)stream));
}

#pragma GCC visibility pop
}  // extern "C"
