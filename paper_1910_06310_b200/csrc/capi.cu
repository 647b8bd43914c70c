// libmgk C-ABI: context, dataset upload/validation, label lowering, device
// preprocessing (octiles, degrees, PBR) and solver dispatch.  See include/mgk.h.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <set>
#include <thread>
#include <limits>
#include <string>
#include <vector>

#include "../../include/mgk.h"
#include "mgk_internal.h"
#include "pbr.h"

using namespace mgk;

namespace {

thread_local std::string g_err;
// cumulative host<->device payload bytes (benchmark accounting)
std::atomic<int64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

cudaError_t d2h(void* dst, const void* src, size_t bytes) {
  g_d2h_bytes += (int64_t)bytes;
  return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
}

// Large device -> host result copies (the N x N Gram outputs: ~0.7 GB for config 2) into pageable caller
// memory: a plain cudaMemcpy stages through the driver's small bounce buffer and first-touches every
// destination page on one thread.  Here chunks go to two pinned buffers (per host thread) with
// cudaMemcpyAsync while host threads move the previous chunk into the destination (page faults in
// parallel); widen = true converts int32 elements to int64 on the way (the Gram iteration counts, whose
// int64 form the result type needs, cross PCIe at half the size).  The source must be complete
// (callers synchronise their solve first).
constexpr size_t kStageBytes = size_t(32) << 20;
constexpr size_t kStageMin = size_t(64) << 20;

struct Stage {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  int device = -1;
};
thread_local Stage g_stage;

static void host_move(char* dst, const char* src, size_t bytes, bool widen, int threads) {
  const size_t unit = widen ? 4 : 1;
  const size_t n = bytes / unit;
  auto part = [&](int t) {
    const size_t a = n * t / threads, b = n * (t + 1) / threads;
    if (widen) {
      const int32_t* s = reinterpret_cast<const int32_t*>(src);
      int64_t* d = reinterpret_cast<int64_t*>(dst);
      for (size_t i = a; i < b; ++i) d[i] = s[i];
    } else {
      std::memcpy(dst + a, src + a, b - a);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(part, t);
  part(0);
  for (auto& th : pool) th.join();
}

cudaError_t d2h_staged(void* dst, const void* src, size_t bytes, bool widen = false) {
  if (bytes < kStageMin) {  // small results (config 1: a 16 x 16 Gram): one plain copy, no staging threads
    if (!widen) return d2h(dst, src, bytes);
    std::vector<int32_t> tmp(bytes / 4);
    cudaError_t r = d2h(tmp.data(), src, bytes);
    if (r != cudaSuccess) return r;
    int64_t* d = static_cast<int64_t*>(dst);
    for (size_t i = 0; i < tmp.size(); ++i) d[i] = tmp[i];
    return cudaSuccess;
  }
  g_d2h_bytes += (int64_t)bytes;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Stage& S = g_stage;
  if (S.device != dev) {
    for (int b = 0; b < 2; ++b) {
      if (!S.buf[b]) {
        e = cudaHostAlloc(&S.buf[b], kStageBytes, cudaHostAllocPortable);
        if (e != cudaSuccess) return e;
      }
      if (S.ev[b]) cudaEventDestroy(S.ev[b]);
      e = cudaEventCreateWithFlags(&S.ev[b], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    if (S.st) cudaStreamDestroy(S.st);
    e = cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    S.device = dev;
  }
  static const int max_threads = getenv("MGK_D2H_THREADS") ? std::max(1, atoi(getenv("MGK_D2H_THREADS"))) : 8;
  const int threads = (int)std::max(1u, std::min((unsigned)max_threads, std::thread::hardware_concurrency()));
  const size_t nchunks = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t k) {
    const size_t off = k * kStageBytes, len = std::min(kStageBytes, bytes - off);
    cudaError_t r = cudaMemcpyAsync(S.buf[k & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                    S.st);
    if (r == cudaSuccess) r = cudaEventRecord(S.ev[k & 1], S.st);
    return r;
  };
  if ((e = issue(0)) != cudaSuccess) return e;
  for (size_t k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks && (e = issue(k + 1)) != cudaSuccess) return e;
    if ((e = cudaEventSynchronize(S.ev[k & 1])) != cudaSuccess) return e;
    const size_t off = k * kStageBytes, len = std::min(kStageBytes, bytes - off);
    host_move(static_cast<char*>(dst) + (widen ? 2 * off : off), static_cast<const char*>(S.buf[k & 1]), len, widen,
              threads);
  }
  return cudaSuccess;
}

int fail(int code, const char* fmt, ...) {
  char buf[4096];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) return fail(MGK_E_CUDA, "CUDA error %s at %s:%d: %s", #x, __FILE__, \
                                       __LINE__, cudaGetErrorString(e_));                    \
  } while (0)

template <typename T>
struct DBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    if (count <= n && ptr) return cudaSuccess;
    release();
    n = count;
    return cudaMalloc(&ptr, std::max<size_t>(count, 1) * sizeof(T));
  }
  cudaError_t upload(const std::vector<T>& v, cudaStream_t s) {
    cudaError_t e = alloc(v.size());
    if (e != cudaSuccess || v.empty()) return e;
    g_h2d_bytes += (int64_t)(v.size() * sizeof(T));
    return cudaMemcpyAsync(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
  }
};

struct Spec {
  int kind = KK_NONE;  // KK_NONE == None
  double h = 1.0, alpha = 1.0;
  std::vector<double> coef;
  std::vector<Spec> sub;  // PROD components / RCONV inner kernel
};

int parse_spec(const char* s, Spec& out);

// Composite grammar (extension of basekernels.py:247-261 for the class-only kernels):
//   prod:K1|K2|...   ProductComposite(K1, K2, ...)   (basekernels.py:175-211)
//   rconv:K          RConvolution(K)                 (basekernels.py:214-244)
// with scalar sub-kernels K in const1 | delta:H | se:A | poly:c0,..
static int parse_composite(const std::string& head, const std::string& rest, Spec& out) {
  std::vector<std::string> parts;
  if (head == "prod") {
    size_t pos = 0;
    for (;;) {
      size_t bar = rest.find('|', pos);
      parts.push_back(rest.substr(pos, bar == std::string::npos ? std::string::npos : bar - pos));
      if (bar == std::string::npos) break;
      pos = bar + 1;
    }
    out.kind = KK_PROD;
  } else {
    parts.push_back(rest);
    out.kind = KK_RCONV;
  }
  if ((int)parts.size() > kMaxSub)
    return fail(MGK_E_UNSUPPORTED, "at most %d composite components on device", kMaxSub);
  int polys = 0;
  for (const std::string& p : parts) {
    Spec sub;
    int rc = parse_spec(p.c_str(), sub);
    if (rc) return rc;
    if (sub.kind == KK_NONE || sub.kind == KK_PROD || sub.kind == KK_RCONV)
      return fail(MGK_E_UNSUPPORTED, "composite components must be scalar kernels, got '%s'", p.c_str());
    if (sub.kind == KK_POLY && ++polys > 1)
      return fail(MGK_E_UNSUPPORTED, "at most one polynomial component on device");
    out.sub.push_back(sub);
  }
  return MGK_OK;
}

int parse_spec(const char* s, Spec& out) {
  out = Spec();
  if (!s || !*s) return MGK_OK;
  std::string str(s);
  auto colon = str.find(':');
  std::string head = str.substr(0, colon);
  std::string rest = colon == std::string::npos ? "" : str.substr(colon + 1);
  if (head == "prod" || head == "rconv") return parse_composite(head, rest, out);
  try {
    if (head == "const1") {
      out.kind = KK_CONST1;
    } else if (head == "delta") {
      out.kind = KK_DELTA;
      out.h = std::stod(rest);
      if (!(out.h > 0 && out.h <= 1)) return fail(MGK_E_INVALID, "delta baseline h must be in (0, 1], got %g", out.h);
    } else if (head == "se") {
      out.kind = KK_SE;
      out.alpha = std::stod(rest);
      if (!(out.alpha > 0)) return fail(MGK_E_INVALID, "alpha must be positive");
    } else if (head == "poly") {
      out.kind = KK_POLY;
      size_t pos = 0;
      while (pos <= rest.size()) {
        size_t c = rest.find(',', pos);
        out.coef.push_back(std::stod(rest.substr(pos, c == std::string::npos ? std::string::npos : c - pos)));
        if (c == std::string::npos) break;
        pos = c + 1;
      }
      if (out.coef.empty()) return fail(MGK_E_INVALID, "need at least one coefficient");
      if ((int)out.coef.size() > kMaxPoly)
        return fail(MGK_E_UNSUPPORTED, "at most %d polynomial coefficients on device", kMaxPoly);
    } else {
      return fail(MGK_E_INVALID, "unknown kernel spec '%s'", s);
    }
  } catch (...) {
    return fail(MGK_E_INVALID, "unknown kernel spec '%s'", s);
  }
  return MGK_OK;
}

KernelDesc to_desc(const Spec& s) {
  KernelDesc d{};
  d.kind = s.kind;
  d.h = (float)s.h;
  d.alpha = (float)s.alpha;
  d.se_scale = (float)std::sqrt(s.alpha * 1.4426950408889634);
  d.ncoef = (int)s.coef.size();
  for (int i = 0; i < d.ncoef; ++i) d.coef[i] = (float)s.coef[i];
  d.nsub = (int)s.sub.size();
  for (int c = 0; c < d.nsub; ++c) {
    d.sub_kind[c] = s.sub[c].kind;
    d.sub_h[c] = (float)s.sub[c].h;
    if (s.sub[c].kind == KK_POLY) {
      d.ncoef = (int)s.sub[c].coef.size();
      for (int i = 0; i < d.ncoef; ++i) d.coef[i] = (float)s.sub[c].coef[i];
    }
  }
  return d;
}

// Labels lowered for the device according to the kernel that reads them.
struct Lowered {
  int kind = LK_NONE;
  int dim = 0;
  std::vector<float> data;
};

// Composite kernels: every component lowered for its scalar sub-kernel.
static int lower_composite(int kind, int dim, const std::vector<int64_t>& cat, const std::vector<double>& vec,
                           size_t count, const Spec& k, Lowered& out) {
  if (kind == LK_CAT) dim = 1;
  auto raw = [&](size_t i, int c) { return kind == LK_CAT ? (double)cat[i] : vec[i * dim + c]; };
  if (k.kind == KK_PROD && dim != (int)k.sub.size())
    return fail(MGK_E_SHAPE, "composite kernel component count mismatch: %d components, labels of dimension %d",
                (int)k.sub.size(), dim);
  if (dim > kMaxLabelDim) return fail(MGK_E_UNSUPPORTED, "label dimension %d > %d", dim, kMaxLabelDim);
  out.kind = LK_VEC;
  out.dim = dim;
  out.data.assign(count * dim, 0.0f);
  // RCONV compares every component with every component: one class map / scale for all of them
  for (int c = 0; c < dim; ++c) {
    const Spec& sub = k.kind == KK_PROD ? k.sub[c] : k.sub[0];
    if (sub.kind == KK_DELTA) {
      if (k.kind == KK_RCONV && c > 0) continue;  // filled below with the shared map
      std::map<double, int32_t> ids;
      const int c0 = c, c1 = k.kind == KK_RCONV ? dim : c + 1;
      for (size_t i = 0; i < count; ++i)
        for (int cc = c0; cc < c1; ++cc) {
          double key = raw(i, cc);
          if (key == 0.0) key = 0.0;
          int32_t v = ids.emplace(key, (int32_t)ids.size()).first->second;
          memcpy(&out.data[i * dim + cc], &v, 4);
        }
    } else {
      const double scale = sub.kind == KK_SE ? std::sqrt(sub.alpha * 1.4426950408889634) : 1.0;
      for (size_t i = 0; i < count; ++i) out.data[i * dim + c] = (float)(raw(i, c) * scale);
    }
  }
  return MGK_OK;
}

int lower_labels(int kind, int dim, const std::vector<int64_t>& cat, const std::vector<double>& vec, size_t count,
                 const Spec& k, Lowered& out, const char* what) {
  out = Lowered();
  if (kind == LK_NONE || k.kind == KK_NONE || k.kind == KK_CONST1) return MGK_OK;
  if (k.kind == KK_PROD || k.kind == KK_RCONV) return lower_composite(kind, dim, cat, vec, count, k, out);
  if (k.kind == KK_DELTA) {
    // equality classes -> dense ids: exact for int64 tokens and float vectors alike
    out.kind = LK_CAT;
    out.dim = 1;
    out.data.resize(count);
    if (kind == LK_CAT) {
      std::map<int64_t, int32_t> ids;
      for (size_t i = 0; i < count; ++i) {
        auto it = ids.emplace(cat[i], (int32_t)ids.size()).first;
        int32_t v = it->second;
        memcpy(&out.data[i], &v, 4);
      }
    } else {
      std::map<std::vector<double>, int32_t> ids;
      for (size_t i = 0; i < count; ++i) {
        std::vector<double> key(vec.begin() + i * dim, vec.begin() + (i + 1) * dim);
        for (double& x : key)
          if (x == 0.0) x = 0.0;  // -0.0 == 0.0 (numpy ==)
        auto it = ids.emplace(key, (int32_t)ids.size()).first;
        int32_t v = it->second;
        memcpy(&out.data[i], &v, 4);
      }
    }
    return MGK_OK;
  }
  if (kind == LK_CAT) dim = 1;
  if (k.kind == KK_POLY && dim != 1)
    return fail(MGK_E_SHAPE, "polynomial kernel expects scalar labels");
  if (dim > kMaxLabelDim) return fail(MGK_E_UNSUPPORTED, "%s label dimension %d > %d", what, dim, kMaxLabelDim);
  double scale = k.kind == KK_SE ? std::sqrt(k.alpha * 1.4426950408889634) : 1.0;
  out.kind = LK_VEC;
  out.dim = dim;
  out.data.resize(count * dim);
  for (size_t i = 0; i < count * dim; ++i) out.data[i] = (float)((kind == LK_CAT ? (double)cat[i] : vec[i]) * scale);
  return MGK_OK;
}

}  // namespace

struct mgk_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side[2] = {nullptr, nullptr};   // warp-class jobs run beside the CTA/grid jobs
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evside[2] = {nullptr, nullptr};
  double last_ms = 0.0;
  int last_launches = 0;
  // host copy of the dataset
  int32_t G = 0;
  std::vector<int64_t> node_off, edge_off;
  std::vector<int32_t> ei, ej;
  std::vector<double> w, p, q;
  int nl_kind = 0, nl_dim = 0, el_kind = 0, el_dim = 0;
  std::vector<int64_t> nl_cat, el_cat;
  std::vector<double> nl_vec, el_vec;
  bool uploaded = false;
  // kernels
  Spec vspec, espec;
  bool prepared = false;
  // device dataset
  std::vector<GraphDesc> graphs;  // host mirror after preprocessing
  int64_t total_tiles = 0;
  DBuf<GraphDesc> d_graphs;
  DBuf<float> d_p, d_q, d_vlabel, d_ew, d_elabel, d_nzw, d_nzlabel;
  DBuf<double> d_q64, d_deg;
  DBuf<float> d_dm;
  DBuf<int32_t> d_status;
  double v_min = 1e-12;  // SolverConfig.v_min (solver.py:39-52), mgk_set_vertex_floor
  float max_dqr = 1.0f;  // largest GraphDesc::dqr of the dataset (precise-mode switch, kPreciseLap)
  std::vector<int32_t> h_hist;  // k_tile_hist per graph (cost counters), filled on first use after prepare
  DBuf<int32_t> d_ei, d_ej, d_egraph, d_ngraph, d_trow, d_segcount, d_segcursor, d_segntiles, d_seggraph, d_segrow;
  DBuf<int64_t> d_gseg, d_segstart, d_segtile;
  DBuf<uint64_t> d_keys, d_keys2;
  DBuf<Octile> d_tiles;
  DBuf<int32_t> d_rowptr, d_panel;
  DBuf<float4> d_rowent;
  DBuf<int2> d_symk;
  DatasetDev ds{};
  KernelDesc vk{}, ek{};
  // solver buffers
  DBuf<unsigned long long> d_queue;
  DBuf<int32_t> d_list_a, d_list_b, d_list_c;
  DBuf<double> d_K, d_value;
  DBuf<int32_t> d_Kit, d_iters;
  DBuf<uint8_t> d_Kconv, d_conv;
  DBuf<float> d_resid, d_scratch, d_nodewise, d_gridvec;
  DBuf<double2> d_gridbuf;
  DBuf<int64_t> d_nwoff;
  DBuf<int32_t> d_pa, d_pb, d_rowcol;
  DBuf<int64_t> d_rowpre;
  // host images of the Gram job lists (host-side pair decoding for streaming)
  std::vector<int32_t> h_lists, h_rowcol;
  std::vector<int64_t> h_rowpre;
  // pinned staging for streamed nodewise chunks (two slots: fields + per-pair records)
  void* h_nw = nullptr;
  size_t h_nw_cap = 0;
};

extern "C" {

const char* mgk_version(void) { return "mgk-b200 0.1.0 (sm_100a)"; }

const char* mgk_last_error(void) { return g_err.c_str(); }

// error hook for the other translation units of the C-ABI (ingest.cu)
int mgk_fail_ingest(int code, const char* msg) { return fail(code, "%s", msg); }

int mgk_ctx_create(mgk_ctx** out, int device) {
  if (!out) return fail(MGK_E_INVALID, "null output pointer");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(MGK_E_CUDA, "no CUDA device available (%s); libmgk has no CPU fallback",
                e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  if (device < 0 || device >= count) return fail(MGK_E_INVALID, "device %d out of range (%d devices)", device, count);
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new mgk_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreate(&c->ev0));
  CUDA_TRY(cudaEventCreate(&c->ev1));
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->side[k], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->evside[k], cudaEventDisableTiming));
  }
  *out = c;
  return MGK_OK;
}

int mgk_ctx_destroy(mgk_ctx* ctx) {
  if (!ctx) return MGK_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  for (int k = 0; k < 2; ++k) {
    if (ctx->side[k]) cudaStreamSynchronize(ctx->side[k]);
    if (ctx->side[k]) cudaStreamDestroy(ctx->side[k]);
    if (ctx->evside[k]) cudaEventDestroy(ctx->evside[k]);
  }
  if (ctx->h_nw) cudaFreeHost(ctx->h_nw);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return MGK_OK;
}

// validate_graph (graphs.py:161-199) for graph g; returns the joined violations
static std::string validate_one(const mgk_ctx* c, int g) {
  std::vector<std::string> v;
  int64_t n0 = c->node_off[g], n = c->node_off[g + 1] - n0;
  int64_t e0 = c->edge_off[g], ne = c->edge_off[g + 1] - e0;
  char buf[256];
  if (n <= 0) v.push_back("node count must be positive");
  for (int64_t k = 0; k < n; ++k)
    if (c->p[n0 + k] < 0) {
      snprintf(buf, sizeof buf, "starting probability must be >= 0 at node %lld", (long long)k);
      v.push_back(buf);
    }
  for (int64_t k = 0; k < n; ++k) {
    double qq = c->q[n0 + k];
    if (!(qq > 0 && qq <= 1)) {
      snprintf(buf, sizeof buf, "stopping probability must be %s at node %lld", qq <= 0 ? "> 0" : "<= 1",
               (long long)k);
      v.push_back(buf);
    }
  }
  for (int64_t k = 0; k < ne; ++k) {
    int a = c->ei[e0 + k], b = c->ej[e0 + k];
    if (a < 0 || a >= n || b < 0 || b >= n) {
      snprintf(buf, sizeof buf, "edge (%d,%d) references unknown node", a, b);
      v.push_back(buf);
    }
  }
  for (int64_t k = 0; k < ne; ++k)
    if (c->ei[e0 + k] == c->ej[e0 + k]) {
      snprintf(buf, sizeof buf, "self-loop at node %d", c->ei[e0 + k]);
      v.push_back(buf);
    }
  for (int64_t k = 0; k < ne; ++k)
    if (!(c->w[e0 + k] > 0)) {
      snprintf(buf, sizeof buf, "edge weight must be > 0 at edge %lld", (long long)k);
      v.push_back(buf);
    }
  std::set<std::pair<int, int>> seen;
  for (int64_t k = 0; k < ne; ++k) {
    auto key = std::make_pair(c->ei[e0 + k], c->ej[e0 + k]);
    if (!seen.insert(key).second) {
      snprintf(buf, sizeof buf, "duplicate edge (%d,%d)", key.first, key.second);
      v.push_back(buf);
    }
  }
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "; " : "") + v[i];
  return s;
}

int mgk_upload(mgk_ctx* c, int32_t N, const int64_t* node_off, const int64_t* edge_off, const int32_t* ei,
               const int32_t* ej, const double* w, const double* p, const double* q, int nl_kind, int nl_dim,
               const void* node_labels, int el_kind, int el_dim, const void* edge_labels) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (N <= 0) return fail(MGK_E_INVALID, "dataset must hold at least one graph");
  if (!node_off || !edge_off || !p || !q) return fail(MGK_E_INVALID, "null dataset array");
  if (nl_kind < 0 || nl_kind > 2 || el_kind < 0 || el_kind > 2) return fail(MGK_E_INVALID, "bad label kind");
  if (nl_kind == LK_CAT) nl_dim = 1;
  if (el_kind == LK_CAT) el_dim = 1;
  if (nl_kind == LK_NONE) nl_dim = 0;
  if (el_kind == LK_NONE) el_dim = 0;
  if ((nl_kind && (!node_labels || nl_dim < 1)) || (el_kind && (!edge_labels || el_dim < 1)))
    return fail(MGK_E_INVALID, "labels declared but missing");
  c->G = N;
  c->node_off.assign(node_off, node_off + N + 1);
  c->edge_off.assign(edge_off, edge_off + N + 1);
  int64_t nn = c->node_off[N], ne = c->edge_off[N];
  if (c->node_off[0] != 0 || c->edge_off[0] != 0) return fail(MGK_E_INVALID, "offsets must start at 0");
  for (int g = 0; g < N; ++g)
    if (c->node_off[g + 1] < c->node_off[g] || c->edge_off[g + 1] < c->edge_off[g])
      return fail(MGK_E_INVALID, "offsets must be non-decreasing");
  if (ne > 0 && (!ei || !ej || !w)) return fail(MGK_E_INVALID, "null edge arrays");
  c->ei.assign(ei, ei + ne);
  c->ej.assign(ej, ej + ne);
  c->w.assign(w, w + ne);
  c->p.assign(p, p + nn);
  c->q.assign(q, q + nn);
  c->nl_kind = nl_kind;
  c->nl_dim = nl_dim;
  c->el_kind = el_kind;
  c->el_dim = el_dim;
  c->nl_cat.clear();
  c->nl_vec.clear();
  c->el_cat.clear();
  c->el_vec.clear();
  if (nl_kind == LK_CAT) c->nl_cat.assign((const int64_t*)node_labels, (const int64_t*)node_labels + nn);
  if (nl_kind == LK_VEC) c->nl_vec.assign((const double*)node_labels, (const double*)node_labels + nn * nl_dim);
  if (el_kind == LK_CAT) c->el_cat.assign((const int64_t*)edge_labels, (const int64_t*)edge_labels + ne);
  if (el_kind == LK_VEC) c->el_vec.assign((const double*)edge_labels, (const double*)edge_labels + ne * el_dim);
  for (int g = 0; g < N; ++g) {
    if (c->node_off[g + 1] - c->node_off[g] > 65535 * 8)
      return fail(MGK_E_UNSUPPORTED, "graph %d has more than %d nodes", g, 65535 * 8);
    std::string v = validate_one(c, g);
    if (!v.empty()) {
      c->uploaded = false;
      return fail(MGK_E_INVALID, "graph %d invalid: %s", g, v.c_str());
    }
  }
  c->uploaded = true;
  c->prepared = false;
  return MGK_OK;
}

int mgk_set_vertex_floor(mgk_ctx* c, double v_min) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (std::isnan(v_min)) return fail(MGK_E_INVALID, "v_min must be a number");
  c->v_min = v_min;
  return MGK_OK;
}

int mgk_set_kernels(mgk_ctx* c, const char* vertex_spec, const char* edge_spec) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  Spec vs, es;
  int rc = parse_spec(vertex_spec, vs);
  if (rc) return rc;
  rc = parse_spec(edge_spec, es);
  if (rc) return rc;
  c->vspec = vs;
  c->espec = es;
  c->prepared = false;
  return MGK_OK;
}

// Octiles + degrees for the current (possibly relabelled) dataset.
static int build_octiles(mgk_ctx* c) {
  cudaStream_t s = c->stream;
  const int G = c->G;
  int64_t ne = c->edge_off[G], nn = c->node_off[G];
  std::vector<int64_t> gseg(G + 1, 0);
  std::vector<int32_t> seg_graph, seg_row;
  for (int g = 0; g < G; ++g) {
    int n = (int)(c->node_off[g + 1] - c->node_off[g]);
    int rows = ceil8(n);
    gseg[g + 1] = gseg[g] + rows;
    for (int r = 0; r < rows; ++r) {
      seg_graph.push_back(g);
      seg_row.push_back(r);
    }
  }
  int64_t nseg = gseg[G];
  CUDA_TRY(c->d_gseg.upload(gseg, s));
  CUDA_TRY(c->d_seggraph.upload(seg_graph, s));
  CUDA_TRY(c->d_segrow.upload(seg_row, s));
  CUDA_TRY(c->d_ei.upload(c->ei, s));
  CUDA_TRY(c->d_ej.upload(c->ej, s));
  CUDA_TRY(c->d_segcount.alloc(nseg));
  CUDA_TRY(c->d_segcursor.alloc(nseg));
  CUDA_TRY(c->d_segntiles.alloc(nseg));
  CUDA_TRY(c->d_segstart.alloc(nseg + 1));
  CUDA_TRY(c->d_segtile.alloc(nseg + 1));
  CUDA_TRY(cudaMemsetAsync(c->d_segcount.ptr, 0, nseg * sizeof(int32_t), s));
  CUDA_TRY(cudaMemsetAsync(c->d_segcursor.ptr, 0, nseg * sizeof(int32_t), s));
  const int64_t nnz = 2 * ne;
  CUDA_TRY(c->d_keys.alloc(nnz));
  CUDA_TRY(c->d_keys2.alloc(2 * nnz));
  CUDA_TRY(c->d_nzw.alloc(nnz));
  CUDA_TRY(c->d_nzlabel.alloc(nnz * std::max(c->ds.el_dim, 1)));
  if (nnz > 0) {
    int tpb = 256;
    unsigned grid = (unsigned)((nnz + tpb - 1) / tpb);
    k_seg_count<<<grid, tpb, 0, s>>>(ne, c->d_ei.ptr, c->d_ej.ptr, c->d_egraph.ptr, c->d_gseg.ptr, c->d_segcount.ptr);
  }
  k_scan_exclusive<<<1, 1024, 0, s>>>(nseg, c->d_segcount.ptr, c->d_segstart.ptr);
  if (nnz > 0) {
    int tpb = 256;
    unsigned grid = (unsigned)((nnz + tpb - 1) / tpb);
    k_seg_scatter<<<grid, tpb, 0, s>>>(ne, c->d_ei.ptr, c->d_ej.ptr, c->d_egraph.ptr, c->d_gseg.ptr,
                                       c->d_segstart.ptr, c->d_segcursor.ptr, c->d_keys.ptr);
    CUDA_TRY(cudaFuncSetAttribute(k_seg_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmemBytes));
    unsigned sg = (unsigned)std::min<int64_t>(nseg, (int64_t)c->num_sms * 3);
    k_seg_sort<<<sg, 256, kSortSmemBytes, s>>>(nseg, c->d_segstart.ptr, c->d_segcount.ptr, c->d_keys.ptr,
                                               c->d_keys2.ptr);
  }
  {
    unsigned wg = (unsigned)std::min<int64_t>((nseg + 7) / 8, 65535);
    k_seg_ntiles<<<std::max(wg, 1u), 256, 0, s>>>(nseg, c->d_segstart.ptr, c->d_segcount.ptr, c->d_keys.ptr,
                                                  c->d_segntiles.ptr);
  }
  k_scan_exclusive<<<1, 1024, 0, s>>>(nseg, c->d_segntiles.ptr, c->d_segtile.ptr);
  int64_t total_tiles = 0;
  CUDA_TRY(cudaMemcpyAsync(&total_tiles, c->d_segtile.ptr + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  c->total_tiles = total_tiles;
  CUDA_TRY(c->d_tiles.alloc(total_tiles));
  CUDA_TRY(cudaMemsetAsync(c->d_tiles.ptr, 0, std::max<int64_t>(total_tiles, 1) * sizeof(Octile), s));
  if (nnz > 0) {
    unsigned wg = (unsigned)std::min<int64_t>((nseg + 7) / 8, 65535);
    k_seg_emit<<<std::max(wg, 1u), 256, 0, s>>>(nseg, c->d_segstart.ptr, c->d_segcount.ptr, c->d_segtile.ptr,
                                               c->d_seggraph.ptr, c->d_segrow.ptr, c->d_keys.ptr, c->d_graphs.ptr,
                                               c->d_ew.ptr, c->d_elabel.ptr, c->ds.el_dim, c->d_tiles.ptr,
                                               c->d_nzw.ptr, c->d_nzlabel.ptr);
  }
  k_trow<<<(G + 127) / 128, 128, 0, s>>>(G, c->d_gseg.ptr, c->d_segtile.ptr, c->d_graphs.ptr, c->d_trow.ptr);
  CUDA_TRY(c->d_deg.alloc(nn));
  CUDA_TRY(c->d_dm.alloc(nn));
  k_degrees<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(nn, c->d_ngraph.ptr, c->d_graphs.ptr, c->d_tiles.ptr,
                                                         c->d_trow.ptr, c->d_nzw.ptr, c->d_q64.ptr, c->d_deg.ptr,
                                                         c->d_dm.ptr);
  CUDA_TRY(cudaGetLastError());
  c->graphs.resize(G);
  CUDA_TRY(cudaMemcpyAsync(c->graphs.data(), c->d_graphs.ptr, G * sizeof(GraphDesc), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  c->ds.tiles = c->d_tiles.ptr;
  c->ds.trow = c->d_trow.ptr;
  c->ds.nz_w = c->d_nzw.ptr;
  c->ds.nz_label = c->d_nzlabel.ptr;
  c->ds.deg = c->d_deg.ptr;
  c->ds.dm = c->d_dm.ptr;
  c->ds.q64 = c->d_q64.ptr;
  return MGK_OK;
}

// Lower labels for the current kernels, upload node/edge arrays, build octiles.
static int prepare(mgk_ctx* c) {
  if (!c->uploaded) return fail(MGK_E_STATE, "no dataset uploaded");
  if (c->prepared) return MGK_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const int G = c->G;
  int64_t nn = c->node_off[G], ne = c->edge_off[G];
  Lowered vl, el;
  int rc = lower_labels(c->nl_kind, c->nl_dim, c->nl_cat, c->nl_vec, nn, c->vspec, vl, "node");
  if (rc) return rc;
  rc = lower_labels(c->el_kind, c->el_dim, c->el_cat, c->el_vec, ne, c->espec, el, "edge");
  if (rc) return rc;
  std::vector<float> p32(nn), q32(nn), w32(ne);
  std::vector<int32_t> egraph(ne), ngraph(nn);
  for (int64_t i = 0; i < nn; ++i) {
    p32[i] = (float)c->p[i];
    q32[i] = (float)c->q[i];
  }
  for (int64_t i = 0; i < ne; ++i) w32[i] = (float)c->w[i];
  std::vector<GraphDesc> gd(G);
  std::vector<int32_t> rowptr(nn + G), panels;
  c->max_dqr = 1.0f;
  int64_t trow_off = 0;
  for (int g = 0; g < G; ++g) {
    GraphDesc d{};
    d.n = (int32_t)(c->node_off[g + 1] - c->node_off[g]);
    d.ne = (int32_t)(c->edge_off[g + 1] - c->edge_off[g]);
    d.node_off = c->node_off[g];
    d.edge_off = c->edge_off[g];
    d.nz_off = 2 * c->edge_off[g];
    d.trow_off = trow_off;
    trow_off += ceil8(d.n) + 1;
    // row pointers of the row-ordered octile expansion + row panels of <= kPanelCap nonzeros
    d.rowptr_off = c->node_off[g] + g;
    int32_t* rp = rowptr.data() + d.rowptr_off;
    std::fill(rp, rp + d.n + 1, 0);
    for (int64_t e = c->edge_off[g]; e < c->edge_off[g + 1]; ++e) {
      ++rp[c->ei[e] + 1];
      ++rp[c->ej[e] + 1];
    }
    d.maxdeg = 0;
    for (int i = 0; i < d.n; ++i) {
      d.maxdeg = std::max(d.maxdeg, rp[i + 1]);
      rp[i + 1] += rp[i];
    }
    d.panel_off = (int64_t)panels.size();
    if (d.maxdeg <= kPanelCap) {
      panels.push_back(0);
      for (int i = 0; i < d.n; ++i)
        if (rp[i + 1] - rp[panels.back()] > kPanelCap) panels.push_back(i);
      panels.push_back(d.n);
      d.npanels = (int32_t)(panels.size() - d.panel_off - 1);
    } else {
      d.npanels = 0;
    }
    {  // max d_i / q_i (host FP64; only steers the Laplacian-splitting switch)
      std::vector<double> dd(d.n, 0.0);
      for (int64_t e = c->edge_off[g]; e < c->edge_off[g + 1]; ++e) {
        dd[c->ei[e]] += c->w[e];
        dd[c->ej[e]] += c->w[e];
      }
      double r = 1.0;
      for (int i = 0; i < d.n; ++i) r = std::max(r, (dd[i] + c->q[c->node_off[g] + i]) / c->q[c->node_off[g] + i]);
      d.dqr = (float)std::min(r, 3.0e38);
    }
    gd[g] = d;
    c->max_dqr = std::max(c->max_dqr, d.dqr);
    for (int64_t i = c->node_off[g]; i < c->node_off[g + 1]; ++i) ngraph[i] = g;
    for (int64_t i = c->edge_off[g]; i < c->edge_off[g + 1]; ++i) egraph[i] = g;
  }
  CUDA_TRY(c->d_p.upload(p32, s));
  CUDA_TRY(c->d_q.upload(q32, s));
  CUDA_TRY(c->d_q64.upload(c->q, s));
  CUDA_TRY(c->d_ew.upload(w32, s));
  CUDA_TRY(c->d_vlabel.upload(vl.data, s));
  CUDA_TRY(c->d_elabel.upload(el.data, s));
  CUDA_TRY(c->d_egraph.upload(egraph, s));
  CUDA_TRY(c->d_ngraph.upload(ngraph, s));
  CUDA_TRY(c->d_graphs.upload(gd, s));
  CUDA_TRY(c->d_trow.alloc(trow_off));
  CUDA_TRY(c->d_rowptr.upload(rowptr, s));
  CUDA_TRY(c->d_panel.upload(panels, s));
  DatasetDev& ds = c->ds;
  ds = DatasetDev{};
  ds.G = G;
  ds.nl_kind = vl.kind;
  ds.nl_dim = vl.dim;
  ds.el_kind = el.kind;
  ds.el_dim = el.dim;
  ds.graphs = c->d_graphs.ptr;
  ds.p = c->d_p.ptr;
  ds.q = c->d_q.ptr;
  ds.vlabel = c->d_vlabel.ptr;
  c->vk = to_desc(c->vspec);
  c->ek = to_desc(c->espec);
  rc = build_octiles(c);
  if (rc) return rc;
  // row-ordered expansion of the octiles (panel solver input)
  CUDA_TRY(c->d_rowent.alloc(2 * ne));
  if (ne > 0)
    k_rows_fill<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(nn, c->d_ngraph.ptr, c->d_graphs.ptr, c->d_tiles.ptr,
                                                              c->d_trow.ptr, c->d_nzw.ptr, c->d_nzlabel.ptr,
                                                              c->ds.el_dim, c->d_rowptr.ptr, c->d_rowent.ptr);
  CUDA_TRY(c->d_symk.alloc(ne));
  if (ne > 0)
    k_sym_fill<<<(unsigned)((ne + 255) / 256), 256, 0, s>>>(ne, c->d_ei.ptr, c->d_ej.ptr, c->d_egraph.ptr,
                                                             c->d_graphs.ptr, c->d_rowptr.ptr, c->d_rowent.ptr,
                                                             c->d_symk.ptr);
  CUDA_TRY(cudaGetLastError());
  ds.rowptr = c->d_rowptr.ptr;
  ds.rowent = c->d_rowent.ptr;
  ds.panel_row = c->d_panel.ptr;
  ds.symk = c->d_symk.ptr;
  c->h_hist.clear();
  c->prepared = true;
  return MGK_OK;
}

int mgk_tiles(mgk_ctx* c, int32_t g, int32_t* ntiles, int32_t* nnz, int32_t* rc_out, uint64_t* bitmap_out,
              float* w_out) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  int rc = prepare(c);
  if (rc) return rc;
  if (g < 0 || g >= c->G) return fail(MGK_E_INVALID, "graph index %d out of range", g);
  const GraphDesc& d = c->graphs[g];
  if (ntiles) *ntiles = d.ntiles;
  if (nnz) *nnz = 2 * d.ne;
  if (!rc_out && !bitmap_out && !w_out) return MGK_OK;
  std::vector<Octile> t(d.ntiles);
  if (d.ntiles)
    CUDA_TRY(d2h(t.data(), c->d_tiles.ptr + d.tile_off, d.ntiles * sizeof(Octile)));
  for (int k = 0; k < d.ntiles; ++k) {
    if (rc_out) {
      rc_out[2 * k] = t[k].row;
      rc_out[2 * k + 1] = t[k].col;
    }
    if (bitmap_out) bitmap_out[k] = t[k].bitmap;
  }
  if (w_out && d.ne)
    CUDA_TRY(d2h(w_out, c->d_nzw.ptr + d.nz_off, 2 * d.ne * sizeof(float)));
  return MGK_OK;
}

int mgk_degrees(mgk_ctx* c, int32_t g, double* d_out) {
  if (!c || !d_out) return fail(MGK_E_INVALID, "null argument");
  int rc = prepare(c);
  if (rc) return rc;
  if (g < 0 || g >= c->G) return fail(MGK_E_INVALID, "graph index %d out of range", g);
  const GraphDesc& d = c->graphs[g];
  CUDA_TRY(d2h(d_out, c->d_deg.ptr + d.node_off, d.n * sizeof(double)));
  return MGK_OK;
}

// ---------------------------------------------------------------------------
// Solver dispatch
// ---------------------------------------------------------------------------

// composite edge kernels (vector labels, per-component sub-kernels) run on the generic CTA solver
static bool composite_edges(const mgk_ctx* c) {
  return c->el_kind != LK_NONE && (c->espec.kind == KK_PROD || c->espec.kind == KK_RCONV);
}

static bool small_graph(const mgk_ctx* c, const GraphDesc& d) {
  return d.n <= SmallClass::NU && 2 * d.ne <= SmallClass::SMAX && c->ds.el_dim <= 1 && !composite_edges(c);
}

// n * m at or below which a small pair is solved by the FP64 tiny kernel
// (clamped to 128: then min(n, m) <= 11 and the smaller graph fits the tiny kernel's 4 lane slots)
static int tiny_nm() {
  const char* t = getenv("MGK_TINY_NM");
  return t ? std::max(0, std::min(128, atoi(t))) : 128;
}

static SolveParams make_params(const mgk_ctx* c, double tol, int64_t max_iter) {
  SolveParams p{};
  p.tol2 = tol * tol;
  p.max_iter = max_iter;
  p.v_min = (float)c->v_min;
  p.tiny_nm = tiny_nm();
  p.lap_mode = getenv("MGK_LAPLACIAN") ? std::max(0, std::min(2, atoi(getenv("MGK_LAPLACIAN")))) : 1;
  p.panel_rpc = getenv("MGK_PANEL_RPC") ? atoi(getenv("MGK_PANEL_RPC")) : 0;
  // product.py:153-161 with dataset-uniform label presence; kappa = 1 when ek is None/const1
  p.labeled = (c->el_kind != LK_NONE && c->espec.kind != KK_NONE && c->espec.kind != KK_CONST1) ? 1 : 0;
  p.fp64 = (!p.labeled && (tol < kPreciseTol || c->max_dqr > 2.0f * kPreciseLap)) ? 1 : 0;
  if (const char* e = getenv("MGK_FP64")) p.fp64 = atoi(e) ? 1 : 0;
  p.factor_ratio4 = getenv("MGK_FACTOR_RATIO4") ? std::max(0, atoi(getenv("MGK_FACTOR_RATIO4"))) : 12;
  return p;
}

// Solver status bits -> the reference's errors (vertex_similarity_matrix, product.py:176-177).
static int check_status(mgk_ctx* c) {
  int32_t st = 0;
  CUDA_TRY(cudaMemcpy(&st, c->d_status.ptr, sizeof st, cudaMemcpyDeviceToHost));
  if (st & kStatusNonPositiveKv) return fail(MGK_E_INVALID, "vertex kernel produced non-positive similarity");
  return MGK_OK;
}

enum JobKernel { JK_BLOCK = 0, JK_WARP = 1, JK_TINY = 2, JK_PANEL = 3, JK_GRID = 4 };

struct JobSpec {
  PairJob job;
  int kernel;         // JobKernel
  int slots = SmallClass::SLOTS;  // warp solver lane-slot capacity
  int64_t max_n, max_m, max_su, max_sl;
};


// Panel solver eligibility: scalar edge labels and row panels for every graph
// (a row of more than kPanelCap nonzeros sends the dataset to the block kernel).
static bool panel_dataset(const mgk_ctx* c) {
  if (c->ds.el_dim > 1 || composite_edges(c)) return false;
  if (getenv("MGK_NO_PANEL")) return false;
  for (const GraphDesc& d : c->graphs)
    if (d.npanels <= 0) return false;
  return true;
}

// Largest n*m the panel solver keeps in shared memory (P and Ap: 2 n m floats).
constexpr int64_t kPanelSmemNM = 8192;
// Jobs whose largest pair reaches this n*m run the 512-thread panel CTAs.
constexpr int64_t kPanelWideNM = 32768;
// Graphs with at least large_n() nodes pair with each other on the whole device
// (grid class); explicit pair lists use n*m >= large_n()^2.  MGK_GRID_N
// overrides the threshold (tests drive the grid path at oracle-sized graphs).
static int large_n() {
  const char* t = getenv("MGK_GRID_N");
  return t ? atoi(t) : 1024;
}

// Per-CTA slab (floats) for the block kernel.
static int64_t block_slab(const mgk_ctx* c, int64_t n, int64_t m, int64_t su, int64_t sl, bool fp64) {
  int64_t el = c->ds.el_dim > 2 ? c->ds.el_dim : 0;
  // 6 vectors (P, AP, R, X, DG, SD); + 6 * 128 + 8: a pair with n m <= tiny_nm (<= 128) runs with FP64
  // vectors (2 floats per element), every pair does in a precise solve
  int64_t f = (fp64 ? 12 : 6) * n * m + 6 * 128 + 8 + 8 + 4 * (su + sl) + el * (su + sl) + (n + m + 2) + 16;
  return (f + 31) / 32 * 32;
}

// Enqueue every job of `jobs` (device time bracketed by e0 / e1, default the context's events); with
// sync the call waits for completion and stores the elapsed time in last_ms.
// Kernel attributes (max dynamic shared memory) are process-wide per function while the panel CTAs'
// dynamic size varies per job: contexts driven from several host threads (mgk_gram_multi) must not
// interleave one thread's attribute update with another's launch.
static std::mutex g_launch_mu;

static int run_jobs(mgk_ctx* c, std::vector<JobSpec>& jobs, const SolveOut& out_base,
                    const std::vector<int64_t>& out_offsets, const SolveParams& prm, bool sync = true,
                    cudaEvent_t e0 = nullptr, cudaEvent_t e1 = nullptr) {
  std::unique_lock<std::mutex> launch_lock(g_launch_mu);
  CUDA_TRY(cudaSetDevice(c->device));  // the calling thread may have last used another context's device
  cudaStream_t s = c->stream;
  if (!e0) e0 = c->ev0;
  if (!e1) e1 = c->ev1;
  CUDA_TRY(c->d_queue.alloc(std::max<size_t>(jobs.size(), 1)));
  CUDA_TRY(cudaMemsetAsync(c->d_queue.ptr, 0, std::max<size_t>(jobs.size(), 1) * sizeof(unsigned long long), s));
  // scratch slabs (block and panel jobs run one after another on the stream and share the buffer)
  std::vector<int64_t> slabs(jobs.size(), 0);
  std::vector<int> ctas(jobs.size(), 0), svec(jobs.size(), 0);
  std::vector<char> big(jobs.size(), 0);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const int64_t budget = (int64_t)(free_b * 0.6) / 4 + (int64_t)c->d_scratch.n;
  int64_t need = 0;
  for (size_t k = 0; k < jobs.size(); ++k) {
    JobSpec& j = jobs[k];
    if (j.job.npairs <= 0) continue;
    if (j.kernel == JK_BLOCK) {
      slabs[k] = block_slab(c, j.max_n, j.max_m, j.max_su, j.max_sl, prm.fp64 != 0);
      ctas[k] = 2 * c->num_sms;
    } else if (j.kernel == JK_PANEL) {
      const int64_t nm = j.max_n * j.max_m;
      slabs[k] = kSlabVectors * ((nm + 31) / 32 * 32);
      // P and Ap in shared memory when every pair of the job fits; else all pairs keep them in HBM/L2
      // and the whole L1 stays available to the gathers
      const int64_t smem_nm = getenv("MGK_PANEL_SMEM_NM") ? atoll(getenv("MGK_PANEL_SMEM_NM")) : kPanelSmemNM;
      svec[k] = nm <= smem_nm ? (int)(2 * nm) : 0;
      // large pairs (P streamed through L2): one 512-thread CTA per SM keeps the resident P
      // vectors within L2; mid-size pairs: two 256-thread CTAs per SM
      big[k] = svec[k] == 0 && nm >= kPanelWideNM && !getenv("MGK_PANEL_NO512");
      int per_sm = big[k] ? p512::panel_ctas_per_sm(0) : p256::panel_ctas_per_sm(svec[k]);
      if (const char* e = getenv("MGK_PANEL_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
      ctas[k] = per_sm * c->num_sms;
      if (const char* e = getenv("MGK_PANEL_MAX_CTAS")) ctas[k] = std::max(1, std::min(ctas[k], atoi(e)));
    } else {
      continue;
    }
    int64_t fit = std::max<int64_t>(budget / std::max<int64_t>(slabs[k], 1), 1);
    if (fit < ctas[k]) ctas[k] = (int)fit;
    need = std::max(need, slabs[k] * ctas[k]);
  }
  if (need > 0) CUDA_TRY(c->d_scratch.alloc((size_t)need));
  int64_t grid_vstride = 0;
  const bool grid512 = getenv("MGK_GRID256") == nullptr;
  const int gblocks = grid512 ? p512::grid_blocks(c->num_sms) : p256::grid_blocks(c->num_sms);
  for (auto& j : jobs)
    if (j.kernel == JK_GRID && j.job.npairs > 0) grid_vstride = std::max(grid_vstride, (j.max_n * j.max_m + 31) / 32 * 32);
  if (grid_vstride > 0) {
    CUDA_TRY(c->d_gridvec.alloc((size_t)(kSlabVectors * grid_vstride)));
    CUDA_TRY(c->d_gridbuf.alloc((size_t)(2 * gblocks)));
  }
  c->last_launches = 0;
  CUDA_TRY(c->d_status.alloc(1));
  // asynchronous callers (the nodewise stream) clear the status once and check it at the end
  if (sync) CUDA_TRY(cudaMemsetAsync(c->d_status.ptr, 0, sizeof(int32_t), s));
  CUDA_TRY(cudaEventRecord(e0, s));
  // Streams: grid and CTA-class jobs in order on the main stream (they share the scratch slabs and the
  // cooperative grid must own the device); warp-class jobs on side stream 0, tiny jobs on side stream
  // 1.  Persistent kernels leave the device as their queues drain, so the concurrent jobs fill each
  // other's tails.  MGK_SERIAL=1 runs everything on the main stream.
  // The cooperative grid jobs go first and alone (their blocks must all be resident).
  const bool serial = getenv("MGK_SERIAL") != nullptr;
  std::vector<size_t> order;
  for (size_t k = 0; k < jobs.size(); ++k)
    if (jobs[k].kernel == JK_GRID) order.push_back(k);
  const size_t ngrid = order.size();
  for (size_t k = 0; k < jobs.size(); ++k)
    if (jobs[k].kernel != JK_GRID) order.push_back(k);
  for (size_t oi = 0; oi < order.size(); ++oi) {
    const size_t k = order[oi];
    if (oi == ngrid) {
      CUDA_TRY(cudaEventRecord(c->evside[0], s));
      for (int q = 0; q < 2; ++q) CUDA_TRY(cudaStreamWaitEvent(c->side[q], c->evside[0], 0));
    }
    JobSpec& j = jobs[k];
    if (j.job.npairs <= 0) continue;
    SolveOut o = out_base;
    o.status = c->d_status.ptr;
    int64_t off = out_offsets[k];
    if (o.value) o.value += off;
    if (o.iters) o.iters += off;
    if (o.conv) o.conv += off;
    if (o.residual) o.residual += off;
    if (o.nodewise_off) o.nodewise_off += off;
    if (o.pair_a) o.pair_a += off;
    if (o.pair_b) o.pair_b += off;
    cudaError_t e;
    const int q = serial ? -1 : (j.kernel == JK_WARP ? 0 : (j.kernel == JK_TINY ? 1 : -1));
    cudaStream_t js = q < 0 ? s : c->side[q];
    if (j.kernel == JK_WARP)
      e = launch_pcg_warp(c->ds, c->vk, c->ek, j.job, prm, o, c->d_queue.ptr + k, c->num_sms, j.slots, js);
    else if (j.kernel == JK_TINY)
      e = launch_pcg_tiny(c->ds, c->vk, c->ek, j.job, prm, o, c->d_queue.ptr + k, c->num_sms, js);
    else if (j.kernel == JK_GRID)
      e = (grid512 ? p512::launch_pcg_grid : p256::launch_pcg_grid)(c->ds, c->vk, c->ek, j.job, prm, o, c->d_gridvec.ptr, grid_vstride, c->d_gridbuf.ptr,
                          gblocks, s);
    else if (j.kernel == JK_PANEL)
      e = (big[k] ? p512::launch_pcg_panel : p256::launch_pcg_panel)(
          c->ds, c->vk, c->ek, j.job, prm, o, c->d_queue.ptr + k, c->d_scratch.ptr, slabs[k], ctas[k], svec[k], s);
    else
      e = launch_pcg_block(c->ds, c->vk, c->ek, j.job, prm, o, c->d_queue.ptr + k, c->d_scratch.ptr, slabs[k],
                           ctas[k], s);
    if (e != cudaSuccess) return fail(MGK_E_CUDA, "solver launch failed: %s", cudaGetErrorString(e));
    ++c->last_launches;
  }
  if (ngrid == order.size()) {  // only grid jobs (or none): the side streams still join below
    CUDA_TRY(cudaEventRecord(c->evside[0], s));
    for (int q = 0; q < 2; ++q) CUDA_TRY(cudaStreamWaitEvent(c->side[q], c->evside[0], 0));
  }
  for (int q = 0; q < 2; ++q) {
    CUDA_TRY(cudaEventRecord(c->evside[q], c->side[q]));
    CUDA_TRY(cudaStreamWaitEvent(s, c->evside[q], 0));
  }
  CUDA_TRY(cudaEventRecord(e1, s));
  launch_lock.unlock();  // everything is enqueued
  if (!sync) return MGK_OK;
  CUDA_TRY(cudaEventSynchronize(e1));
  CUDA_TRY(cudaGetLastError());
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  c->last_ms = ms;
  return check_status(c);
}

// Gram jobs (all pairs a <= b, gram.py:57-95), cost-descending within each:
//   small graphs sorted by (n, S) descending; the pairs of row u are split at
//   c(u) = first column whose n_u * n_v <= tiny_nm into a main ragged job
//   [warp kernel, FP32] and a tiny ragged job [tiny kernel, FP64];
//   pairs with a larger graph: TRI(other) + RECT(other x small) [block kernel].
static int gram_jobs(mgk_ctx* c, std::vector<JobSpec>& jobs, const SolveParams& prm) {
  std::vector<int32_t> small, mid, large;
  // a precise solve (prm.fp64) runs every pair on the FP64 block solver: one mid triangle
  const bool precise = prm.fp64 != 0;
  const bool panel = !precise && panel_dataset(c);
  for (int g = 0; g < c->G; ++g) {
    const GraphDesc& d = c->graphs[g];
    if (!precise && small_graph(c, d))
      small.push_back(g);
    else if (panel && d.n >= large_n())
      large.push_back(g);
    else
      mid.push_back(g);
  }
  auto by_size = [c](int32_t a, int32_t b) {
    const GraphDesc &x = c->graphs[a], &y = c->graphs[b];
    if (x.n != y.n) return x.n > y.n;
    if (x.ne != y.ne) return x.ne > y.ne;
    return a < b;
  };
  // small list = [wide graphs (> 32 * kNarrowSlots nonzeros)] ++ [narrow graphs], each size-sorted:
  // wide x wide pairs form the triangle of the prefix (wide warp instantiation); every other small
  // pair has a narrow graph for the lane side (narrow instantiation)
  auto is_wide = [c](int32_t g) { return (2 * c->graphs[g].ne + 31) / 32 > kNarrowSlots; };
  std::stable_partition(small.begin(), small.end(), is_wide);
  const int64_t P = std::count_if(small.begin(), small.end(), is_wide);
  std::stable_sort(small.begin(), small.begin() + P, by_size);
  std::stable_sort(small.begin() + P, small.end(), by_size);
  std::stable_sort(mid.begin(), mid.end(), by_size);
  std::stable_sort(large.begin(), large.end(), by_size);
  const int64_t ns = (int64_t)small.size(), nmid = (int64_t)mid.size(), nl = (int64_t)large.size();
  const int T = tiny_nm();
  // ragged rows over the small list: row u pairs with columns [start(u), split(u)) on the narrow
  // warp kernel and [split(u), ns) on the FP64 tiny kernel; start(u) = P for wide rows (their
  // wide partners are in the prefix triangle), u otherwise.  Wide graphs are never tiny
  // (S > 128 needs n >= 12), so tiny columns are a suffix of the n-sorted narrow part.
  std::vector<int64_t> mpre(ns + 1, 0), tpre(ns + 1, 0);
  std::vector<int32_t> mcol(ns), tcol(ns);
  for (int64_t u = 0; u < ns; ++u) {
    const int64_t nu = c->graphs[small[u]].n;
    const int64_t start = u < P ? P : u;
    int64_t lo = std::max<int64_t>(start, P), hi = ns;  // first narrow column with n_u * n_v <= T
    while (lo < hi) {
      const int64_t mid_ = (lo + hi) / 2;
      if ((int64_t)c->graphs[small[mid_]].n * nu > T) lo = mid_ + 1; else hi = mid_;
    }
    const int64_t split = std::max<int64_t>(start, lo);
    mcol[u] = (int32_t)start;
    mpre[u + 1] = mpre[u] + (split - start);
    tcol[u] = (int32_t)split;
    tpre[u + 1] = tpre[u] + (ns - split);
  }
  // mid x mid pairs split the same way by n_u * n_v <= kPanelSmemNM: the second part keeps P and Ap in
  // shared memory, the first streams them through L1/L2
  std::vector<int64_t> bpre(nmid + 1, 0), spre(nmid + 1, 0);
  std::vector<int32_t> bcol(nmid), scol(nmid);
  for (int64_t u = 0; u < nmid; ++u) {
    const int64_t nu = c->graphs[mid[u]].n;
    int64_t lo = u, hi = nmid;
    while (lo < hi) {
      const int64_t md = (lo + hi) / 2;
      if ((int64_t)c->graphs[mid[md]].n * nu > kPanelSmemNM) lo = md + 1; else hi = md;
    }
    bcol[u] = (int32_t)u;
    bpre[u + 1] = bpre[u] + (lo - u);
    scol[u] = (int32_t)lo;
    spre[u + 1] = spre[u] + (nmid - lo);
  }
  // mid x small pairs: row u of the mid list pairs with small columns [0, x(u)) on the CTA solver
  // and [x(u), ns) -- n_u n_v <= tiny_nm, a dense small graph (n <= NU but too many nonzeros for the
  // warp class) against a tiny partner -- on the block solver's FP64 vectors, the same predicate as
  // mgk_pairs.  Mid graphs have n >= 19, so tiny partners have n <= 6 and lie in the narrow suffix.
  std::vector<int64_t> rpre(nmid + 1, 0), xpre(nmid + 1, 0);
  std::vector<int32_t> rcol(nmid), xcol(nmid);
  for (int64_t u = 0; u < nmid; ++u) {
    const int64_t nu = c->graphs[mid[u]].n;
    int64_t lo = P, hi = ns;
    while (lo < hi) {
      const int64_t md = (lo + hi) / 2;
      if ((int64_t)c->graphs[small[md]].n * nu > T) lo = md + 1; else hi = md;
    }
    rcol[u] = (int32_t)nmid;  // columns index the combined [mid ++ small] list
    rpre[u + 1] = rpre[u] + lo;
    xcol[u] = (int32_t)(nmid + lo);
    xpre[u + 1] = xpre[u] + (ns - lo);
  }
  cudaStream_t s = c->stream;
  std::vector<int32_t> lists;  // large, mid, small (mid ++ small contiguous for the ragged mid x small jobs)
  lists.insert(lists.end(), large.begin(), large.end());
  lists.insert(lists.end(), mid.begin(), mid.end());
  lists.insert(lists.end(), small.begin(), small.end());
  CUDA_TRY(c->d_list_a.upload(lists, s));
  std::vector<int64_t> pre(mpre);
  for (auto* v : {&tpre, &bpre, &spre, &rpre, &xpre}) pre.insert(pre.end(), v->begin(), v->end());
  std::vector<int32_t> col(mcol);
  for (auto* v : {&tcol, &bcol, &scol, &rcol, &xcol}) col.insert(col.end(), v->begin(), v->end());
  CUDA_TRY(c->d_rowpre.upload(pre, s));
  CUDA_TRY(c->d_rowcol.upload(col, s));
  c->h_lists = lists;
  c->h_rowpre = pre;
  c->h_rowcol = col;
  const int32_t* dlarge = c->d_list_a.ptr;
  const int32_t* dmid = dlarge + nl;
  const int32_t* dsmall = dmid + nmid;
  auto mx = [c](const std::vector<int32_t>& vv, bool nodes) {
    int64_t r = 0;
    for (int32_t g : vv) r = std::max<int64_t>(r, nodes ? c->graphs[g].n : 2 * c->graphs[g].ne);
    return r;
  };
  auto tri = [&](const std::vector<int32_t>& l, const int32_t* dl, int kernel) {
    JobSpec j{};
    const int64_t n = (int64_t)l.size();
    j.job = PairJob{PM_TRI, (int32_t)n, 0, n * (n + 1) / 2, 0, 1, dl, nullptr, nullptr, nullptr};
    j.kernel = kernel;
    j.max_n = j.max_m = mx(l, true);
    j.max_su = j.max_sl = mx(l, false);
    return j;
  };
  auto rect = [&](const std::vector<int32_t>& la, const int32_t* da, const std::vector<int32_t>& lb,
                  const int32_t* db, int kernel) {
    JobSpec j{};
    j.job = PairJob{PM_RECT, (int32_t)la.size(), (int32_t)lb.size(), (int64_t)la.size() * (int64_t)lb.size(), 0, 1,
                    da, db, nullptr, nullptr};
    j.kernel = kernel;
    j.max_n = mx(la, true);
    j.max_m = mx(lb, true);
    j.max_su = mx(la, false);
    j.max_sl = mx(lb, false);
    return j;
  };
  const int cta = panel ? JK_PANEL : JK_BLOCK;
  std::vector<int32_t> wide(small.begin(), small.begin() + P);
  JobSpec jw = tri(wide, dsmall, JK_WARP);
  jw.slots = SmallClass::SLOTS;
  JobSpec jm{};
  jm.job = PairJob{PM_RAGGED, (int32_t)ns, 0, mpre[ns], 0, 1, dsmall, nullptr, c->d_rowpre.ptr, c->d_rowcol.ptr};
  jm.kernel = JK_WARP;
  jm.slots = kNarrowSlots;
  JobSpec jt{};
  jt.job = PairJob{PM_RAGGED, (int32_t)ns, 0, tpre[ns], 0, 1, dsmall, nullptr, c->d_rowpre.ptr + ns + 1,
                   c->d_rowcol.ptr + ns};
  jt.kernel = JK_TINY;
  JobSpec jmb = tri(mid, dmid, cta), jms = tri(mid, dmid, cta);
  if (cta == JK_PANEL) {
    const int64_t* bp = c->d_rowpre.ptr + 2 * (ns + 1);
    const int32_t* bc = c->d_rowcol.ptr + 2 * ns;
    jmb.job = PairJob{PM_RAGGED, (int32_t)nmid, 0, bpre[nmid], 0, 1, dmid, nullptr, bp, bc};
    jms.job = PairJob{PM_RAGGED, (int32_t)nmid, 0, spre[nmid], 0, 1, dmid, nullptr, bp + nmid + 1, bc + nmid};
    jms.max_n = std::min<int64_t>(jms.max_n * jms.max_m, kPanelSmemNM);  // every pair has n m <= kPanelSmemNM
    jms.max_m = 1;
  } else {
    jms.job.npairs = 0;
  }
  JobSpec jr = rect(mid, dmid, small, dsmall, cta), jx = rect(mid, dmid, small, dsmall, JK_BLOCK);
  {
    const int64_t* rp = c->d_rowpre.ptr + 2 * (ns + 1) + 2 * (nmid + 1);
    const int32_t* rc = c->d_rowcol.ptr + 2 * ns + 2 * nmid;
    jr.job = PairJob{PM_RAGGED, (int32_t)nmid, 0, rpre[nmid], 0, 1, dmid, nullptr, rp, rc};
    jx.job = PairJob{PM_RAGGED, (int32_t)nmid, 0, xpre[nmid], 0, 1, dmid, nullptr, rp + nmid + 1, rc + nmid};
  }
  // big pairs first (longest job first across classes)
  jobs = {tri(large, dlarge, JK_GRID), rect(large, dlarge, mid, dmid, cta), rect(large, dlarge, small, dsmall, cta),
          jmb, jms, jr, jw, jm, jt, jx};
  return MGK_OK;
}

int mgk_gram(mgk_ctx* c, double tol, int64_t max_iter, double* K, int32_t* iters, uint8_t* conv) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (!(tol > 0)) return fail(MGK_E_INVALID, "tolerance must be positive");
  int rc = prepare(c);
  if (rc) return rc;
  const SolveParams prm = make_params(c, tol, max_iter);
  std::vector<JobSpec> jobs;
  rc = gram_jobs(c, jobs, prm);
  if (rc) return rc;
  int64_t G = c->G;
  CUDA_TRY(c->d_K.alloc(G * G));
  CUDA_TRY(c->d_Kit.alloc(G * G));
  CUDA_TRY(c->d_Kconv.alloc(G * G));
  SolveOut o{};
  o.K = c->d_K.ptr;
  o.K_iters = c->d_Kit.ptr;
  o.K_conv = c->d_Kconv.ptr;
  o.G = G;
  std::vector<int64_t> offs(jobs.size(), 0);
  rc = run_jobs(c, jobs, o, offs, prm);
  if (rc) return rc;
  if (K) CUDA_TRY(d2h_staged(K, c->d_K.ptr, G * G * sizeof(double)));
  if (iters) CUDA_TRY(d2h_staged(iters, c->d_Kit.ptr, G * G * sizeof(int32_t)));
  if (conv) CUDA_TRY(d2h_staged(conv, c->d_Kconv.ptr, G * G));
  return MGK_OK;
}

int mgk_gram_iterations64(mgk_ctx* c, int64_t* iters) {
  if (!c || !iters) return fail(MGK_E_INVALID, "null argument");
  const int64_t G = c->G;
  if (c->d_Kit.n < (size_t)(G * G)) return fail(MGK_E_STATE, "no Gram solved on this context");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // int32 counts cross PCIe and are widened by the host threads that move the staged chunks
  CUDA_TRY(d2h_staged(iters, c->d_Kit.ptr, G * G * sizeof(int32_t), true));
  return MGK_OK;
}

int mgk_gram_normalized(mgk_ctx* c, double tol, int64_t max_iter, double* K, int32_t* iters, uint8_t* conv) {
  int rc = mgk_gram(c, tol, max_iter, nullptr, iters, conv);
  if (rc) return rc;
  const int64_t G = c->G;
  DBuf<double> diag;
  DBuf<int> bad;
  CUDA_TRY(diag.alloc(G));
  CUDA_TRY(bad.alloc(1));
  bool nonpositive = false;
  CUDA_TRY(launch_gram_normalize(c->d_K.ptr, G, diag.ptr, bad.ptr, c->num_sms, c->stream, &nonpositive));
  if (nonpositive) return fail(MGK_E_INVALID, "Gram diagonal must be strictly positive");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (K) CUDA_TRY(d2h_staged(K, c->d_K.ptr, G * G * sizeof(double)));
  return MGK_OK;
}

static int64_t shard_len(int64_t total, int rank, int world) {
  return total > rank ? (total - rank + world - 1) / world : 0;
}

// Shard jobs of the Gram (pair ids congruent to rank mod world of every class job) solved into the
// per-pair device outputs `o` (null: count only).
static int gram_shard_run(mgk_ctx* c, int rank, int world, double tol, int64_t max_iter, int64_t* npairs_out,
                          SolveOut* o) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (world < 1 || rank < 0 || rank >= world) return fail(MGK_E_INVALID, "bad rank/world");
  if (!(tol > 0)) return fail(MGK_E_INVALID, "tolerance must be positive");
  int rc = prepare(c);
  if (rc) return rc;
  const SolveParams prm = make_params(c, tol, max_iter);
  std::vector<JobSpec> jobs;
  rc = gram_jobs(c, jobs, prm);
  if (rc) return rc;
  std::vector<int64_t> offs;
  int64_t total = 0;
  for (auto& j : jobs) {
    int64_t len = shard_len(j.job.npairs, rank, world);
    j.job.offset = rank;
    j.job.stride = world;
    j.job.npairs = len;
    offs.push_back(total);
    total += len;
  }
  if (npairs_out) *npairs_out = total;
  if (!o) return MGK_OK;
  return run_jobs(c, jobs, *o, offs, prm);
}

int mgk_gram_shard(mgk_ctx* c, int rank, int world, double tol, int64_t max_iter, int64_t* npairs_out,
                   int32_t* pair_a, int32_t* pair_b, double* value, int32_t* iters, uint8_t* conv) {
  int64_t total = 0;
  int rc = gram_shard_run(c, rank, world, tol, max_iter, &total, nullptr);
  if (rc) return rc;
  if (npairs_out) *npairs_out = total;
  if (!pair_a && !pair_b && !value && !iters && !conv) return MGK_OK;
  CUDA_TRY(c->d_value.alloc(total));
  CUDA_TRY(c->d_iters.alloc(total));
  CUDA_TRY(c->d_conv.alloc(total));
  CUDA_TRY(c->d_pa.alloc(total));
  CUDA_TRY(c->d_pb.alloc(total));
  SolveOut o{};
  o.value = c->d_value.ptr;
  o.iters = c->d_iters.ptr;
  o.conv = c->d_conv.ptr;
  o.pair_a = c->d_pa.ptr;
  o.pair_b = c->d_pb.ptr;
  rc = gram_shard_run(c, rank, world, tol, max_iter, nullptr, &o);
  if (rc) return rc;
  if (pair_a) CUDA_TRY(d2h(pair_a, c->d_pa.ptr, total * sizeof(int32_t)));
  if (pair_b) CUDA_TRY(d2h(pair_b, c->d_pb.ptr, total * sizeof(int32_t)));
  if (value) CUDA_TRY(d2h(value, c->d_value.ptr, total * sizeof(double)));
  if (iters) CUDA_TRY(d2h(iters, c->d_iters.ptr, total * sizeof(int32_t)));
  if (conv) CUDA_TRY(d2h(conv, c->d_conv.ptr, total));
  return MGK_OK;
}

int mgk_gram_shard_device(mgk_ctx* c, int rank, int world, double tol, int64_t max_iter, int64_t* npairs_out,
                          int32_t* d_pair_a, int32_t* d_pair_b, double* d_value, int32_t* d_iters, uint8_t* d_conv) {
  if (!d_pair_a && !d_pair_b && !d_value && !d_iters && !d_conv)
    return gram_shard_run(c, rank, world, tol, max_iter, npairs_out, nullptr);
  SolveOut o{};
  o.value = d_value;
  o.iters = d_iters;
  o.conv = d_conv;
  o.pair_a = d_pair_a;
  o.pair_b = d_pair_b;
  return gram_shard_run(c, rank, world, tol, max_iter, npairs_out, &o);
}

int mgk_gram_assemble(int device, int64_t npairs, const int32_t* d_pair_a, const int32_t* d_pair_b,
                      const double* d_value, const int32_t* d_iters, const uint8_t* d_conv, int64_t G, double* d_K,
                      int32_t* d_K_iters, uint8_t* d_K_conv) {
  if (npairs < 0 || G < 0) return fail(MGK_E_INVALID, "negative size");
  if (npairs > 0 && (!d_pair_a || !d_pair_b || !d_conv || (d_K && !d_value) || (d_K_iters && !d_iters)))
    return fail(MGK_E_INVALID, "null record array");
  CUDA_TRY(cudaSetDevice(device));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t s;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = launch_gram_assemble(npairs, d_pair_a, d_pair_b, d_value, d_iters, d_conv, G, d_K, d_K_iters,
                                       d_K_conv, sms, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(MGK_E_CUDA, "gram assembly: %s", cudaGetErrorString(e));
  return MGK_OK;
}

int mgk_gram_multi(mgk_ctx* const* ctxs, int nctx, double tol, int64_t max_iter, double* K, int32_t* iters,
                   uint8_t* conv) {
  if (!ctxs || nctx < 1) return fail(MGK_E_INVALID, "need at least one context");
  for (int k = 0; k < nctx; ++k) {
    if (!ctxs[k]) return fail(MGK_E_INVALID, "null context %d", k);
    if (!ctxs[k]->uploaded) return fail(MGK_E_STATE, "context %d has no dataset", k);
    if (ctxs[k]->G != ctxs[0]->G) return fail(MGK_E_INVALID, "contexts hold different datasets");
  }
  const int64_t G = ctxs[0]->G;
  // one host thread per context: solve shard k of nctx, copy the compact records back, scatter them
  // (mirrored, NaN where not converged) into the caller's matrices -- shards are disjoint pair sets,
  // so the threads never write the same entry
  std::vector<int> rcs(nctx, MGK_OK);
  std::vector<std::string> errs(nctx);
  std::vector<double> ms(nctx, 0.0);
  std::vector<int> launches(nctx, 0);
  auto work = [&](int k) {
    mgk_ctx* c = ctxs[k];
    cudaSetDevice(c->device);
    std::vector<int32_t> pa, pb, it;
    std::vector<double> v;
    std::vector<uint8_t> cv;
    int64_t n = 0;
    int rc = mgk_gram_shard(c, k, nctx, tol, max_iter, &n, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (!rc) {
      pa.resize(n);
      pb.resize(n);
      v.resize(n);
      it.resize(n);
      cv.resize(n);
      rc = mgk_gram_shard(c, k, nctx, tol, max_iter, &n, pa.data(), pb.data(), v.data(), it.data(), cv.data());
    }
    rcs[k] = rc;
    if (rc) {
      errs[k] = g_err;
      return;
    }
    ms[k] = c->last_ms;
    launches[k] = c->last_launches;
    for (int64_t q = 0; q < n; ++q) {
      const int64_t a = pa[q], b = pb[q];
      const double kv = cv[q] ? v[q] : std::numeric_limits<double>::quiet_NaN();
      if (K) K[a * G + b] = K[b * G + a] = kv;
      if (iters) iters[a * G + b] = iters[b * G + a] = it[q];
      if (conv) conv[a * G + b] = conv[b * G + a] = cv[q];
    }
  };
  std::vector<std::thread> th;
  for (int k = 1; k < nctx; ++k) th.emplace_back(work, k);
  work(0);
  for (auto& t : th) t.join();
  for (int k = 0; k < nctx; ++k)
    if (rcs[k]) return fail(rcs[k], "device %d: %s", ctxs[k]->device, errs[k].c_str());
  // device time of the group = the slowest shard (max over devices); launches summed
  const double mx = *std::max_element(ms.begin(), ms.end());
  int nl = 0;
  for (int x : launches) nl += x;
  for (int k = 0; k < nctx; ++k) {
    ctxs[k]->last_ms = mx;
    ctxs[k]->last_launches = nl;
  }
  return MGK_OK;
}

// Host image of a Gram job (device list pointers rebased onto the host copies).
static PairJob host_job(const mgk_ctx* c, const PairJob& j) {
  PairJob h = j;
  auto rebase32 = [&](const int32_t* p, const DBuf<int32_t>& d, const std::vector<int32_t>& hv) -> const int32_t* {
    return p ? hv.data() + (p - d.ptr) : nullptr;
  };
  h.list_a = rebase32(j.list_a, c->d_list_a, c->h_lists);
  h.list_b = rebase32(j.list_b, c->d_list_a, c->h_lists);
  h.row_col0 = rebase32(j.row_col0, c->d_rowcol, c->h_rowcol);
  h.row_prefix = j.row_prefix ? c->h_rowpre.data() + (j.row_prefix - c->d_rowpre.ptr) : nullptr;
  return h;
}

int mgk_gram_nodewise(mgk_ctx* c, int rank, int world, double tol, int64_t max_iter, int64_t chunk_bytes,
                      mgk_nodewise_sink sink, void* user, int64_t* npairs_out, int64_t* nfloats_out) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (world < 1 || rank < 0 || rank >= world) return fail(MGK_E_INVALID, "bad rank/world");
  if (!(tol > 0)) return fail(MGK_E_INVALID, "tolerance must be positive");
  if (!sink) return fail(MGK_E_INVALID, "null sink");
  int rc = prepare(c);
  if (rc) return rc;
  const SolveParams prm = make_params(c, tol, max_iter);
  std::vector<JobSpec> jobs;
  rc = gram_jobs(c, jobs, prm);
  if (rc) return rc;
  int64_t max_pair = 0;
  for (const GraphDesc& d : c->graphs) max_pair = std::max<int64_t>(max_pair, d.n);
  max_pair *= max_pair;
  const int64_t cap = std::max<int64_t>(chunk_bytes / 4, max_pair);
  const int64_t pair_cap = 1 << 22;
  // Two slots: the device solves chunk k + 1 while the host hands chunk k (already copied into pinned
  // memory) to the sink.  Per slot: field floats, per-pair records, offsets.
  constexpr int64_t kRec = 4 + 4 + 8 + 4 + 1;  // a, b, value, iterations, converged
  const size_t host_need = (size_t)(2 * cap) * sizeof(float) + (size_t)(2 * pair_cap) * kRec;
  if (c->h_nw_cap < host_need) {
    if (c->h_nw) cudaFreeHost(c->h_nw);
    c->h_nw = nullptr;
    c->h_nw_cap = 0;
    CUDA_TRY(cudaMallocHost(&c->h_nw, host_need));
    c->h_nw_cap = host_need;
  }
  CUDA_TRY(c->d_nodewise.alloc(2 * cap));
  CUDA_TRY(c->d_value.alloc(2 * pair_cap));
  CUDA_TRY(c->d_iters.alloc(2 * pair_cap));
  CUDA_TRY(c->d_conv.alloc(2 * pair_cap));
  CUDA_TRY(c->d_pa.alloc(2 * pair_cap));
  CUDA_TRY(c->d_pb.alloc(2 * pair_cap));
  CUDA_TRY(c->d_nwoff.alloc(2 * (pair_cap + 1)));
  struct Slot {
    float* nw;
    int32_t *a, *b, *it;
    double* v;
    uint8_t* cv;
    std::vector<int64_t> offs;
    int64_t np = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr, done = nullptr;
  } slot[2];
  {
    char* h = reinterpret_cast<char*>(c->h_nw);
    for (int k = 0; k < 2; ++k) {
      slot[k].nw = reinterpret_cast<float*>(h) + k * cap;
    }
    char* r = h + (size_t)(2 * cap) * sizeof(float);
    for (int k = 0; k < 2; ++k) {
      slot[k].v = reinterpret_cast<double*>(r);
      r += pair_cap * 8;
      slot[k].a = reinterpret_cast<int32_t*>(r);
      r += pair_cap * 4;
      slot[k].b = reinterpret_cast<int32_t*>(r);
      r += pair_cap * 4;
      slot[k].it = reinterpret_cast<int32_t*>(r);
      r += pair_cap * 4;
      slot[k].cv = reinterpret_cast<uint8_t*>(r);
      r += pair_cap;
    }
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaEventCreate(&slot[k].t0));
      CUDA_TRY(cudaEventCreate(&slot[k].t1));
      CUDA_TRY(cudaEventCreateWithFlags(&slot[k].done, cudaEventDisableTiming));
    }
  }
  auto destroy = [&]() {
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(slot[k].t0);
      cudaEventDestroy(slot[k].t1);
      cudaEventDestroy(slot[k].done);
    }
  };
  CUDA_TRY(c->d_status.alloc(1));
  CUDA_TRY(cudaMemsetAsync(c->d_status.ptr, 0, sizeof(int32_t), c->stream));
  int64_t total_pairs = 0, total_floats = 0;
  double ms_total = 0.0;
  int launches = 0, pending = -1, chunk = 0;
  cudaStream_t s = c->stream;
  // hand a finished slot to the sink
  auto drain = [&](int k) -> int {
    Slot& z = slot[k];
    cudaError_t e = cudaEventSynchronize(z.done);
    if (e != cudaSuccess) return fail(MGK_E_CUDA, "nodewise stream: %s", cudaGetErrorString(e));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, z.t0, z.t1);
    ms_total += ms;
    if (sink(user, z.np, z.a, z.b, z.v, z.it, z.cv, z.offs.data(), z.nw) != 0)
      return fail(MGK_E_STATE, "nodewise sink aborted the stream");
    total_pairs += z.np;
    total_floats += z.offs.back();
    return MGK_OK;
  };
  for (const JobSpec& js : jobs) {
    if (js.job.npairs <= 0) continue;
    const PairJob hj = host_job(c, js.job);
    const int64_t local = shard_len(js.job.npairs, rank, world);
    for (int64_t q0 = 0; q0 < local; ++chunk) {
      const int k = chunk & 1;
      Slot& z = slot[k];
      // chunk [q0, q1): field floats <= cap and pairs <= pair_cap
      z.offs.assign(1, 0);
      int64_t q1 = q0;
      while (q1 < local && q1 - q0 < pair_cap) {
        int32_t a, b;
        decode_pair(hj, rank + q1 * (int64_t)world, a, b);
        const int64_t f = (int64_t)c->graphs[a].n * c->graphs[b].n;
        if (z.offs.back() + f > cap) break;
        z.offs.push_back(z.offs.back() + f);
        ++q1;
      }
      z.np = q1 - q0;
      int64_t* d_off = c->d_nwoff.ptr + k * (pair_cap + 1);
      CUDA_TRY(cudaMemcpyAsync(d_off, z.offs.data(), z.offs.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      g_h2d_bytes += (int64_t)(z.offs.size() * sizeof(int64_t));
      JobSpec chunkjob = js;
      chunkjob.job.offset = rank + q0 * (int64_t)world;
      chunkjob.job.stride = world;
      chunkjob.job.npairs = z.np;
      std::vector<JobSpec> one = {chunkjob};
      SolveOut o{};
      o.value = c->d_value.ptr + k * pair_cap;
      o.iters = c->d_iters.ptr + k * pair_cap;
      o.conv = c->d_conv.ptr + k * pair_cap;
      o.pair_a = c->d_pa.ptr + k * pair_cap;
      o.pair_b = c->d_pb.ptr + k * pair_cap;
      o.nodewise = c->d_nodewise.ptr + k * cap;
      o.nodewise_off = d_off;
      rc = run_jobs(c, one, o, {0}, prm, false, z.t0, z.t1);
      if (rc) {
        destroy();
        return rc;
      }
      launches += c->last_launches;
      const int64_t np = z.np;
      auto cp = [&](void* dst, const void* src, size_t bytes) {
        g_d2h_bytes += (int64_t)bytes;
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
      };
      cudaError_t e = cp(z.a, o.pair_a, np * 4);
      if (e == cudaSuccess) e = cp(z.b, o.pair_b, np * 4);
      if (e == cudaSuccess) e = cp(z.v, o.value, np * 8);
      if (e == cudaSuccess) e = cp(z.it, o.iters, np * 4);
      if (e == cudaSuccess) e = cp(z.cv, o.conv, np);
      if (e == cudaSuccess) e = cp(z.nw, o.nodewise, z.offs.back() * sizeof(float));
      if (e == cudaSuccess) e = cudaEventRecord(z.done, s);
      if (e != cudaSuccess) {
        destroy();
        return fail(MGK_E_CUDA, "nodewise stream: %s", cudaGetErrorString(e));
      }
      if (pending >= 0) {
        rc = drain(pending);
        if (rc) {
          cudaStreamSynchronize(s);
          destroy();
          return rc;
        }
      }
      pending = k;
      q0 = q1;
    }
  }
  if (pending >= 0) {
    rc = drain(pending);
    if (rc) {
      destroy();
      return rc;
    }
  }
  destroy();
  rc = check_status(c);
  if (rc) return rc;
  c->last_ms = ms_total;
  c->last_launches = launches;
  if (npairs_out) *npairs_out = total_pairs;
  if (nfloats_out) *nfloats_out = total_floats;
  return MGK_OK;
}

int mgk_pairs(mgk_ctx* c, int64_t npairs, const int32_t* a, const int32_t* b, double tol, int64_t max_iter,
              double* value, int32_t* iters, double* residual, uint8_t* conv, double* nodewise) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (!(tol > 0)) return fail(MGK_E_INVALID, "tolerance must be positive");
  if (npairs <= 0) return MGK_OK;
  if (!a || !b) return fail(MGK_E_INVALID, "null pair arrays");
  int rc = prepare(c);
  if (rc) return rc;
  for (int64_t k = 0; k < npairs; ++k)
    if (a[k] < 0 || a[k] >= c->G || b[k] < 0 || b[k] >= c->G)
      return fail(MGK_E_INVALID, "pair %lld references unknown graph", (long long)k);
  // split into tiny / warp-class / block-class pairs; outputs in job order, remapped below
  std::vector<int32_t> ta, tb, wa, wb, ba, bb, ga_, gb_, xa, xb;
  std::vector<int64_t> tidx, widx, bidx, gidx, xidx;
  int64_t bn = 0, bm = 0, bsu = 0, bsl = 0, gn = 0, gm = 0, xn = 0, xm = 0, xsu = 0, xsl = 0;
  const SolveParams prm = make_params(c, tol, max_iter);
  const bool precise = prm.fp64 != 0;  // every pair on the FP64 block solver
  const bool panel = !precise && panel_dataset(c);
  const int T = tiny_nm();
  for (int64_t k = 0; k < npairs; ++k) {
    const GraphDesc &A = c->graphs[a[k]], &B = c->graphs[b[k]];
    if (!precise && small_graph(c, A) && small_graph(c, B)) {
      const bool tiny = (int64_t)A.n * B.n <= T;
      (tiny ? ta : wa).push_back(a[k]);
      (tiny ? tb : wb).push_back(b[k]);
      (tiny ? tidx : widx).push_back(k);
    } else if (panel && (int64_t)A.n * B.n <= T) {
      // tiny n m with a graph outside the warp class (a dense small graph): the block solver's FP64
      // vectors instead of the FP32 panel kernel
      xa.push_back(a[k]);
      xb.push_back(b[k]);
      xidx.push_back(k);
      xn = std::max<int64_t>(xn, A.n);
      xm = std::max<int64_t>(xm, B.n);
      xsu = std::max<int64_t>(xsu, 2 * A.ne);
      xsl = std::max<int64_t>(xsl, 2 * B.ne);
    } else if (panel && (int64_t)A.n * B.n >= (int64_t)large_n() * large_n()) {
      ga_.push_back(a[k]);
      gb_.push_back(b[k]);
      gidx.push_back(k);
      gn = std::max<int64_t>(gn, A.n);
      gm = std::max<int64_t>(gm, B.n);
    } else {
      ba.push_back(a[k]);
      bb.push_back(b[k]);
      bidx.push_back(k);
      bn = std::max<int64_t>(bn, A.n);
      bm = std::max<int64_t>(bm, B.n);
      bsu = std::max<int64_t>(bsu, 2 * A.ne);
      bsl = std::max<int64_t>(bsl, 2 * B.ne);
    }
  }
  std::vector<int32_t> la(wa), lb(wb);
  la.insert(la.end(), ta.begin(), ta.end());
  lb.insert(lb.end(), tb.begin(), tb.end());
  la.insert(la.end(), ba.begin(), ba.end());
  lb.insert(lb.end(), bb.begin(), bb.end());
  la.insert(la.end(), ga_.begin(), ga_.end());
  lb.insert(lb.end(), gb_.begin(), gb_.end());
  la.insert(la.end(), xa.begin(), xa.end());
  lb.insert(lb.end(), xb.begin(), xb.end());
  std::vector<int64_t> order(widx);
  order.insert(order.end(), tidx.begin(), tidx.end());
  order.insert(order.end(), bidx.begin(), bidx.end());
  order.insert(order.end(), gidx.begin(), gidx.end());
  order.insert(order.end(), xidx.begin(), xidx.end());
  cudaStream_t s = c->stream;
  CUDA_TRY(c->d_list_b.upload(la, s));
  CUDA_TRY(c->d_list_c.upload(lb, s));
  const int64_t nw0 = (int64_t)wa.size(), nt0 = (int64_t)ta.size();
  std::vector<JobSpec> jobs(5);
  jobs[0].job = PairJob{PM_LIST, 0, 0, nw0, 0, 1, c->d_list_b.ptr, c->d_list_c.ptr, nullptr, nullptr};
  jobs[0].kernel = JK_WARP;
  jobs[1].job = PairJob{PM_LIST, 0, 0, nt0, 0, 1, c->d_list_b.ptr + nw0, c->d_list_c.ptr + nw0, nullptr, nullptr};
  jobs[1].kernel = JK_TINY;
  jobs[2].job = PairJob{PM_LIST, 0, 0, (int64_t)ba.size(), 0, 1, c->d_list_b.ptr + nw0 + nt0,
                        c->d_list_c.ptr + nw0 + nt0, nullptr, nullptr};
  jobs[2].kernel = panel ? JK_PANEL : JK_BLOCK;
  jobs[2].max_n = bn;
  jobs[2].max_m = bm;
  jobs[2].max_su = bsu;
  jobs[2].max_sl = bsl;
  const int64_t nb0 = (int64_t)ba.size();
  jobs[3].job = PairJob{PM_LIST, 0, 0, (int64_t)ga_.size(), 0, 1, c->d_list_b.ptr + nw0 + nt0 + nb0,
                        c->d_list_c.ptr + nw0 + nt0 + nb0, nullptr, nullptr};
  jobs[3].kernel = JK_GRID;
  jobs[3].max_n = gn;
  jobs[3].max_m = gm;
  const int64_t nx0 = nw0 + nt0 + nb0 + (int64_t)ga_.size();
  jobs[4].job = PairJob{PM_LIST, 0, 0, (int64_t)xa.size(), 0, 1, c->d_list_b.ptr + nx0, c->d_list_c.ptr + nx0,
                        nullptr, nullptr};
  jobs[4].kernel = JK_BLOCK;
  jobs[4].max_n = xn;
  jobs[4].max_m = xm;
  jobs[4].max_su = xsu;
  jobs[4].max_sl = xsl;
  std::vector<int64_t> offs = {0, nw0, nw0 + nt0, nw0 + nt0 + nb0, nx0};
  CUDA_TRY(c->d_value.alloc(npairs));
  CUDA_TRY(c->d_iters.alloc(npairs));
  CUDA_TRY(c->d_conv.alloc(npairs));
  CUDA_TRY(c->d_resid.alloc(npairs));
  SolveOut o{};
  o.value = c->d_value.ptr;
  o.iters = c->d_iters.ptr;
  o.conv = c->d_conv.ptr;
  o.residual = c->d_resid.ptr;
  std::vector<int64_t> nwoff(npairs + 1, 0);
  if (nodewise) {
    for (int64_t k = 0; k < npairs; ++k)
      nwoff[k + 1] = nwoff[k] + (int64_t)c->graphs[la[k]].n * c->graphs[lb[k]].n;
    CUDA_TRY(c->d_nwoff.upload(nwoff, s));
    CUDA_TRY(c->d_nodewise.alloc(nwoff[npairs]));
    o.nodewise = c->d_nodewise.ptr;
    o.nodewise_off = c->d_nwoff.ptr;
  }
  rc = run_jobs(c, jobs, o, offs, prm);
  if (rc) return rc;
  std::vector<double> hv(npairs);
  std::vector<int32_t> hi(npairs);
  std::vector<uint8_t> hc(npairs);
  std::vector<float> hr(npairs);
  CUDA_TRY(d2h(hv.data(), c->d_value.ptr, npairs * sizeof(double)));
  CUDA_TRY(d2h(hi.data(), c->d_iters.ptr, npairs * sizeof(int32_t)));
  CUDA_TRY(d2h(hc.data(), c->d_conv.ptr, npairs));
  CUDA_TRY(d2h(hr.data(), c->d_resid.ptr, npairs * sizeof(float)));
  std::vector<float> hn;
  if (nodewise) {
    hn.resize(nwoff[npairs]);
    CUDA_TRY(d2h(hn.data(), c->d_nodewise.ptr, hn.size() * sizeof(float)));
  }
  // output offsets of the caller's order
  std::vector<int64_t> caller_off(npairs + 1, 0);
  if (nodewise)
    for (int64_t k = 0; k < npairs; ++k)
      caller_off[k + 1] = caller_off[k] + (int64_t)c->graphs[a[k]].n * c->graphs[b[k]].n;
  for (int64_t j = 0; j < npairs; ++j) {
    int64_t k = order[j];
    if (value) value[k] = hv[j];
    if (iters) iters[k] = hi[j];
    if (conv) conv[k] = hc[j];
    if (residual) residual[k] = hr[j];
    if (nodewise)
      for (int64_t e = 0; e < nwoff[j + 1] - nwoff[j]; ++e) nodewise[caller_off[k] + e] = hn[nwoff[j] + e];
  }
  return MGK_OK;
}

int mgk_kernel(mgk_ctx* c, int32_t a, int32_t b, double tol, int64_t max_iter, double* value, double* nodewise,
               int32_t* iters, double* residual, uint8_t* conv) {
  return mgk_pairs(c, 1, &a, &b, tol, max_iter, value, iters, residual, conv, nodewise);
}

int mgk_counters(mgk_ctx* c, int32_t a, int32_t b, int64_t applies, const double* model, const int32_t* thresholds,
                 int force_dense, double* out) {
  if (!c || !model || !thresholds || !out) return fail(MGK_E_INVALID, "null argument");
  if (applies < 0) return fail(MGK_E_INVALID, "applies must be >= 0");
  int rc = prepare(c);
  if (rc) return rc;
  if (a < 0 || a >= c->G || b < 0 || b >= c->G) return fail(MGK_E_INVALID, "graph index out of range");
  if (c->h_hist.empty()) {
    DBuf<int32_t> d;
    CUDA_TRY(d.alloc((size_t)c->G * kHistBins));
    k_tile_hist<<<c->G, 128, 0, c->stream>>>(c->d_graphs.ptr, c->d_tiles.ptr, c->d_trow.ptr, d.ptr);
    CUDA_TRY(cudaGetLastError());
    c->h_hist.resize((size_t)c->G * kHistBins);
    CUDA_TRY(cudaMemcpyAsync(c->h_hist.data(), d.ptr, c->h_hist.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  const int32_t* ha = c->h_hist.data() + (size_t)a * kHistBins;
  const int32_t* hb = c->h_hist.data() + (size_t)b * kHistBins;
  const double E = model[0], F = model[1], X = model[2], r = model[3], t = 8.0;
  const int s1 = thresholds[0], s2 = thresholds[1], dmin = thresholds[2];
  // per-apply increments of ProductOperator._build_plan (product.py:224-266), summed over the tile-pair
  // density classes (na, nb) with multiplicity count_a[na] * count_b[nb]; every term is an integer, so the
  // sums equal the reference's tile-pair-by-tile-pair accumulation exactly
  double flops = 0, t1l = 0, t2l = 0, t2s = 0, pairs = 0;
  for (int na = 1; na <= 64; ++na) {
    if (!ha[na]) continue;
    for (int nb = 1; nb <= 64; ++nb) {
      if (!hb[nb]) continue;
      const double mult = (double)ha[na] * (double)hb[nb];
      pairs += mult;
      if (force_dense) {
        flops += mult * (t * t * t * t * X);
        t1l += mult * (t * t * (E + 2 * F));
        t2s += mult * (t * t * (E + F));
        t2l += mult * (t * t * t * t * (E + F) * (1.0 / t + 1.0 / r));
        continue;
      }
      t1l += mult * (8.0 + nb * (E + F) + t * t * F);
      const int lo = std::min(na, nb), hi = std::max(na, nb);
      double contrib;
      if (lo <= s1 && hi <= s2) {  // select_tile_kernel (product.py:56-66)
        contrib = (double)na * nb;
        t2s += mult * ((na + nb) * (E + F));
      } else if (lo >= dmin) {
        contrib = t * t * t * t;
        t2s += mult * (t * t * (E + F));
      } else {
        contrib = t * t * lo;
        t2s += mult * (t * t * (E + F));
      }
      flops += mult * contrib * X;
      t2l += mult * contrib * (E + 2 * F);
    }
  }
  const double t1s = (double)ha[65] * (double)hb[65] * t * t * F;
  const double k = (double)applies;
  out[0] = k * flops;
  out[1] = k * t1l;
  out[2] = k * t1s;
  out[3] = k * t2l;
  out[4] = k * t2s;
  out[5] = k * pairs;
  return MGK_OK;
}

int mgk_transfer_bytes(int64_t* h2d, int64_t* d2h_out) {
  if (h2d) *h2d = g_h2d_bytes.load();
  if (d2h_out) *d2h_out = g_d2h_bytes.load();
  return MGK_OK;
}

int mgk_last_timing(mgk_ctx* c, double* solve_ms, int32_t* launches) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (solve_ms) *solve_ms = c->last_ms;
  if (launches) *launches = c->last_launches;
  return MGK_OK;
}

int mgk_reorder(mgk_ctx* c, int method, uint64_t seed, int apply, int64_t* perms_out) {
  if (!c) return fail(MGK_E_INVALID, "null context");
  if (!c->uploaded) return fail(MGK_E_STATE, "no dataset uploaded");
  if (method == MGK_REORDER_NONE) {
    if (perms_out)
      for (int g = 0; g < c->G; ++g)
        for (int64_t i = c->node_off[g]; i < c->node_off[g + 1]; ++i) perms_out[i] = i - c->node_off[g];
    return MGK_OK;
  }
  if (method != MGK_REORDER_PBR && method != MGK_REORDER_RCM && method != MGK_REORDER_MORTON)
    return fail(MGK_E_INVALID, "unknown reorder method %d", method);
  if (method == MGK_REORDER_MORTON && !(c->nl_kind == LK_VEC && (c->nl_dim == 2 || c->nl_dim == 3)))
    return fail(MGK_E_INVALID, "morton reordering needs 2D/3D coordinate node labels");
  int rc = prepare(c);  // octiles of the current order drive the PBR tile-count fallback
  if (rc) return rc;
  std::vector<int64_t> fwd;
  if (method == MGK_REORDER_PBR)
    rc = pbr_device(c->G, c->node_off, c->edge_off, c->ei, c->ej, seed, c->d_tiles.ptr, c->graphs, c->d_trow.ptr,
                    c->device, c->stream, fwd, g_err);
  else
    rc = order_device(method, c->G, c->graphs, c->d_graphs.ptr, c->d_ngraph.ptr, c->d_rowptr.ptr, c->d_rowent.ptr,
                      c->nl_vec, c->nl_dim, c->stream, fwd, g_err);
  if (rc) return rc;
  if (perms_out) std::copy(fwd.begin(), fwd.end(), perms_out);
  if (apply) {
    // apply_permutation (reorder.py:86-109): edges (min, max) of forward images, node arrays via inverse
    std::vector<double> p2(c->p.size()), q2(c->q.size()), nlv(c->nl_vec.size());
    std::vector<int64_t> nlc(c->nl_cat.size());
    for (int g = 0; g < c->G; ++g) {
      int64_t n0 = c->node_off[g];
      for (int64_t i = n0; i < c->node_off[g + 1]; ++i) {
        int64_t dst = n0 + fwd[i];
        p2[dst] = c->p[i];
        q2[dst] = c->q[i];
        if (!c->nl_cat.empty()) nlc[dst] = c->nl_cat[i];
        for (int d = 0; d < c->nl_dim && !c->nl_vec.empty(); ++d) nlv[dst * c->nl_dim + d] = c->nl_vec[i * c->nl_dim + d];
      }
      for (int64_t e = c->edge_off[g]; e < c->edge_off[g + 1]; ++e) {
        int32_t x = (int32_t)fwd[n0 + c->ei[e]], y = (int32_t)fwd[n0 + c->ej[e]];
        c->ei[e] = std::min(x, y);
        c->ej[e] = std::max(x, y);
      }
    }
    c->p.swap(p2);
    c->q.swap(q2);
    if (!c->nl_cat.empty()) c->nl_cat.swap(nlc);
    if (!c->nl_vec.empty()) c->nl_vec.swap(nlv);
    c->prepared = false;
  }
  return MGK_OK;
}

}  // extern "C"
