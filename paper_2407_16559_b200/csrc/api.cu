// api.cu — the C ABI (include/agk/agk.h): handles, device memory layout, graph caching.
//
// Device memory layout per handle (HBM, fp64):
//   ut  r x m   U transposed: rank a's column contiguous (the FFT loads and the death epilogue
//               read it unit-stride; the reference's m x r layout would be stride r)
//   v   r x m   V as in the reference
//   y   g x P   complex intermediate of one rank group (sized to stay L2-resident)
//   acc (N1/2+1) x N2 complex: Hermitian half of the summed product spectrum, then G
//   state 2 x m, K1..K6, K1b, stage, full, mid (stepper vectors, m each)
// The rank dedupe of birth_term (rhs.cpp:96-124) is evaluated once at create time with the
// reference's bitwise comparison rule.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"
#include "steps.cuh"

using namespace agk;

namespace {
// NVTX range around each C-ABI entry point (domain "agk"): host-side API spans for a timeline
// tool; header-only NVTX v3, a no-op pointer check when no tool is attached.
struct NvtxRange {
  static nvtxDomainHandle_t domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("agk");
    return d;
  }
  explicit NvtxRange(const char* name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(domain(), &a);
  }
  ~NvtxRange() { nvtxDomainRangePop(domain()); }
};
}  // namespace

struct agk_rhs {
  int device = 0;
  cudaStream_t stream = nullptr;
  int kind = AGK_RHS_MODEL;
  double fake_param = 0.0;
  int64_t m = 0;
  int r = 0, rf = 0;
  int variant = 0;
  double lambda = 0.0;
  int nsrc = 0;
  std::vector<double> host_weight;
  RhsPlan plan{};
  RhsArgs base{};  // model arguments with n/out unset
  std::vector<void*> allocs;
  double2* tw_all = nullptr;
  StepBuffers sb{};
  DevCtl* ctl = nullptr;
  double* d_in = nullptr;
  double* d_out = nullptr;
  double* d_scalar = nullptr;
  uint64_t evals = 0;
  std::string err;
  std::map<int, cudaGraphExec_t> graphs;
  std::map<int, int> graph_kernels;
  cudaGraphExec_t rhs_graph = nullptr;
  cudaGraphExec_t rhs_graph_b = nullptr;  // kTimedBatch evaluations back to back in one graph
  const double* rhs_graph_in = nullptr;
  double* rhs_graph_out = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  agk_record* rec_ring = nullptr;  // device record ring of agk_run (allocated on first use)
  ~agk_rhs();
};

namespace {

thread_local std::string g_create_error;
constexpr int kSwap = 1000000;

agk_status fail(agk_rhs* h, agk_status st, const std::string& msg) {
  if (h) h->err = msg;
  else g_create_error = msg;
  return st;
}

agk_status cuda_fail(agk_rhs* h, cudaError_t e, const char* what) {
  return fail(h, e == cudaErrorMemoryAllocation ? AGK_ERR_OUT_OF_MEMORY : AGK_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK_H(h, x, what)                             \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, what); \
  } while (0)

template <typename T>
cudaError_t dalloc(agk_rhs* h, T** p, size_t n) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, (n ? n : 1) * sizeof(T));
  if (e == cudaSuccess) {
    h->allocs.push_back(q);
    *p = static_cast<T*>(q);
  }
  return e;
}

// exp(-2 pi i k / n) for k < n, computed in long double and rounded once
void fill_table(std::vector<double2>& t, size_t off, int64_t n, int64_t stride_num = 1) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int64_t k = 0; k < n; ++k) {
    const long double ang = -2.0L * pi * (long double)(k * stride_num) / (long double)(n * stride_num);
    t[off + k] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
}

agk_status select_device(agk_rhs* h, int device) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(h, AGK_ERR_NO_DEVICE, "no CUDA device visible: the B200 path has no CPU fallback");
  if (device < 0) {
    e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaGetDevice");
  }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaGetDeviceProperties");
  if (prop.major < 10)
    return fail(h, AGK_ERR_NO_DEVICE, std::string("device ") + prop.name + " is not sm_100: kernels are built for sm_100a only");
  h->device = device;  // made current only inside each call (DeviceGuard)
  return AGK_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

// Releases everything the handle owns (also on a failed create: unique_ptr<agk_rhs>).
agk_rhs::~agk_rhs() {
  DeviceGuard dg(device);
  if (stream) cudaStreamSynchronize(stream);
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  if (rhs_graph) cudaGraphExecDestroy(rhs_graph);
  if (rhs_graph_b) cudaGraphExecDestroy(rhs_graph_b);
  for (void* p : allocs) cudaFree(p);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (stream) cudaStreamDestroy(stream);
}

namespace {

agk_status alloc_common(agk_rhs* h) {
  const int64_t m = h->m;
  // blocking stream: ordered after (and before) work on the legacy default stream, so device
  // inputs produced there (torch's default stream) are complete when a kernel reads them
  CK_H(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamDefault), "cudaStreamCreate");
  CK_H(h, cudaEventCreate(&h->ev0), "cudaEventCreate");
  CK_H(h, cudaEventCreate(&h->ev1), "cudaEventCreate");
  CK_H(h, dalloc(h, &h->d_in, m), "alloc in");
  CK_H(h, dalloc(h, &h->d_out, m), "alloc out");
  CK_H(h, dalloc(h, &h->d_scalar, 8), "alloc scalar");
  CK_H(h, dalloc(h, &h->ctl, 1), "alloc ctl");
  StepBuffers& b = h->sb;
  CK_H(h, dalloc(h, &b.state, 2 * m), "alloc state");
  for (int q = 0; q < 7; ++q) CK_H(h, dalloc(h, &b.k[q], m), "alloc k");
  CK_H(h, dalloc(h, &b.stg, m), "alloc stage");
  CK_H(h, dalloc(h, &b.full, m), "alloc full");
  CK_H(h, dalloc(h, &b.mid, m), "alloc mid");
  CK_H(h, dalloc(h, &b.n5, m), "alloc n5");
  b.nred = red_blocks_for(m);
  CK_H(h, dalloc(h, &b.red, (size_t)b.nred * RF_N), "alloc red");
  b.naux = b.nred;
  CK_H(h, dalloc(h, &b.aux, (size_t)b.naux * (4 + (h->r > 0 ? h->r : 1))), "alloc aux");
  CK_H(h, cudaMemsetAsync(h->ctl, 0, sizeof(DevCtl), h->stream), "memset ctl");
  return AGK_OK;
}

// Enqueue the handle's RHS: the model's kernels or the injected fake.
struct HandleRhs final : RhsEnqueue {
  agk_rhs* h;
  explicit HandleRhs(agk_rhs* hh) : h(hh) {}
  cudaError_t operator()(VecRef in, double* out, const int* skip, cudaStream_t s) const override {
    if (h->kind != AGK_RHS_MODEL) return fake_rhs_launch(h->kind, h->fake_param, in, out, h->m, skip, s);
    RhsArgs a = h->base;
    a.n = in;
    a.out = out;
    a.skip = skip;
    return rhs_launch(h->plan, a, s);
  }
  int launches() const override { return h->kind == AGK_RHS_MODEL ? h->plan.launches : 1; }
  bool stage_fusable() const override { return h->kind == AGK_RHS_MODEL && !h->plan.dense && knob("AGK_FUSE_STAGES", 1) != 0; }
  cudaError_t stage(VecRef x, const StageIn& st, double* stg, double* out, cudaStream_t s) const override {
    RhsArgs a = h->base;
    a.n = x;
    a.st = st;
    a.stg_out = stg;
    a.out = out;
    a.skip = nullptr;
    return rhs_launch(h->plan, a, s);
  }
};

int body_for(const agk_control* c) {
  if (c->stepper == AGK_RKF45) return BODY_FEHLBERG;
  return c->mode == AGK_FIXED ? BODY_FIXED : BODY_DOUBLING;
}

agk_status get_graph(agk_rhs* h, int body, int stepper, cudaGraphExec_t* out) {
  const int key = body * 4 + stepper;
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    *out = it->second;
    return AGK_OK;
  }
  HandleRhs rhs(h);
  cudaGraphExec_t ex = nullptr;
  int nk = 0;
  const RhsArgs* model = h->kind == AGK_RHS_MODEL ? &h->base : nullptr;
  CK_H(h, build_step_graph(body, stepper, rhs, h->sb, h->ctl, h->m, model, h->stream, &ex, &nk),
       "building the step graph");
  h->graphs[key] = ex;
  h->graph_kernels[key] = nk;
  *out = ex;
  return AGK_OK;
}

void control_to_ctl(const agk_control* c, DevCtl* d) {
  d->stepper = c->stepper;
  d->mode = c->mode;
  d->max_rejects = c->max_rejects;
  d->relative_error = c->relative_error;
  d->tol = c->tol;
  d->safety = c->safety;
  d->growth_max = c->growth_max;
  d->shrink_min = c->shrink_min;
  d->tau_min = c->tau_min;
  d->tau_fixed = c->tau;
  d->body = body_for(c);
}

agk_status copy_in(agk_rhs* h, const double* n, int where, double* dst) {
  CK_H(h, cudaMemcpyAsync(dst, n, h->m * sizeof(double),
                          where == AGK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream),
       "copy in");
  return AGK_OK;
}

agk_status copy_out(agk_rhs* h, double* out, int where, const double* src) {
  CK_H(h, cudaMemcpyAsync(out, src, h->m * sizeof(double),
                          where == AGK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream),
       "copy out");
  return AGK_OK;
}

agk_status run_terms(agk_rhs* h, const double* n, double* out, int where, int flags, double lambda) {
  if (!h || !n || !out) return fail(h, AGK_ERR_INVALID_ARGUMENT, "null argument");
  if (h->kind != AGK_RHS_MODEL) return fail(h, AGK_ERR_INVALID_ARGUMENT, "term functions need a model handle");
  DeviceGuard dg(h->device);
  const double* din = n;
  double* dout = out;
  if (where == AGK_MEM_HOST) {
    agk_status st = copy_in(h, n, where, h->d_in);
    if (st) return st;
    din = h->d_in;
    dout = h->d_out;
  }
  RhsArgs a = h->base;
  a.n = VecRef{din, nullptr, 0};
  a.out = dout;
  a.skip = nullptr;
  a.flags = flags;
  a.lambda = lambda;
  CK_H(h, rhs_launch(h->plan, a, h->stream), "rhs launch");
  if (where == AGK_MEM_HOST) {
    agk_status st = copy_out(h, out, where, h->d_out);
    if (st) return st;
  }
  CK_H(h, cudaStreamSynchronize(h->stream), "rhs sync");
  return AGK_OK;
}

int model_flags(const agk_rhs* h) {
  int f = T_BIRTH | T_DEATH;
  if (h->variant == AGK_AGGREGATION_SOURCES) f |= T_SOURCES;
  if (h->variant == AGK_AGGREGATION_SHATTERING) f |= T_SHATTER;
  return f;
}

}  // namespace

// DenseKernel model (rhs.cpp dense branches; rhs_dense.cu): K is copied to the device once.
static agk_status create_dense(const agk_model_desc* d, std::unique_ptr<agk_rhs> h, agk_rhs** out) {
  const int64_t m = (int64_t)d->m;
  if (d->m > ((size_t)1 << 17)) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "dense kernel m > 2^17 is not supported");
  h->kind = AGK_RHS_MODEL;
  h->m = m;
  h->r = 0;
  h->rf = 0;
  h->variant = d->variant;
  h->lambda = d->shatter_rate;
  RhsPlan& p = h->plan;
  p = RhsPlan{};
  p.dense = 1;
  p.launches = 3 + (d->variant == AGK_AGGREGATION_SHATTERING ? 1 : 0);
  agk_status st = alloc_common(h.get());
  agk_rhs* hp = h.get();
  auto cleanup_fail = [&](agk_status s2) {
    g_create_error = hp->err;
    for (void* q : hp->allocs) cudaFree(q);
    hp->allocs.clear();
    return s2;
  };
  if (st) return cleanup_fail(st);
#define CK_D(x, what)                                                        \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) return cleanup_fail(cuda_fail(hp, e_, what));     \
  } while (0)
  RhsArgs& a = h->base;
  double *kd, *drow, *dpair, *dpart, *scalars;
  CK_D(dalloc(hp, &kd, (size_t)m * m), "alloc dense kernel");
  CK_D(cudaMemcpy(kd, d->k, (size_t)m * m * sizeof(double), cudaMemcpyHostToDevice), "upload dense kernel");
  CK_D(dalloc(hp, &drow, (size_t)m), "alloc row sums");
  CK_D(dalloc(hp, &dpair, (size_t)m), "alloc gain terms");
  CK_D(dalloc(hp, &dpart, (size_t)dense_chunks(m) * m), "alloc birth partials");
  CK_D(dalloc(hp, &scalars, 8), "alloc scalars");
  int64_t* sk = nullptr;
  double* sr = nullptr;
  if (d->variant == AGK_AGGREGATION_SOURCES && d->num_sources > 0) {
    std::vector<int64_t> hk(d->num_sources);
    for (size_t q = 0; q < d->num_sources; ++q) hk[q] = (int64_t)d->source_k[q];
    CK_D(dalloc(hp, &sk, d->num_sources), "alloc sources");
    CK_D(dalloc(hp, &sr, d->num_sources), "alloc sources");
    CK_D(cudaMemcpy(sk, hk.data(), hk.size() * sizeof(int64_t), cudaMemcpyHostToDevice), "upload sources");
    CK_D(cudaMemcpy(sr, d->source_rate, d->num_sources * sizeof(double), cudaMemcpyHostToDevice), "upload sources");
    h->nsrc = (int)d->num_sources;
  }
  a.m = m;
  a.r = 0;
  a.rf = 0;
  a.kd = kd;
  a.drow = drow;
  a.dpair = dpair;
  a.dpart = dpart;
  a.scalars = scalars;
  a.flags = model_flags(hp);
  a.lambda = d->shatter_rate;
  a.src_k = sk;
  a.src_rate = sr;
  a.nsrc = h->nsrc;
  CK_D(cudaStreamSynchronize(hp->stream), "create sync");
#undef CK_D
  *out = h.release();
  return AGK_OK;
}

extern "C" {

void agk_control_defaults(agk_control* c) {
  c->stepper = AGK_RKF45;
  c->mode = AGK_ADAPTIVE;
  c->tau = 0.0;
  c->tol = 1e-6;
  c->safety = 0.0;
  c->growth_max = 2.0;
  c->shrink_min = 0.5;
  c->tau_min = 1e-12;
  c->max_rejects = 40;
  c->relative_error = 0;
}

agk_status agk_control_validate(const agk_control* c) {
  if (!c) return AGK_ERR_INVALID_ARGUMENT;
  if (c->stepper < 0 || c->stepper > 2 || c->mode < 0 || c->mode > 1) return AGK_ERR_INVALID_ARGUMENT;
  if (c->mode == AGK_FIXED && !(c->tau > 0.0)) return AGK_ERR_INVALID_ARGUMENT;
  if (c->mode == AGK_ADAPTIVE && !(c->tol > 0.0)) return AGK_ERR_INVALID_ARGUMENT;
  if (c->safety < 0.0 || c->safety >= 1.0) return AGK_ERR_INVALID_ARGUMENT;
  if (!(c->tau_min > 0.0)) return AGK_ERR_INVALID_ARGUMENT;
  if (!(c->shrink_min < 1.0 && 1.0 < c->growth_max)) return AGK_ERR_INVALID_ARGUMENT;
  if (c->max_rejects < 1) return AGK_ERR_INVALID_ARGUMENT;
  return AGK_OK;
}

const char* agk_describe_status(int s) {
  switch (s) {
    case AGK_STEP_OK: return "ok";
    case AGK_STEP_NONFINITE: return "non-finite state";
    case AGK_STEP_TOO_MANY_REJECTS: return "step reject limit exceeded";
    case AGK_STEP_TAU_UNDERFLOW: return "step size underflow";
    default: return "unknown";
  }
}

const char* agk_last_error(const agk_rhs* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

agk_status agk_rhs_create(const agk_model_desc* d, agk_rhs** out) {
  NvtxRange nvtx_("agk_rhs_create");
  if (!d || !out) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  // ModelSpec::validate (rhs.cpp:63-72) and SourceTerm::validate (rhs.cpp:48-61)
  if (d->m < 2) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "truncation size m must be >= 2");
  if (!d->k && (d->r < 1 || !d->u || !d->v)) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "kernel factors missing");
  if (d->m > ((size_t)1 << 22)) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "m > 2^22 is not supported");
  if (d->variant < 0 || d->variant > 2) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "unknown model variant");
  if (d->variant == AGK_AGGREGATION_SOURCES) {
    for (size_t q = 0; q < d->num_sources; ++q) {
      if (d->source_k[q] < 1 || d->source_k[q] > d->m)
        return fail(nullptr, AGK_ERR_INVALID_ARGUMENT,
                    "source index " + std::to_string(d->source_k[q]) + " outside 1.." + std::to_string(d->m));
      if (!std::isfinite(d->source_rate[q]) || d->source_rate[q] < 0.0)
        return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "source rate must be finite and >= 0");
    }
  }
  if (d->variant == AGK_AGGREGATION_SHATTERING && (!std::isfinite(d->shatter_rate) || d->shatter_rate < 0.0))
    return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "shattering rate lambda must be finite and >= 0");

  std::unique_ptr<agk_rhs> h(new agk_rhs());
  agk_status st = select_device(h.get(), d->device);
  if (st) {
    g_create_error = h->err;
    return st;
  }
  DeviceGuard dg(h->device);  // restores the caller's current device on every return path
  if (d->k) return create_dense(d, std::move(h), out);
  const int64_t m = (int64_t)d->m;
  const int r = (int)d->r;
  h->kind = AGK_RHS_MODEL;
  h->m = m;
  h->r = r;
  h->variant = d->variant;
  h->lambda = d->shatter_rate;

  // rank dedupe, reference rule (rhs.cpp:96-124)
  std::vector<double> weight(r, 1.0);
  std::vector<char> skip(r, 0);
  std::vector<int> swapped_into(r, -1), same_into(r, -1);
  auto ucol_eq = [&](int a, const double* other, int64_t stride) {
    for (int64_t i = 0; i < m; ++i)
      if (d->u[i * r + a] != other[i * stride]) return false;
    return true;
  };
  for (int a = 1; a < r; ++a) {
    for (int b = 0; b < a; ++b) {
      if (skip[b]) continue;
      const bool sw = ucol_eq(a, d->v + (int64_t)b * m, 1) && ucol_eq(b, d->v + (int64_t)a * m, 1);
      bool same = ucol_eq(a, d->u + b, r);
      if (same)
        for (int64_t j = 0; j < m; ++j)
          if (d->v[(int64_t)a * m + j] != d->v[(int64_t)b * m + j]) {
            same = false;
            break;
          }
      if (sw || same) {
        weight[b] += 1.0;
        skip[a] = 1;
        if (sw) swapped_into[a] = b;
        else same_into[a] = b;
        break;
      }
    }
  }
  std::vector<int> uniq_rank, rank_map(r), uindex(r, -1);
  std::vector<double> uniq_weight;
  for (int a = 0; a < r; ++a)
    if (!skip[a]) {
      uindex[a] = (int)uniq_rank.size();
      uniq_rank.push_back(a);
      uniq_weight.push_back(weight[a]);
    }
  for (int a = 0; a < r; ++a) {
    if (!skip[a]) rank_map[a] = uindex[a];
    else if (swapped_into[a] >= 0) rank_map[a] = uindex[swapped_into[a]] + kSwap;
    else rank_map[a] = uindex[same_into[a]];
  }
  h->rf = (int)uniq_rank.size();
  h->host_weight = weight;

  rhs_make_plan(m, h->rf, &h->plan);
  st = alloc_common(h.get());
  if (st) {
    g_create_error = h->err;
    for (void* p : h->allocs) cudaFree(p);
    return st;
  }
  agk_rhs* hp = h.get();
  auto cleanup_fail = [&](agk_status s2) {
    g_create_error = hp->err;
    for (void* p : hp->allocs) cudaFree(p);
    hp->allocs.clear();
    return s2;
  };
#define CK_C(x, what)                                                        \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) return cleanup_fail(cuda_fail(hp, e_, what));     \
  } while (0)

  // factors: U transposed to rank-major, V as is
  RhsArgs& a = h->base;
  double *ut, *vv, *u0, *v0, *uw, *partials, *scalars;
  int *ur, *rm;
  int64_t* sk = nullptr;
  double* sr = nullptr;
  CK_C(dalloc(hp, &ut, (size_t)r * m), "alloc U");
  CK_C(dalloc(hp, &vv, (size_t)r * m), "alloc V");
  {
    std::vector<double> tmp((size_t)m);
    for (int q = 0; q < r; ++q) {
      for (int64_t i = 0; i < m; ++i) tmp[i] = d->u[i * r + q];
      CK_C(cudaMemcpy(ut + (int64_t)q * m, tmp.data(), m * sizeof(double), cudaMemcpyHostToDevice), "upload U");
    }
    CK_C(cudaMemcpy(vv, d->v, (size_t)r * m * sizeof(double), cudaMemcpyHostToDevice), "upload V");
    std::vector<double> hu0(r), hv0(r);
    for (int q = 0; q < r; ++q) {
      hu0[q] = d->u[q];
      hv0[q] = d->v[(int64_t)q * m];
    }
    CK_C(dalloc(hp, &u0, r), "alloc u0");
    CK_C(dalloc(hp, &v0, r), "alloc v0");
    CK_C(cudaMemcpy(u0, hu0.data(), r * sizeof(double), cudaMemcpyHostToDevice), "upload u0");
    CK_C(cudaMemcpy(v0, hv0.data(), r * sizeof(double), cudaMemcpyHostToDevice), "upload v0");
  }
  CK_C(dalloc(hp, &ur, h->rf), "alloc ranks");
  CK_C(dalloc(hp, &uw, h->rf), "alloc weights");
  CK_C(dalloc(hp, &rm, r), "alloc rank map");
  CK_C(cudaMemcpy(ur, uniq_rank.data(), h->rf * sizeof(int), cudaMemcpyHostToDevice), "upload ranks");
  CK_C(cudaMemcpy(uw, uniq_weight.data(), h->rf * sizeof(double), cudaMemcpyHostToDevice), "upload weights");
  CK_C(cudaMemcpy(rm, rank_map.data(), r * sizeof(int), cudaMemcpyHostToDevice), "upload rank map");
  if (d->variant == AGK_AGGREGATION_SOURCES && d->num_sources > 0) {
    std::vector<int64_t> hk(d->num_sources);
    for (size_t q = 0; q < d->num_sources; ++q) hk[q] = (int64_t)d->source_k[q];
    CK_C(dalloc(hp, &sk, d->num_sources), "alloc sources");
    CK_C(dalloc(hp, &sr, d->num_sources), "alloc sources");
    CK_C(cudaMemcpy(sk, hk.data(), hk.size() * sizeof(int64_t), cudaMemcpyHostToDevice), "upload sources");
    CK_C(cudaMemcpy(sr, d->source_rate, d->num_sources * sizeof(double), cudaMemcpyHostToDevice), "upload sources");
    h->nsrc = (int)d->num_sources;
  }
  const RhsPlan& p = h->plan;
  double2 *y, *acc;
  CK_C(dalloc(hp, &y, rhs_y_elems(p)), "alloc Y");
  CK_C(dalloc(hp, &acc, rhs_acc_elems(p)), "alloc acc");
  CK_C(dalloc(hp, &partials, rhs_partial_elems(p, h->rf)), "alloc partials");
  CK_C(dalloc(hp, &scalars, (size_t)r + 2 + 4 * (size_t)h->rf), "alloc scalars");

  // twiddle tables: per-size W_N (N = 2..8192) at offset N, plus the two-level W_P tables
  const int64_t P = (int64_t)1 << p.log2p;
  const int s_lo = (p.log2p + 1) / 2;
  const int64_t nlo = (int64_t)1 << s_lo, nhi = P >> s_lo;
  std::vector<double2> tw((size_t)(16384 + nlo + nhi));
  for (int64_t n = 2; n <= 8192; n <<= 1) fill_table(tw, (size_t)n, n);
  {
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int64_t k = 0; k < nlo; ++k) {
      const long double ang = -2.0L * pi * (long double)k / (long double)P;
      tw[16384 + k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    for (int64_t k = 0; k < nhi; ++k) {
      const long double ang = -2.0L * pi * (long double)(k * nlo) / (long double)P;
      tw[16384 + nlo + k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
  }
  if (p.fast) {
    // warp fast path: column-major (U_a, V_a) pairs per unique rank, the n grid buffer and the
    // 32x32 / radix-2 tables
    const int64_t N1 = p.n1, N2 = p.n2, H = N1 / 2;
    double2* uvg;
    double* ng;
    CK_C(dalloc(hp, &uvg, (size_t)h->rf * N2 * H), "alloc UV grid");
    CK_C(dalloc(hp, &ng, (size_t)N2 * H), "alloc n grid");
    std::vector<double2> col((size_t)N2 * H);
    for (int ub = 0; ub < h->rf; ++ub) {
      const int ra = uniq_rank[ub];
      for (int64_t n2 = 0; n2 < N2; ++n2)
        for (int64_t n1 = 0; n1 < H; ++n1) {
          const int64_t i = n1 * N2 + n2;
          col[n2 * H + n1] = i < m ? make_double2(d->u[i * r + ra], d->v[(int64_t)ra * m + i]) : make_double2(0.0, 0.0);
        }
      CK_C(cudaMemcpy(uvg + (size_t)ub * N2 * H, col.data(), col.size() * sizeof(double2), cudaMemcpyHostToDevice),
           "upload UV grid");
    }
    std::vector<double2> t32(2048);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k1 = 0; k1 < 32; ++k1)
      for (int l = 0; l < 32; ++l) {
        const long double ang = -2.0L * pi * (long double)(l * k1) / 1024.0L;
        t32[k1 * 32 + l] = make_double2((double)cosl(ang), (double)sinl(ang));
      }
    for (int rr = 0; rr < 32; ++rr)
      for (int l = 0; l < 32; ++l) {
        const long double ang = -2.0L * pi * (long double)(l + 32 * rr) / 2048.0L;
        t32[1024 + rr * 32 + l] = make_double2((double)cosl(ang), (double)sinl(ang));
      }
    double2* dt32;
    CK_C(dalloc(hp, &dt32, t32.size()), "alloc tables");
    CK_C(cudaMemcpy(dt32, t32.data(), t32.size() * sizeof(double2), cudaMemcpyHostToDevice), "upload tables");
    double* dvec;
    CK_C(dalloc(hp, &dvec, (size_t)m), "alloc D");
    a.dvec = dvec;
    {
      int nsm = 0;
      CK_C(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, hp->device), "SM count");
      h->plan.nsm = nsm;
    }
    a.uvg = uvg;
    a.ng = ng;
    a.tw32 = dt32;
    a.tw2048h = dt32 + 1024;
  }
  CK_C(dalloc(hp, &h->tw_all, tw.size()), "alloc twiddles");
  CK_C(cudaMemcpy(h->tw_all, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice), "upload twiddles");

  a.m = m;
  a.r = r;
  a.rf = h->rf;
  a.ut = ut;
  a.v = vv;
  a.uniq_rank = ur;
  a.uniq_weight = uw;
  a.rank_map = rm;
  a.u0 = u0;
  a.v0 = v0;
  a.flags = model_flags(hp);
  a.lambda = d->shatter_rate;
  a.src_k = sk;
  a.src_rate = sr;
  a.nsrc = h->nsrc;
  a.log2p = p.log2p;
  a.n1 = p.n1;
  a.n2 = p.n2;
  a.y = y;
  a.acc = acc;
  a.partials = partials;
  a.scalars = scalars;
  a.nblk_colfwd = p.small ? 1 : p.n2 / p.c;
  a.tw_n1 = TwTable{h->tw_all + p.n1, ilog2(p.n1)};
  a.tw_n2 = TwTable{h->tw_all + p.n2, ilog2(p.n2)};
  a.tw_small = TwTable{h->tw_all + (p.small ? P : 2), p.small ? p.log2p : 1};
  a.twp = TwoLevel{h->tw_all + 16384 + nlo, h->tw_all + 16384, s_lo};

  CK_C(rhs_set_smem_limits(), "cudaFuncSetAttribute");
  CK_C(cudaStreamSynchronize(hp->stream), "create sync");
#undef CK_C
  *out = h.release();
  return AGK_OK;
}

agk_status agk_rhs_create_fake(int kind, size_t m, double param, int device, agk_rhs** out) {
  if (!out) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (kind <= AGK_RHS_MODEL || kind > AGK_RHS_BURST_NAN) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "unknown fake kind");
  if (m < 1) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "m must be >= 1");
  std::unique_ptr<agk_rhs> h(new agk_rhs());
  agk_status st = select_device(h.get(), device);
  if (st) {
    g_create_error = h->err;
    return st;
  }
  DeviceGuard dg(h->device);
  h->kind = kind;
  h->fake_param = param;
  h->m = (int64_t)m;
  h->r = 0;
  st = alloc_common(h.get());
  if (st) {
    g_create_error = h->err;
    for (void* p : h->allocs) cudaFree(p);
    return st;
  }
  cudaStreamSynchronize(h->stream);
  *out = h.release();
  return AGK_OK;
}

void agk_rhs_destroy(agk_rhs* h) { delete h; }

size_t agk_rhs_size(const agk_rhs* h) { return h ? (size_t)h->m : 0; }
size_t agk_rhs_unique_ranks(const agk_rhs* h) { return h ? (size_t)h->rf : 0; }
uint64_t agk_rhs_evals(const agk_rhs* h) { return h ? h->evals : 0; }
void agk_rhs_reset_evals(agk_rhs* h) {
  if (h) h->evals = 0;
}
int agk_rhs_launches_per_eval(const agk_rhs* h) { return h ? (h->kind == AGK_RHS_MODEL ? h->plan.launches : 1) : 0; }

agk_status agk_rhs_eval(agk_rhs* h, const double* n, double* out, int where) {
  NvtxRange nvtx_("agk_rhs_eval");
  if (!h) return fail(nullptr, AGK_ERR_INVALID_ARGUMENT, "null handle");
  if (h->kind != AGK_RHS_MODEL) {
    DeviceGuard dg(h->device);
    const double* din = n;
    double* dout = out;
    if (where == AGK_MEM_HOST) {
      agk_status st = copy_in(h, n, where, h->d_in);
      if (st) return st;
      din = h->d_in;
      dout = h->d_out;
    }
    CK_H(h, fake_rhs_launch(h->kind, h->fake_param, VecRef{din, nullptr, 0}, dout, h->m, nullptr, h->stream), "fake");
    if (where == AGK_MEM_HOST) {
      agk_status st = copy_out(h, out, where, h->d_out);
      if (st) return st;
    }
    CK_H(h, cudaStreamSynchronize(h->stream), "sync");
    h->evals += 1;
    return AGK_OK;
  }
  agk_status st = run_terms(h, n, out, where, model_flags(h), h->lambda);
  if (st == AGK_OK) h->evals += 1;  // eval_rhs counts one evaluation (rhs.cpp:218)
  return st;
}

agk_status agk_rhs_eval_async(agk_rhs* h, const double* n_dev, double* out_dev) {
  if (!h || h->kind != AGK_RHS_MODEL) return fail(h, AGK_ERR_INVALID_ARGUMENT, "model handle required");
  DeviceGuard dg(h->device);
  RhsArgs a = h->base;
  a.n = VecRef{n_dev, nullptr, 0};
  a.out = out_dev;
  CK_H(h, rhs_launch(h->plan, a, h->stream), "rhs launch");
  h->evals += 1;
  return AGK_OK;
}

agk_status agk_birth_term(agk_rhs* h, const double* n, double* out, int where) {
  return run_terms(h, n, out, where, T_BIRTH, 0.0);
}
agk_status agk_death_term(agk_rhs* h, const double* n, double* out, int where) {
  return run_terms(h, n, out, where, T_DEATH_POS, 0.0);
}
agk_status agk_shattering_terms(agk_rhs* h, const double* n, double lambda, double* out, int where) {
  if (!std::isfinite(lambda) || lambda < 0.0)
    return fail(h, AGK_ERR_INVALID_ARGUMENT, "shattering rate lambda must be finite and >= 0");
  return run_terms(h, n, out, where, T_SHATTER, lambda);
}

agk_status agk_euler_stability_bound(agk_rhs* h, const double* n, double a, double* bound, int where) {
  if (!h || !n || !bound) return fail(h, AGK_ERR_INVALID_ARGUMENT, "null argument");
  if (!(a > 0.0)) return fail(h, AGK_ERR_INVALID_ARGUMENT, "euler bound factor a must be > 0");
  if (h->kind != AGK_RHS_MODEL) return fail(h, AGK_ERR_INVALID_ARGUMENT, "model handle required");
  DeviceGuard dg(h->device);
  const double* din = n;
  if (where == AGK_MEM_HOST) {
    agk_status st = copy_in(h, n, where, h->d_in);
    if (st) return st;
    din = h->d_in;
  }
  CK_H(h, launch_euler_bound(h->base, VecRef{din, nullptr, 0}, a, h->sb.aux, h->sb.naux, h->d_scalar, h->stream),
       "euler bound");
  CK_H(h, cudaMemcpyAsync(bound, h->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, h->stream), "copy");
  CK_H(h, cudaStreamSynchronize(h->stream), "sync");
  return AGK_OK;
}

// One trial loop on the device: agk_advance / agk_rk_step share it (RUN_ADVANCE mode).
static agk_status advance_impl(agk_rhs* h, const double* n, double tau, const agk_control* c, agk_outcome* o,
                               double* state_out, int where, bool store_n5, double* n5_out, double* err_out) {
  DeviceGuard dg(h->device);
  const int body = body_for(c);
  cudaGraphExec_t ex;
  agk_status st = get_graph(h, body, c->stepper, &ex);
  if (st) return st;
  st = copy_in(h, n, where, h->sb.state);
  if (st) return st;
  DevCtl d{};
  control_to_ctl(c, &d);
  d.run_mode = RUN_ADVANCE;
  d.tau_try = tau;
  d.store_n5 = store_n5 ? 1 : 0;
  d.has_model = h->kind == AGK_RHS_MODEL;
  d.cur = 0;
  CK_H(h, cudaMemcpyAsync(h->ctl, &d, sizeof(DevCtl), cudaMemcpyHostToDevice, h->stream), "ctl upload");
  CK_H(h, cudaGraphLaunch(ex, h->stream), "graph launch");
  DevCtl r;
  CK_H(h, cudaMemcpyAsync(&r, h->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, h->stream), "ctl download");
  CK_H(h, cudaStreamSynchronize(h->stream), "advance sync");
  o->tau_used = r.tau_used;
  o->tau_next = r.tau_next;
  o->error_estimate = r.err;
  o->rejects = r.step_rejects;
  o->rhs_evals = r.step_evals;
  o->status = r.status;
  h->evals += r.evals;
  if (state_out && r.status == AGK_STEP_OK) {
    st = copy_out(h, state_out, where, h->sb.state + (int64_t)r.cur * h->m);
    if (st) return st;
  }
  if (n5_out) {
    st = copy_out(h, n5_out, where, h->sb.n5);
    if (st) return st;
  }
  if (err_out) *err_out = r.err;
  CK_H(h, cudaStreamSynchronize(h->stream), "advance sync");
  return AGK_OK;
}

agk_status agk_advance(agk_rhs* h, const double* n, double tau, const agk_control* c, agk_outcome* o,
                       double* state_out, int where) {
  NvtxRange nvtx_("agk_advance");
  if (!h || !n || !c || !o) return fail(h, AGK_ERR_INVALID_ARGUMENT, "null argument");
  if (c->stepper < 0 || c->stepper > 2 || c->mode < 0 || c->mode > 1)
    return fail(h, AGK_ERR_INVALID_ARGUMENT, "unknown stepper or mode");
  if (!(tau > 0.0)) return fail(h, AGK_ERR_INVALID_ARGUMENT, "step size must be > 0");
  return advance_impl(h, n, tau, c, o, state_out, where, false, nullptr, nullptr);
}

agk_status agk_rk_step(agk_rhs* h, int stepper, const double* n, double tau, double* out, double* out5, double* err,
                       int where) {
  NvtxRange nvtx_("agk_rk_step");
  if (!h || !n || !out) return fail(h, AGK_ERR_INVALID_ARGUMENT, "null argument");
  if (stepper < 0 || stepper > 2) return fail(h, AGK_ERR_INVALID_ARGUMENT, "unknown stepper");
  if (!(tau > 0.0)) return fail(h, AGK_ERR_INVALID_ARGUMENT, "step size must be > 0");
  agk_control c;
  agk_control_defaults(&c);
  c.stepper = stepper;
  c.mode = AGK_FIXED;
  c.tau = tau;
  agk_outcome o;
  const bool want5 = stepper == AGK_RKF45 && out5;
  agk_status st = advance_impl(h, n, tau, &c, &o, nullptr, where, want5, want5 ? out5 : nullptr, err);
  if (st) return st;
  // the step's result whatever its finiteness (rk*_step do not check, steppers.hpp:79-80)
  DeviceGuard dg(h->device);
  st = copy_out(h, out, where, h->sb.state + h->m);  // candidate of the first trial (cur was 0)
  if (st) return st;
  CK_H(h, cudaStreamSynchronize(h->stream), "sync");
  return AGK_OK;
}

agk_status agk_run(agk_rhs* h, const agk_run_desc* d, agk_run_report* rep) {
  NvtxRange nvtx_("agk_run");
  if (!h || !d || !rep) return fail(h, AGK_ERR_INVALID_ARGUMENT, "null argument");
  if (h->kind != AGK_RHS_MODEL) return fail(h, AGK_ERR_INVALID_ARGUMENT, "run() drives the model right-hand side");
  // SimulationConfig::validate (simulator.cpp:23-49)
  if (agk_control_validate(&d->control) != AGK_OK) return fail(h, AGK_ERR_INVALID_ARGUMENT, "invalid step control");
  if (!(d->t_end >= 0.0) || !std::isfinite(d->t_end)) return fail(h, AGK_ERR_INVALID_ARGUMENT, "t_end must be finite and >= 0");
  if (d->record == AGK_RECORD_INTERVAL && !(d->record_interval > 0.0))
    return fail(h, AGK_ERR_INVALID_ARGUMENT, "interval recording needs record_interval > 0");
  if (d->record < 0 || d->record > 2) return fail(h, AGK_ERR_INVALID_ARGUMENT, "unknown record mode");
  double prev = -1.0;
  for (size_t q = 0; q < d->num_snapshots; ++q) {
    const double s = d->snapshot_times[q];
    if (!(s >= 0.0) || s > d->t_end) return fail(h, AGK_ERR_INVALID_ARGUMENT, "snapshot times must lie in [0, t_end]");
    if (s <= prev) return fail(h, AGK_ERR_INVALID_ARGUMENT, "snapshot times must be strictly ascending");
    prev = s;
  }
  if (!d->initial) return fail(h, AGK_ERR_INVALID_ARGUMENT, "custom initial state size does not match m");
  if (d->initial_tau < 0.0 || !std::isfinite(d->initial_tau))
    return fail(h, AGK_ERR_INVALID_ARGUMENT, "initial_tau must be finite and >= 0");

  const auto wall0 = std::chrono::steady_clock::now();
  DeviceGuard dg(h->device);
  const int body = body_for(&d->control);
  cudaGraphExec_t ex;
  agk_status st = get_graph(h, body, d->control.stepper, &ex);
  if (st) return st;
  const int64_t m = h->m;
  // per-run device buffers, freed on every return path
  struct TmpBufs {
    std::vector<void*> p;
    ~TmpBufs() {
      for (void* q : p) cudaFree(q);
    }
  } tmp;
  double* snap_times = nullptr;
  double* snap_buf = nullptr;
  if (d->num_snapshots) {
    CK_H(h, cudaMalloc(&snap_times, d->num_snapshots * sizeof(double)), "alloc snapshots");
    tmp.p.push_back(snap_times);
    CK_H(h, cudaMemcpyAsync(snap_times, d->snapshot_times, d->num_snapshots * sizeof(double), cudaMemcpyHostToDevice,
                            h->stream), "upload snapshots");
    if (rep->snapshots) {
      CK_H(h, cudaMalloc(&snap_buf, d->num_snapshots * m * sizeof(double)), "alloc snapshot buffer");
      tmp.p.push_back(snap_buf);
    }
  }
  // records: a device ring of kRing records, drained to the host whenever it fills (the
  // controller then leaves the WHILE loop with `paused`, the graph is relaunched in resume mode)
  constexpr int64_t kRing = 1 << 16;
  const bool want_rec = d->record != AGK_RECORD_NONE && (rep->record_sink || (rep->records && rep->records_capacity));
  if (want_rec && !h->rec_ring) CK_H(h, dalloc(h, &h->rec_ring, (size_t)kRing), "alloc record ring");
  st = copy_in(h, d->initial, AGK_MEM_HOST, h->sb.state);
  if (st) return st;
  DevCtl c{};
  control_to_ctl(&d->control, &c);
  c.run_mode = RUN_LOOP;
  c.t_end = d->t_end;
  c.initial_tau = d->initial_tau;
  c.nsnap = (int)d->num_snapshots;
  c.snap_times = snap_times;
  c.snap_buf = snap_buf;
  c.record = d->record;
  c.record_interval = d->record_interval;
  c.rec_buf = want_rec ? h->rec_ring : nullptr;
  c.rec_cap = want_rec ? kRing : 0;
  c.has_model = 1;
  c.cur = 0;
  CK_H(h, cudaMemcpyAsync(h->ctl, &c, sizeof(DevCtl), cudaMemcpyHostToDevice, h->stream), "ctl upload");
  size_t delivered = 0;  // records handed to the caller so far
  std::vector<agk_record> chunk;
  auto deliver = [&](const agk_record* r, size_t n) {
    if (!n) return;
    if (rep->records) {
      for (size_t q = 0; q < n && delivered + q < rep->records_capacity; ++q) rep->records[delivered + q] = r[q];
    }
    if (rep->record_sink) rep->record_sink(rep->sink_user, r, n);
    delivered += n;
  };
  DevCtl r;
  for (;;) {
    CK_H(h, cudaGraphLaunch(ex, h->stream), "graph launch");
    CK_H(h, cudaMemcpyAsync(&r, h->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, h->stream), "ctl download");
    CK_H(h, cudaStreamSynchronize(h->stream), "run");
    if (want_rec) {
      // drain [rec_drained, nrec) of the ring (one or two contiguous pieces)
      const long long from = r.rec_drained, to = r.nrec;
      chunk.resize((size_t)(to - from));
      for (long long q = from; q < to;) {
        const long long slot = q % kRing, n = std::min<long long>(to - q, kRing - slot);
        CK_H(h, cudaMemcpyAsync(chunk.data() + (q - from), h->rec_ring + slot, (size_t)n * sizeof(agk_record),
                                cudaMemcpyDeviceToHost, h->stream), "copy records");
        q += n;
      }
      CK_H(h, cudaStreamSynchronize(h->stream), "copy records");
      deliver(chunk.data(), chunk.size());
    }
    if (!r.paused) break;
    // resume: the loop state stays on the device; only the drain mark and the resume flag change
    const long long drained = r.nrec;
    const int one = 1;
    CK_H(h, cudaMemcpyAsync(&h->ctl->rec_drained, &drained, sizeof(drained), cudaMemcpyHostToDevice, h->stream),
         "ctl update");
    CK_H(h, cudaMemcpyAsync(&h->ctl->resume, &one, sizeof(one), cudaMemcpyHostToDevice, h->stream), "ctl update");
  }
  rep->termination = r.status == AGK_STEP_OK ? 0 : 1;
  rep->abort_status = r.status;
  rep->abort_t = rep->termination ? r.abort_t : 0.0;
  rep->abort_tau = rep->termination ? r.abort_tau : 0.0;
  rep->final_t = r.t;
  rep->total_rhs_evals = r.evals;
  rep->total_accepted = r.accepted;
  rep->total_rejects = r.rejects_total;
  if (rep->final_state)
    CK_H(h, cudaMemcpyAsync(rep->final_state, h->sb.state + (int64_t)r.cur * m, m * sizeof(double),
                            cudaMemcpyDeviceToHost, h->stream), "copy final state");
  rep->num_snapshots_taken = (size_t)r.snap_idx;
  if (snap_buf && r.snap_idx > 0)
    CK_H(h, cudaMemcpyAsync(rep->snapshots, snap_buf, (size_t)r.snap_idx * m * sizeof(double), cudaMemcpyDeviceToHost,
                            h->stream), "copy snapshots");
  CK_H(h, cudaStreamSynchronize(h->stream), "run copy-out");
  size_t nrec = (size_t)r.nrec;
  // closing record (simulator.cpp:219-222): when the run completed and the last record is not at t
  if (d->record != AGK_RECORD_NONE && rep->termination == 0 && (nrec == 0 || r.last_rec_t < r.t)) {
    agk_record x{};
    x.t = r.t;
    x.tau = 0.0;
    x.density = r.mom[0];
    x.mass = r.mom[1];
    x.m2 = r.mom[2];
    x.error_estimate = NAN;
    x.rhs_evals = r.evals;
    x.rejects = r.rejects_total;
    if (want_rec) deliver(&x, 1);
    nrec += 1;
  }
  rep->num_records = nrec;
  h->evals += r.evals;
  rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  return AGK_OK;
}

agk_status agk_rhs_eval_timed(agk_rhs* h, const double* n_dev, double* out_dev, int count, float* elapsed_ms) {
  if (!h || h->kind != AGK_RHS_MODEL || count < 1) return fail(h, AGK_ERR_INVALID_ARGUMENT, "bad timing request");
  DeviceGuard dg(h->device);
  // back-to-back evaluations (BASELINE config 4 runs 1000 of them): one graph holds kTimedBatch
  // chained evaluations, so consecutive evaluations are joined by programmatic dependent launch
  // like the RHS evaluations inside a stepping graph, not by a graph-launch boundary
  constexpr int kTimedBatch = 10;
  if (h->rhs_graph && (h->rhs_graph_in != n_dev || h->rhs_graph_out != out_dev)) {
    cudaGraphExecDestroy(h->rhs_graph);
    h->rhs_graph = nullptr;
    if (h->rhs_graph_b) cudaGraphExecDestroy(h->rhs_graph_b);
    h->rhs_graph_b = nullptr;
  }
  if (!h->rhs_graph) {
    h->rhs_graph_in = n_dev;
    h->rhs_graph_out = out_dev;
    RhsArgs a = h->base;
    a.n = VecRef{n_dev, nullptr, 0};
    a.out = out_dev;
    for (int b = 0; b < 2; ++b) {
      cudaGraph_t g;
      CK_H(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal), "capture");
      cudaError_t e = cudaSuccess;
      for (int q = 0; q < (b ? kTimedBatch : 1) && e == cudaSuccess; ++q) e = rhs_launch(h->plan, a, h->stream);
      cudaError_t e2 = cudaStreamEndCapture(h->stream, &g);
      if (e != cudaSuccess) return cuda_fail(h, e, "capture rhs");
      if (e2 != cudaSuccess) return cuda_fail(h, e2, "capture end");
      CK_H(h, cudaGraphInstantiate(b ? &h->rhs_graph_b : &h->rhs_graph, g, 0), "instantiate");
      cudaGraphDestroy(g);
    }
  }
  CK_H(h, cudaEventRecord(h->ev0, h->stream), "event");
  for (int q = 0; q < count / kTimedBatch; ++q) CK_H(h, cudaGraphLaunch(h->rhs_graph_b, h->stream), "graph launch");
  for (int q = 0; q < count % kTimedBatch; ++q) CK_H(h, cudaGraphLaunch(h->rhs_graph, h->stream), "graph launch");
  CK_H(h, cudaEventRecord(h->ev1, h->stream), "event");
  CK_H(h, cudaEventSynchronize(h->ev1), "event sync");
  CK_H(h, cudaEventElapsedTime(elapsed_ms, h->ev0, h->ev1), "elapsed");
  h->evals += (uint64_t)count;
  return AGK_OK;
}

agk_status agk_rhs_profile(agk_rhs* h, const double* n_dev, double* out_dev, int reps, double* ms, int* cls, int cap,
                           int* n, int* plan4) {
  if (!h || h->kind != AGK_RHS_MODEL || reps < 1 || cap < 1) return fail(h, AGK_ERR_INVALID_ARGUMENT, "bad profile request");
  DeviceGuard dg(h->device);
  std::vector<cudaEvent_t> ev(cap + 1);
  for (auto& e : ev) CK_H(h, cudaEventCreate(&e), "event");
  std::vector<double> acc(cap, 0.0);
  int nk = 0;
  RhsArgs a = h->base;
  a.n = VecRef{n_dev, nullptr, 0};
  a.out = out_dev;
  for (int q = 0; q < reps; ++q) {
    CK_H(h, cudaEventRecord(ev[0], h->stream), "event");
    CK_H(h, rhs_launch_marked(h->plan, a, h->stream, ev.data() + 1, cls, cap, &nk), "rhs launch");
    CK_H(h, cudaStreamSynchronize(h->stream), "sync");
    for (int k = 0; k < nk; ++k) {
      float t = 0.f;
      CK_H(h, cudaEventElapsedTime(&t, ev[k], ev[k + 1]), "elapsed");
      acc[k] += t;
    }
  }
  for (int k = 0; k < nk; ++k) ms[k] = acc[k] / reps;
  *n = nk;
  if (plan4) {
    plan4[0] = h->plan.log2p;
    plan4[1] = h->plan.small ? 0 : h->plan.n1;
    plan4[2] = h->plan.small ? 0 : h->plan.n2;
    plan4[3] = h->plan.gsize;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  h->evals += (uint64_t)reps;
  return AGK_OK;
}

}  // extern "C"
