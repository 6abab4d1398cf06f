// tracker.cu -- the C-ABI (include/pathtrack_b200.h): plan compilation,
// engine choice, launches.  The kernels live in kernels.cuh and are
// instantiated per precision in kern_{d,dd,qd}.cu; they are launched here
// through the KernelSet tables.  There is no host fallback: every compute
// entry point needs an sm_100 device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "work.hpp"

using namespace ptdev;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define PT_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return fail(PT_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

inline int limbs(pt_prec p) { return p == PT_D ? 1 : (p == PT_DD ? 2 : 4); }
inline const KernelSet& kset(pt_prec p) { return p == PT_D ? kset_d : (p == PT_DD ? kset_dd : kset_qd); }
// kernels that follow the reference's non-finite rules exactly: the DD set
// differs (kset_dd skips dd_norm's non-finite select); D and QD are exact as is
inline const KernelSet& kset_exact(pt_prec p) { return p == PT_DD ? kset_dd_exact : kset(p); }
inline const KernelSet& kset_mode(pt_prec p, int arith) { return (p == PT_QD && arith == 1) ? kset_qd_fast : kset_exact(p); }

// Launch a kernel (as a cluster of `cluster` CTAs when cluster > 0) from its
// untyped pointer.
cudaError_t launch_ex(const void* fn, int grid, size_t smem, cudaStream_t s, int cluster, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cluster > 0 ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace

// ---------------------------------------------------------------------------
// plan object
// ---------------------------------------------------------------------------
struct pt_plan {
  int device = 0;
  pt_prec prec = PT_DD;
  int L = 2;
  int n = 0, N = 0, M = 0;
  long n_ctr = 0;
  cudaStream_t stream = nullptr;
  DevPlan dp{};
  Layout lay{};
  void* dtables = nullptr;  // plan tables
  double* dwork = nullptr;  // single-path workspace (slice 0)
  unsigned long long* uwork = nullptr;
  int grid_blocks = 1;
  size_t grid_dyn_smem = 0;   // dynamic smem of k_track_grid / k_eval
  int grid_warp = 0, cluster_warp = 0, batch_warp = 0;  // warp-per-column MGS per engine
  const ptplan::SlotTask* tasks_b = nullptr;            // batch partition of the slot tasks
  int class_beg_b[6] = {0, 0, 0, 0, 0, 0};
  // batch bundles over lane-interleaved contribution streams (plan.hpp Bundle)
  const ptplan::Bundle* bundles = nullptr;
  int n_bundles = 0;
  const int32_t* splits = nullptr;
  int n_splits = 0, scratch_units = 0;
  const ptplan::SlotTask* btasks = nullptr;
  const int32_t* s_ws = nullptr;
  const double* s_coef = nullptr;
  long s_len = 0;
  int s_hi = 0;
  int arith = 0;              // PT_ARITH_REFERENCE / PT_ARITH_FAST (QD only)
  int engine = 0;             // 0 grid, 1 cluster (single path)
  int cluster_size = 0;       // CTAs of the cluster engine (0: unavailable)
  size_t cluster_dyn_smem = 0;
  size_t batch_dyn_smem = 0;  // dynamic smem of k_track_batch
  int batch_mgs = 0;          // k_track_batch runs mgs_batch (N <= kBmMaxN)
  int batch_mgs_smem = 0;     // the batch's MGS stages its columns in the dynamic smem
  // staging for the host-buffer API
  double* d_start = nullptr;
  double* d_end = nullptr;
  pt_path_stats* d_stats = nullptr;
  pt_trace_event* d_trace = nullptr;
  int* d_trace_len = nullptr;
  int trace_cap = 0;
  // batch
  double* bwork = nullptr;
  unsigned long long* bu = nullptr;
  int batch_blocks = 0;
  unsigned long long* d_queue = nullptr;
  double* b_starts = nullptr;
  double* b_ends = nullptr;
  pt_path_stats* b_stats = nullptr;
  long b_cap = 0;
  unsigned long long launches = 0;
  ptwork::OpCount w_eval, w_solve;
};

namespace {


// the plan's tracking kernels, and those that follow the reference's
// non-finite rules (the DD re-track set; the same set otherwise)
inline const KernelSet& tset(const pt_plan* p) { return p->arith ? kset_qd_fast : kset(p->prec); }
inline const KernelSet& tset_exact(const pt_plan* p) { return p->arith ? kset_qd_fast : kset_exact(p->prec); }

int occupancy_blocks(const void* fn, int device, int* per_sm, int* sms) {
  cudaDeviceProp prop;
  PT_CUDA(cudaGetDeviceProperties(&prop, device));
  *sms = prop.multiProcessorCount;
  PT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, kThreads, 0));
  return PT_OK;
}

int check_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(PT_E_NODEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
  if (device < 0 || device >= count) return fail(PT_E_NODEVICE, "device index out of range");
  cudaDeviceProp prop;
  PT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return fail(PT_E_NODEVICE, "device is not sm_100 class");
  return PT_OK;
}

constexpr size_t kSmemBudget = 200 * 1024;  // dynamic smem ceiling per CTA (227 KB minus static)

// bytes of owned MGS columns per CTA, 0 when they do not fit (global fallback)
size_t mgs_smem_bytes(int L, int N, int n, int nblocks) {
  const int cols = (n + 1 + nblocks - 1) / nblocks;
  const size_t bytes = mgs_stage_doubles(L, N, n, cols) * 8;
  return bytes <= kSmemBudget ? bytes : 0;
}

// MGS variant of an engine with `nblocks` CTAs (DevPlan::mgs_warp) and its
// dynamic shared memory:
//   2  warp-per-column MGS, q_k pushed by st.async into every consuming CTA
//      (cluster / block teams; needs the whole Q buffer in shared memory);
//   1  warp-per-column MGS, q_k through shared memory / DSMEM / L2 + flags;
//   0  group MGS of device.cuh (any N up to 1024).
// QD keeps the group MGS: its column chain is issue bound, and groups of
// 2+ warps put one element per thread on it.  PT_MGS_WARP=<0|1|2> caps it.
size_t engine_smem(int L, int N, int n, int nblocks, bool cluster_or_block, int* warp, int cap_default = 2) {
  const char* e = getenv("PT_MGS_WARP");
  int cap = e ? atoi(e) : (L == 4 ? 0 : cap_default);
  if (!cluster_or_block) cap = std::min(cap, 1);
  *warp = 0;
  if (N <= kWarpMgsMaxN) {
    if (cap >= 2 && mgs_warp_bytes(L, N, n, nblocks, true) <= kSmemBudget) *warp = 2;
    else if (cap >= 1 && mgs_warp_bytes(L, N, n, nblocks, false) <= kSmemBudget) *warp = 1;
  }
  return *warp ? mgs_warp_bytes(L, N, n, nblocks, *warp == 2) : mgs_smem_bytes(L, N, n, nblocks);
}
// Default block: 8 columns per CTA block in D (chandra-64 D 2.58 vs 2.63 ms
// per path with 4), 4 in DD / QD (chandra-64 DD 11.84 vs 11.97 ms with 8;
// deterministic build, same box, twice: DESIGN.md §5.1).
int warp_mgs_block(int L) {
  const int def = L == 1 ? 8 : 4;
  const char* e = getenv("PT_MGS_B");
  const int b = e ? atoi(e) : def;
  return (b == 1 || b == 2 || b == 4 || b == 8) ? b : def;
}

int set_dyn_smem(const void* fn, size_t bytes) {
  PT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(bytes, 1)));
  return PT_OK;
}

int dispatch_grid_size(pt_plan* p) {
  const void* fn = kset(p->prec).track_grid;
  int per_sm = 0, sms = 0;
  int rc = occupancy_blocks(fn, p->device, &per_sm, &sms);
  if (rc) return rc;
  const int cap = std::max(1, per_sm) * sms;
  // enough CTAs that each phase has about one unit of work per warp / group
  const long ntasks = p->dp.class_beg[5];
  const int gpc_mgs = kWarps / p->dp.mgs_gw;
  long want = 1;
  want = std::max(want, (long)(p->M + kThreads - 1) / kThreads);
  want = std::max(want, (ntasks + kWarps - 1) / kWarps);
  want = std::max(want, (long)(p->n + 1 + gpc_mgs - 1) / gpc_mgs);
  // cap = resident CTAs without dynamic smem (kGridCtasPerSm per SM); the
  // cooperative launch needs every CTA resident WITH the MGS staging, so the
  // grid shrinks until the occupancy at that staging size covers it
  p->grid_blocks = (int)std::min<long>(want, cap);
  for (int round = 0;; ++round) {
    p->grid_dyn_smem = engine_smem(p->L, p->N, p->n, p->grid_blocks, false, &p->grid_warp);
    for (const void* f : {fn, kset_exact(p->prec).eval}) {
      rc = set_dyn_smem(f, p->grid_dyn_smem);
      if (rc) return rc;
    }
    int per_sm2 = 0;
    PT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, fn, kThreads, p->grid_dyn_smem));
    if (per_sm2 < 1) return fail(PT_E_INVAL, "tracker CTA does not fit on an SM");
    if (per_sm2 * sms >= p->grid_blocks) return PT_OK;
    if (round >= 4) return fail(PT_E_INVAL, "grid engine: no co-resident grid size found");
    p->grid_blocks = per_sm2 * sms;
  }
}

// Largest cluster (<= 16 CTAs) the device can schedule for this kernel with
// the MGS columns staged in shared memory.
int setup_cluster(pt_plan* p) {
  const void* fn = kset(p->prec).track_cluster;
  PT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  PT_CUDA(cudaFuncSetAttribute(kset_exact(p->prec).track_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  p->cluster_size = 0;
  const char* ce = getenv("PT_CLUSTER_MAX");  // tuning knob: cap the cluster size
  const int cmax = ce ? atoi(ce) : 16;
  for (int c : {16, 8, 4, 2, 1}) {
    if (c > cmax) continue;
    int warp = 0;
    const size_t dyn = engine_smem(p->L, p->N, p->n, c, true, &warp);
    if (dyn == 0) continue;
    if (set_dyn_smem(fn, dyn)) return PT_E_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters >= 1) {
      p->cluster_size = c;
      p->cluster_dyn_smem = dyn;
      p->cluster_warp = warp;
      break;
    }
    cudaGetLastError();
  }
  // engine choice: systems whose MGS fits one cluster and whose evaluation is
  // small enough that 16 SMs do not starve it run on the cluster engine
  const double contributions = (double)p->n_ctr;
  // QD always takes the grid: its column chain is QD-latency bound either way
  // and the grid engine measured 6-14 % faster (chandra-64 QD 233 vs 255 ms,
  // fast 74 vs 86 ms; cyclic-16 QD 796 vs 848 ms) -- D / DD keep the cluster
  p->engine = (p->cluster_size >= 8 && p->n <= 192 && contributions <= 2e5 && p->prec != PT_QD) ? 1 : 0;
  const char* ee = getenv("PT_ENGINE");  // tuning knob: 0 grid, 1 cluster
  if (ee && (ee[0] == '0' || (ee[0] == '1' && p->cluster_size > 0))) p->engine = ee[0] - '0';
  return PT_OK;
}

template <class T>
T* dev_alloc(size_t count, int* rc) {
  T* ptr = nullptr;
  cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    *rc = fail(PT_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return nullptr;
  }
  return ptr;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    return fail(PT_E_INVAL, e.what());
  }
}

// the warp back substitution can stage R in the engine's dynamic smem
int stage_fits(const pt_plan* p, size_t dyn_bytes) {
  const char* e = getenv("PT_BS_SMEM");  // tuning knob: 0 reads R from L2 in the back substitution
  if (e && e[0] == '0') return 0;
  return backsub_stage_doubles(p->L, p->n) * 8 <= dyn_bytes ? 1 : 0;
}
// the monomial evaluation can read x from a shared-memory copy
int x_fits(const pt_plan* p, size_t dyn_bytes) { return (size_t)2 * p->L * p->n * 8 <= dyn_bytes ? 1 : 0; }

// One single-path launch of kernel set `ks` on the plan's engine.
void launch_engine(pt_plan* p, const KernelSet& ks, const pt_step_params& sp, const TrackIO& io, cudaStream_t s,
                   cudaError_t* err) {
  Work W = carve(p->dwork, p->uwork, p->lay, 0);
  unsigned long long epoch = (++p->launches) << 40;
  // barrier / abort / rank words start clean on every launch (a watchdog
  // abort of an earlier launch must not poison this one)
  *err = cudaMemsetAsync(W.ctl, 0, CTL_WORDS * sizeof(unsigned long long), s);
  if (*err != cudaSuccess) return;
  // the max-dynamic-smem attribute belongs to the kernel function, not to the
  // plan: set this plan's value right before its launch (another live plan
  // of the same precision may have lowered it since)
  const void* fn = p->engine == 1 ? ks.track_cluster : ks.track_grid;
  *err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)std::max<size_t>(p->engine == 1 ? p->cluster_dyn_smem : p->grid_dyn_smem, 1));
  if (*err != cudaSuccess) return;
  pt_step_params spc = sp;
  TrackIO ioc = io;
  if (p->engine == 1) {
    DevPlan dp = p->dp;
    dp.mgs_smem = p->cluster_dyn_smem > 0;
    dp.dyn_smem = dp.mgs_smem;
    dp.mgs_warp = p->cluster_warp;
    dp.bs_smem = stage_fits(p, p->cluster_dyn_smem);
    dp.x_smem = x_fits(p, p->cluster_dyn_smem);
    void* args[] = {&dp, &W, &spc, &ioc, &epoch};
    *err = launch_ex(fn, p->cluster_size, p->cluster_dyn_smem, s, p->cluster_size, args);
    return;
  }
  DevPlan dp = p->dp;
  dp.mgs_smem = p->grid_dyn_smem > 0;
  dp.dyn_smem = dp.mgs_smem;
  dp.mgs_warp = p->grid_warp;
  dp.bs_smem = stage_fits(p, p->grid_dyn_smem);
  dp.x_smem = x_fits(p, p->grid_dyn_smem);
  void* args[] = {&dp, &W, &spc, &ioc, &epoch};
  *err = cudaLaunchCooperativeKernel(fn, dim3(p->grid_blocks), dim3(kThreads), args, p->grid_dyn_smem, s);
}

// track_path on the device: the fast kernels, then (DD) the exact re-track
// launch, which exits at once unless the fast run flagged PT_STAT_NONFINITE.
void launch_grid(pt_plan* p, const pt_step_params& sp, const TrackIO& io, cudaStream_t s, cudaError_t* err) {
  launch_engine(p, tset(p), sp, io, s, err);
  if (*err != cudaSuccess || &tset_exact(p) == &tset(p)) return;
  TrackIO re = io;
  re.retrack = 1;
  launch_engine(p, tset_exact(p), sp, re, s, err);
}

int validate_params(const pt_step_params* sp) {
  if (!sp) return fail(PT_E_INVAL, "null step params");
  if (sp->pred_degree < 0 || sp->pred_degree > kMaxDegree) return fail(PT_E_INVAL, "pred_degree must be 0..8");
  if (sp->newton_max_iter < 1) return fail(PT_E_INVAL, "newton_max_iter must be >= 1");
  if (!(sp->min_step > 0.0) || !(sp->max_step >= sp->min_step) || !(sp->max_step <= 1.0))
    return fail(PT_E_INVAL, "need 0 < min_step <= max_step <= 1");
  if (sp->max_steps < 0) return fail(PT_E_INVAL, "max_steps must be >= 0");
  return PT_OK;
}

int read_abort(pt_plan* p, unsigned long long* ctl) {
  unsigned long long h[CTL_WORDS];
  PT_CUDA(cudaMemcpy(h, ctl, sizeof h, cudaMemcpyDeviceToHost));
  if (h[CTL_ABORT]) {
    // reset barrier state so the plan stays usable
    PT_CUDA(cudaMemset(ctl, 0, sizeof h));
    return fail(PT_E_TIMEOUT, "device watchdog fired (grid barrier or MGS flag stalled)");
  }
  return PT_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* pt_last_error(void) { return g_err.c_str(); }
const char* pt_version(void) { return "pathtrack_b200 0.1 (sm_100a)"; }

int pt_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int pt_default_params(pt_prec prec, pt_step_params* out) {
  if (!out) return PT_E_INVAL;
  out->max_step = 0.1;
  out->min_step = 1e-6;
  out->max_steps = prec == PT_QD ? 1500 : 500;
  out->pred_degree = 4;
  out->newton_max_iter = 6;
  out->reserved = 0;
  out->newton_tol = prec == PT_D ? 1e-8 : (prec == PT_DD ? 1e-20 : 1e-44);
  return PT_OK;
}

int pt_plan_create(int device, pt_prec prec, const pt_system_desc* g, const pt_system_desc* f,
                   const double* gamma, int32_t relax_k, pt_plan** out) {
  return guarded([&]() -> int {
    if (!out || !gamma || relax_k < 1) return fail(PT_E_INVAL, "bad plan arguments");
    if (prec != PT_D && prec != PT_DD && prec != PT_QD) return fail(PT_E_INVAL, "bad precision");
    int rc = check_device(device);
    if (rc) return rc;
    const int L = limbs(prec);
    ptplan::HostPlan hp = ptplan::compile(g, f, L);
    if (hp.n > kMaxRowsPerThread * kThreads) return fail(PT_E_INVAL, "n_vars > 512 not supported");
    if (hp.N > kMaxElems * 256) return fail(PT_E_INVAL, "n_eqs > 1024 not supported");
    PT_CUDA(cudaSetDevice(device));
    auto p = std::make_unique<pt_plan>();
    p->device = device;
    p->prec = prec;
    p->L = L;
    p->n = hp.n;
    p->N = hp.N;
    p->M = (int)hp.mono_size.size();
    p->n_ctr = (long)hp.ctr_coef.size();
    p->w_eval = ptwork::eval_work(hp, relax_k);
    p->w_solve = ptwork::solve_work(hp.N, hp.n);
    PT_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    // tables: one allocation, 256-byte aligned pieces
    std::vector<std::pair<const void*, size_t>> pieces = {
        {hp.mono_size.data(), hp.mono_size.size() * 4}, {hp.mono_vbeg.data(), hp.mono_vbeg.size() * 4},
        {hp.mono_out.data(), hp.mono_out.size() * 4},   {hp.mono_flags.data(), hp.mono_flags.size() * 4},
        {hp.mono_var.data(), hp.mono_var.size() * 4},   {hp.mono_exp.data(), hp.mono_exp.size() * 4},
        {hp.tasks.data(), hp.tasks.size() * sizeof(ptplan::SlotTask)},
        {hp.ctr_coef.data(), hp.ctr_coef.size() * 4},   {hp.ctr_ws.data(), hp.ctr_ws.size() * 4},
        {hp.coef.data(), hp.coef.size() * 8},           {gamma, (size_t)2 * L * 8},
        {hp.tasks_b.data(), hp.tasks_b.size() * sizeof(ptplan::SlotTask)},
        {hp.bundles.data(), hp.bundles.size() * sizeof(ptplan::Bundle)},
        {hp.btasks.data(), hp.btasks.size() * sizeof(ptplan::SlotTask)},
        {hp.s_ws.data(), hp.s_ws.size() * 4},
        {hp.s_coef.data(), hp.s_coef.size() * 8},
        {hp.splits.data(), hp.splits.size() * 4}};
    size_t total = 0;
    std::vector<size_t> offs;
    for (auto& pc : pieces) {
      offs.push_back(total);
      total += (pc.second + 255) & ~(size_t)255;
    }
    rc = 0;
    char* base = dev_alloc<char>(total, &rc);
    if (rc) return rc;
    p->dtables = base;
    for (size_t q = 0; q < pieces.size(); ++q)
      if (pieces[q].second) PT_CUDA(cudaMemcpy(base + offs[q], pieces[q].first, pieces[q].second, cudaMemcpyHostToDevice));
    DevPlan& dp = p->dp;
    dp.n = hp.n;
    dp.N = hp.N;
    dp.M = p->M;
    dp.mono_long = 0;  // device order is size-descending: count the long ones
    const int split = prec == PT_QD ? kMonoSplit<qd> : kMonoSplit<dd>;
    while (dp.mono_long < p->M && hp.mono_size[dp.mono_long] >= split) ++dp.mono_long;
    dp.P_mgs = ptplan::width_mgs(hp.N);
    dp.mgs_gw = ptplan::mgs_group_warps(hp.N);
    dp.mgs_B = warp_mgs_block(p->L);
    dp.mono_size = (const int32_t*)(base + offs[0]);
    dp.mono_vbeg = (const int32_t*)(base + offs[1]);
    dp.mono_out = (const int32_t*)(base + offs[2]);
    dp.mono_flags = (const int32_t*)(base + offs[3]);
    dp.mono_var = (const int32_t*)(base + offs[4]);
    dp.mono_exp = (const int32_t*)(base + offs[5]);
    dp.ws_len = hp.ws_len;
    dp.tasks = (const ptplan::SlotTask*)(base + offs[6]);
    for (int c = 0; c < 6; ++c) dp.class_beg[c] = hp.class_beg[c];
    p->tasks_b = (const ptplan::SlotTask*)(base + offs[11]);
    for (int c = 0; c < 6; ++c) p->class_beg_b[c] = hp.class_beg_b[c];
    if (!hp.bundles.empty()) {
      p->bundles = (const ptplan::Bundle*)(base + offs[12]);
      p->n_bundles = (int)hp.bundles.size();
      p->splits = (const int32_t*)(base + offs[16]);
      p->n_splits = (int)(hp.splits.size() / 4);
      p->scratch_units = hp.scratch_units;
      p->btasks = (const ptplan::SlotTask*)(base + offs[13]);
      p->s_ws = (const int32_t*)(base + offs[14]);
      p->s_coef = (const double*)(base + offs[15]);
      p->s_len = (long)hp.s_len;
      p->s_hi = hp.s_hi;
    }
    dp.ctr_coef = (const int32_t*)(base + offs[7]);
    dp.ctr_ws = (const int32_t*)(base + offs[8]);
    dp.coef = (const double*)(base + offs[9]);
    dp.n_coef = hp.n_coef;
    dp.gamma = (const double*)(base + offs[10]);
    dp.relax_k = relax_k;
    // single-path workspace
    p->lay = make_layout(L, hp.n, hp.N, hp.ws_len);
    p->dwork = dev_alloc<double>(p->lay.dslice, &rc);
    if (rc) return rc;
    p->uwork = dev_alloc<unsigned long long>(p->lay.uslice, &rc);
    if (rc) return rc;
    PT_CUDA(cudaMemset(p->dwork, 0, p->lay.dslice * 8));
    PT_CUDA(cudaMemset(p->uwork, 0, p->lay.uslice * 8));
    const size_t vec = (size_t)2 * L * hp.n;
    p->d_start = dev_alloc<double>(vec, &rc);
    if (rc) return rc;
    p->d_end = dev_alloc<double>(vec, &rc);
    if (rc) return rc;
    p->d_stats = dev_alloc<pt_path_stats>(1, &rc);
    if (rc) return rc;
    p->d_trace_len = dev_alloc<int>(1, &rc);
    if (rc) return rc;
    rc = dispatch_grid_size(p.get());
    if (rc) return rc;
    rc = setup_cluster(p.get());
    if (rc) return rc;
    *out = p.release();
    return PT_OK;
  });
}

void pt_plan_destroy(pt_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  for (void* q : {(void*)p->dtables, (void*)p->dwork, (void*)p->uwork, (void*)p->d_start, (void*)p->d_end,
                  (void*)p->d_stats, (void*)p->d_trace, (void*)p->d_trace_len, (void*)p->bwork, (void*)p->bu,
                  (void*)p->d_queue, (void*)p->b_starts, (void*)p->b_ends, (void*)p->b_stats})
    if (q) cudaFree(q);
  if (p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

int64_t pt_plan_info(const pt_plan* p, int32_t what) {
  if (!p) return -1;
  switch (what) {
    case 0: return p->n;
    case 1: return p->N;
    case 2: return p->M;
    case 3: return p->n_ctr;
    case 4: return p->grid_blocks;
    case 5: return p->prec;
    case 6: return p->batch_blocks;
    case 7: return p->dp.ws_len;
    case 8: return p->engine;
    case 9: return p->cluster_size;
  }
  return -1;
}

int pt_plan_set_engine(pt_plan* p, int32_t engine) {
  if (!p || engine < 0 || engine > 1) return fail(PT_E_INVAL, "engine must be 0 (grid) or 1 (cluster)");
  if (engine == 1 && p->cluster_size == 0) return fail(PT_E_INVAL, "no schedulable cluster for this plan");
  p->engine = engine;
  return PT_OK;
}

int pt_plan_set_arith(pt_plan* p, int32_t arith) {
  if (!p || (arith != PT_ARITH_REFERENCE && arith != PT_ARITH_FAST)) return fail(PT_E_INVAL, "bad arithmetic");
  if (arith == PT_ARITH_FAST && p->prec != PT_QD) return fail(PT_E_INVAL, "PT_ARITH_FAST exists for QD plans only");
  if (arith == PT_ARITH_FAST)  // the fast set is launched with the reference set's geometry
    PT_CUDA(cudaFuncSetAttribute(kset_qd_fast.track_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  p->arith = arith;
  return PT_OK;
}

int pt_plan_work(const pt_plan* p, int32_t kind, int32_t degree, double* out) {
  if (!p || !out || kind < 0 || kind > 2 || degree < 0) return PT_E_INVAL;
  const ptwork::OpCount o = kind == 0 ? p->w_eval : kind == 1 ? p->w_solve : ptwork::predict_work(p->n, degree);
  out[0] = o.radd;
  out[1] = o.rmul;
  out[2] = o.rdiv;
  out[3] = o.rsqrt;
  out[4] = o.hypot;
  out[5] = ptwork::fp64_instructions(o, p->L);
  return PT_OK;
}

int pt_fp64_peak(int device, double* instr_per_s, double* ms_out) {
  if (!instr_per_s) return PT_E_INVAL;
  int rc = check_device(device);
  if (rc) return rc;
  PT_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  PT_CUDA(cudaGetDeviceProperties(&prop, device));
  const int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 4096;
  double* d = dev_alloc<double>((size_t)blocks * threads, &rc);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  PT_CUDA(cudaEventCreate(&e0));
  PT_CUDA(cudaEventCreate(&e1));
  int it = iters;
  void* args[] = {&d, &it};
  PT_CUDA(cudaLaunchKernel(kmisc.fp64_peak, dim3(blocks), dim3(threads), args, 0, 0));  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    PT_CUDA(cudaEventRecord(e0));
    PT_CUDA(cudaLaunchKernel(kmisc.fp64_peak, dim3(blocks), dim3(threads), args, 0, 0));
    PT_CUDA(cudaEventRecord(e1));
    PT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    PT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  *instr_per_s = (double)blocks * threads * iters * kPeakChains / (best * 1e-3);
  if (ms_out) *ms_out = best;
  return PT_OK;
}

int pt_plan_profile(pt_plan* p, double* out, int32_t reset) {
  if (!p || !out) return PT_E_INVAL;
  PT_CUDA(cudaSetDevice(p->device));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  unsigned long long* prof = carve(p->dwork, p->uwork, p->lay, 0).prof;
  unsigned long long h[kProfSlots];
  PT_CUDA(cudaMemcpy(h, prof, sizeof h, cudaMemcpyDeviceToHost));
  for (int i = 0; i < kProfSlots; ++i) out[i] = (double)h[i];
  if (reset) PT_CUDA(cudaMemset(prof, 0, sizeof h));
  return PT_OK;
}

int pt_plan_batch_profile(pt_plan* p, int32_t slice, double* out, int32_t reset) {
  if (!p || !out || slice < 0) return PT_E_INVAL;
  if (!p->bu || slice >= p->batch_blocks) return fail(PT_E_INVAL, "no such batch workspace slice");
  PT_CUDA(cudaSetDevice(p->device));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  unsigned long long* prof = carve(p->bwork, p->bu, p->lay, slice).prof;
  unsigned long long h[kProfSlots];
  PT_CUDA(cudaMemcpy(h, prof, sizeof h, cudaMemcpyDeviceToHost));
  for (int i = 0; i < kProfSlots; ++i) out[i] = (double)h[i];
  if (reset) PT_CUDA(cudaMemset(prof, 0, sizeof h));
  return PT_OK;
}

int pt_microbench(int device, int32_t what, double* out) {
  if (!out) return PT_E_INVAL;
  int rc = check_device(device);
  if (rc) return rc;
  PT_CUDA(cudaSetDevice(device));
  double* d = dev_alloc<double>(32, &rc);
  unsigned long long* u = dev_alloc<unsigned long long>(64, &rc);
  if (rc) return rc;
  PT_CUDA(cudaMemset(d, 0, 32 * 8));
  PT_CUDA(cudaMemset(u, 0, 64 * 8));
  cudaDeviceProp prop;
  PT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (what == 0) {
    double seed = 1.25;
    void* args[] = {&d, &seed};
    PT_CUDA(cudaLaunchKernel(kmisc.latency, dim3(1), dim3(1), args, 0, 0));
    PT_CUDA(cudaDeviceSynchronize());
    PT_CUDA(cudaLaunchKernel(kmisc.latency, dim3(1), dim3(1), args, 0, 0));
  } else if (what == 1) {
    int iters = 2000;
    int blocks = prop.multiProcessorCount;
    void* args[] = {&u, &iters, &d};
    PT_CUDA(cudaLaunchCooperativeKernel(kmisc.barrier, dim3(blocks), dim3(kThreads), args, 0, 0));
  } else if (what == 2) {
    int iters = 10000;
    void* args[] = {&u, &iters, &d};
    PT_CUDA(cudaLaunchKernel(kmisc.pingpong, dim3(prop.multiProcessorCount), dim3(32), args, 0, 0));
  } else if (what == 3) {
    void* args[] = {&d};
    PT_CUDA(cudaLaunchKernel(kmisc.mgs_pieces, dim3(1), dim3(32), args, 0, 0));
    PT_CUDA(cudaDeviceSynchronize());
    PT_CUDA(cudaLaunchKernel(kmisc.mgs_pieces, dim3(1), dim3(32), args, 0, 0));
  } else {
    return fail(PT_E_INVAL, "unknown microbenchmark");
  }
  PT_CUDA(cudaGetLastError());
  PT_CUDA(cudaDeviceSynchronize());
  PT_CUDA(cudaMemcpy(out, d, 16 * 8, cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(u);
  return PT_OK;
}

int pt_plan_mgs_timeline(pt_plan* p, double* out, int32_t count) {
  if (!p || !out) return PT_E_INVAL;
  PT_CUDA(cudaSetDevice(p->device));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  const int m = std::min(count, 14 * (p->n + 2));
  std::vector<unsigned long long> h(m);
  PT_CUDA(cudaMemcpy(h.data(), carve(p->dwork, p->uwork, p->lay, 0).prof + kProfSlots, m * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < m; ++i) out[i] = (double)h[i];
  return PT_OK;
}

int pt_plan_set_trace(pt_plan* p, int32_t capacity) {
  if (!p || capacity < 0) return PT_E_INVAL;
  PT_CUDA(cudaSetDevice(p->device));
  if (p->d_trace) cudaFree(p->d_trace);
  p->d_trace = nullptr;
  p->trace_cap = 0;
  if (capacity > 0) {
    int rc = 0;
    p->d_trace = dev_alloc<pt_trace_event>(capacity, &rc);
    if (rc) return rc;
    p->trace_cap = capacity;
  }
  return PT_OK;
}

int pt_plan_get_trace(pt_plan* p, pt_trace_event* out, int32_t capacity, int32_t* count) {
  if (!p || !count) return PT_E_INVAL;
  PT_CUDA(cudaSetDevice(p->device));
  int len = 0;
  PT_CUDA(cudaMemcpy(&len, p->d_trace_len, sizeof(int), cudaMemcpyDeviceToHost));
  *count = len;
  const int m = std::min({len, capacity, p->trace_cap});
  if (m > 0 && out) PT_CUDA(cudaMemcpy(out, p->d_trace, m * sizeof(pt_trace_event), cudaMemcpyDeviceToHost));
  return PT_OK;
}

int pt_track_path_device(pt_plan* p, const double* d_start, const pt_step_params* sp, double* d_end,
                         pt_path_stats* d_stats, void* stream) {
  if (!p || !d_start || !d_end || !d_stats) return fail(PT_E_INVAL, "null argument");
  int rc = validate_params(sp);
  if (rc) return rc;
  PT_CUDA(cudaSetDevice(p->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : p->stream;
  TrackIO io{d_start, d_end, d_stats, p->d_trace, p->trace_cap, p->d_trace_len, 0};
  cudaError_t err = cudaSuccess;
  launch_grid(p, *sp, io, s, &err);
  if (err != cudaSuccess) return fail(PT_E_CUDA, std::string("track launch: ") + cudaGetErrorString(err));
  return PT_OK;
}

int pt_track_path(pt_plan* p, const double* start, const pt_step_params* sp, double* end, pt_path_stats* stats) {
  if (!p || !start || !end || !stats) return fail(PT_E_INVAL, "null argument");
  PT_CUDA(cudaSetDevice(p->device));
  const size_t bytes = (size_t)2 * p->L * p->n * sizeof(double);
  PT_CUDA(cudaMemcpyAsync(p->d_start, start, bytes, cudaMemcpyHostToDevice, p->stream));
  int rc = pt_track_path_device(p, p->d_start, sp, p->d_end, p->d_stats, p->stream);
  if (rc) return rc;
  PT_CUDA(cudaMemcpyAsync(end, p->d_end, bytes, cudaMemcpyDeviceToHost, p->stream));
  PT_CUDA(cudaMemcpyAsync(stats, p->d_stats, sizeof(pt_path_stats), cudaMemcpyDeviceToHost, p->stream));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  return read_abort(p, carve(p->dwork, p->uwork, p->lay, 0).ctl);
}

static int ensure_batch(pt_plan* p) {
  if (p->bwork) return PT_OK;
  int per_sm = 0, sms = 0;
  const void* fn = kset(p->prec).track_batch;
  // batch: the warp MGS hands q_k on through shared memory + flags (mode 1):
  // one CTA has no remote consumer for the TMA multicast, and without the Q
  // buffer each CTA leaves 33 KB more of the SM to L1 (C5: 7.30-7.38 s vs
  // 7.47-7.49 s per 2368 paths, same box)
  p->batch_dyn_smem = engine_smem(p->L, p->N, p->n, 1, true, &p->batch_warp, 1);
  // split-bundle scratch (eval_bundles) after the x copy in the dynamic smem
  const size_t scratch_end = (((size_t)2 * p->L * p->n + 31) & ~(size_t)31) + (size_t)p->scratch_units * 32 * 2 * p->L;
  // PT_MGS_BATCH=1: the column-item MGS (mgs_batch.cuh) instead of the warp MGS.
  // Measured on C5 (same box, A/B x2): warp MGS 8.11 s, column items 8.51 s
  // per 2368 paths -- the warp MGS stays the default.
  const char* be = getenv("PT_MGS_BATCH");
  p->batch_mgs = (p->N <= kBmMaxN && be && be[0] == '1') ? 1 : 0;
  if (p->batch_mgs) {  // the padded matrix, then (after the MGS) the staged R and the x copy reuse it
    p->batch_warp = 0;
    p->batch_dyn_smem = std::max({bm_smem_doubles(p->L, p->N, p->n), backsub_stage_doubles(p->L, p->n),
                                  (size_t)2 * p->L * p->n}) * 8;
  }
  p->batch_mgs_smem = p->batch_dyn_smem > 0;  // before the x copy / split scratch may enlarge it
  p->batch_dyn_smem = std::max(p->batch_dyn_smem, scratch_end * 8);
  int rc = set_dyn_smem(fn, p->batch_dyn_smem);
  if (rc) return rc;
  cudaDeviceProp prop;
  PT_CUDA(cudaGetDeviceProperties(&prop, p->device));
  sms = prop.multiProcessorCount;
  PT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, p->batch_dyn_smem));
  p->batch_blocks = std::max(1, per_sm) * sms;
  p->bwork = dev_alloc<double>((size_t)p->lay.dslice * p->batch_blocks, &rc);
  if (rc) return rc;
  p->bu = dev_alloc<unsigned long long>((size_t)p->lay.uslice * p->batch_blocks, &rc);
  if (rc) return rc;
  p->d_queue = dev_alloc<unsigned long long>(2, &rc);  // [0] path queue, [1] watchdog abort
  if (rc) return rc;
  PT_CUDA(cudaMemset(p->bwork, 0, (size_t)p->lay.dslice * p->batch_blocks * 8));
  PT_CUDA(cudaMemset(p->bu, 0, (size_t)p->lay.uslice * p->batch_blocks * 8));
  return PT_OK;
}

int pt_track_batch_device(pt_plan* p, int32_t n_paths, const double* d_starts, const pt_step_params* sp,
                          double* d_ends, pt_path_stats* d_stats, void* stream) {
  if (!p || n_paths < 0 || (n_paths > 0 && (!d_starts || !d_ends || !d_stats))) return fail(PT_E_INVAL, "bad batch args");
  int rc = validate_params(sp);
  if (rc) return rc;
  if (n_paths == 0) return PT_OK;
  PT_CUDA(cudaSetDevice(p->device));
  rc = ensure_batch(p);
  if (rc) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : p->stream;
  PT_CUDA(cudaMemsetAsync(p->d_queue, 0, 16, s));
  const void* fn_fast = tset(p).track_batch;
  const void* fn_exact = tset_exact(p).track_batch;
  rc = set_dyn_smem(fn_fast, p->batch_dyn_smem);  // per-function attribute: this plan's value
  if (rc) return rc;
  const unsigned long long epoch = (++p->launches) << 40;
  const int blocks = std::min(p->batch_blocks, n_paths);
  DevPlan bdp = p->dp;
  bdp.mgs_smem = p->batch_mgs_smem;
  bdp.dyn_smem = p->batch_dyn_smem > 0;
  bdp.mgs_warp = p->batch_warp;
  bdp.mgs_batch = p->batch_mgs;
  bdp.bs_smem = stage_fits(p, p->batch_dyn_smem);
  bdp.x_smem = x_fits(p, p->batch_dyn_smem);
  bdp.tasks = p->tasks_b;
  for (int c = 0; c < 6; ++c) bdp.class_beg[c] = p->class_beg_b[c];
  bdp.bundles = p->bundles;
  bdp.n_bundles = p->n_bundles;
  bdp.splits = p->splits;
  bdp.n_splits = p->n_splits;
  bdp.scratch_units = p->scratch_units;
  bdp.btasks = p->btasks;
  bdp.s_ws = p->s_ws;
  bdp.s_coef = p->s_coef;
  bdp.s_len = p->s_len;
  bdp.s_hi = p->s_hi;
  // launched as clusters of one CTA: the warp MGS pushes q_k with st.async,
  // which needs a cluster launch even when the cluster is the CTA itself
  Layout lay = p->lay;
  pt_step_params spc = *sp;
  int np = n_paths;
  unsigned long long ep = epoch;
  int retrack = 0;
  void* args[] = {&bdp, &p->bwork, &p->bu, &lay, &spc, &d_starts, &d_ends, &d_stats, &np, &p->d_queue, &ep, &retrack};
  PT_CUDA(launch_ex(fn_fast, blocks, p->batch_dyn_smem, s, 1, args));
  if (fn_exact != fn_fast) {
    // exact re-track of the paths whose fast run met a non-finite value
    // (PT_STAT_NONFINITE): the queue restarts, the abort word is kept
    PT_CUDA(cudaMemsetAsync(p->d_queue, 0, 8, s));
    rc = set_dyn_smem(fn_exact, p->batch_dyn_smem);
    if (rc) return rc;
    retrack = 1;
    ep = (++p->launches) << 40;
    PT_CUDA(launch_ex(fn_exact, blocks, p->batch_dyn_smem, s, 1, args));
  }
  PT_CUDA(cudaGetLastError());
  return PT_OK;
}

int pt_track_batch(pt_plan* p, int32_t n_paths, const double* starts, const pt_step_params* sp, double* ends,
                   pt_path_stats* stats) {
  if (!p || n_paths < 0) return fail(PT_E_INVAL, "bad batch args");
  if (n_paths == 0) return PT_OK;
  PT_CUDA(cudaSetDevice(p->device));
  const size_t vec = (size_t)2 * p->L * p->n;
  if (p->b_cap < n_paths) {
    for (void* q : {(void*)p->b_starts, (void*)p->b_ends, (void*)p->b_stats})
      if (q) cudaFree(q);
    int rc = 0;
    p->b_starts = dev_alloc<double>(vec * n_paths, &rc);
    if (rc) return rc;
    p->b_ends = dev_alloc<double>(vec * n_paths, &rc);
    if (rc) return rc;
    p->b_stats = dev_alloc<pt_path_stats>(n_paths, &rc);
    if (rc) return rc;
    p->b_cap = n_paths;
  }
  PT_CUDA(cudaMemcpyAsync(p->b_starts, starts, vec * n_paths * 8, cudaMemcpyHostToDevice, p->stream));
  int rc = pt_track_batch_device(p, n_paths, p->b_starts, sp, p->b_ends, p->b_stats, p->stream);
  if (rc) return rc;
  PT_CUDA(cudaMemcpyAsync(ends, p->b_ends, vec * n_paths * 8, cudaMemcpyDeviceToHost, p->stream));
  PT_CUDA(cudaMemcpyAsync(stats, p->b_stats, sizeof(pt_path_stats) * n_paths, cudaMemcpyDeviceToHost, p->stream));
  unsigned long long abort_flag = 0;
  PT_CUDA(cudaMemcpyAsync(&abort_flag, p->d_queue + 1, 8, cudaMemcpyDeviceToHost, p->stream));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  if (abort_flag)
    return fail(PT_E_TIMEOUT, "device watchdog fired in the batch (paths with failure_kind PT_FAIL_ABORT)");
  return PT_OK;
}

int pt_eval_homotopy(pt_plan* p, const double* x, double t, double* h, double* J, double* rmax) {
  if (!p || !x) return fail(PT_E_INVAL, "null argument");
  PT_CUDA(cudaSetDevice(p->device));
  const int L = p->L, n = p->n, N = p->N;
  int rc = 0;
  double* dx = dev_alloc<double>((size_t)2 * L * n, &rc);
  if (rc) return rc;
  double* dh = dev_alloc<double>((size_t)2 * L * N, &rc);
  double* dJ = dev_alloc<double>((size_t)2 * L * N * n, &rc);
  double* dr = dev_alloc<double>(1, &rc);
  if (rc) return rc;
  PT_CUDA(cudaMemcpy(dx, x, (size_t)2 * L * n * 8, cudaMemcpyHostToDevice));
  Work W = carve(p->dwork, p->uwork, p->lay, 0);
  DevPlan dp = p->dp;
  dp.mgs_smem = 0;
  dp.mgs_warp = 0;
  void* args[] = {&dp, &W, &dx, &t, &dh, &dJ, &dr};
  const void* fn = tset_exact(p).eval;
  rc = set_dyn_smem(fn, p->grid_dyn_smem);
  if (rc) return rc;
  PT_CUDA(cudaMemset(W.ctl, 0, CTL_WORDS * sizeof(unsigned long long)));
  PT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(p->grid_blocks), dim3(kThreads), args, p->grid_dyn_smem, p->stream));
  PT_CUDA(cudaStreamSynchronize(p->stream));
  if (h) PT_CUDA(cudaMemcpy(h, dh, (size_t)2 * L * N * 8, cudaMemcpyDeviceToHost));
  if (J) PT_CUDA(cudaMemcpy(J, dJ, (size_t)2 * L * N * n * 8, cudaMemcpyDeviceToHost));
  if (rmax) PT_CUDA(cudaMemcpy(rmax, dr, 8, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dh);
  cudaFree(dJ);
  cudaFree(dr);
  return read_abort(p, W.ctl);
}

int pt_eval_bench(pt_plan* p, const double* x, double t, int32_t reps, double* ms_per_eval) {
  if (!p || !x || reps < 1 || !ms_per_eval) return fail(PT_E_INVAL, "bad eval-bench arguments");
  PT_CUDA(cudaSetDevice(p->device));
  const int L = p->L, n = p->n;
  int rc = 0;
  double* dx = dev_alloc<double>((size_t)2 * L * n, &rc);
  if (rc) return rc;
  std::unique_ptr<double, decltype(&cudaFree)> gx(dx, &cudaFree);
  PT_CUDA(cudaMemcpy(dx, x, (size_t)2 * L * n * 8, cudaMemcpyHostToDevice));
  Work W = carve(p->dwork, p->uwork, p->lay, 0);
  DevPlan dp = p->dp;
  dp.mgs_smem = 0;
  dp.mgs_warp = 0;
  double* null = nullptr;
  void* args[] = {&dp, &W, &dx, &t, &null, &null, &null};
  const void* fn = tset_exact(p).eval;
  rc = set_dyn_smem(fn, p->grid_dyn_smem);
  if (rc) return rc;
  PT_CUDA(cudaMemset(W.ctl, 0, CTL_WORDS * sizeof(unsigned long long)));
  cudaEvent_t e0, e1;
  PT_CUDA(cudaEventCreate(&e0));
  PT_CUDA(cudaEventCreate(&e1));
  // one untimed warm-up pass, then `reps` passes between events on the plan's stream
  cudaError_t err = cudaLaunchCooperativeKernel(fn, dim3(p->grid_blocks), dim3(kThreads), args, p->grid_dyn_smem,
                                                p->stream);
  if (err == cudaSuccess) err = cudaEventRecord(e0, p->stream);
  for (int r = 0; r < reps && err == cudaSuccess; ++r)
    err = cudaLaunchCooperativeKernel(fn, dim3(p->grid_blocks), dim3(kThreads), args, p->grid_dyn_smem, p->stream);
  if (err == cudaSuccess) err = cudaEventRecord(e1, p->stream);
  if (err == cudaSuccess) err = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err != cudaSuccess) return fail(PT_E_CUDA, std::string("eval bench: ") + cudaGetErrorString(err));
  *ms_per_eval = ms / reps;
  return read_abort(p, W.ctl);
}

int pt_lstsq(int device, pt_prec prec, int32_t N, int32_t n, const double* A, const double* b, double* x) {
  return guarded([&]() -> int {
    if (!A || !b || !x || n < 1 || N < n || n > kMaxRowsPerThread * kThreads || N > kMaxElems * 256)
      return fail(PT_E_INVAL, "bad lstsq arguments");
    int rc = check_device(device);
    if (rc) return rc;
    PT_CUDA(cudaSetDevice(device));
    const int L = limbs(prec);
    Layout lay = make_layout(L, n, N, 1);
    double* dw = dev_alloc<double>(lay.dslice, &rc);
    if (rc) return rc;
    unsigned long long* uw = dev_alloc<unsigned long long>(lay.uslice, &rc);
    int* dstat = dev_alloc<int>(1, &rc);
    if (rc) return rc;
    PT_CUDA(cudaMemset(dw, 0, lay.dslice * 8));
    PT_CUDA(cudaMemset(uw, 0, lay.uslice * 8));
    Work W = carve(dw, uw, lay, 0);
    const long SA = (long)N * (n + 1), SJ = (long)N * n;
    // [A | b] into SoA with stride SA
    std::vector<double> hA((size_t)2 * L * SA);
    for (int q = 0; q < 2 * L; ++q) {
      std::memcpy(&hA[(size_t)q * SA], A + (size_t)q * SJ, SJ * 8);
      std::memcpy(&hA[(size_t)q * SA + SJ], b + (size_t)q * N, (size_t)N * 8);
    }
    PT_CUDA(cudaMemcpy(W.A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice));
    DevPlan dp{};
    dp.n = n;
    dp.N = N;
    dp.P_mgs = ptplan::width_mgs(N);
    dp.mgs_gw = ptplan::mgs_group_warps(N);
    const int gpc = kWarps / dp.mgs_gw;
    int per_sm = 0, sms = 0;
    const void* fn = kset_exact(prec).lstsq;
    rc = occupancy_blocks(fn, device, &per_sm, &sms);
    if (rc) return rc;
    int blocks = std::min(std::min(sms, std::max(1, per_sm) * sms), std::max(1, (n + 1 + gpc - 1) / gpc));
    const size_t dyn = mgs_smem_bytes(L, N, n, blocks);
    rc = set_dyn_smem(fn, dyn);
    if (rc) return rc;
    dp.mgs_smem = dyn > 0;
    unsigned long long epoch = 1;
    void* args[] = {&dp, &W, &epoch, &dstat};
    PT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kThreads), args, dyn, 0));
    PT_CUDA(cudaDeviceSynchronize());
    int st = 0;
    PT_CUDA(cudaMemcpy(&st, dstat, 4, cudaMemcpyDeviceToHost));
    if (st == 0) PT_CUDA(cudaMemcpy(x, W.dx, (size_t)2 * L * n * 8, cudaMemcpyDeviceToHost));
    cudaFree(dw);
    cudaFree(uw);
    cudaFree(dstat);
    if (st == PT_E_RANK) return fail(PT_E_RANK, "rank-deficient least-squares matrix");
    if (st) return fail(st, "lstsq kernel failed");
    return PT_OK;
  });
}

int pt_arith_host(pt_prec prec, int32_t op, int64_t count, const double* a, const double* b, double* out) {
  if (!a || !b || !out || count < 0) return PT_E_INVAL;
  const int L = limbs(prec);
  for (int64_t i = 0; i < count; ++i) {
    const double* pa = a + i * 2 * L;
    const double* pb = b + i * 2 * L;
    double* po = out + i * 2 * L;
    switch (prec) {
      case PT_D: arith_one<double>(op, pa, pb, po); break;
      case PT_DD: arith_one<dd>(op, pa, pb, po); break;
      default: arith_one<qd>(op, pa, pb, po); break;
    }
  }
  return PT_OK;
}

int pt_arith_device(int device, pt_prec prec, int32_t op, int64_t count, const double* a, const double* b,
                    double* out) {
  return pt_arith_device_mode(device, prec, PT_ARITH_REFERENCE, op, count, a, b, out);
}

int pt_arith_device_mode(int device, pt_prec prec, int32_t arith, int32_t op, int64_t count, const double* a,
                         const double* b, double* out) {
  if (arith != PT_ARITH_REFERENCE && !(arith == PT_ARITH_FAST && prec == PT_QD))
    return fail(PT_E_INVAL, "PT_ARITH_FAST exists for QD only");
  if (!a || !b || !out || count < 0) return fail(PT_E_INVAL, "bad arith args");
  int rc = check_device(device);
  if (rc) return rc;
  PT_CUDA(cudaSetDevice(device));
  const size_t bytes = (size_t)count * 2 * limbs(prec) * 8;
  double *da = dev_alloc<double>(bytes / 8, &rc), *db = dev_alloc<double>(bytes / 8, &rc),
         *dout = dev_alloc<double>(bytes / 8, &rc);
  if (rc) return rc;
  PT_CUDA(cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice));
  PT_CUDA(cudaMemcpy(db, b, bytes, cudaMemcpyHostToDevice));
  PT_CUDA(cudaMemset(dout, 0, bytes));
  const int blocks = (int)std::min<int64_t>(4096, (count + 255) / 256 + 1);
  long cnt = (long)count;
  int opc = op;
  void* args[] = {&opc, &cnt, &da, &db, &dout};
  PT_CUDA(cudaLaunchKernel(kset_mode(prec, arith).arith, dim3(blocks), dim3(256), args, 0, 0));
  PT_CUDA(cudaGetLastError());
  PT_CUDA(cudaDeviceSynchronize());
  PT_CUDA(cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost));
  cudaFree(da);
  cudaFree(db);
  cudaFree(dout);
  return PT_OK;
}

}  // extern "C"
