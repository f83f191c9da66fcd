// Runtime half of libispc: NVRTC compilation to sm_100a cubins, module
// management, problem binding (seeded inputs, golden expected outputs, GLOBAL
// temporary scratch), CUDA-event-timed launches with a device watchdog, and
// on-device output checks. Replaces the reference's analytic evaluate()
// (proj/core/src/simulate.cpp:118-133) with a measurement on a B200.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include "builtins.hpp"
#include "ispc.h"
#include "nest_view.hpp"

namespace ispc {
std::string emit_cuda_kernel(const NestView& v, const ispc_emit_opts& opts, const std::string& fn,
                             ispc_launch& L);
}

struct ispc_module {
  std::vector<char> cubin;
  std::string log;
};

namespace {

struct Buffer {
  float* ptr = nullptr;
  int64_t elems = 0;
};

struct Loaded {
  CUmodule mod = nullptr;
  std::unordered_map<std::string, CUfunction> fns;
  CUdeviceptr timeout_flag = 0;
  CUfunction arm = nullptr;  // ispc_arm of the prelude (device-side watchdog deadline)
};


// Driver API entry points, resolved through the runtime at first device open
// so the library loads (and its symbols can be inspected) on hosts without a
// CUDA driver.
struct DriverTable {
  decltype(&::cuCtxGetCurrent) CtxGetCurrent = nullptr;
  decltype(&::cuDeviceGet) DeviceGet = nullptr;
  decltype(&::cuFuncSetAttribute) FuncSetAttribute = nullptr;
  decltype(&::cuGetErrorName) GetErrorName = nullptr;
  decltype(&::cuInit) Init = nullptr;
  decltype(&::cuLaunchKernel) LaunchKernel = nullptr;
  decltype(&::cuMemcpyDtoH) MemcpyDtoH = nullptr;
  decltype(&::cuModuleGetFunction) ModuleGetFunction = nullptr;
  decltype(&::cuModuleGetGlobal) ModuleGetGlobal = nullptr;
  decltype(&::cuModuleLoadData) ModuleLoadData = nullptr;
  decltype(&::cuModuleUnload) ModuleUnload = nullptr;
  decltype(&::cuMemsetD32Async) MemsetD32Async = nullptr;
  decltype(&::cuLaunchKernelEx) LaunchKernelEx = nullptr;
  decltype(&::cuTensorMapEncodeTiled) TensorMapEncodeTiled = nullptr;
  // optional (eager loading of a module's kernels on the thread that loads it)
  decltype(&::cuModuleGetFunctionCount) ModuleGetFunctionCount = nullptr;
  decltype(&::cuModuleEnumerateFunctions) ModuleEnumerateFunctions = nullptr;
  decltype(&::cuFuncLoad) FuncLoad = nullptr;
  decltype(&::cuFuncGetAttribute) FuncGetAttribute = nullptr;
};
DriverTable drv;

bool resolve_driver(std::string& why) {
  static std::once_flag once;
  static bool ok = false;
  static std::string err;
  std::call_once(once, [] {
    ok = true;
    auto get = [](const char* sym, void** fp) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(sym, fp, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        ok = false;
        err += std::string(sym) + " ";
      }
    };
    get("cuCtxGetCurrent", reinterpret_cast<void**>(&drv.CtxGetCurrent));
    get("cuDeviceGet", reinterpret_cast<void**>(&drv.DeviceGet));
    get("cuFuncSetAttribute", reinterpret_cast<void**>(&drv.FuncSetAttribute));
    get("cuGetErrorName", reinterpret_cast<void**>(&drv.GetErrorName));
    get("cuInit", reinterpret_cast<void**>(&drv.Init));
    get("cuLaunchKernel", reinterpret_cast<void**>(&drv.LaunchKernel));
    get("cuMemcpyDtoH", reinterpret_cast<void**>(&drv.MemcpyDtoH));
    get("cuModuleGetFunction", reinterpret_cast<void**>(&drv.ModuleGetFunction));
    get("cuModuleGetGlobal", reinterpret_cast<void**>(&drv.ModuleGetGlobal));
    get("cuModuleLoadData", reinterpret_cast<void**>(&drv.ModuleLoadData));
    get("cuModuleUnload", reinterpret_cast<void**>(&drv.ModuleUnload));
    get("cuMemsetD32Async", reinterpret_cast<void**>(&drv.MemsetD32Async));
    get("cuLaunchKernelEx", reinterpret_cast<void**>(&drv.LaunchKernelEx));
    get("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&drv.TensorMapEncodeTiled));
    auto opt = [](const char* sym, void** fp) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(sym, fp, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        *fp = nullptr;
    };
    opt("cuModuleGetFunctionCount", reinterpret_cast<void**>(&drv.ModuleGetFunctionCount));
    opt("cuModuleEnumerateFunctions", reinterpret_cast<void**>(&drv.ModuleEnumerateFunctions));
    opt("cuFuncLoad", reinterpret_cast<void**>(&drv.FuncLoad));
    opt("cuFuncGetAttribute", reinterpret_cast<void**>(&drv.FuncGetAttribute));
  });
  if (!ok) why = "CUDA driver entry points unavailable: " + err;
  return ok;
}

double host_ns() {
  return double(std::chrono::duration_cast<std::chrono::nanoseconds>(
                    std::chrono::steady_clock::now().time_since_epoch())
                    .count());
}

}  // namespace

struct ispc_dev {
  int ordinal = 0;
  CUdevice cu_dev = 0;
  CUcontext ctx = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  int sm_count = 0, sm_clock_khz = 0;
  int64_t l2_bytes = 0, hbm_bytes = 0;
  double gt_offset_ns = 0;  // device globaltimer - host steady clock
  void* flush = nullptr;
  size_t flush_bytes = 0;
  void* cmp_res = nullptr;
  unsigned long long* timer_buf = nullptr;

  ispc_problem prob{};
  bool bound = false;
  std::map<std::string, Buffer> regions;  // inputs and outputs by name
  std::map<std::string, Buffer> expected;  // golden outputs by name
  std::map<std::string, Buffer> scale;     // golden sum of |products| per output element (reductions)
  std::vector<std::string> outputs;
  std::vector<Buffer> scratch;
  // rotation copies of the input regions (timing with inputs larger than L2)
  std::vector<std::map<std::string, Buffer>> rot;

  std::map<int, Loaded> modules;  // guarded by mod_mu (loads may come from compile threads)
  std::mutex mod_mu;
  int next_handle = 1;
  std::vector<cudaEvent_t> evpool;  // timing events of batched launches
  void* slots = nullptr;            // per-item ispc::CmpResult of batched launches
  size_t slot_cap = 0;
  cudaEvent_t marks[8] = {};
};

namespace {
unsigned flush_counter_ = 0;
}

namespace {

int fail(ispc_dev* d, int code, const std::string& msg) {
  if (d) d->err = msg;
  ispc::set_thread_error(msg);
  return code;
}

bool sticky(cudaError_t e) {
  return e == cudaErrorIllegalAddress || e == cudaErrorLaunchFailure || e == cudaErrorIllegalInstruction ||
         e == cudaErrorMisalignedAddress || e == cudaErrorInvalidAddressSpace || e == cudaErrorInvalidPc ||
         e == cudaErrorHardwareStackError || e == cudaErrorAssert || e == cudaErrorLaunchTimeout;
}

int cuda_fail(ispc_dev* d, cudaError_t e, const char* what) {
  return fail(d, sticky(e) ? ISPC_E_STICKY : ISPC_E_CUDA,
              std::string(what) + ": " + cudaGetErrorName(e) + " " + cudaGetErrorString(e));
}

int cu_fail(ispc_dev* d, CUresult r, const char* what) {
  const char* name = nullptr;
  if (drv.GetErrorName) drv.GetErrorName(r, &name);
  bool st = r == CUDA_ERROR_ILLEGAL_ADDRESS || r == CUDA_ERROR_LAUNCH_FAILED ||
            r == CUDA_ERROR_ILLEGAL_INSTRUCTION || r == CUDA_ERROR_MISALIGNED_ADDRESS ||
            r == CUDA_ERROR_HARDWARE_STACK_ERROR || r == CUDA_ERROR_ASSERT;
  int code = st ? ISPC_E_STICKY
                : (r == CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES || r == CUDA_ERROR_INVALID_VALUE) ? ISPC_E_LAUNCH
                                                                                                : ISPC_E_CUDA;
  return fail(d, code, std::string(what) + ": " + (name ? name : "CUDA error"));
}

#define CK(d, expr)                                   \
  do {                                                \
    cudaError_t e_ = (expr);                          \
    if (e_ != cudaSuccess) return cuda_fail(d, e_, #expr); \
  } while (0)
#define CU(d, expr)                                   \
  do {                                                \
    CUresult r_ = (expr);                             \
    if (r_ != CUDA_SUCCESS) return cu_fail(d, r_, #expr); \
  } while (0)

int bind_ctx(ispc_dev* d) {
  CK(d, cudaSetDevice(d->ordinal));
  return ISPC_OK;
}

uint32_t tag_of(const std::string& name) { return uint32_t(static_cast<unsigned char>(name[0])); }

int alloc(ispc_dev* d, Buffer& b, int64_t elems) {
  b.elems = elems;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&b.ptr), size_t(std::max<int64_t>(elems, 1)) * 4);
  if (e != cudaSuccess) {
    b.ptr = nullptr;
    cudaGetLastError();
    return fail(d, ISPC_E_NOMEM, "cudaMalloc of " + std::to_string(elems * 4) + " bytes failed");
  }
  return ISPC_OK;
}

void free_problem(ispc_dev* d) {
  for (auto& [k, b] : d->regions) cudaFree(b.ptr);
  for (auto& [k, b] : d->expected) cudaFree(b.ptr);
  for (auto& [k, b] : d->scale) cudaFree(b.ptr);
  for (auto& b : d->scratch) cudaFree(b.ptr);
  for (auto& m : d->rot)
    for (auto& [k, b] : m) cudaFree(b.ptr);
  d->rot.clear();
  d->regions.clear();
  d->expected.clear();
  d->scale.clear();
  d->scratch.clear();
  d->outputs.clear();
  d->bound = false;
}

int calibrate_timer(ispc_dev* d) {
  double best_gap = 1e30;
  for (int i = 0; i < 5; ++i) {
    double t0 = host_ns();
    CK(d, ispc::launch_timer(d->timer_buf, d->stream));
    CK(d, cudaStreamSynchronize(d->stream));
    double t1 = host_ns();
    unsigned long long gt = 0;
    CK(d, cudaMemcpy(&gt, d->timer_buf, 8, cudaMemcpyDeviceToHost));
    if (t1 - t0 < best_gap) {
      best_gap = t1 - t0;
      d->gt_offset_ns = double(gt) - 0.5 * (t0 + t1);
    }
  }
  return ISPC_OK;
}

// Expected outputs of the bound problem, from the golden kernels.
int recompute_expected(ispc_dev* d) {
  const ispc_problem* p = &d->prob;
  const int64_t m = p->m, n = p->n, k = p->k, s = std::max<int64_t>(p->a_stride, 1);
  const int64_t batch = std::max<int64_t>(p->batch, 1);
  auto R_ = [&](const char* nm) { return d->regions.at(nm).ptr; };
  auto E_ = [&](const char* nm) { return d->expected.at(nm).ptr; };
  auto S_ = [&](const char* nm) { return d->scale.count(nm) ? d->scale.at(nm).ptr : nullptr; };
  switch (p->kind) {
    case ISPC_PROB_AXPY: CK(d, ispc::launch_axpy_golden(R_("x"), R_("y"), E_("z"), n, p->alpha, d->stream)); break;
    case ISPC_PROB_OUTER: CK(d, ispc::launch_outer_golden(R_("a"), R_("b"), E_("c"), m, n, d->stream)); break;
    case ISPC_PROB_MATMUL:
      CK(d, ispc::launch_matmul_golden(R_("a"), R_("b"), E_("c"), m, n, k, s, 1, S_("c"), d->stream));
      break;
    case ISPC_PROB_GEMV: CK(d, ispc::launch_gemv_golden(R_("a"), R_("x"), E_("y"), m, n, S_("y"), d->stream)); break;
    case ISPC_PROB_BATCHED:
      CK(d, ispc::launch_matmul_golden(R_("a"), R_("b"), E_("c"), m, n, k, 1, batch, S_("c"), d->stream));
      break;
  }
  CK(d, cudaStreamSynchronize(d->stream));
  return ISPC_OK;
}

}  // namespace

extern "C" {

const char* ispc_last_error(const ispc_dev* d) { return d ? d->err.c_str() : ispc::thread_error(); }

int ispc_dev_open(int ordinal, ispc_dev** out) {
  if (!out) return fail(nullptr, ISPC_E_ARG, "null out");
  auto d = std::make_unique<ispc_dev>();
  d->ordinal = ordinal;
  CK(d.get(), cudaSetDevice(ordinal));
  CK(d.get(), cudaFree(nullptr));  // create the primary context
  std::string why;
  if (!resolve_driver(why)) return fail(d.get(), ISPC_E_CUDA, why);
  CU(d.get(), drv.Init(0));
  CU(d.get(), drv.DeviceGet(&d->cu_dev, ordinal));
  CU(d.get(), drv.CtxGetCurrent(&d->ctx));
  CK(d.get(), cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  CK(d.get(), cudaEventCreate(&d->ev0));
  CK(d.get(), cudaEventCreate(&d->ev1));
  cudaDeviceProp p{};
  CK(d.get(), cudaGetDeviceProperties(&p, ordinal));
  d->sm_count = p.multiProcessorCount;
  d->l2_bytes = p.l2CacheSize;
  d->hbm_bytes = int64_t(p.totalGlobalMem);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, ordinal);
  d->sm_clock_khz = clk;
  d->flush_bytes = size_t(std::max<int64_t>(d->l2_bytes, 64 << 20)) * 2;
  CK(d.get(), cudaMalloc(&d->flush, d->flush_bytes));
  CK(d.get(), cudaMalloc(&d->cmp_res, sizeof(ispc::CmpResult)));
  CK(d.get(), cudaMalloc(reinterpret_cast<void**>(&d->timer_buf), 8));
  int rc = calibrate_timer(d.get());
  if (rc) return rc;
  *out = d.release();
  return ISPC_OK;
}

void ispc_dev_close(ispc_dev* d) {
  if (!d) return;
  cudaSetDevice(d->ordinal);
  cudaStreamSynchronize(d->stream);
  for (auto& [h, m] : d->modules) drv.ModuleUnload(m.mod);
  free_problem(d);
  for (cudaEvent_t e : d->evpool) cudaEventDestroy(e);
  if (d->slots) cudaFree(d->slots);
  cudaFree(d->flush);
  cudaFree(d->cmp_res);
  cudaFree(d->timer_buf);
  cudaEventDestroy(d->ev0);
  cudaEventDestroy(d->ev1);
  cudaStreamDestroy(d->stream);
  delete d;
}

int ispc_dev_inject_fault(ispc_dev* d) {
  if (!d) return ISPC_E_ARG;
  int rc = bind_ctx(d);
  if (rc) return rc;
  CK(d, ispc::launch_fault(d->stream));
  CK(d, cudaStreamSynchronize(d->stream));
  return fail(d, ISPC_E_CUDA, "the injected fault did not fault");
}

int ispc_dev_info(const ispc_dev* d, int* sm_count, int64_t* l2_bytes, int64_t* hbm_bytes, int* sm_clock_khz) {
  if (!d) return ISPC_E_ARG;
  if (sm_count) *sm_count = d->sm_count;
  if (l2_bytes) *l2_bytes = d->l2_bytes;
  if (hbm_bytes) *hbm_bytes = d->hbm_bytes;
  if (sm_clock_khz) *sm_clock_khz = d->sm_clock_khz;
  return ISPC_OK;
}

int ispc_bind_problem(ispc_dev* d, const ispc_problem* p) {
  if (!d || !p) return fail(d, ISPC_E_ARG, "null argument");
  int rc = bind_ctx(d);
  if (rc) return rc;
  CK(d, cudaStreamSynchronize(d->stream));
  free_problem(d);
  d->prob = *p;
  struct R {
    const char* name;
    int64_t elems;
    bool input;
  };
  R rs_buf[3];
  const int64_t m = p->m, n = p->n, k = p->k, s = std::max<int64_t>(p->a_stride, 1);
  const int64_t batch = std::max<int64_t>(p->batch, 1);
  switch (p->kind) {
    case ISPC_PROB_AXPY: rs_buf[0] = {"x", n, true}, rs_buf[1] = {"y", n, true}, rs_buf[2] = {"z", n, false}; break;
    case ISPC_PROB_OUTER: rs_buf[0] = {"a", m, true}, rs_buf[1] = {"b", n, true}, rs_buf[2] = {"c", m * n, false}; break;
    case ISPC_PROB_MATMUL: rs_buf[0] = {"a", m * k * s, true}, rs_buf[1] = {"b", k * n, true}, rs_buf[2] = {"c", m * n, false}; break;
    case ISPC_PROB_GEMV: rs_buf[0] = {"a", m * n, true}, rs_buf[1] = {"x", n, true}, rs_buf[2] = {"y", m, false}; break;
    case ISPC_PROB_BATCHED:
      rs_buf[0] = {"a", batch * m * k, true}, rs_buf[1] = {"b", batch * k * n, true}, rs_buf[2] = {"c", batch * m * n, false};
      break;
    default: return fail(d, ISPC_E_ARG, "unknown problem kind");
  }
  for (const R& r : rs_buf) {
    if (r.elems <= 0) return fail(d, ISPC_E_ARG, std::string("empty region ") + r.name);
    Buffer b;
    if ((rc = alloc(d, b, r.elems))) return rc;
    d->regions[r.name] = b;
    if (r.input) {
      CK(d, ispc::launch_fill(b.ptr, b.elems, p->seed, tag_of(r.name), d->stream));
    } else {
      Buffer e;
      if ((rc = alloc(d, e, r.elems))) return rc;
      d->expected[r.name] = e;
      d->outputs.push_back(r.name);
      if (p->kind == ISPC_PROB_MATMUL || p->kind == ISPC_PROB_GEMV || p->kind == ISPC_PROB_BATCHED) {
        Buffer sc;
        if ((rc = alloc(d, sc, r.elems))) return rc;
        d->scale[r.name] = sc;
      }
    }
  }
  d->bound = true;
  return recompute_expected(d);
}

int ispc_problem_region(ispc_dev* d, const char* name, uint64_t* dev_ptr, int64_t* elems) {
  if (!d || !name) return ISPC_E_ARG;
  auto it = d->regions.find(name);
  if (it == d->regions.end()) return fail(d, ISPC_E_ARG, std::string("no region ") + name);
  if (dev_ptr) *dev_ptr = reinterpret_cast<uint64_t>(it->second.ptr);
  if (elems) *elems = it->second.elems;
  return ISPC_OK;
}

int ispc_read_region(ispc_dev* d, const char* name, void* host, size_t bytes) {
  if (!d || !name || !host) return ISPC_E_ARG;
  int rc = bind_ctx(d);
  if (rc) return rc;
  auto it = d->regions.find(name);
  if (it == d->regions.end()) return fail(d, ISPC_E_ARG, std::string("no region ") + name);
  size_t n = std::min(bytes, size_t(it->second.elems) * 4);
  CK(d, cudaStreamSynchronize(d->stream));
  CK(d, cudaMemcpy(host, it->second.ptr, n, cudaMemcpyDeviceToHost));
  return ISPC_OK;
}

int ispc_write_region(ispc_dev* d, const char* name, const void* host, size_t bytes) {
  if (!d || !name || !host) return ISPC_E_ARG;
  if (!d->bound) return fail(d, ISPC_E_ARG, "no problem bound");
  int rc = bind_ctx(d);
  if (rc) return rc;
  auto it = d->regions.find(name);
  if (it == d->regions.end()) return fail(d, ISPC_E_ARG, std::string("no region ") + name);
  if (d->expected.count(name)) return fail(d, ISPC_E_ARG, std::string("region ") + name + " is an output");
  size_t n = std::min(bytes, size_t(it->second.elems) * 4);
  CK(d, cudaMemcpyAsync(it->second.ptr, host, n, cudaMemcpyHostToDevice, d->stream));
  for (auto& m : d->rot)  // rotation copies are stale now; rebuilt on demand
    for (auto& [k, b] : m) cudaFree(b.ptr);
  d->rot.clear();
  return recompute_expected(d);
}

int ispc_read_expected(ispc_dev* d, const char* name, void* host, size_t bytes) {
  if (!d || !name || !host) return ISPC_E_ARG;
  int rc = bind_ctx(d);
  if (rc) return rc;
  auto it = d->expected.find(name);
  if (it == d->expected.end()) return fail(d, ISPC_E_ARG, std::string("no expected output ") + name);
  size_t n = std::min(bytes, size_t(it->second.elems) * 4);
  CK(d, cudaStreamSynchronize(d->stream));
  CK(d, cudaMemcpy(host, it->second.ptr, n, cudaMemcpyDeviceToHost));
  return ISPC_OK;
}

// ---- compilation --------------------------------------------------------------

int ispc_compile(const char* const* srcs, int n, const char* arch, ispc_module** out) {
  if (!srcs || n <= 0 || !out) return fail(nullptr, ISPC_E_ARG, "bad compile arguments");
  std::string text = ispc_cuda_prelude();
  for (int i = 0; i < n; ++i) {
    if (!srcs[i]) return fail(nullptr, ISPC_E_ARG, "null source");
    text += srcs[i];
    text += "\n";
  }
  auto m = std::make_unique<ispc_module>();
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, text.c_str(), "ispc_candidates.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(nullptr, ISPC_E_NVRTC, "nvrtcCreateProgram failed");
  std::string arch_opt = std::string("--gpu-architecture=") + (arch ? arch : "sm_100a");
  std::vector<std::string> extra;  // ISPC_NVRTC_OPTS: space separated extra options (tuning experiments)
  if (const char* e = std::getenv("ISPC_NVRTC_OPTS")) {
    std::string cur;
    for (const char* p = e;; ++p) {
      if (*p == ' ' || *p == 0) {
        if (!cur.empty()) extra.push_back(cur);
        cur.clear();
        if (!*p) break;
      } else {
        cur += *p;
      }
    }
  }
  std::vector<const char*> opts = {arch_opt.c_str(), "--device-as-default-execution-space", "--std=c++17"};
  for (const std::string& x : extra) opts.push_back(x.c_str());
  nvrtcResult r = nvrtcCompileProgram(prog, int(opts.size()), opts.data());
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  m->log.resize(log_size);
  if (log_size) nvrtcGetProgramLog(prog, m->log.data());
  if (!m->log.empty() && m->log.back() == 0) m->log.pop_back();
  if (r != NVRTC_SUCCESS) {
    std::string msg = std::string("NVRTC: ") + nvrtcGetErrorString(r) + "\n" + m->log;
    nvrtcDestroyProgram(&prog);
    return fail(nullptr, ISPC_E_NVRTC, msg);
  }
  size_t cubin_size = 0;
  if (nvrtcGetCUBINSize(prog, &cubin_size) != NVRTC_SUCCESS || cubin_size == 0) {
    nvrtcDestroyProgram(&prog);
    return fail(nullptr, ISPC_E_NVRTC, "NVRTC produced no cubin (is the arch a real sm_?)");
  }
  m->cubin.resize(cubin_size);
  nvrtcGetCUBIN(prog, m->cubin.data());
  nvrtcDestroyProgram(&prog);
  *out = m.release();
  return ISPC_OK;
}

int ispc_module_cubin(const ispc_module* m, const void** data, size_t* size) {
  if (!m) return ISPC_E_ARG;
  if (data) *data = m->cubin.data();
  if (size) *size = m->cubin.size();
  return ISPC_OK;
}

const char* ispc_module_log(const ispc_module* m) { return m ? m->log.c_str() : ""; }
void ispc_module_free(ispc_module* m) { delete m; }

int ispc_module_load(ispc_dev* d, const ispc_module* m, int* handle) {
  if (!d || !m || !handle) return fail(d, ISPC_E_ARG, "null argument");
  int rc = bind_ctx(d);
  if (rc) return rc;
  Loaded L;
  CU(d, drv.ModuleLoadData(&L.mod, m->cubin.data()));
  size_t sz = 0;
  if (drv.ModuleGetGlobal(&L.timeout_flag, &sz, L.mod, "ispc_timeout_flag") != CUDA_SUCCESS) L.timeout_flag = 0;
  if (drv.ModuleGetFunction(&L.arm, L.mod, "ispc_arm") != CUDA_SUCCESS) L.arm = nullptr;
  // lazy module loading would upload each kernel at its first launch, on the
  // launching thread; load them all here (a compile thread, off the device's
  // critical path) instead
  unsigned nf = 0;
  if (drv.ModuleGetFunctionCount && drv.ModuleEnumerateFunctions && drv.FuncLoad &&
      drv.ModuleGetFunctionCount(&nf, L.mod) == CUDA_SUCCESS && nf > 0) {
    std::vector<CUfunction> fs(nf);
    if (drv.ModuleEnumerateFunctions(fs.data(), nf, L.mod) == CUDA_SUCCESS)
      for (CUfunction f : fs) drv.FuncLoad(f);
  }
  std::lock_guard<std::mutex> lk(d->mod_mu);
  *handle = d->next_handle++;
  d->modules[*handle] = std::move(L);
  return ISPC_OK;
}

int ispc_module_unload(ispc_dev* d, int handle) {
  if (!d) return ISPC_E_ARG;
  bind_ctx(d);
  CUmodule mod = nullptr;
  {
    std::lock_guard<std::mutex> lk(d->mod_mu);
    auto it = d->modules.find(handle);
    if (it == d->modules.end()) return fail(d, ISPC_E_ARG, "unknown module handle");
    mod = it->second.mod;
    d->modules.erase(it);
  }
  drv.ModuleUnload(mod);
  return ISPC_OK;
}

// ---- check ----------------------------------------------------------------------

int ispc_check(ispc_dev* d, double rtol, int bit_exact, double* max_err, int64_t* mismatches, int* ok) {
  if (!d || !d->bound) return fail(d, ISPC_E_ARG, "no problem bound");
  int rc = bind_ctx(d);
  if (rc) return rc;
  double worst = 0;
  int64_t bad = 0;
  for (const std::string& o : d->outputs) {
    CK(d, cudaMemsetAsync(d->cmp_res, 0, sizeof(ispc::CmpResult), d->stream));
    const Buffer& out = d->regions.at(o);
    const Buffer& exp = d->expected.at(o);
    auto sc = d->scale.find(o);
    const float* scale = (!bit_exact && sc != d->scale.end()) ? sc->second.ptr : nullptr;
    CK(d, ispc::launch_compare(out.ptr, exp.ptr, scale, out.elems, bit_exact, float(rtol), d->cmp_res, d->stream));
    ispc::CmpResult h{};
    CK(d, cudaMemcpyAsync(&h, d->cmp_res, sizeof(h), cudaMemcpyDeviceToHost, d->stream));
    CK(d, cudaStreamSynchronize(d->stream));
    float e;
    std::memcpy(&e, &h.max_err_bits, 4);
    worst = std::max(worst, double(e));
    bad += int64_t(h.mismatches);
  }
  if (max_err) *max_err = worst;
  if (mismatches) *mismatches = bad;
  if (ok) *ok = bad == 0;
  return ISPC_OK;
}

// ---- timed launches -------------------------------------------------------------------
//
// A batch of candidates of one module is evaluated with two host round trips
// in total, however many kernels it holds:
//   screen   per item: NaN-fill the outputs, [L2 flush], ispc_arm(budget),
//            event, the kernel, event, check (skipped on the device when the
//            watchdog fired) into the item's result slot
//   refine   per item whose screened time is at most `refine_below_ns` and
//            whose output checked: warmup launches, then `reps` timed groups
//            (one launch each, or R back-to-back launches over R input copies),
//            each group armed with its own budget and its watchdog flag
//            collected into the item's second slot
// Everything of a phase is enqueued before the host waits once on its last
// event; the watchdog deadline of each launch is set on the device by
// ispc_arm (emitted in every module's prelude) right before the launch, so a
// kernel queued behind others still gets its whole budget.

namespace {

struct Bound {  // one kernel with its parameters bound per rotation copy
  CUfunction fn = nullptr;
  const ispc_launch* L = nullptr;
  uint32_t R = 1;
  std::vector<std::vector<uint64_t>> stores;     // [copy][param]
  std::vector<std::vector<CUtensorMap>> tmaps;   // [copy][tmap]
  std::vector<int> tmap_of;                      // param -> tmap index or -1
  int deadline_slot = -1;
  bool clustered = false;
};

int get_function(ispc_dev* d, Loaded& mod, const ispc_launch* L, CUfunction* out) {
  auto fit = mod.fns.find(L->name);
  if (fit != mod.fns.end()) {
    *out = fit->second;
    return ISPC_OK;
  }
  CUfunction fn;
  CU(d, drv.ModuleGetFunction(&fn, mod.mod, L->name));
  if (L->static_smem > 48 * 1024)
    CU(d, drv.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, int(L->static_smem)));
  mod.fns[L->name] = fn;
  *out = fn;
  return ISPC_OK;
}

int ensure_rotation(ispc_dev* d, uint32_t R) {
  if (R <= 1 || d->rot.size() + 1 >= R) return ISPC_OK;
  CK(d, cudaStreamSynchronize(d->stream));
  while (d->rot.size() + 1 < R) {
    std::map<std::string, Buffer> copy;
    for (auto& [name, b] : d->regions) {
      if (d->expected.count(name)) continue;  // outputs are shared
      Buffer c;
      int rc = alloc(d, c, b.elems);
      if (rc) return rc;
      CK(d, cudaMemcpy(c.ptr, b.ptr, size_t(b.elems) * 4, cudaMemcpyDeviceToDevice));
      copy[name] = c;
    }
    d->rot.push_back(std::move(copy));
  }
  return ISPC_OK;
}

int bind_kernel(ispc_dev* d, Loaded& mod, const ispc_launch* L, uint32_t rotate, Bound& B) {
  int rc = get_function(d, mod, L, &B.fn);
  if (rc) return rc;
  if (L->grid_x == 0 || L->grid_x > 0x7fffffffull) return fail(d, ISPC_E_ILLEGAL, "grid out of range");
  // the hardware's per-dimension block limits (a schedule mapping a thread
  // level of 128 to threadIdx.z is not launchable: CUDA_ERROR_INVALID_VALUE)
  if (L->block[0] > 1024 || L->block[1] > 1024 || L->block[2] > 64)
    return fail(d, ISPC_E_ILLEGAL, "block dims " + std::to_string(L->block[0]) + " x " + std::to_string(L->block[1]) +
                                       " x " + std::to_string(L->block[2]) + " exceed x, y <= 1024, z <= 64");
  // the block the candidate asks for must fit the registers ptxas gave the
  // kernel (a static property of the compiled candidate, not a launch error)
  if (drv.FuncGetAttribute) {
    int max_threads = 0, regs = 0;
    if (drv.FuncGetAttribute(&max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, B.fn) == CUDA_SUCCESS &&
        drv.FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, B.fn) == CUDA_SUCCESS) {
      const uint64_t threads = uint64_t(L->block[0]) * std::max(1u, L->block[1]) * std::max(1u, L->block[2]);
      if (max_threads > 0 && threads > uint64_t(max_threads))
        return fail(d, ISPC_E_ILLEGAL, "block of " + std::to_string(threads) + " threads exceeds the " +
                                           std::to_string(max_threads) + " that " + std::to_string(regs) +
                                           " registers per thread allow");
    }
  }
  B.L = L;
  B.R = std::max<uint32_t>(1, std::min<uint32_t>(rotate, 16));
  if ((rc = ensure_rotation(d, B.R))) return rc;
  auto region_ptr = [&](uint32_t copy, const std::string& name) -> float* {
    if (copy > 0) {
      auto it = d->rot[copy - 1].find(name);
      if (it != d->rot[copy - 1].end()) return it->second.ptr;
    }
    auto it = d->regions.find(name);
    return it == d->regions.end() ? nullptr : it->second.ptr;
  };
  B.stores.assign(B.R, std::vector<uint64_t>(L->num_params, 0));
  B.tmaps.assign(B.R, std::vector<CUtensorMap>(L->num_tmaps));
  B.tmap_of.assign(L->num_params, -1);
  size_t next_scratch = 0;
  for (uint32_t i = 0; i < L->num_params; ++i) {
    const ispc_param& prm = L->params[i];
    if (prm.kind == ISPC_PARAM_REGION) {
      if (prm.is_input) {
        auto it = d->regions.find(prm.name);
        if (it == d->regions.end())
          return fail(d, ISPC_E_ARG, std::string("kernel region '") + prm.name + "' not in the bound problem");
        if (it->second.elems < prm.elems)
          return fail(d, ISPC_E_ARG, std::string("region '") + prm.name + "' smaller than the kernel's");
        for (uint32_t c = 0; c < B.R; ++c) B.stores[c][i] = reinterpret_cast<uint64_t>(region_ptr(c, prm.name));
      } else {
        // sized by grow_scratch() for every kernel of the batch beforehand
        if (next_scratch >= d->scratch.size() || d->scratch[next_scratch].elems < prm.elems)
          return fail(d, ISPC_E_ARG, "scratch pool not sized for the batch");
        Buffer& b = d->scratch[next_scratch++];
        for (uint32_t c = 0; c < B.R; ++c) B.stores[c][i] = reinterpret_cast<uint64_t>(b.ptr);
      }
    } else if (prm.kind == ISPC_PARAM_INPUT) {
      if (std::strcmp(prm.name, "alpha") != 0)
        return fail(d, ISPC_E_ARG, std::string("unknown scalar input ") + prm.name);
      float a = d->prob.alpha;
      for (uint32_t c = 0; c < B.R; ++c) std::memcpy(&B.stores[c][i], &a, 4);
    } else if (prm.kind == ISPC_PARAM_TMAP) {
      const ispc_tmap* tm = nullptr;
      uint32_t ti = 0;
      for (; ti < L->num_tmaps && ti < ISPC_MAX_TMAPS; ++ti)
        if (L->tmaps[ti].param == i) {
          tm = &L->tmaps[ti];
          break;
        }
      if (!tm) return fail(d, ISPC_E_ARG, "tensor-map parameter without a descriptor");
      if (!d->regions.count(tm->region))
        return fail(d, ISPC_E_ARG, std::string("tensor map over unknown region ") + tm->region);
      if (tm->rank < 2 || tm->rank > 3) return fail(d, ISPC_E_ARG, "tensor map rank");
      cuuint64_t dims[3] = {tm->dims[0], tm->dims[1], tm->dims[2]};
      cuuint64_t strides[2] = {tm->strides[0], tm->strides[1]};
      cuuint32_t box[3] = {tm->box[0], tm->box[1], tm->box[2]};
      cuuint32_t estr[3] = {1, 1, 1};
      static const CUtensorMapSwizzle sw[5] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                               CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B,
                                               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B};
      if (tm->swizzle > 4) return fail(d, ISPC_E_ARG, "tensor map swizzle mode");
      for (uint32_t c = 0; c < B.R; ++c)
        CU(d, drv.TensorMapEncodeTiled(&B.tmaps[c][ti], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, tm->rank,
                                       region_ptr(c, tm->region), dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw[tm->swizzle],
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
      B.tmap_of[i] = int(ti);
    } else {
      B.deadline_slot = int(i);
    }
  }
  B.clustered = L->cluster[0] * std::max(1u, L->cluster[1]) * std::max(1u, L->cluster[2]) > 1;
  if (B.clustered && L->grid_x % L->cluster[0] != 0) return fail(d, ISPC_E_ILLEGAL, "grid not a multiple of the cluster");
  return ISPC_OK;
}

// Enqueues one launch over rotation copy `copy`. `deadline`: the absolute
// deadline parameter (0: the device-armed one).
int enqueue(ispc_dev* d, Bound& B, uint32_t copy, uint64_t deadline) {
  const ispc_launch* L = B.L;
  void* args[ISPC_MAX_PARAMS];
  for (uint32_t i = 0; i < L->num_params; ++i) {
    if (int(i) == B.deadline_slot) B.stores[copy][i] = deadline;
    args[i] = B.tmap_of[i] >= 0 ? static_cast<void*>(&B.tmaps[copy][size_t(B.tmap_of[i])])
                                : static_cast<void*>(&B.stores[copy][i]);
  }
  if (B.clustered || L->pdl) {
    CUlaunchConfig cfg{};
    cfg.gridDimX = unsigned(L->grid_x);
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = L->block[0];
    cfg.blockDimY = L->block[1];
    cfg.blockDimZ = L->block[2];
    cfg.sharedMemBytes = L->static_smem;
    cfg.hStream = reinterpret_cast<CUstream>(d->stream);
    CUlaunchAttribute attr[2]{};
    unsigned na = 0;
    if (B.clustered) {
      attr[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      attr[na].value.clusterDim.x = L->cluster[0];
      attr[na].value.clusterDim.y = std::max(1u, L->cluster[1]);
      attr[na].value.clusterDim.z = std::max(1u, L->cluster[2]);
      ++na;
    }
    if (L->pdl) {  // the kernel opens with griddepcontrol.wait (ispc.h: ispc_launch.pdl)
      attr[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      attr[na].value.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CU(d, drv.LaunchKernelEx(&cfg, B.fn, args, nullptr));
  } else {
    CU(d, drv.LaunchKernel(B.fn, unsigned(L->grid_x), 1, 1, L->block[0], L->block[1], L->block[2], L->static_smem,
                           reinterpret_cast<CUstream>(d->stream), args, nullptr));
  }
  return ISPC_OK;
}

// Sets the device deadline `budget_ns` from now (when the stream reaches it)
// and clears the module's watchdog flag. Without an arm kernel (a module not
// built from the prelude) the deadline is computed on the host instead.
int arm(ispc_dev* d, Loaded& mod, double budget_ns, uint64_t* host_deadline) {
  *host_deadline = 0;
  if (mod.arm) {
    unsigned long long b = (unsigned long long)std::max(0.0, budget_ns);
    void* args[1] = {&b};
    CU(d, drv.LaunchKernel(mod.arm, 1, 1, 1, 1, 1, 1, 0, reinterpret_cast<CUstream>(d->stream), args, nullptr));
  } else {
    if (mod.timeout_flag) CU(d, drv.MemsetD32Async(mod.timeout_flag, 0, 1, reinterpret_cast<CUstream>(d->stream)));
    *host_deadline = uint64_t(host_ns() + d->gt_offset_ns + budget_ns);
  }
  return ISPC_OK;
}

// GLOBAL temporaries come from a per-device pool: the j-th temporary of every
// kernel shares buffer j (the kernels of a stream never overlap), sized for
// the largest j-th temporary of the batch before anything is enqueued.
int grow_scratch(ispc_dev* d, int n, const ispc_batch_item* items) {
  std::vector<int64_t> need;
  for (int i = 0; i < n; ++i) {
    size_t j = 0;
    const ispc_launch* L = items[i].launch;
    for (uint32_t p = 0; p < L->num_params; ++p)
      if (L->params[p].kind == ISPC_PARAM_REGION && !L->params[p].is_input) {
        if (need.size() <= j) need.push_back(0);
        need[j] = std::max(need[j], L->params[p].elems);
        ++j;
      }
  }
  bool synced = false;
  for (size_t j = 0; j < need.size(); ++j) {
    if (j == d->scratch.size()) d->scratch.push_back(Buffer{});
    Buffer& b = d->scratch[j];
    if (b.elems >= need[j]) continue;
    if (!synced) {  // the pool may be in use by kernels still queued
      CK(d, cudaStreamSynchronize(d->stream));
      synced = true;
    }
    cudaFree(b.ptr);
    b = Buffer{};
    int rc = alloc(d, b, need[j]);
    if (rc) return rc;
  }
  return ISPC_OK;
}

cudaEvent_t event_at(ispc_dev* d, size_t i) {
  while (d->evpool.size() <= i) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    d->evpool.push_back(e);
  }
  return d->evpool[i];
}

int slots_for(ispc_dev* d, size_t n) {
  if (d->slot_cap >= n) return ISPC_OK;
  CK(d, cudaStreamSynchronize(d->stream));
  if (d->slots) cudaFree(d->slots);
  d->slots = nullptr;
  d->slot_cap = 0;
  size_t cap = std::max<size_t>(64, n);
  CK(d, cudaMalloc(&d->slots, cap * sizeof(ispc::CmpResult)));
  d->slot_cap = cap;
  return ISPC_OK;
}

// Waits for `ev`, polling so that a kernel outliving every watchdog is
// reported as a context-killing fault instead of blocking forever.
int wait_event(ispc_dev* d, cudaEvent_t ev, double limit_ns, const char* what) {
  const double t_wait = host_ns();
  for (int spin = 0;; ++spin) {
    cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return ISPC_OK;
    if (q != cudaErrorNotReady) return cuda_fail(d, q, "kernel");
    if (host_ns() - t_wait > limit_ns)
      return fail(d, ISPC_E_STICKY, std::string("kernel ") + what + " still running after " +
                                        std::to_string(int(limit_ns / 1e9)) + " s (host guard)");
    if (spin < 64) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(10));
  }
}

int flush_l2(ispc_dev* d) {
  // write a buffer larger than L2, then read it back (clean L2, no pending write-backs)
  CK(d, cudaMemsetAsync(d->flush, int(flush_counter_++ & 0xff), d->flush_bytes, d->stream));
  CK(d, ispc::launch_flush_read(d->flush, d->flush_bytes, d->cmp_res, d->stream));
  return ISPC_OK;
}

}  // namespace

int ispc_launch_batch(ispc_dev* d, int handle, int n, const ispc_batch_item* items, double refine_below_ns,
                      ispc_time_result* res) {
  if (!d || n < 0 || (n > 0 && (!items || !res))) return fail(d, ISPC_E_ARG, "null argument");
  if (!d->bound) return fail(d, ISPC_E_ARG, "no problem bound");
  if (n == 0) return ISPC_OK;
  int rc = bind_ctx(d);
  if (rc) return rc;
  Loaded* modp = nullptr;
  {
    std::lock_guard<std::mutex> lk(d->mod_mu);
    auto mit = d->modules.find(handle);
    if (mit == d->modules.end()) return fail(d, ISPC_E_ARG, "unknown module handle");
    modp = &mit->second;
  }
  Loaded& mod = *modp;
  const int* flag = reinterpret_cast<const int*>(mod.timeout_flag);
  for (int i = 0; i < n; ++i) {
    std::memset(&res[i], 0, sizeof(res[i]));
    if (!items[i].launch) return fail(d, ISPC_E_ARG, "null launch");
  }
  if ((rc = slots_for(d, size_t(2 * n)))) return rc;
  auto* slots = static_cast<ispc::CmpResult*>(d->slots);
  CK(d, cudaMemsetAsync(slots, 0, size_t(2 * n) * sizeof(ispc::CmpResult), d->stream));

  if ((rc = grow_scratch(d, n, items))) return rc;
  std::vector<Bound> B(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i)
    if ((rc = bind_kernel(d, mod, items[i].launch, items[i].opts.rotate, B[size_t(i)]))) {
      // report the failing item, keep the others
      res[i].status = rc;
    }

  // ---- screen -------------------------------------------------------------------
  double guard_ns = 0;
  size_t ev = 0;
  std::vector<size_t> first_ev(size_t(n), SIZE_MAX);
  for (int i = 0; i < n; ++i) {
    if (res[i].status) continue;
    const ispc_time_opts& o = items[i].opts;
    const double budget = o.budget_ns > 0 ? o.budget_ns : 2e9;
    for (const std::string& out : d->outputs) {
      const Buffer& b = d->regions.at(out);
      CK(d, cudaMemsetAsync(b.ptr, 0xff, size_t(b.elems) * 4, d->stream));
    }
    if (o.flush_l2 && (rc = flush_l2(d))) return rc;
    uint64_t dl = 0;
    if ((rc = arm(d, mod, budget, &dl))) return rc;
    cudaEvent_t e0 = event_at(d, ev), e1 = event_at(d, ev + 1);
    if (!e0 || !e1) return fail(d, ISPC_E_CUDA, "cudaEventCreate failed");
    first_ev[size_t(i)] = ev;
    ev += 2;
    CK(d, cudaEventRecord(e0, d->stream));
    if ((rc = enqueue(d, B[size_t(i)], 0, dl))) {
      if (rc == ISPC_E_STICKY) return rc;
      res[i].status = rc;  // this kernel alone cannot launch; the batch goes on
      first_ev[size_t(i)] = SIZE_MAX;
      ev -= 2;
      continue;
    }
    CK(d, cudaEventRecord(e1, d->stream));
    guard_ns += std::max(5e9, 40.0 * budget);
    ispc::CmpResult* slot = slots + i;
    if (o.check) {
      for (const std::string& out_name : d->outputs) {
        const Buffer& out = d->regions.at(out_name);
        const Buffer& exp = d->expected.at(out_name);
        auto sc = d->scale.find(out_name);
        const float* scale = (!o.bit_exact && sc != d->scale.end()) ? sc->second.ptr : nullptr;
        CK(d, ispc::launch_check(out.ptr, exp.ptr, scale, out.elems, int(o.bit_exact), float(o.rtol), flag, slot,
                                 d->stream));
      }
    } else if (flag) {
      CK(d, ispc::launch_collect(flag, slot, d->stream));
    }
  }
  if (ev == 0) return ISPC_OK;
  if ((rc = wait_event(d, d->evpool[ev - 1], guard_ns, items[0].launch->name))) return rc;
  std::vector<ispc::CmpResult> h(size_t(2 * n));
  CK(d, cudaMemcpy(h.data(), slots, size_t(n) * sizeof(ispc::CmpResult), cudaMemcpyDeviceToHost));
  std::vector<char> refine(size_t(n), 0);
  bool any_refine = false;
  for (int i = 0; i < n; ++i) {
    if (res[i].status) continue;
    const ispc_time_opts& o = items[i].opts;
    const double budget = o.budget_ns > 0 ? o.budget_ns : 2e9;
    float ms = 0;
    CK(d, cudaEventElapsedTime(&ms, d->evpool[first_ev[size_t(i)]], d->evpool[first_ev[size_t(i)] + 1]));
    res[i].first_ns = double(ms) * 1e6;
    if (h[size_t(i)].timeout) {
      res[i].status = ISPC_E_TIMEOUT;
      res[i].median_ns = res[i].min_ns = std::max(res[i].first_ns, budget);
      continue;
    }
    if (o.check) {
      float e;
      std::memcpy(&e, &h[size_t(i)].max_err_bits, 4);
      res[i].max_err = e;
      res[i].mismatches = int64_t(h[size_t(i)].mismatches);
      if (res[i].mismatches) {
        res[i].status = ISPC_E_MISMATCH;
        res[i].median_ns = res[i].min_ns = res[i].first_ns;
        continue;
      }
    }
    res[i].median_ns = res[i].min_ns = res[i].first_ns;
    if (o.reps > 0 && !(res[i].first_ns > refine_below_ns)) {
      refine[size_t(i)] = 1;
      any_refine = true;
    }
  }
  if (!any_refine) return ISPC_OK;

  // ---- refine -------------------------------------------------------------------
  guard_ns = 0;
  ev = 0;
  struct Group {
    int item;
    size_t ev;
    uint32_t count;
  };
  std::vector<Group> groups;
  for (int i = 0; i < n; ++i) {
    if (!refine[size_t(i)]) continue;
    const ispc_time_opts& o = items[i].opts;
    const double budget = o.budget_ns > 0 ? o.budget_ns : 2e9;
    Bound& b = B[size_t(i)];
    ispc::CmpResult* slot = slots + n + i;
    uint64_t dl = 0;
    for (uint32_t w = 0; w < o.warmup; ++w) {
      if (o.flush_l2 && (rc = flush_l2(d))) return rc;
      if ((rc = arm(d, mod, budget, &dl))) return rc;
      if ((rc = enqueue(d, b, 0, dl))) return rc;
      if (flag) CK(d, ispc::launch_collect(flag, slot, d->stream));
      guard_ns += std::max(5e9, 40.0 * budget);
    }
    // rotation: groups of R back-to-back launches over the R input copies
    // (each launch reads inputs untouched for R-1 launches, i.e. not in L2),
    // mean per launch; else one launch per event pair
    const uint32_t R = b.R;
    const uint32_t ngroups = R > 1 ? std::max<uint32_t>(1, (o.reps + R - 1) / R) : o.reps;
    for (uint32_t g = 0; g < ngroups; ++g) {
      if (R == 1 && o.flush_l2 && (rc = flush_l2(d))) return rc;
      if ((rc = arm(d, mod, budget * R, &dl))) return rc;  // R launches share one armed deadline
      cudaEvent_t e0 = event_at(d, ev), e1 = event_at(d, ev + 1);
      if (!e0 || !e1) return fail(d, ISPC_E_CUDA, "cudaEventCreate failed");
      CK(d, cudaEventRecord(e0, d->stream));
      for (uint32_t k = 0; k < R; ++k)
        if ((rc = enqueue(d, b, k % R, dl))) return rc;
      CK(d, cudaEventRecord(e1, d->stream));
      if (flag) CK(d, ispc::launch_collect(flag, slot, d->stream));
      groups.push_back(Group{i, ev, R});
      ev += 2;
      guard_ns += std::max(5e9, 40.0 * budget * R);
    }
  }
  if (ev == 0) return ISPC_OK;
  if ((rc = wait_event(d, d->evpool[ev - 1], guard_ns, items[0].launch->name))) return rc;
  CK(d, cudaMemcpy(h.data() + n, slots + n, size_t(n) * sizeof(ispc::CmpResult), cudaMemcpyDeviceToHost));
  std::vector<std::vector<double>> times(static_cast<size_t>(n));
  for (const Group& g : groups) {
    float ms = 0;
    CK(d, cudaEventElapsedTime(&ms, d->evpool[g.ev], d->evpool[g.ev + 1]));
    times[size_t(g.item)].push_back(double(ms) * 1e6 / g.count);
  }
  for (int i = 0; i < n; ++i) {
    if (!refine[size_t(i)] || times[size_t(i)].empty()) continue;
    std::vector<double>& t = times[size_t(i)];
    std::sort(t.begin(), t.end());
    res[i].median_ns = t[t.size() / 2];
    res[i].min_ns = t.front();
    if (h[size_t(n + i)].timeout) res[i].status = ISPC_E_TIMEOUT;
  }
  return ISPC_OK;
}

int ispc_launch_timed(ispc_dev* d, int handle, const ispc_launch* L, const ispc_time_opts* o,
                      ispc_time_result* res) {
  if (!d || !L || !o || !res) return fail(d, ISPC_E_ARG, "null argument");
  ispc_batch_item it{};
  it.launch = L;
  it.opts = *o;
  int rc = ispc_launch_batch(d, handle, 1, &it, std::numeric_limits<double>::infinity(), res);
  if (rc) return rc;
  // a launch-level failure of the single item is the call's failure
  if (res->status != ISPC_OK && res->status != ISPC_E_TIMEOUT && res->status != ISPC_E_MISMATCH) return res->status;
  return ISPC_OK;
}

int ispc_dev_mark(ispc_dev* d, int slot) {
  if (!d || slot < 0 || slot >= 8) return fail(d, ISPC_E_ARG, "bad mark slot");
  int rc = bind_ctx(d);
  if (rc) return rc;
  if (!d->marks[slot]) CK(d, cudaEventCreate(&d->marks[slot]));
  CK(d, cudaEventRecord(d->marks[slot], d->stream));
  return ISPC_OK;
}

int ispc_dev_mark_elapsed(ispc_dev* d, int a, int b, double* ms) {
  if (!d || a < 0 || a >= 8 || b < 0 || b >= 8 || !d->marks[a] || !d->marks[b] || !ms)
    return fail(d, ISPC_E_ARG, "bad mark slots");
  int rc = bind_ctx(d);
  if (rc) return rc;
  CK(d, cudaEventSynchronize(d->marks[b]));
  float f = 0;
  CK(d, cudaEventElapsedTime(&f, d->marks[a], d->marks[b]));
  *ms = f;
  return ISPC_OK;
}

int ispc_host_register(void* p, size_t bytes) {
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, ISPC_E_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  }
  return ISPC_OK;
}

int ispc_host_unregister(void* p) {
  cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, ISPC_E_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
  }
  return ISPC_OK;
}

// ---- one-shot evaluate -----------------------------------------------------------------

int ispc_evaluate(ispc_dev* d, const ispc_nest* nest, const ispc_emit_opts* eopts, const ispc_time_opts* topts,
                  ispc_time_result* res, ispc_launch* launch) {
  if (!d || !nest || !topts || !res) return fail(d, ISPC_E_ARG, "null argument");
  ispc_launch L{};
  size_t len = 0;
  int rc = ispc_emit_cuda(nest, eopts, nullptr, nullptr, 0, &len, &L);
  if (rc) return fail(d, rc, ispc::thread_error());
  std::string src(len + 1, '\0');
  if ((rc = ispc_emit_cuda(nest, eopts, nullptr, src.data(), src.size(), &len, &L)))
    return fail(d, rc, ispc::thread_error());
  src.resize(len);
  if (launch) *launch = L;
  const char* srcs[] = {src.c_str()};
  ispc_module* m = nullptr;
  if ((rc = ispc_compile(srcs, 1, nullptr, &m))) return fail(d, rc, ispc::thread_error());
  std::unique_ptr<ispc_module, void (*)(ispc_module*)> guard(m, ispc_module_free);
  int h = 0;
  if ((rc = ispc_module_load(d, m, &h))) return rc;
  rc = ispc_launch_timed(d, h, &L, topts, res);
  ispc_module_unload(d, h);
  return rc;
}

int ispc_evaluate_tiles(ispc_dev* d, const ispc_tile_config* cfg, const ispc_time_opts* topts,
                        ispc_time_result* res, ispc_launch* launch) {
  if (!d || !cfg || !topts || !res) return fail(d, ISPC_E_ARG, "null argument");
  ispc_launch L{};
  size_t len = 0;
  int rc = ispc_emit_tiles(cfg, nullptr, nullptr, 0, &len, &L);
  if (rc) return fail(d, rc, ispc::thread_error());
  std::string src(len + 1, '\0');
  if ((rc = ispc_emit_tiles(cfg, nullptr, src.data(), src.size(), &len, &L))) return fail(d, rc, ispc::thread_error());
  src.resize(len);
  if (launch) *launch = L;
  const char* srcs[] = {src.c_str()};
  ispc_module* m = nullptr;
  if ((rc = ispc_compile(srcs, 1, nullptr, &m))) return fail(d, rc, ispc::thread_error());
  std::unique_ptr<ispc_module, void (*)(ispc_module*)> guard(m, ispc_module_free);
  int h = 0;
  if ((rc = ispc_module_load(d, m, &h))) return rc;
  rc = ispc_launch_timed(d, h, &L, topts, res);
  ispc_module_unload(d, h);
  return rc;
}

}  // extern "C"
