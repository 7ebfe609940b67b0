// libdpia_rt: NVRTC + CUDA driver API + NCCL behind a C ABI (include/dpia_rt.h).
#include "dpia_rt.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

// ---------------------------------------------------------------------------
// The CUDA driver is loaded with dlopen so the library itself loads (and its
// symbols can be inspected) on machines without a GPU driver.  Names go
// through the cuda.h macros (e.g. cuMemAlloc -> cuMemAlloc_v2) before lookup.
#define DPIA_STR2(x) #x
#define DPIA_STR(x) DPIA_STR2(x)
#define DPIA_DRIVER_FUNCS(X)                                                              \
  X(cuInit) X(cuGetErrorString) X(cuDeviceGet) X(cuDeviceGetCount) X(cuDeviceGetAttribute)   \
  X(cuDeviceGetName) X(cuDevicePrimaryCtxRetain) X(cuCtxSetCurrent) X(cuCtxSynchronize)      \
  X(cuModuleLoadData) X(cuModuleUnload) X(cuModuleGetFunction) X(cuFuncSetAttribute)         \
  X(cuFuncGetAttribute) X(cuMemAlloc) X(cuMemFree) X(cuMemAllocHost) X(cuMemFreeHost)        \
  X(cuMemcpyHtoD) X(cuMemcpyDtoH) X(cuMemcpyHtoDAsync) X(cuMemcpyDtoHAsync)                  \
  X(cuMemcpyDtoDAsync) X(cuMemsetD8Async) X(cuMemsetD32Async) X(cuLaunchKernel)              \
  X(cuStreamCreate) X(cuStreamDestroy) X(cuStreamSynchronize) X(cuEventCreate)               \
  X(cuEventDestroy) X(cuEventRecord) X(cuEventSynchronize) X(cuEventElapsedTime)          \
  X(cuIpcGetMemHandle) X(cuIpcOpenMemHandle) X(cuIpcCloseMemHandle) X(cuStreamWaitEvent)   \
  X(cuCtxGetCurrent) X(cuMemcpy2DAsync)

namespace drv {
#define DPIA_DECL(f) decltype(&::f) f = nullptr;
DPIA_DRIVER_FUNCS(DPIA_DECL)
#undef DPIA_DECL
// optional: without it, dpia_launch_pdl degrades to an ordinary launch (the
// kernels' griddepcontrol.wait is then a no-op and ordering is the stream's)
decltype(&::cuLaunchKernelEx) cuLaunchKernelEx = nullptr;
decltype(&::cuTensorMapEncodeTiled) cuTensorMapEncodeTiled = nullptr;
}  // namespace drv

// NVRTC is loaded the same way, by the absolute path of the toolkit the
// runtime was built against (DPIA_NVRTC_PATH, set by runtime.build_lib;
// $DPIA_NVRTC overrides), with RTLD_LOCAL: a process that already loaded an
// older libnvrtc.so.12 (PyTorch ships one) would otherwise bind these calls
// to it by SONAME, and an older NVRTC rejects sm_100 PTX such as the 256-bit
// ld.global.v8.f32 the emitter uses.
#define DPIA_NVRTC_FUNCS(X)                                                              \
  X(nvrtcCreateProgram) X(nvrtcCompileProgram) X(nvrtcGetProgramLogSize)                  \
  X(nvrtcGetProgramLog) X(nvrtcDestroyProgram) X(nvrtcGetCUBINSize) X(nvrtcGetCUBIN)      \
  X(nvrtcGetErrorString) X(nvrtcVersion)

#ifndef DPIA_NVRTC_PATH
#define DPIA_NVRTC_PATH "libnvrtc.so.12"
#endif

namespace rtc {
#define DPIA_DECL(f) decltype(&::f) f = nullptr;
DPIA_NVRTC_FUNCS(DPIA_DECL)
#undef DPIA_DECL
}  // namespace rtc

namespace {

thread_local std::string g_err;
void* g_libcuda = nullptr;
void* g_libnvrtc = nullptr;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code ? code : -1;
}

int load_driver() {
  if (g_libcuda) return 0;
  g_libcuda = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!g_libcuda) g_libcuda = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
  if (!g_libcuda) return fail(-1, "cannot load the CUDA driver (libcuda.so.1): %s", dlerror());
#define DPIA_LOAD(f)                                                         \
  drv::f = reinterpret_cast<decltype(drv::f)>(dlsym(g_libcuda, DPIA_STR(f))); \
  if (!drv::f) return fail(-1, "CUDA driver lacks %s", DPIA_STR(f));
  DPIA_DRIVER_FUNCS(DPIA_LOAD)
#undef DPIA_LOAD
  drv::cuLaunchKernelEx =
      reinterpret_cast<decltype(drv::cuLaunchKernelEx)>(dlsym(g_libcuda, DPIA_STR(cuLaunchKernelEx)));
  drv::cuTensorMapEncodeTiled = reinterpret_cast<decltype(drv::cuTensorMapEncodeTiled)>(
      dlsym(g_libcuda, DPIA_STR(cuTensorMapEncodeTiled)));
  return 0;
}

int load_nvrtc() {
  if (g_libnvrtc) return 0;
  static std::mutex m;
  std::lock_guard<std::mutex> lock(m);
  if (g_libnvrtc) return 0;
  const char* env = getenv("DPIA_NVRTC");
  void* h = dlopen(env && *env ? env : DPIA_NVRTC_PATH, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(-1, "cannot load NVRTC (%s): %s", DPIA_NVRTC_PATH, dlerror());
#define DPIA_LOAD(f)                                                    \
  rtc::f = reinterpret_cast<decltype(rtc::f)>(dlsym(h, DPIA_STR(f)));   \
  if (!rtc::f) return fail(-1, "NVRTC lacks %s", DPIA_STR(f));
  DPIA_NVRTC_FUNCS(DPIA_LOAD)
#undef DPIA_LOAD
  g_libnvrtc = h;
  return 0;
}

int cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return 0;
  const char* s = nullptr;
  drv::cuGetErrorString(r, &s);
  return fail(static_cast<int>(r), "%s: %s (%d)", what, s ? s : "?", static_cast<int>(r));
}

#define CU(call)                                \
  do {                                          \
    int _e = cu((call), #call);                 \
    if (_e) return _e;                          \
  } while (0)

constexpr int kMaxDev = 64;
CUcontext g_ctx[kMaxDev] = {};
std::mutex g_mu;

int bind(int dev) {
  if (dev < 0 || dev >= kMaxDev) return fail(-1, "bad device %d", dev);
  if (!g_ctx[dev]) {
    int e = dpia_init(dev);
    if (e) return e;
  }
  CU(drv::cuCtxSetCurrent(g_ctx[dev]));
  return 0;
}

// ------------------------------------------------------------ hash filler
const char* kFillSrc = R"(
extern "C" __global__ void dpia_fill_hash_f32(float* out, unsigned long long n,
    unsigned long long offset, unsigned int seed, float lo, float hi) {
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    unsigned long long k = offset + i;
    unsigned int h = (unsigned int)(k) * 0x9E3779B1u ^ (unsigned int)(k >> 32) * 0x85EBCA77u ^ seed;
    h ^= h >> 16; h *= 0x7FEB352Du; h ^= h >> 15; h *= 0x846CA68Bu; h ^= h >> 16;
    out[i] = __fadd_rn(lo, __fmul_rn(hi - lo, (float)(h >> 8) * (1.0f / 16777216.0f)));
  }
}
)";
// L2 eviction by *reading* a 2x-L2 buffer: leaves only clean lines behind, so
// the next timed kernel pays no write-back for the flush itself.
const char* kScrubSrc = R"(
extern "C" __global__ void dpia_l2_scrub(const uint4* p, unsigned long long n, unsigned int* sink) {
  unsigned int acc = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}
)";
CUmodule g_fill_mod[kMaxDev] = {};
CUfunction g_fill_fn[kMaxDev] = {};
CUfunction g_scrub_fn[kMaxDev] = {};
CUdeviceptr g_flush_buf[kMaxDev] = {};
size_t g_flush_bytes[kMaxDev] = {};

// ------------------------------------------------------------------ NCCL
typedef struct { char internal[128]; } ncclUniqueId_t;
typedef void* ncclComm_t;
typedef int (*nccl_get_id_fn)(ncclUniqueId_t*);
typedef int (*nccl_init_rank_fn)(ncclComm_t*, int, ncclUniqueId_t, int);
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, ncclComm_t, CUstream);
typedef int (*nccl_destroy_fn)(ncclComm_t);
typedef const char* (*nccl_err_fn)(int);
void* g_nccl = nullptr;
nccl_get_id_fn p_get_id = nullptr;
nccl_init_rank_fn p_init_rank = nullptr;
nccl_allreduce_fn p_allreduce = nullptr;
nccl_destroy_fn p_destroy = nullptr;
nccl_err_fn p_errstr = nullptr;
ncclComm_t g_comm = nullptr;

int load_nccl() {
  if (g_nccl) return 0;
  const char* env = getenv("DPIA_NCCL_LIB");
  const char* cands[] = {env, "libnccl.so.2", "libnccl.so",
                         "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
  for (const char* c : cands) {
    if (!c) continue;
    g_nccl = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl) break;
  }
  if (!g_nccl) return fail(-1, "cannot dlopen libnccl.so.2 (set DPIA_NCCL_LIB)");
  p_get_id = (nccl_get_id_fn)dlsym(g_nccl, "ncclGetUniqueId");
  p_init_rank = (nccl_init_rank_fn)dlsym(g_nccl, "ncclCommInitRank");
  p_allreduce = (nccl_allreduce_fn)dlsym(g_nccl, "ncclAllReduce");
  p_destroy = (nccl_destroy_fn)dlsym(g_nccl, "ncclCommDestroy");
  p_errstr = (nccl_err_fn)dlsym(g_nccl, "ncclGetErrorString");
  if (!p_get_id || !p_init_rank || !p_allreduce || !p_destroy)
    return fail(-1, "libnccl is missing required symbols");
  return 0;
}

int nccl(int r, const char* what) {
  if (r == 0) return 0;
  return fail(r, "%s: %s", what, p_errstr ? p_errstr(r) : "nccl error");
}

}  // namespace

extern "C" {

const char* dpia_last_error(void) { return g_err.c_str(); }

int dpia_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (device < 0 || device >= kMaxDev) return fail(-1, "bad device %d", device);
  if (int e = load_driver()) return e;
  CU(drv::cuInit(0));
  if (!g_ctx[device]) {
    CUdevice d;
    CU(drv::cuDeviceGet(&d, device));
    CU(drv::cuDevicePrimaryCtxRetain(&g_ctx[device], d));
  }
  CU(drv::cuCtxSetCurrent(g_ctx[device]));
  return 0;
}

int dpia_device_count(int* count) {
  if (int e = load_driver()) return e;
  CU(drv::cuInit(0));
  CU(drv::cuDeviceGetCount(count));
  return 0;
}

int dpia_device_attribute(int device, int attr, int* value) {
  if (int e = load_driver()) return e;
  CU(drv::cuInit(0));
  CUdevice d;
  CU(drv::cuDeviceGet(&d, device));
  CU(drv::cuDeviceGetAttribute(value, static_cast<CUdevice_attribute>(attr), d));
  return 0;
}

int dpia_device_name(int device, char* buf, int len) {
  if (int e = load_driver()) return e;
  CU(drv::cuInit(0));
  CUdevice d;
  CU(drv::cuDeviceGet(&d, device));
  CU(drv::cuDeviceGetName(buf, len, d));
  return 0;
}

int dpia_nvrtc_version(int* major, int* minor) {
  if (int e = load_nvrtc()) return e;
  nvrtcResult r = rtc::nvrtcVersion(major, minor);
  return r == NVRTC_SUCCESS ? 0 : fail(r, "nvrtcVersion: %s", rtc::nvrtcGetErrorString(r));
}

int dpia_compile(const char* source, const char* program_name, const char* arch,
                 const char* options, void** image, size_t* size, char* log, size_t logcap) {
  if (log && logcap) log[0] = 0;
  if (int e = load_nvrtc()) return e;
  nvrtcProgram prog;
  nvrtcResult r = rtc::nvrtcCreateProgram(&prog, source, program_name, 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(r, "nvrtcCreateProgram: %s", rtc::nvrtcGetErrorString(r));
  std::vector<std::string> opts;
  opts.push_back(std::string("--gpu-architecture=") + (arch && *arch ? arch : "sm_100a"));
  opts.push_back("--std=c++17");
  if (options) {
    std::string all(options);
    size_t pos = 0;
    while (pos <= all.size()) {
      size_t nl = all.find('\n', pos);
      std::string o = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
      if (!o.empty()) opts.push_back(o);
      if (nl == std::string::npos) break;
      pos = nl + 1;
    }
  }
  std::vector<const char*> cops;
  for (auto& o : opts) cops.push_back(o.c_str());
  r = rtc::nvrtcCompileProgram(prog, static_cast<int>(cops.size()), cops.data());
  size_t lsz = 0;
  rtc::nvrtcGetProgramLogSize(prog, &lsz);
  if (log && logcap && lsz > 1) {
    std::string l(lsz, '\0');
    rtc::nvrtcGetProgramLog(prog, &l[0]);
    size_t n = lsz < logcap ? lsz : logcap - 1;
    memcpy(log, l.data(), n);
    log[n] = 0;
  }
  if (r != NVRTC_SUCCESS) {
    rtc::nvrtcDestroyProgram(&prog);
    return fail(r, "nvrtcCompileProgram: %s (see log)", rtc::nvrtcGetErrorString(r));
  }
  size_t n = 0;
  r = rtc::nvrtcGetCUBINSize(prog, &n);
  if (r != NVRTC_SUCCESS) {
    rtc::nvrtcDestroyProgram(&prog);
    return fail(r, "nvrtcGetCUBINSize: %s", rtc::nvrtcGetErrorString(r));
  }
  void* buf = malloc(n);
  r = rtc::nvrtcGetCUBIN(prog, static_cast<char*>(buf));
  rtc::nvrtcDestroyProgram(&prog);
  if (r != NVRTC_SUCCESS) {
    free(buf);
    return fail(r, "nvrtcGetCUBIN: %s", rtc::nvrtcGetErrorString(r));
  }
  *image = buf;
  *size = n;
  return 0;
}

void dpia_free_host(void* ptr) { free(ptr); }

int dpia_module_load(int device, const void* image, void** module) {
  if (int e = bind(device)) return e;
  CUmodule m;
  CU(drv::cuModuleLoadData(&m, image));
  *module = m;
  return 0;
}

int dpia_module_unload(void* module) {
  CU(drv::cuModuleUnload(static_cast<CUmodule>(module)));
  return 0;
}

int dpia_get_kernel(void* module, const char* name, void** function) {
  CUfunction f;
  CU(drv::cuModuleGetFunction(&f, static_cast<CUmodule>(module), name));
  *function = f;
  return 0;
}

int dpia_kernel_set_smem(void* function, int bytes) {
  CU(drv::cuFuncSetAttribute(static_cast<CUfunction>(function),
                        CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, bytes));
  return 0;
}

int dpia_kernel_attribute(void* function, int attr, int* value) {
  CU(drv::cuFuncGetAttribute(value, static_cast<CUfunction_attribute>(attr),
                        static_cast<CUfunction>(function)));
  return 0;
}

int dpia_malloc(int device, size_t bytes, uint64_t* dptr) {
  if (int e = bind(device)) return e;
  CUdeviceptr p = 0;
  CU(drv::cuMemAlloc(&p, bytes ? bytes : 16));
  *dptr = static_cast<uint64_t>(p);
  return 0;
}

int dpia_free(int device, uint64_t dptr) {
  if (int e = bind(device)) return e;
  CU(drv::cuMemFree(static_cast<CUdeviceptr>(dptr)));
  return 0;
}

int dpia_host_alloc(size_t bytes, void** ptr) {
  // page-locked memory belongs to a context: use the current one, or bind
  // device 0 when the caller has not initialised any device yet
  if (int e = load_driver()) return e;
  CU(drv::cuInit(0));
  CUcontext cur = nullptr;
  if (drv::cuCtxGetCurrent(&cur) != CUDA_SUCCESS || !cur) {
    if (int e = bind(0)) return e;
  }
  CU(drv::cuMemAllocHost(ptr, bytes ? bytes : 16));
  return 0;
}

int dpia_host_free(void* ptr) {
  CU(drv::cuMemFreeHost(ptr));
  return 0;
}

int dpia_memcpy_htod(int device, uint64_t dst, const void* src, size_t bytes, void* stream) {
  if (int e = bind(device)) return e;
  if (stream) CU(drv::cuMemcpyHtoDAsync(dst, src, bytes, static_cast<CUstream>(stream)));
  else CU(drv::cuMemcpyHtoD(dst, src, bytes));
  return 0;
}

int dpia_memcpy_dtoh(int device, void* dst, uint64_t src, size_t bytes, void* stream) {
  if (int e = bind(device)) return e;
  if (stream) CU(drv::cuMemcpyDtoHAsync(dst, src, bytes, static_cast<CUstream>(stream)));
  else CU(drv::cuMemcpyDtoH(dst, src, bytes));
  return 0;
}

// Strided (pitched) copies: `height` rows of `width` bytes, consecutive rows
// `spitch` bytes apart in the source and `dpitch` bytes apart in the
// destination (a column panel of a row-major host matrix <-> a contiguous
// device panel).  Asynchronous on `stream`.
int dpia_memcpy2d_htod(int device, uint64_t dst, size_t dpitch, const void* src, size_t spitch,
                       size_t width, size_t height, void* stream) {
  if (int e = bind(device)) return e;
  CUDA_MEMCPY2D c;
  std::memset(&c, 0, sizeof(c));
  c.srcMemoryType = CU_MEMORYTYPE_HOST;
  c.srcHost = src;
  c.srcPitch = spitch;
  c.dstMemoryType = CU_MEMORYTYPE_DEVICE;
  c.dstDevice = dst;
  c.dstPitch = dpitch;
  c.WidthInBytes = width;
  c.Height = height;
  CU(drv::cuMemcpy2DAsync(&c, static_cast<CUstream>(stream)));
  return 0;
}

int dpia_memcpy2d_dtoh(int device, void* dst, size_t dpitch, uint64_t src, size_t spitch,
                       size_t width, size_t height, void* stream) {
  if (int e = bind(device)) return e;
  CUDA_MEMCPY2D c;
  std::memset(&c, 0, sizeof(c));
  c.srcMemoryType = CU_MEMORYTYPE_DEVICE;
  c.srcDevice = src;
  c.srcPitch = spitch;
  c.dstMemoryType = CU_MEMORYTYPE_HOST;
  c.dstHost = dst;
  c.dstPitch = dpitch;
  c.WidthInBytes = width;
  c.Height = height;
  CU(drv::cuMemcpy2DAsync(&c, static_cast<CUstream>(stream)));
  return 0;
}

int dpia_memcpy_dtod(int device, uint64_t dst, uint64_t src, size_t bytes, void* stream) {
  if (int e = bind(device)) return e;
  CU(drv::cuMemcpyDtoDAsync(dst, src, bytes, static_cast<CUstream>(stream)));
  return 0;
}

int dpia_memset(int device, uint64_t dst, int value, size_t bytes, void* stream) {
  if (int e = bind(device)) return e;
  CU(drv::cuMemsetD8Async(dst, static_cast<unsigned char>(value), bytes, static_cast<CUstream>(stream)));
  return 0;
}

int dpia_launch(void* function, int device, unsigned gx, unsigned gy, unsigned bx, unsigned by,
                unsigned smem, void** args, void* stream) {
  if (int e = bind(device)) return e;
  CU(drv::cuLaunchKernel(static_cast<CUfunction>(function), gx, gy, 1, bx, by, 1, smem,
                    static_cast<CUstream>(stream), args, nullptr));
  return 0;
}

// Launch with programmatic dependent launch allowed: the kernel may start
// while the previous kernel on `stream` is still running; it must execute
// griddepcontrol.wait before touching that kernel's results, and the previous
// kernel may trigger it early with griddepcontrol.launch_dependents.
int dpia_launch_pdl(void* function, int device, unsigned gx, unsigned gy, unsigned bx, unsigned by,
                    unsigned smem, void** args, void* stream) {
  if (int e = bind(device)) return e;
  if (!drv::cuLaunchKernelEx)
    return dpia_launch(function, device, gx, gy, bx, by, smem, args, stream);
  CUlaunchAttribute attr[1];
  std::memset(attr, 0, sizeof(attr));
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  CUlaunchConfig cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = gx;
  cfg.gridDimY = gy;
  cfg.gridDimZ = 1;
  cfg.blockDimX = bx;
  cfg.blockDimY = by;
  cfg.blockDimZ = 1;
  cfg.sharedMemBytes = smem;
  cfg.hStream = static_cast<CUstream>(stream);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CU(drv::cuLaunchKernelEx(&cfg, static_cast<CUfunction>(function), args, nullptr));
  return 0;
}

// TMA descriptor of a row-major matrix of 4-byte (fp32) or 8-byte (int64)
// elements (rows x cols, row pitch in bytes) read in boxes of box_rows x
// box_cols into the 128-byte CUtensorMap at `out` (passed to kernels by
// value); swizzle 0 (plain box layout) or 128 (16-byte chunks of each
// 128-byte row XOR-permuted by the row index mod 8).  The toLocal k-tiles
// (cuda/emit.py KernelEmitter._tma_plan) and the work-item row folds
// (KernelEmitter._finish_rows) the emitter lowers to cp.async.bulk.tensor.2d.
int dpia_tensor_map_2d(void* out, int elem_bytes, uint64_t base, uint64_t rows, uint64_t cols,
                       uint64_t pitch, unsigned box_rows, unsigned box_cols, int swizzle) {
  if (int e = load_driver()) return e;
  if (!drv::cuTensorMapEncodeTiled) return fail(-1, "CUDA driver lacks cuTensorMapEncodeTiled");
  if (elem_bytes != 4 && elem_bytes != 8) return fail(-1, "tensor map: element size must be 4 or 8");
  if (base % 16 || pitch % 16 || (box_cols * elem_bytes) % 16 || box_cols > 256 || box_rows > 256 ||
      box_cols == 0 || box_rows == 0)
    return fail(-1, "tensor map: base/pitch/box violate the TMA alignment or size rules");
  if (swizzle != 0 && !(swizzle == 128 && box_cols * elem_bytes <= 128))
    return fail(-1, "tensor map: swizzle must be 0, or 128 with rows of at most 128 bytes");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CU(drv::cuTensorMapEncodeTiled(
      static_cast<CUtensorMap*>(out),
      elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT64, 2,
      reinterpret_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return 0;
}

int dpia_tensor_map_2d_f32(void* out, uint64_t base, uint64_t rows, uint64_t cols, uint64_t pitch,
                           unsigned box_rows, unsigned box_cols) {
  return dpia_tensor_map_2d(out, 4, base, rows, cols, pitch, box_rows, box_cols, 0);
}

int dpia_stream_create(int device, void** stream) {
  if (int e = bind(device)) return e;
  CUstream s;
  CU(drv::cuStreamCreate(&s, CU_STREAM_NON_BLOCKING));
  *stream = s;
  return 0;
}

int dpia_stream_destroy(void* stream) {
  CU(drv::cuStreamDestroy(static_cast<CUstream>(stream)));
  return 0;
}

int dpia_stream_sync(void* stream) {
  CU(drv::cuStreamSynchronize(static_cast<CUstream>(stream)));
  return 0;
}

int dpia_device_sync(int device) {
  if (int e = bind(device)) return e;
  CU(drv::cuCtxSynchronize());
  return 0;
}

int dpia_event_create(int device, void** event) {
  if (int e = bind(device)) return e;
  CUevent ev;
  CU(drv::cuEventCreate(&ev, CU_EVENT_DEFAULT));
  *event = ev;
  return 0;
}

int dpia_event_destroy(void* event) {
  CU(drv::cuEventDestroy(static_cast<CUevent>(event)));
  return 0;
}

int dpia_event_record(void* event, void* stream) {
  CU(drv::cuEventRecord(static_cast<CUevent>(event), static_cast<CUstream>(stream)));
  return 0;
}

int dpia_stream_wait_event(void* stream, void* event) {
  CU(drv::cuStreamWaitEvent(static_cast<CUstream>(stream), static_cast<CUevent>(event), 0));
  return 0;
}

int dpia_event_elapsed(void* start, void* stop, float* ms) {
  CU(drv::cuEventSynchronize(static_cast<CUevent>(stop)));
  CU(drv::cuEventElapsedTime(ms, static_cast<CUevent>(start), static_cast<CUevent>(stop)));
  return 0;
}

static int load_helper(int device, const char* src, const char* name, CUmodule* mod, CUfunction* fn) {
  void* img = nullptr;
  size_t sz = 0;
  char log[4096];
  int major = 0, minor = 0;
  CUdevice d;
  CU(drv::cuDeviceGet(&d, device));
  CU(drv::cuDeviceGetAttribute(&major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, d));
  CU(drv::cuDeviceGetAttribute(&minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, d));
  char arch[32];
  snprintf(arch, sizeof arch, "sm_%d%d%s", major, minor, major >= 9 ? "a" : "");
  if (int e = dpia_compile(src, "dpia_helper.cu", arch, "", &img, &sz, log, sizeof log)) return e;
  CUresult r = drv::cuModuleLoadData(mod, img);
  free(img);
  CU(r);
  CU(drv::cuModuleGetFunction(fn, *mod, name));
  return 0;
}

// grid of the runtime's own streaming helpers (L2 scrub, hash fill): 8
// resident blocks per SM over the device's SM count (148 on a B200)
static int helper_blocks(int device) {
  CUdevice d;
  int sms = 0;
  if (drv::cuDeviceGet(&d, device) != CUDA_SUCCESS ||
      drv::cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, d) != CUDA_SUCCESS ||
      sms <= 0)
    sms = 148;
  return sms * 8;
}

int dpia_l2_flush(int device, void* stream) {
  if (int e = bind(device)) return e;
  if (!g_flush_buf[device]) {
    int l2 = 0;
    CUdevice d;
    CU(drv::cuDeviceGet(&d, device));
    CU(drv::cuDeviceGetAttribute(&l2, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, d));
    g_flush_bytes[device] = static_cast<size_t>(l2 > 0 ? l2 : (128 << 20)) * 2;
    CU(drv::cuMemAlloc(&g_flush_buf[device], g_flush_bytes[device] + 256));
    CU(drv::cuMemsetD32Async(g_flush_buf[device], 0x5a5a5a5a, (g_flush_bytes[device] + 256) / 4,
                             static_cast<CUstream>(stream)));
    CUmodule m;
    if (int e = load_helper(device, kScrubSrc, "dpia_l2_scrub", &m, &g_scrub_fn[device])) return e;
  }
  CUdeviceptr sink = g_flush_buf[device] + g_flush_bytes[device];
  unsigned long long n = g_flush_bytes[device] / 16;
  void* args[] = {&g_flush_buf[device], &n, &sink};
  CU(drv::cuLaunchKernel(g_scrub_fn[device], helper_blocks(device), 1, 1, 512, 1, 1, 0,
                         static_cast<CUstream>(stream), args, nullptr));
  return 0;
}

int dpia_fill_hash_f32(int device, uint64_t dptr, uint64_t count, uint64_t offset, uint32_t seed,
                       float lo, float hi, void* stream) {
  if (int e = bind(device)) return e;
  if (!g_fill_fn[device]) {
    void* img = nullptr;
    size_t sz = 0;
    char log[4096];
    int major = 0, minor = 0;
    CUdevice d;
    CU(drv::cuDeviceGet(&d, device));
    CU(drv::cuDeviceGetAttribute(&major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, d));
    CU(drv::cuDeviceGetAttribute(&minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, d));
    char arch[32];
    snprintf(arch, sizeof arch, "sm_%d%d%s", major, minor, major >= 9 ? "a" : "");
    if (int e = dpia_compile(kFillSrc, "dpia_fill.cu", arch, "", &img, &sz, log, sizeof log)) return e;
    CUresult r = drv::cuModuleLoadData(&g_fill_mod[device], img);
    free(img);
    CU(r);
    CU(drv::cuModuleGetFunction(&g_fill_fn[device], g_fill_mod[device], "dpia_fill_hash_f32"));
  }
  unsigned long long n = count, off = offset;
  void* args[] = {&dptr, &n, &off, &seed, &lo, &hi};
  CU(drv::cuLaunchKernel(g_fill_fn[device], helper_blocks(device), 1, 1, 256, 1, 1, 0,
                    static_cast<CUstream>(stream), args, nullptr));
  return 0;
}

// ------------------------------------------------- peer (NVLink) mailboxes
int dpia_ipc_alloc(int device, size_t bytes, uint64_t* dptr, char handle[64]) {
  if (int e = bind(device)) return e;
  CUdeviceptr p = 0;
  CU(drv::cuMemAlloc(&p, bytes ? bytes : 16));
  CU(drv::cuMemsetD8Async(p, 0, bytes ? bytes : 16, nullptr));
  CU(drv::cuCtxSynchronize());
  CUipcMemHandle h;
  CU(drv::cuIpcGetMemHandle(&h, p));
  static_assert(sizeof(CUipcMemHandle) == 64, "CUipcMemHandle is 64 bytes");
  memcpy(handle, &h, 64);
  *dptr = static_cast<uint64_t>(p);
  return 0;
}

int dpia_ipc_open(int device, const char handle[64], uint64_t* dptr) {
  if (int e = bind(device)) return e;
  CUipcMemHandle h;
  memcpy(&h, handle, 64);
  CUdeviceptr p = 0;
  CU(drv::cuIpcOpenMemHandle(&p, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS));
  *dptr = static_cast<uint64_t>(p);
  return 0;
}

int dpia_ipc_close(int device, uint64_t dptr) {
  if (int e = bind(device)) return e;
  CU(drv::cuIpcCloseMemHandle(static_cast<CUdeviceptr>(dptr)));
  return 0;
}

int dpia_nccl_available(void) { return load_nccl() == 0 ? 1 : 0; }

int dpia_nccl_unique_id(char out[128]) {
  if (int e = load_nccl()) return e;
  ncclUniqueId_t id;
  if (int e = nccl(p_get_id(&id), "ncclGetUniqueId")) return e;
  memcpy(out, id.internal, 128);
  return 0;
}

int dpia_nccl_init(int device, int nranks, int rank, const char id[128]) {
  if (int e = load_nccl()) return e;
  if (int e = bind(device)) return e;
  ncclUniqueId_t uid;
  memcpy(uid.internal, id, 128);
  return nccl(p_init_rank(&g_comm, nranks, uid, rank), "ncclCommInitRank");
}

int dpia_nccl_allreduce(uint64_t dptr, size_t count, int dtype, void* stream) {
  if (!g_comm) return fail(-1, "NCCL communicator not initialised");
  // ncclDataType_t: ncclFloat32 = 7, ncclFloat64 = 8, ncclInt64 = 4; ncclSum = 0
  int nd = dtype == 0 ? 7 : dtype == 1 ? 8 : 4;
  void* p = reinterpret_cast<void*>(dptr);
  return nccl(p_allreduce(p, p, count, nd, 0, g_comm, static_cast<CUstream>(stream)),
              "ncclAllReduce");
}

int dpia_nccl_destroy(void) {
  if (g_comm && p_destroy) {
    int r = p_destroy(g_comm);
    g_comm = nullptr;
    return nccl(r, "ncclCommDestroy");
  }
  return 0;
}

}  // extern "C"
