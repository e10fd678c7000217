// context.cu — device/stream setup, error plumbing, scratch workspace,
// launch accounting and per-phase CUDA-event timing for libgtb200.so.
#include "common.cuh"

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace gt {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_last_error(const std::string& m) { g_last_error = m; }

[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  fail(e == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA, buf);
}

static Context g_lanes[GT_LANES];
static thread_local int t_lane = 0;
static std::atomic<bool> g_profiling{false};
static std::mutex g_init_mu;
static int init_locked(int device);  // gt_init body; caller holds g_init_mu
Context& ctx() { return g_lanes[t_lane]; }

// Library streams are created BLOCKING (no cudaStreamNonBlocking): work on
// them is ordered after everything queued before on the legacy default
// stream — torch's default stream — so device buffers a caller just wrote
// with torch ops are complete before a library kernel reads them. (Callers on
// another stream order themselves: the Python layer waits on it, see
// _native.order_after_torch.)
static constexpr unsigned kStreamFlags = cudaStreamDefault;

void require_init() {
  if (ctx().stream != nullptr) return;
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (g_lanes[0].stream == nullptr) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const int lane = t_lane;
    t_lane = 0;
    const int rc = init_locked(dev);
    t_lane = lane;
    if (rc != GT_OK) fail(GT_ENODEV, std::string("gt_init failed: ") + g_last_error);
  }
  Context& c = ctx();
  if (c.stream == nullptr) {  // a further lane: lane 0's device, its own stream
    const Context& z = g_lanes[0];
    GT_CUDA(cudaSetDevice(z.device));
    c.device = z.device;
    c.sm_count = z.sm_count;
    c.l2_bytes = z.l2_bytes;
    c.smem_optin = z.smem_optin;
    GT_CUDA(cudaStreamCreateWithFlags(&c.stream, kStreamFlags));
  }
}

void after_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof buf, "launch of %s failed: %s", name, cudaGetErrorString(e));
    fail(GT_ECUDA, buf);
  }
}

void* dalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMallocAsync(&p, bytes, ctx().stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[256];
    snprintf(buf, sizeof buf, "device allocation of %zu bytes failed: %s", bytes,
             cudaGetErrorString(e));
    fail(GT_ENOMEM, buf);
  }
  return p;
}

void dfree(void* p) {
  if (p) cudaFreeAsync(p, ctx().stream);
}

struct SlotBuf { void* p = nullptr; size_t cap = 0; };
static SlotBuf g_slots[GT_LANES][WS_NSLOTS];

void* ws_get(Slot s, size_t bytes) {
  SlotBuf& b = g_slots[t_lane][s];
  if (b.cap < bytes) {
    dfree(b.p);
    size_t cap = bytes + bytes / 8;  // headroom so slightly larger inputs reuse
    b.p = dalloc(cap);
    b.cap = cap;
    if (s == WS_LOOKBACK) GT_CUDA(cudaMemsetAsync(b.p, 0, cap, ctx().stream));
  }
  return b.p;
}

void ws_release_all() {
  for (auto& b : g_slots[t_lane]) { dfree(b.p); b.p = nullptr; b.cap = 0; }
}

static uint32_t g_epoch[GT_LANES] = {};
uint32_t next_epoch() {  // per lane: each lane has its own look-back words
  uint32_t& ep = g_epoch[t_lane];
  ep = (ep + 1) & 0x3FFFFFu;
  if (ep == 0) {  // wrapped: clear stale words so old epochs cannot alias
    SlotBuf& b = g_slots[t_lane][WS_LOOKBACK];
    if (b.p) GT_CUDA(cudaMemsetAsync(b.p, 0, b.cap, ctx().stream));
    ep = 1;
  }
  return ep;
}

void d2h(void* h, const void* d, size_t bytes) {
  if (bytes) GT_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx().stream));
}
void h2d(void* d, const void* h, size_t bytes) {
  if (bytes) GT_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx().stream));
}
void sync() { GT_CUDA(cudaStreamSynchronize(ctx().stream)); }

// ---------------------------------------------------------------- profiling --
struct PhaseStat {
  std::string name;
  double ms = 0.0;
  int64_t launches = 0;
  double bytes = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};
static std::vector<PhaseStat> g_phases;
static std::vector<cudaEvent_t> g_event_pool;
static std::mutex g_prof_mu;

static cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  GT_CUDA(cudaEventCreate(&e));
  return e;
}

static int phase_index(const char* name) {
  for (size_t i = 0; i < g_phases.size(); ++i)
    if (g_phases[i].name == name) return static_cast<int>(i);
  g_phases.push_back(PhaseStat{});
  g_phases.back().name = name;
  return static_cast<int>(g_phases.size() - 1);
}

static void resolve_pending() {
  for (auto& p : g_phases) {
    for (auto& ev : p.pending) {
      GT_CUDA(cudaEventSynchronize(ev.second));
      float ms = 0.f;
      GT_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
      p.ms += ms;
      g_event_pool.push_back(ev.first);
      g_event_pool.push_back(ev.second);
    }
    p.pending.clear();
  }
}

Phase::Phase(const char* name, double bytes) {
  if (!g_profiling.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  idx = phase_index(name);
  g_phases[idx].bytes += bytes;
  g_phases[idx].launches += 1;
  start = get_event();
  GT_CUDA(cudaEventRecord(start, ctx().stream));
}

void profile_add_bytes(const char* name, double bytes) {
  if (!g_profiling.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_phases[phase_index(name)].bytes += bytes;
}

Phase::~Phase() {
  if (idx < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t end = get_event();
  if (cudaEventRecord(end, ctx().stream) != cudaSuccess) return;
  g_phases[idx].pending.emplace_back(start, end);
}

static int init_locked(int device) {
  try {
    Context& c = ctx();
    if (c.stream != nullptr && c.device == device) return GT_OK;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(GT_ENODEV, "no CUDA device visible (libgtb200 has no CPU fallback)");
    }
    if (device < 0 || device >= n) fail(GT_EINVAL, "device ordinal out of range");
    if (c.stream != nullptr) {
      // switching devices: this lane's workspace and stream belong to the old
      // one — release them there before re-initialising
      GT_CUDA(cudaSetDevice(c.device));
      ws_release_all();
      GT_CUDA(cudaStreamSynchronize(c.stream));
      GT_CUDA(cudaStreamDestroy(c.stream));
      c.stream = nullptr;
    }
    GT_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    GT_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) {
      char buf[160];
      snprintf(buf, sizeof buf, "device %d is sm_%d%d; libgtb200 is built for sm_100a only",
               device, prop.major, prop.minor);
      fail(GT_ENODEV, buf);
    }
    c.device = device;
    c.sm_count = prop.multiProcessorCount;
    c.l2_bytes = prop.l2CacheSize;
    c.smem_optin = int(prop.sharedMemPerBlockOptin);
    GT_CUDA(cudaStreamCreateWithFlags(&c.stream, kStreamFlags));
    cudaMemPool_t pool;
    GT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    GT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    return GT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

}  // namespace gt

using namespace gt;

extern "C" {

int gt_init(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  return init_locked(device);
}

const char* gt_version(void) { return "gtb200 0.1.0 (sm_100a)"; }

void* gt_stream(void) {
  try {
    require_init();
  } catch (const Error& e) {
    set_last_error(e.what());
    return nullptr;
  }
  return ctx().stream;
}

const char* gt_last_error(void) { return g_last_error.c_str(); }

int gt_release_workspace(void) {
  try {
    if (ctx().stream == nullptr) return GT_OK;
    ws_release_all();
    sync();
    // the pool keeps freed blocks (release threshold raised at init); hand
    // them back to the driver so other allocators (torch) can use the memory
    cudaMemPool_t pool;
    GT_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx().device));
    GT_CUDA(cudaMemPoolTrimTo(pool, 0));
    return GT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int64_t gt_launch_count(void) { return g_launches.load(); }

int gt_profile_enable(int on) {
  g_profiling.store(on != 0);
  return GT_OK;
}

int gt_set_lane(int lane) {
  if (lane < 0 || lane >= GT_LANES) {
    set_last_error("lane must be in [0, GT_LANES)");
    return GT_EINVAL;
  }
  t_lane = lane;
  return GT_OK;
}

int gt_profile_reset(void) {
  try {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    resolve_pending();
    for (auto& p : g_phases) { p.ms = 0; p.launches = 0; p.bytes = 0; }
    return GT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int gt_profile_read(int cap, const char** names, double* total_ms, int64_t* launches,
                    double* bytes) {
  try {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    resolve_pending();
    int n = 0;
    for (auto& p : g_phases) {
      if (p.launches == 0) continue;
      if (n < cap) {
        if (names) names[n] = p.name.c_str();
        if (total_ms) total_ms[n] = p.ms;
        if (launches) launches[n] = p.launches;
        if (bytes) bytes[n] = p.bytes;
      }
      ++n;
    }
    return n;
  } catch (const Error& e) {
    set_last_error(e.what());
    return -e.code;
  }
}

}  // extern "C"
