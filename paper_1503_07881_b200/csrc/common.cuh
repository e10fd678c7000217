// common.cuh — context, errors, scratch workspace, launch accounting and
// per-phase device timing shared by every translation unit of libgtb200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gtb200.h"

namespace gt {

// ---------------------------------------------------------------- errors --
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void set_last_error(const std::string& m);

#define GT_CUDA(call) ::gt::cuda_check((call), #call, __FILE__, __LINE__)

// Wrap the body of every extern "C" entry point: C++ errors become status codes.
#define GT_API_BEGIN try {
#define GT_API_END                                                             \
  }                                                                            \
  catch (const ::gt::Error& e) {                                               \
    ::gt::set_last_error(e.what());                                            \
    return e.code;                                                             \
  }                                                                            \
  catch (const std::exception& e) {                                            \
    ::gt::set_last_error(e.what());                                            \
    return GT_ECUDA;                                                           \
  }                                                                            \
  return GT_OK;

// ---------------------------------------------------------------- context --
// Lanes: each calling thread works on a lane (gt_set_lane; default 0) with
// its own stream and workspace slots, so two threads can run independent
// calls on one graph concurrently (e.g. PageRank next to the triangle count).
constexpr int GT_LANES = 2;

struct Context {
  int device = -1;
  int sm_count = 148;
  size_t l2_bytes = 0;
  int smem_optin = 227 * 1024;  // max dynamic shared memory per block (opt-in)
  cudaStream_t stream = nullptr;
  bool profiling = false;
};
Context& ctx();
void require_init();

// Every kernel launch goes through this: counts it and surfaces launch errors.
void after_launch(const char* name);

#define GT_LAUNCH(kernel, grid, block, smem, ...)                              \
  do {                                                                         \
    kernel<<<(grid), (block), (smem), ::gt::ctx().stream>>>(__VA_ARGS__);      \
    ::gt::after_launch(#kernel);                                               \
  } while (0)

// ----------------------------------------------------------- device memory --
// Stream-ordered allocation from the device's default pool (kept warm: the
// pool release threshold is raised at init so repeated builds reuse memory).
void* dalloc(size_t bytes);
void dfree(void* p);

template <typename T>
T* dalloc_n(size_t n) { return static_cast<T*>(dalloc(n * sizeof(T) + (n == 0 ? 8 : 0))); }

// Growable named scratch slots (radix-sort ping-pong buffers, look-back
// status words, histograms ...). Contents are undefined on return.
enum Slot {
  WS_KEYS_A = 0, WS_KEYS_B, WS_LOOKBACK, WS_HIST, WS_COUNTERS, WS_SMALL,
  WS_RANKMAP, WS_COLS, WS_TMP0, WS_TMP1, WS_TMP2, WS_TMP3, WS_TMP4,
  WS_PART,  // partition_pass's segment table and cursors (its callers own TMP0-4)
  WS_NSLOTS
};
void* ws_get(Slot s, size_t bytes);
template <typename T>
T* ws_n(Slot s, size_t n) { return static_cast<T*>(ws_get(s, n * sizeof(T) + 16)); }
void ws_release_all();

// Look-back status words carry an epoch so that they never need clearing
// between passes; a fresh epoch is handed out per decoupled-look-back scan.
uint32_t next_epoch();

// Copy helpers on the library stream.
void d2h(void* h, const void* d, size_t bytes);
void h2d(void* d, const void* h, size_t bytes);
void sync();

// ---------------------------------------------------------------- profiling --
// RAII phase marker: records CUDA events around a group of launches when
// profiling is enabled; `bytes` is the algorithmic traffic credited to it.
struct Phase {
  int idx = -1;
  cudaEvent_t start = nullptr;
  Phase(const char* name, double bytes);
  ~Phase();
};
// Credit extra algorithmic bytes to a phase once sizes are known (e.g. E).
void profile_add_bytes(const char* name, double bytes);

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gt

// ------------------------------------------------------------ device helpers --
namespace gtd {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Streaming 64-bit load that does not allocate in L1 (read-once data).
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_stream_s64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Look-back status words: the flag and the value travel in ONE 64-bit word,
// so readers need no ordering beyond the single-copy atomicity of the word:
// relaxed gpu-scope accesses (served by L2). acquire/release here would make
// ptxas emit an L1 invalidate (CCTL.IVALL) per spin iteration and a memory
// barrier per publish — measured as ~30% of the radix pass's stall samples.
__device__ __forceinline__ uint64_t ld_status_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// Look-back word: [63:62] flag (1 aggregate, 2 inclusive) [61:40] epoch, [39:0] value.
constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_INC = 2ull << 62;
__device__ __forceinline__ uint64_t lb_pack(uint64_t flag, uint32_t epoch, uint64_t v) {
  return flag | (uint64_t(epoch & 0x3FFFFFu) << 40) | (v & ((1ull << 40) - 1));
}

// Decoupled look-back for a single running total: called by ONE thread of the
// tile; publishes `aggregate`, walks predecessors, publishes the inclusive
// value and returns the exclusive prefix of this tile.
__device__ __forceinline__ uint64_t lookback_single(uint64_t* status, int tile, uint32_t epoch,
                                                    uint64_t aggregate) {
  if (tile == 0) {
    st_status_u64(&status[0], lb_pack(LB_INC, epoch, aggregate));
    return 0;
  }
  st_status_u64(&status[tile], lb_pack(LB_AGG, epoch, aggregate));
  uint64_t excl = 0;
  int t = tile - 1;
  const uint64_t ep = uint64_t(epoch & 0x3FFFFFu);
  while (true) {
    uint64_t s = ld_status_u64(&status[t]);
    if (((s >> 40) & 0x3FFFFFu) != ep || (s >> 62) == 0) continue;  // not yet published
    excl += s & ((1ull << 40) - 1);
    if ((s >> 62) == 2) break;
    --t;
  }
  st_status_u64(&status[tile], lb_pack(LB_INC, epoch, excl + aggregate));
  return excl;
}

// Warp-parallel decoupled look-back (called by all 32 lanes of ONE warp):
// 32 predecessors polled per round trip, consumed up to the nearest
// inclusive value (or up to the first one not yet published). Returns the
// exclusive prefix of `tile` to every lane and publishes its inclusive value.
// For chains whose tiles finish out of order (variable-size work units).
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, int tile, uint32_t epoch,
                                                  uint64_t aggregate) {
  const int lane = threadIdx.x & 31;
  const uint64_t ep = uint64_t(epoch & 0x3FFFFFu);
  if (lane == 0)
    st_status_u64(&status[tile], lb_pack(tile == 0 ? LB_INC : LB_AGG, epoch, aggregate));
  uint64_t excl = 0;
  int t = tile - 1;
  while (t >= 0) {
    const int idx = t - lane;
    uint64_t v = idx >= 0 ? ld_status_u64(&status[idx]) : (LB_INC | (ep << 40));
    const bool ready = ((v >> 40) & 0x3FFFFFu) == ep && (v >> 62) != 0;
    const uint32_t inc = __ballot_sync(0xffffffffu, ready && (v >> 62) == 2);
    const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
    // lanes [0, lim] are needed: up to the nearest inclusive value, else all
    const int lim = inc ? __ffs(inc) - 1 : 31;
    const uint32_t need = lim == 31 ? 0xffffffffu : ((2u << lim) - 1u);
    int take;  // lanes consumed this round
    bool done;
    if (notready & need) {
      take = __ffs(notready & need) - 1;  // all-aggregate prefix before the first gap
      done = false;
    } else {
      take = lim + 1;
      done = inc != 0;
    }
    uint64_t x = lane < take ? (v & ((1ull << 40) - 1)) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    excl += x;
    t -= take;
    if (done) break;
  }
  if (lane == 0 && tile > 0) st_status_u64(&status[tile], lb_pack(LB_INC, epoch, excl + aggregate));
  return excl;
}

}  // namespace gtd
