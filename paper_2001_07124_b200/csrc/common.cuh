// common.cuh -- shared host/device plumbing of librtucker (errors, launch context,
// profiling hooks, workspace arena).  No method arithmetic lives here.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace rt {

// Thrown inside the library, converted to an rt_status at the C-ABI boundary.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define RT_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw ::rt::Error(-4, std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" +      \
                                std::to_string(__LINE__));                                   \
  } while (0)

#define RT_REQUIRE(cond, status, msg)                                                        \
  do {                                                                                       \
    if (!(cond)) throw ::rt::Error((status), std::string(msg));                              \
  } while (0)

constexpr int kEINVAL = -1, kERANK = -2, kENOMEM = -3, kECUDA = -4, kENCCL = -5, kENUMERIC = -6,
              kEUNSUPPORTED = -7;

// device status bits (latched by kernels, read by rt_sync)
constexpr int kStatusCholBreakdown = 1;
constexpr int kStatusNonFinite = 2;
constexpr int kStatusBadHash = 4;     // count-sketch code outside [-K, -1] U [1, K]

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- profiling
struct Profiler {
  bool enabled = false;
  struct Rec { const char* name; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  int64_t launches = 0;     // counted even when timing is disabled
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    RT_CUDA(cudaEventCreate(&e));
    return e;
  }
  ~Profiler() {
    for (auto& r : recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

class Arena;

// Pool of reusable CUDA events (fork / join of the side stream); reset at the start of every call.
struct EventPool {
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  cudaEvent_t get() {
    if (next == ev.size()) {
      cudaEvent_t e;
      RT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    return ev[next++];
  }
  void reset() { next = 0; }
  ~EventPool() { for (auto e : ev) cudaEventDestroy(e); }
};

// ---------------------------------------------------------------- launch context
struct Ctx {
  cudaStream_t stream = nullptr;
  int* d_status = nullptr;      // device status latch
  Profiler* prof = nullptr;
  int num_sms = 148;
  int ttm_impl = 0;             // 0 auto, 1 SIMT, 2 tcgen05 (error if unavailable), 3 SIMT with fp64
                                // accumulation of every X pass (the strict reference-precision mode)
  bool simt() const { return ttm_impl == 1 || ttm_impl == 3; }
  bool acc64() const { return ttm_impl == 3; }
  int omega_tf32 = 0;           // caller asserts Gaussian Omega entries are tf32-representable
  int tc_seg = 16;              // tcgen05: 32-element chunks per TMEM accumulator segment (drained to fp32 regs)
  int tc_ablate = 0;            // profiling only (RT_OPT_TC_ABLATE): 1 no MMA, 2 no split; results invalid
  int tc_skew = -1;             // ttm_s_tc: chunk-order rotation per M-tile (-1 = default)
  int force_dist = 0;           // run the slab exchanges on a 1-rank communicator (tests)
  mutable const char* label = nullptr;   // profiler name override for the next TC launches
  int tc_presplit_z = 0;        // power iteration: write Z R^-1 pre-split [hi | lo] (ablation 200 toggles)
  int tc_h16 = 1;               // fp16-split X passes (R29; ablation 210/211 toggles; 212 = on with the
                                // device gate forced closed, so the tf32 twins run: tests)
  int hooi_tc = 1;              // RP-HOOI: X pass of the S chain on the tensor cores (ablation 220/221 toggles)
  int power_qrz = 0;            // power iteration: orthonormalize Z (shifted CholeskyQR) instead of R31's
                                // power-of-two scale (ablation 240 / 241 toggle)
  int omega_h16_off = 0;        // Omega sketches of later modes: 1 = keep tf32 (ablation 250 / 251 toggle)
  int tc_xfirst = 0;            // wide X rows with L2::evict_first (ablation 280 / 281: first / normal)
  int fuse_off = 0;             // HOSVD: 1 = no fused mode-1 sketch + mode-0 core pass (ablation 290 / 291)
  int fuse2_off = 0;            // HOSVD: 1 = one fused pass (S1 + G1) instead of two (Z0 + S1, G1 + S2) (298 / 299)
  int fused_nbb = 3;            // fused pass: B slots (chunk pairs) 2 or 3 (ablation 292 / 293)
  int resid_tf32 = 0;           // residual pass: 1 = the 3xTF32 kernel only (ablation 294 / 295)
  int split_resid_off = 0;      // HOSVD: 1 = truncate, then the rank-R residual (no R35 overlap; 296 / 297)
  int resid_slab_off = 0;       // 1: a slab's residual pass keeps the J x R_N form of P (ablation 350)
  int core_early_off = 0;       // 1: the core's second stage waits for every Q~ (ablation 340)
  int qr3_always = 0;           // 1: the power steps' intermediate QRs keep 3 CholeskyQR steps (ablation 330)
  int thin_slab_off = 0;        // 1: thin slabs keep the fp16 forms of the slab mode (ablation 320; tests)
  int tc_waves = 4;             // ttm_s split-K grids: CTA waves over the SMs (ablation 301..308)
  int fused_seg = 16;           // fused pass: chunks per accumulator segment (ablation 316 / 332: 16 / 32)
  int tc_xw = 2;                // ttm_s strided modes: chunks per wide-row X stage (1 = swizzled 128 B rows;
                                // ablation 231/232/234 select 1/2/4; cfg5 modes 1/2: 2 is fastest)
  cudaStream_t side_stream = nullptr;   // second stream of the handle (high priority): overlapped QRs
  cudaStream_t comm_stream = nullptr;   // third stream: the slab mode's Z allreduce (C3) on the side communicator
  Arena* side_ws = nullptr;             // its workspace arena
  EventPool* events = nullptr;          // fork / join events
  int overlap = 1;              // HOSVD: thin QRs on the side stream (ablation 270 / 271 toggle)
  int sm_reserve = 0;           // SMs the persistent X-pass grids leave free (set while side work is pending)
  unsigned int* d_runs = nullptr;  // device counters: [0] fp16-split X passes that did their work,
                                   // [1] tf32 twins that ran in their place (R29; rt_profile_read),
                                   // [2] Jacobi sweeps run (all matrices)
};

// Launch a kernel (given as a lambda issuing <<<...>>> on ctx.stream) with optional
// CUDA-event timing per kernel class.
// Scoped profiler label: TC TTM launches inside the scope are recorded under `name`.
struct LabelScope {
  const Ctx& c;
  const char* prev;
  LabelScope(const Ctx& ctx, const char* name) : c(ctx), prev(ctx.label) { ctx.label = name; }
  ~LabelScope() { c.label = prev; }
};

template <typename F>
inline void launch(const Ctx& ctx, const char* name, F&& f) {
  Profiler* p = ctx.prof;
  cudaEvent_t a = nullptr, b = nullptr;
  if (p && p->enabled) { a = p->get(); b = p->get(); RT_CUDA(cudaEventRecord(a, ctx.stream)); }
  f();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(kECUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
  if (p) {
    p->launches++;
    if (p->enabled) { RT_CUDA(cudaEventRecord(b, ctx.stream)); p->recs.push_back({name, a, b}); }
  }
}

// ---------------------------------------------------------------- workspace arena
// Bump allocator over device blocks.  A call may grow it (cudaMalloc); at the start of
// the next call all blocks are coalesced into one so the steady state never allocates.
class Arena {
 public:
  ~Arena() { release(); }
  void begin_call() {
    if (blocks_.size() > 1 || (blocks_.size() == 1 && high_ > blocks_[0].size)) {
      size_t total = 0;
      for (auto& b : blocks_) total += b.size;
      total = std::max(total, high_);
      release_sync();
      add_block(total);
    }
    for (auto& b : blocks_) b.used = 0;
    cur_ = 0;
    used_total_ = 0;
  }
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    while (cur_ < blocks_.size()) {
      Block& b = blocks_[cur_];
      if (b.used + bytes <= b.size) {
        void* p = static_cast<char*>(b.ptr) + b.used;
        b.used += bytes;
        used_total_ += bytes;
        high_ = std::max(high_, used_total_);
        return p;
      }
      ++cur_;
    }
    size_t last = blocks_.empty() ? 0 : blocks_.back().size;
    add_block(std::max(bytes, std::max(last, size_t(64) << 20)));
    cur_ = blocks_.size() - 1;
    return alloc(bytes);
  }
  template <typename T> T* alloc_n(int64_t n) { return static_cast<T*>(alloc(sizeof(T) * size_t(n))); }
  // Mark/rewind (scoped reuse inside one call; safe because kernels are stream-ordered).
  struct Mark { size_t cur, used, total; };
  Mark mark() const { return {cur_, cur_ < blocks_.size() ? blocks_[cur_].used : 0, used_total_}; }
  void rewind(const Mark& m) {
    for (size_t i = m.cur + 1; i < blocks_.size(); ++i) blocks_[i].used = 0;
    cur_ = m.cur;
    if (cur_ < blocks_.size()) blocks_[cur_].used = m.used;
    used_total_ = m.total;
  }
  void release() {
    for (auto& b : blocks_) cudaFree(b.ptr);
    blocks_.clear();
  }

 private:
  struct Block { void* ptr; size_t size; size_t used; };
  void add_block(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw Error(kENOMEM, "workspace cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    blocks_.push_back({p, bytes, 0});
  }
  void release_sync() {
    cudaDeviceSynchronize();
    release();
  }
  std::vector<Block> blocks_;
  size_t cur_ = 0, used_total_ = 0, high_ = 0;
};

}  // namespace rt
