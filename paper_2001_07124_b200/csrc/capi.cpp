// capi.cpp -- the extern "C" boundary of librtucker (declared in include/rtucker.h).
// Validation, handle/workspace management and status conversion; no arithmetic.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/rtucker.h"
#include "engine.h"

struct rt_handle {
  rt::Ctx ctx;
  rt::Arena ws;
  rt::Arena ws_side;                 // workspace of the side stream (overlapped QRs)
  rt::EventPool events;
  cudaStream_t side = nullptr;
  cudaStream_t cstream = nullptr;   // C3 overlap (distributed HOSVD)
  rt::Profiler prof;
  std::unique_ptr<rt::Comm> comm;
  std::string err;
  int device = 0;
  int* d_status = nullptr;
  unsigned int* d_runs = nullptr;   // [3] fp16-split / tf32-twin run counters, Jacobi sweeps (rt_profile_read)
};

namespace {

thread_local std::string g_err;

rt_status fail(rt_handle* h, int st, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return static_cast<rt_status>(st);
}

template <typename F>
rt_status guard(rt_handle* h, F&& f) {
  try {
    if (h) {
      cudaSetDevice(h->device);
      h->ws.begin_call();
      h->ws_side.begin_call();
      h->events.reset();
    }
    f();
    return RT_OK;
  } catch (const rt::Error& e) {
    return fail(h, e.status, e.what());
  } catch (const std::bad_alloc&) {
    return fail(h, RT_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(h, RT_ECUDA, e.what());
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

rt::TView check_tensor(const rt_tensor* X) {
  RT_REQUIRE(X != nullptr, rt::kEINVAL, "X is NULL");
  RT_REQUIRE(X->order >= 2 && X->order <= 5, rt::kEINVAL, "order must be in [2,5]");
  RT_REQUIRE(X->dtype == RT_F32 || X->dtype == RT_F64, rt::kEINVAL, "dtype must be RT_F32 or RT_F64");
  RT_REQUIRE(X->data != nullptr && aligned16(X->data), rt::kEINVAL, "X->data must be a 16-byte aligned device pointer");
  rt::TView v;
  v.dtype = X->dtype == RT_F64 ? 1 : 0;
  v.N = X->order;
  for (int k = 0; k < v.N; ++k) {
    RT_REQUIRE(X->dims[k] >= 1, rt::kEINVAL, "dims must be >= 1");
    v.d[k] = X->dims[k];
  }
  v.off = X->last_offset;
  v.glob = X->last_global == 0 ? X->dims[v.N - 1] : X->last_global;
  RT_REQUIRE(v.off >= 0 && v.off + v.d[v.N - 1] <= v.glob, rt::kEINVAL, "inconsistent slab (last_offset/last_global)");
  v.data = X->data;
  return v;
}

// strict: K_n <= min(I_n, J_n) (needed by the thin QR); a bare sketch (q = 0) accepts any K <= 128
int64_t local_rows(const rt::TView& X, int n) {
  int64_t s = 1;
  for (int k = 0; k < X.N; ++k) if (k != n) s *= X.d[k];
  return s;
}

void check_gauss_omega(const rt::TView& X, int n, const void* om, int64_t K, int64_t ld, bool strict = true) {
  RT_REQUIRE(om != nullptr && (reinterpret_cast<uintptr_t>(om) % (X.dtype ? 8 : 4)) == 0, rt::kEINVAL,
             "Omega_n must be an aligned device pointer");
  RT_REQUIRE(K >= 1, rt::kEINVAL, "omega_cols must be >= 1");
  RT_REQUIRE(ld >= K, rt::kEINVAL, "omega_ld (row pitch of the row-major Omega_n) must be >= K_n");
  (void)local_rows;
  RT_REQUIRE(!strict || (K <= X.Ig(n) && K <= X.Jg(n)), rt::kERANK, "K_n must be <= min(I_n, J_n)");
  RT_REQUIRE(K <= 128, rt::kEUNSUPPORTED, "K_n > 128 not supported");
}

// Khatri-Rao factors: every Omega_k (k != n) is I_k x K row-major with the same K
int64_t check_kr_omega(const rt::TView& X, int n, const void* const* om, const int64_t* cols, const int64_t* lds,
                       bool strict = true) {
  const int k0 = n == 0 ? 1 : 0;
  const int64_t K = cols[k0];
  RT_REQUIRE(K >= 1 && K <= 128, rt::kEUNSUPPORTED, "Khatri-Rao width must be in [1, 128]");
  for (int k = 0; k < X.N; ++k) {
    if (k == n) continue;
    RT_REQUIRE(om[k] != nullptr, rt::kEINVAL, "Khatri-Rao factor must be a device pointer");
    RT_REQUIRE(cols[k] == K, rt::kEINVAL, "Khatri-Rao factors must share their column count K_n");
    RT_REQUIRE(lds[k] >= K, rt::kEINVAL, "Khatri-Rao factor row pitch must be >= K_n");
  }
  RT_REQUIRE(!strict || (K <= X.Ig(n) && K <= X.Jg(n)), rt::kERANK, "K_n must be <= min(I_n, J_n)");
  return K;
}

// count sketch: one int32 code per (local) column of X_(n), K_n groups
void check_count_omega(const rt::TView& X, int n, const void* om, int64_t K, bool strict = true) {
  RT_REQUIRE(om != nullptr && (reinterpret_cast<uintptr_t>(om) % 4) == 0, rt::kEINVAL,
             "count-sketch codes must be an aligned device pointer");
  RT_REQUIRE(K >= 1, rt::kEINVAL, "omega_cols (number of count-sketch groups) must be >= 1");
  RT_REQUIRE(!strict || (K <= X.Ig(n) && K <= X.Jg(n)), rt::kERANK, "K_n must be <= min(I_n, J_n)");
  RT_REQUIRE(K <= 128, rt::kEUNSUPPORTED, "K_n > 128 not supported");
}

int64_t check_kron_omega(const rt::TView& X, int n, const void* const* om, const int64_t* cols, const int64_t* lds,
                         bool strict = true) {
  int64_t K = 1;
  for (int k = 0; k < X.N; ++k) {
    if (k == n) continue;
    RT_REQUIRE(om[k] != nullptr, rt::kEINVAL, "Kronecker factor must be a device pointer");
    RT_REQUIRE(cols[k] >= 1, rt::kEINVAL, "Kronecker widths must be >= 1");
    RT_REQUIRE(lds[k] >= cols[k], rt::kEINVAL, "Kronecker factor ld (row pitch) must be >= its width L_k");
    K *= cols[k];
  }
  RT_REQUIRE(!strict || K <= X.Ig(n), rt::kERANK, "Kronecker sketch width prod L_k must be <= I_n");
  RT_REQUIRE(K <= 128, rt::kEUNSUPPORTED, "Kronecker sketch width > 128 not supported");
  return K;
}


}  // namespace

extern "C" {

rt_status rt_get_unique_id(uint8_t id[128]) {
  if (!id) return RT_EINVAL;
  int r = rt::nccl_get_unique_id(id);
  if (r != 0) { g_err = rt::nccl_last_error(); return RT_ENCCL; }
  return RT_OK;
}

static rt_status create_common(rt_handle** h, void* stream) {
  if (!h) return RT_EINVAL;
  auto* hh = new (std::nothrow) rt_handle();
  if (!hh) return RT_ENOMEM;
  cudaGetDevice(&hh->device);
  hh->ctx.stream = static_cast<cudaStream_t>(stream);
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, hh->device) == cudaSuccess) hh->ctx.num_sms = sms;
  if (cudaMalloc(&hh->d_status, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    delete hh;
    return fail(nullptr, RT_ECUDA, "cudaMalloc(status) failed (no CUDA device?)");
  }
  cudaMemset(hh->d_status, 0, sizeof(int));
  hh->ctx.d_status = hh->d_status;
  if (cudaMalloc(&hh->d_runs, 3 * sizeof(unsigned int)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(hh->d_status);
    delete hh;
    return fail(nullptr, RT_ECUDA, "cudaMalloc(run counters) failed");
  }
  cudaMemset(hh->d_runs, 0, 3 * sizeof(unsigned int));
  hh->ctx.d_runs = hh->d_runs;
  // side stream (highest priority: its latency-bound QR kernels take SMs ahead of the X passes)
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  if (cudaStreamCreateWithPriority(&hh->side, cudaStreamNonBlocking, hi_prio) != cudaSuccess) {
    cudaGetLastError();
    hh->side = nullptr;               // no overlap: every step on the main stream
  }
  hh->ctx.side_stream = hh->side;
  if (cudaStreamCreateWithFlags(&hh->cstream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    hh->cstream = nullptr;
  }
  hh->ctx.comm_stream = hh->cstream;
  hh->ctx.side_ws = &hh->ws_side;
  hh->ctx.events = &hh->events;
  hh->ctx.prof = &hh->prof;
  *h = hh;
  return RT_OK;
}

rt_status rt_create(rt_handle** h, void* cuda_stream, const uint8_t* id, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, RT_EINVAL, "bad nranks/rank");
  rt_status s = create_common(h, cuda_stream);
  if (s != RT_OK) return s;
  if (id) {                              // a 1-rank NCCL communicator is allowed (tests)
    rt_status st = guard(*h, [&] { (*h)->comm = rt::make_nccl_comm(id, nranks, rank); });
    if (st != RT_OK) { g_err = (*h)->err; rt_destroy(*h); *h = nullptr; return st; }
  }
  return RT_OK;
}

rt_status rt_loopback_group_create(void** group, int nranks) {
  if (!group) return RT_EINVAL;
  return guard(nullptr, [&] { *group = rt::loopback_group_create(nranks); });
}

rt_status rt_loopback_group_destroy(void* group) {
  rt::loopback_group_destroy(static_cast<rt::LoopbackGroup*>(group));
  return RT_OK;
}

rt_status rt_create_loopback(rt_handle** h, void* cuda_stream, void* group, int rank) {
  rt_status s = create_common(h, cuda_stream);
  if (s != RT_OK) return s;
  rt_status st = guard(*h, [&] { (*h)->comm = rt::make_loopback_comm(static_cast<rt::LoopbackGroup*>(group), rank); });
  if (st != RT_OK) { rt_destroy(*h); *h = nullptr; }
  return st;
}

rt_status rt_destroy(rt_handle* h) {
  if (!h) return RT_OK;
  cudaSetDevice(h->device);
  if (h->ctx.stream) cudaStreamSynchronize(h->ctx.stream); else cudaDeviceSynchronize();
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->cstream) cudaStreamSynchronize(h->cstream);
  h->comm.reset();
  if (h->side) cudaStreamDestroy(h->side);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->d_status) cudaFree(h->d_status);
  if (h->d_runs) cudaFree(h->d_runs);
  delete h;
  return RT_OK;
}

const char* rt_last_error(const rt_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }

rt_status rt_sync(rt_handle* h) {
  if (!h) return RT_EINVAL;
  int st = 0;
  rt_status r = guard(h, [&] {
    RT_CUDA(cudaStreamSynchronize(h->ctx.stream));
    RT_CUDA(cudaMemcpy(&st, h->d_status, sizeof(int), cudaMemcpyDeviceToHost));
    RT_CUDA(cudaMemset(h->d_status, 0, sizeof(int)));
  });
  if (r != RT_OK) return r;
  if (st & rt::kStatusNonFinite) return fail(h, RT_ENUMERIC, "non-finite values in the input or a sketch");
  if (st & rt::kStatusBadHash) return fail(h, RT_EINVAL, "count-sketch code outside [-K, -1] U [1, K]");
  if (st & rt::kStatusCholBreakdown) return fail(h, RT_ENUMERIC, "Cholesky breakdown in the thin QR after the shift");
  return RT_OK;
}

rt_status rt_set_option(rt_handle* h, rt_option opt, int64_t value) {
  if (!h) return RT_EINVAL;
  switch (opt) {
    case RT_OPT_TTM_IMPL: h->ctx.ttm_impl = int(value); return RT_OK;
    case RT_OPT_PROFILE: h->prof.enabled = value != 0; return RT_OK;
    case RT_OPT_QR_FALLBACK: return RT_OK;
    case RT_OPT_OMEGA_TF32: h->ctx.omega_tf32 = int(value != 0); return RT_OK;
    case RT_OPT_TC_SEGMENT: h->ctx.tc_seg = int(value > 0 ? value : 16); return RT_OK;
    case RT_OPT_TC_ABLATE:
      if (value == 200 || value == 201) { h->ctx.tc_presplit_z = int(value == 201); return RT_OK; }
      if (value >= 210 && value <= 212) { h->ctx.tc_h16 = int(value - 210); return RT_OK; }
      if (value == 220 || value == 221) { h->ctx.hooi_tc = int(value == 221); return RT_OK; }
      if (value == 231 || value == 232 || value == 234) { h->ctx.tc_xw = int(value - 230); return RT_OK; }
      if (value == 240 || value == 241) { h->ctx.power_qrz = int(value == 240); return RT_OK; }
      if (value == 250 || value == 251) { h->ctx.omega_h16_off = int(value == 250); return RT_OK; }
      if (value == 270 || value == 271) { h->ctx.overlap = int(value == 271); return RT_OK; }
      if (value == 280 || value == 281) { h->ctx.tc_xfirst = int(value == 280); return RT_OK; }
      if (value == 290 || value == 291) { h->ctx.fuse_off = int(value == 290); return RT_OK; }
      if (value == 292 || value == 293) { h->ctx.fused_nbb = int(value - 290); return RT_OK; }
      if (value == 294 || value == 295) { h->ctx.resid_tf32 = int(value == 294); return RT_OK; }
      if (value == 296 || value == 297) { h->ctx.split_resid_off = int(value == 296); return RT_OK; }
      if (value == 298 || value == 299) { h->ctx.fuse2_off = int(value == 298); return RT_OK; }
      if (value >= 301 && value <= 308) { h->ctx.tc_waves = int(value - 300); return RT_OK; }
      if (value == 320 || value == 321) { h->ctx.thin_slab_off = int(value == 320); return RT_OK; }
      if (value == 330 || value == 331) { h->ctx.qr3_always = int(value == 330); return RT_OK; }
      if (value == 340 || value == 341) { h->ctx.core_early_off = int(value == 340); return RT_OK; }
      if (value == 350 || value == 351) { h->ctx.resid_slab_off = int(value == 350); return RT_OK; }
      if (value == 316 || value == 332 || value == 364) { h->ctx.fused_seg = int(value - 300); return RT_OK; }
      h->ctx.tc_ablate = int(value);
      return RT_OK;
    case RT_OPT_TC_SKEW: h->ctx.tc_skew = int(value); return RT_OK;
    case RT_OPT_FORCE_COLLECTIVES: h->ctx.force_dist = int(value != 0); return RT_OK;
  }
  return fail(h, RT_EINVAL, "unknown option");
}

rt_status rt_profile_read(rt_handle* h, rt_profile_entry* out, int cap, int* n, int64_t* launches) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    RT_CUDA(cudaStreamSynchronize(h->ctx.stream));
    int cnt = 0;
    auto& P = h->prof;
    // RT_TIMELINE=<file> (measurement aid, tools/timeline.py): every recorded launch as
    // "name start_ms end_ms" relative to the first one, whatever stream it ran on
    FILE* tl = nullptr;
    if (const char* tp = getenv("RT_TIMELINE")) tl = P.recs.empty() ? nullptr : std::fopen(tp, "a");
    if (tl) std::fprintf(tl, "# read\n");
    for (auto& r : P.recs) {
      float ms = 0.f;
      RT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      if (tl) {
        float t0 = 0.f;
        RT_CUDA(cudaEventElapsedTime(&t0, P.recs[0].a, r.a));
        std::fprintf(tl, "%s %.4f %.4f\n", r.name, t0, t0 + ms);
      }
      int idx = -1;
      for (int i = 0; i < cnt && i < cap; ++i)
        if (std::strncmp(out[i].name, r.name, sizeof(out[i].name)) == 0) { idx = i; break; }
      if (idx < 0 && cnt < cap) {
        idx = cnt++;
        std::memset(out[idx].name, 0, sizeof(out[idx].name));
        std::strncpy(out[idx].name, r.name, sizeof(out[idx].name) - 1);
        out[idx].count = 0;
        out[idx].ms = 0;
      }
      if (idx >= 0) { out[idx].count += 1; out[idx].ms += ms; }
      P.pool.push_back(r.a);
      P.pool.push_back(r.b);
    }
    P.recs.clear();
    if (tl) std::fclose(tl);
    // device run counters of the fp16-split X passes and their tf32 twins (R29): which one of each
    // gated pair did the work since the last read
    unsigned int runs[3] = {0, 0, 0};
    RT_CUDA(cudaMemcpy(runs, h->d_runs, sizeof(runs), cudaMemcpyDeviceToHost));
    RT_CUDA(cudaMemset(h->d_runs, 0, sizeof(runs)));
    const char* rn[3] = {"h16_ran", "tf32_twin_ran", "jacobi_sweeps"};
    for (int k = 0; k < 3; ++k) {
      if (runs[k] == 0 || cnt >= cap) continue;
      std::memset(out[cnt].name, 0, sizeof(out[cnt].name));
      std::strncpy(out[cnt].name, rn[k], sizeof(out[cnt].name) - 1);
      out[cnt].count = int64_t(runs[k]);
      out[cnt].ms = 0;
      ++cnt;
    }
    if (n) *n = cnt;
    if (launches) *launches = P.launches;
    P.launches = 0;
  });
}

rt_status rtucker_sketch(rt_handle* h, const rt_tensor* X, int mode, rt_omega_kind kind, const void* const* omega,
                         const int64_t* omega_cols, const int64_t* omega_ld, int q, double* Y, int64_t ldy) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    RT_REQUIRE(mode >= 0 && mode < v.N, rt::kEINVAL, "mode out of range");
    RT_REQUIRE(q >= 0, rt::kEINVAL, "q must be >= 0");
    RT_REQUIRE(omega && omega_cols && omega_ld && Y, rt::kEINVAL, "NULL omega/omega_cols/omega_ld/Y");
    RT_REQUIRE(ldy >= v.d[mode], rt::kEINVAL, "ldy < I_n");
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist() && q > 0), rt::kEINVAL,
               "power iterations on a slab need a communicator");
    int64_t K;
    if (kind == RT_OMEGA_GAUSS) { K = omega_cols[mode]; check_gauss_omega(v, mode, omega[mode], K, omega_ld[mode], q > 0); }
    else if (kind == RT_OMEGA_KRON) K = check_kron_omega(v, mode, omega, omega_cols, omega_ld, q > 0);
    else if (kind == RT_OMEGA_KR) K = check_kr_omega(v, mode, omega, omega_cols, omega_ld, q > 0);
    else if (kind == RT_OMEGA_COUNT) { K = omega_cols[mode]; check_count_omega(v, mode, omega[mode], K, q > 0); }
    else throw rt::Error(rt::kEINVAL, "unknown omega kind");
    const int64_t In = v.d[mode];
    double* Yt = (ldy == In) ? Y : h->ws.alloc_n<double>(In * K);
    if (v.dtype == 0)
      eng.sketch<float>(v, static_cast<const float*>(v.data), mode, kind, omega, omega_cols, omega_ld, q, Yt);
    else
      eng.sketch<double>(v, static_cast<const double*>(v.data), mode, kind, omega, omega_cols, omega_ld, q, Yt);
    if (Yt != Y) RT_CUDA(cudaMemcpy2DAsync(Y, ldy * sizeof(double), Yt, In * sizeof(double), In * sizeof(double), K,
                                           cudaMemcpyDeviceToDevice, h->ctx.stream));
  });
}

rt_status rtucker_qr(rt_handle* h, int64_t m, int64_t k, rt_dtype dtype, const void* Y, int64_t ldy, double* Q,
                     int64_t ldq, double* R, int rows_distributed) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    RT_REQUIRE(Y && Q, rt::kEINVAL, "NULL Y/Q");
    RT_REQUIRE(k >= 1 && m >= 0 && ldy >= m && ldq >= m, rt::kEINVAL, "bad m/k/ld");
    RT_REQUIRE(k <= 128, rt::kEUNSUPPORTED, "k > 128 not supported");
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    const bool dist = rows_distributed && eng.dist();
    double* shift_dev = nullptr;
    int64_t* row0_dev = nullptr;
    if (dist) {
      // global row count and this rank's first row from an allgather of the local counts, kept on
      // the device (enqueue-only: no host sync).  A global m < k makes the Cholesky break down
      // (RT_ENUMERIC at rt_sync).
      double* cnt = h->ws.alloc_n<double>(1);
      double* all = h->ws.alloc_n<double>(eng.comm->nranks());
      shift_dev = h->ws.alloc_n<double>(1);
      row0_dev = h->ws.alloc_n<int64_t>(1);
      rt::fill_value(h->ctx, cnt, double(m));
      eng.comm->allgather(cnt, all, 1, h->ctx.stream);
      rt::dist_rows_info(h->ctx, all, eng.comm->nranks(), eng.comm->rank(), int(k), shift_dev, row0_dev);
    } else {
      RT_REQUIRE(m >= k, rt::kERANK, "thin QR needs m >= k");
    }
    // m_glob = max(m, k) only passes the host-side check when distributed; the device values rule
    const int64_t mg = std::max<int64_t>(m, k);
    if (dtype == RT_F64)
      eng.qr_rows<double>(static_cast<const double*>(Y), m, mg, int(k), ldy, Q, ldq, R, dist, 0, shift_dev, row0_dev);
    else if (dtype == RT_F32)
      eng.qr_rows<float>(static_cast<const float*>(Y), m, mg, int(k), ldy, Q, ldq, R, dist, 0, shift_dev, row0_dev);
    else throw rt::Error(rt::kEINVAL, "bad dtype");
  });
}

rt_status rtucker_core(rt_handle* h, const rt_tensor* X, const double* const* Q, const int64_t* C, double* G,
                       double* rel_err, double* rel_err_gram) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    RT_REQUIRE(Q && C && G, rt::kEINVAL, "NULL Q/C/G");
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist() && (rel_err || rel_err_gram)), rt::kEINVAL,
               "relative error of a slab needs a communicator");
    int64_t ldq[5];
    for (int n = 0; n < v.N; ++n) {
      RT_REQUIRE(Q[n] != nullptr, rt::kEINVAL, "NULL Q_n");
      RT_REQUIRE(C[n] >= 1 && C[n] <= v.Ig(n), rt::kERANK, "C_n must be in [1, I_n]");
      RT_REQUIRE(C[n] <= 128, rt::kEUNSUPPORTED, "C_n > 128 not supported");
      ldq[n] = v.d[n];
    }
    if (v.dtype == 0) {
      eng.core<float>(v, static_cast<const float*>(v.data), Q, ldq, C, G);
      if (rel_err || rel_err_gram) eng.rel_error<float>(v, static_cast<const float*>(v.data), G, C, Q, rel_err, rel_err_gram);
    } else {
      eng.core<double>(v, static_cast<const double*>(v.data), Q, ldq, C, G);
      if (rel_err || rel_err_gram) eng.rel_error<double>(v, static_cast<const double*>(v.data), G, C, Q, rel_err, rel_err_gram);
    }
  });
}

static void check_driver_args(const rt::TView& v, const int64_t* R, int p, int q, rt_omega_kind kind,
                              const void* const* omega, const int64_t* omega_cols, const int64_t* omega_ld,
                              double* const* Q_out, double* G_out, const int64_t* cur_dims) {
  RT_REQUIRE(R && omega && omega_cols && omega_ld && Q_out && G_out, rt::kEINVAL, "NULL argument");
  RT_REQUIRE(p >= 0 && q >= 0, rt::kEINVAL, "p and q must be >= 0");
  RT_REQUIRE(kind == RT_OMEGA_GAUSS || kind == RT_OMEGA_KRON || kind == RT_OMEGA_KR || kind == RT_OMEGA_COUNT, rt::kEINVAL,
             "unknown omega kind");
  const int N = v.N;
  for (int n = 0; n < N; ++n) {
    RT_REQUIRE(Q_out[n] != nullptr, rt::kEINVAL, "NULL Q_out[n]");
    rt::TView w = v;
    if (cur_dims) {
      for (int k = 0; k < N; ++k) w.d[k] = cur_dims[n * N + k];
      // the slab mode keeps its global size until it is processed (it is last when sharded)
      if (w.d[N - 1] != v.d[N - 1] || !v.sharded()) { w.glob = w.d[N - 1]; w.off = 0; }
    }
    const void* const* om = omega + n * N;
    const int64_t* oc = omega_cols + n * N;
    const int64_t* ol = omega_ld + n * N;
    int64_t K;
    if (kind == RT_OMEGA_GAUSS) {
      K = oc[n];
      check_gauss_omega(w, n, om[n], K, ol[n]);
      RT_REQUIRE(K == std::min<int64_t>(R[n] + p, std::min(w.Ig(n), w.Jg(n))), rt::kEINVAL,
                 "Gaussian width must be K_n = min(R_n + p, I_n, J_n)");
    } else if (kind == RT_OMEGA_COUNT) {
      K = oc[n];
      check_count_omega(w, n, om[n], K);
      RT_REQUIRE(K == std::min<int64_t>(R[n] + p, std::min(w.Ig(n), w.Jg(n))), rt::kEINVAL,
                 "count-sketch width must be K_n = min(R_n + p, I_n, J_n)");
    } else if (kind == RT_OMEGA_KR) {
      K = check_kr_omega(w, n, om, oc, ol);
      RT_REQUIRE(K == std::min<int64_t>(R[n] + p, std::min(w.Ig(n), w.Jg(n))), rt::kEINVAL,
                 "Khatri-Rao width must be K_n = min(R_n + p, I_n, J_n)");
    } else {
      K = check_kron_omega(w, n, om, oc, ol);
      RT_REQUIRE(K >= std::min<int64_t>(R[n] + p, w.Ig(n)), rt::kEINVAL,
                 "Kronecker width prod L_k must be >= min(R_n + p, I_n)");
    }
    RT_REQUIRE(R[n] >= 1 && R[n] <= K, rt::kERANK, "need 1 <= R_n <= K_n");
  }
}

rt_status rtucker_hosvd(rt_handle* h, const rt_tensor* X, const int64_t* R, int p, int q, rt_omega_kind kind,
                        const void* const* omega, const int64_t* omega_cols, const int64_t* omega_ld,
                        double* const* Q_out, double* G_out, double* rel_err, double* rel_err_gram) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    check_driver_args(v, R, p, q, kind, omega, omega_cols, omega_ld, Q_out, G_out, nullptr);
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist()), rt::kEINVAL, "a sharded tensor needs a communicator");
    if (v.dtype == 0) eng.hosvd<float>(v, R, q, kind, omega, omega_cols, omega_ld, Q_out, G_out, rel_err, rel_err_gram);
    else eng.hosvd<double>(v, R, q, kind, omega, omega_cols, omega_ld, Q_out, G_out, rel_err, rel_err_gram);
  });
}

rt_status rtucker_sthosvd(rt_handle* h, const rt_tensor* X, const int64_t* R, int p, int q, rt_omega_kind kind,
                          const void* const* omega, const int64_t* omega_cols, const int64_t* omega_ld,
                          const int* mode_order, double* const* Q_out, double* G_out, double* rel_err,
                          double* rel_err_gram) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist()), rt::kEINVAL, "a sharded tensor needs a communicator");
    const int N = v.N;
    int order[5];
    bool seen[5] = {false, false, false, false, false};
    for (int s = 0; s < N; ++s) {
      order[s] = mode_order ? mode_order[s] : s;
      RT_REQUIRE(order[s] >= 0 && order[s] < N && !seen[order[s]], rt::kEINVAL, "mode_order must be a permutation");
      seen[order[s]] = true;
    }
    RT_REQUIRE(!v.sharded() || order[N - 1] == N - 1, rt::kEUNSUPPORTED,
               "sharded R-STHOSVD processes the slab mode last (mode_order[N-1] == N-1)");
    RT_REQUIRE(R != nullptr, rt::kEINVAL, "NULL R");
    for (int n = 0; n < N; ++n) RT_REQUIRE(R[n] >= 1 && R[n] <= v.Ig(n), rt::kERANK, "need 1 <= R_n <= I_n");
    // sizes of the working tensor when each mode is processed (already-processed modes have R_m)
    int64_t cur[25];
    int64_t d[5];
    for (int k = 0; k < N; ++k) d[k] = v.d[k];
    for (int s = 0; s < N; ++s) {
      const int n = order[s];
      for (int k = 0; k < N; ++k) cur[n * N + k] = d[k];
      d[n] = R[n];
    }
    check_driver_args(v, R, p, q, kind, omega, omega_cols, omega_ld, Q_out, G_out, cur);
    if (v.dtype == 0)
      eng.sthosvd<float>(v, R, q, kind, omega, omega_cols, omega_ld, order, Q_out, G_out, rel_err, rel_err_gram);
    else
      eng.sthosvd<double>(v, R, q, kind, omega, omega_cols, omega_ld, order, Q_out, G_out, rel_err, rel_err_gram);
  });
}

rt_status rtucker_pet(rt_handle* h, const rt_tensor* X, const int64_t* R, const void* const* omega,
                      const int64_t* omega_cols, const int64_t* omega_ld, const void* const* omega_tilde,
                      const int64_t* S, const int64_t* omega_tilde_ld, double* const* Q_out, double* G_out,
                      double* rel_err, double* rel_err_gram) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    RT_REQUIRE(R && omega && omega_cols && omega_ld && omega_tilde && S && omega_tilde_ld && Q_out && G_out,
               rt::kEINVAL, "NULL argument");
    const int N = v.N;
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist()), rt::kEINVAL, "a sharded tensor needs a communicator");
    int64_t hsz = 1;
    for (int n = 0; n < N; ++n) {
      const rt::TView w = v;
      const int64_t K = omega_cols[n * N + n];
      check_gauss_omega(w, n, omega[n * N + n], K, omega_ld[n * N + n]);
      RT_REQUIRE(R[n] >= 1 && R[n] <= K, rt::kERANK, "need 1 <= R_n <= K_n");
      RT_REQUIRE(S[n] >= K, rt::kERANK, "need K_n <= S_n");
      RT_REQUIRE(omega_tilde[n] != nullptr && (reinterpret_cast<uintptr_t>(omega_tilde[n]) % (v.dtype ? 8 : 4)) == 0,
                 rt::kEINVAL, "Omega~_n must be an aligned device pointer");
      RT_REQUIRE(omega_tilde_ld[n] >= v.d[n], rt::kEINVAL, "Omega~_n row pitch must be >= I_n (local)");
      RT_REQUIRE(Q_out[n] != nullptr, rt::kEINVAL, "NULL Q_out");
      hsz *= S[n];
    }
    RT_REQUIRE(hsz <= (int64_t(1) << 31), rt::kEUNSUPPORTED, "core sketch H too large");
    if (v.dtype == 0)
      eng.pet<float>(v, R, omega, omega_cols, omega_ld, omega_tilde, S, omega_tilde_ld, Q_out, G_out, rel_err,
                     rel_err_gram);
    else
      eng.pet<double>(v, R, omega, omega_cols, omega_ld, omega_tilde, S, omega_tilde_ld, Q_out, G_out, rel_err,
                      rel_err_gram);
  });
}

rt_status rtucker_rp_hooi(rt_handle* h, const rt_tensor* X, const int64_t* R, int sweeps,
                          const double* const* Q_init, const double* const* omega, const int64_t* omega_ld,
                          double* const* Q_out, double* G_out, double* rel_err, double* rel_err_gram) {
  if (!h) return RT_EINVAL;
  return guard(h, [&] {
    rt::TView v = check_tensor(X);
    RT_REQUIRE(R && Q_init && Q_out && G_out && (sweeps == 0 || (omega && omega_ld)), rt::kEINVAL, "NULL argument");
    RT_REQUIRE(sweeps >= 0, rt::kEINVAL, "sweeps must be >= 0");
    const int N = v.N;
    rt::Engine eng(h->ctx, h->ws, h->comm.get());
    RT_REQUIRE(!(v.sharded() && !eng.dist()), rt::kEINVAL, "a sharded tensor needs a communicator");
    for (int n = 0; n < N; ++n) {
      RT_REQUIRE(R[n] >= 1 && R[n] <= v.Ig(n) && R[n] <= 128, rt::kERANK, "need 1 <= R_n <= min(I_n, 128)");
      RT_REQUIRE(Q_init[n] && Q_out[n], rt::kEINVAL, "NULL factor pointer");
      int64_t rows = 1;
      for (int p = 0; p < N; ++p) if (p != n) rows *= R[p];
      RT_REQUIRE(rows >= R[n], rt::kERANK, "need prod_{p!=n} R_p >= R_n");
      for (int it = 0; it < sweeps; ++it) {
        RT_REQUIRE(omega[it * N + n] != nullptr, rt::kEINVAL, "NULL Omega");
        RT_REQUIRE(omega_ld[it * N + n] >= R[n], rt::kEINVAL, "Omega row pitch must be >= R_n");
      }
    }
    if (v.dtype == 0) eng.rp_hooi<float>(v, R, sweeps, Q_init, omega, omega_ld, Q_out, G_out, rel_err, rel_err_gram);
    else eng.rp_hooi<double>(v, R, sweeps, Q_init, omega, omega_ld, Q_out, G_out, rel_err, rel_err_gram);
  });
}

}  // extern "C"
