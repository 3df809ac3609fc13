// fif.cu -- C ABI of the B200 FIF hot path (include/fif.h): plan creation
// (validation, device tables), dispatch to the sm_100a kernels, the host-buffer
// end-to-end path and the test hooks.  No torch types, no CPU compute fallback:
// every step of the decomposition runs in the kernels of fif_resident.cuh (resident
// regime, launchers in fif_res_f64.cu / fif_res_f32.cu) and fif_streamed.cuh (fif_st.cu).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "fif_plan.h"

using namespace fifgpu;
using namespace fifhost;

namespace {

template <typename Real>
fif_status upload_tables(fif_plan_s* p) {
  std::vector<Real> sint, isin;
  std::vector<typename Cx<Real>::V> tw;
  build_tables<Real>(p->n, p->NC, sint, isin, tw);
  if (cudaMalloc(&p->d_sin, sizeof(Real) * sint.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMalloc(&p->d_isin, sizeof(Real) * isin.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMalloc(&p->d_tw, sizeof(tw[0]) * tw.size()) != cudaSuccess) return FIF_ERR_OOM;
  if (cudaMemcpy(p->d_sin, sint.data(), sizeof(Real) * sint.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_isin, isin.data(), sizeof(Real) * isin.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_tw, tw.data(), sizeof(tw[0]) * tw.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return FIF_ERR_CUDA;
  return FIF_OK;
}

size_t elem_size(fif_dtype d) { return d == FIF_F64 ? 8 : 4; }

fif_status launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "fif: CUDA error: %s\n", cudaGetErrorString(e));
    return FIF_ERR_CUDA;
  }
  return FIF_OK;
}


void free_plan(fif_plan_s* p) {
  if (!p) return;
  cudaFree(p->d_sin);
  cudaFree(p->d_isin);
  cudaFree(p->d_tw);
  cudaFree(p->d_wtab);
  st_free(p);
  dist_free(p);
  cl_free(p);
  for (int i = 0; i < p->nstages; ++i) {
    cudaFree(p->st[i].d_in);
    cudaFree(p->st[i].d_out);
    cudaFree(p->st[i].d_meta);
    if (p->st[i].stream) cudaStreamDestroy(p->st[i].stream);
    if (p->st[i].done) cudaEventDestroy(p->st[i].done);
  }
  delete p;
}

}  // namespace

extern "C" {

const char* fif_status_string(fif_status s) {
  switch (s) {
    case FIF_OK: return "FIF_OK";
    case FIF_ERR_INVALID_ARG: return "FIF_ERR_INVALID_ARG";
    case FIF_ERR_UNSUPPORTED_N: return "FIF_ERR_UNSUPPORTED_N";
    case FIF_ERR_OOM: return "FIF_ERR_OOM";
    case FIF_ERR_CUDA: return "FIF_ERR_CUDA";
    case FIF_ERR_NCCL: return "FIF_ERR_NCCL";
  }
  return "FIF_ERR_UNKNOWN";
}

fif_status fif_plan_create(fif_plan_t* out, int64_t n, int64_t batch, fif_dtype dtype, fif_window window, double xi,
                           double delta, int32_t max_inner, int32_t max_imfs) {
  return fif_plan_create_ex(out, n, batch, dtype, window, xi, delta, max_inner, max_imfs, FIF_REGIME_AUTO);
}

fif_status fif_plan_create_ex(fif_plan_t* out, int64_t n, int64_t batch, fif_dtype dtype, fif_window window,
                              double xi, double delta, int32_t max_inner, int32_t max_imfs, fif_regime regime) {
  if (!out) return FIF_ERR_INVALID_ARG;
  *out = nullptr;
  if (n < 9 || batch < 0 || !(xi > 0.0) || !isfinite(xi) || !(delta > 0.0) || !isfinite(delta) || max_inner < 1 ||
      max_imfs < 1 || (dtype != FIF_F64 && dtype != FIF_F32) ||
      (window != FIF_WINDOW_TRI_SQ && window != FIF_WINDOW_TRI_SQ_WIDE) ||
      (regime != FIF_REGIME_AUTO && regime != FIF_REGIME_RESIDENT && regime != FIF_REGIME_STREAMED &&
       regime != FIF_REGIME_ITERATIVE && regime != FIF_REGIME_CLUSTER))
    return FIF_ERR_INVALID_ARG;
  if (n % 2 != 0) return FIF_ERR_UNSUPPORTED_N;
  const int64_t NC = n / 2;
  const bool resident_ok = (NC & (NC - 1)) == 0 && NC >= 256 && (NC <= 4096 || (NC == 8192 && dtype == FIF_F32));
  int reg;
  if (regime == FIF_REGIME_RESIDENT) {
    if (!resident_ok) return FIF_ERR_UNSUPPORTED_N;
    reg = 0;
  } else if (regime == FIF_REGIME_STREAMED) {
    reg = 1;
  } else if (regime == FIF_REGIME_ITERATIVE) {
    if (dtype != FIF_F64 || n > 4096) return FIF_ERR_UNSUPPORTED_N;
    reg = 3;
  } else if (regime == FIF_REGIME_CLUSTER) {
    if (!cl_cluster_size(n, dtype)) return FIF_ERR_UNSUPPORTED_N;
    reg = 4;
  } else {
    reg = resident_ok ? 0 : (cl_cluster_size(n, dtype) ? 4 : 1);
  }
  if (reg == 1) {  // host-side check of the streamed factorisation before any CUDA call
    st::Geo g;
    if (!st_geometry(n, dtype == FIF_F64, g)) return FIF_ERR_UNSUPPORTED_N;
  }
  fif_plan_s* p = new fif_plan_s();
  p->n = n; p->batch = batch; p->dtype = dtype; p->window = window; p->xi = xi; p->delta = delta;
  p->max_inner = max_inner; p->max_imfs = max_imfs; p->NC = (int)(NC < (1 << 30) ? NC : 0); p->regime = reg;
  // test-only knob: cap every persistent grid (other CTA schedules of the same decomposition must give the
  // same bits -- the determinism / race check that stands in for compute-sanitizer, closed on this pool)
  if (const char* gc = getenv("FIF_GRID_CAP")) p->grid_cap = atoi(gc) > 0 ? atoi(gc) : 0;
  if (cudaGetDevice(&p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) {
    free_plan(p);
    return FIF_ERR_CUDA;
  }
  if (reg == 3) {
    fif_status st = it_setup(p);
    if (st != FIF_OK) { free_plan(p); return st; }
    *out = p;
    return FIF_OK;
  }
  if (reg == 1) {
    fif_status st = st_setup(p);
    if (st != FIF_OK) { free_plan(p); return st; }
    *out = p;
    return FIF_OK;
  }
  if (reg == 4) {
    fif_status st = cl_setup(p);
    if (st == FIF_ERR_UNSUPPORTED_N && regime == FIF_REGIME_AUTO) {  // no cluster fits: the streamed regime
      cl_free(p);
      p->d_cl_scr = nullptr;
      p->regime = reg = 1;
      st::Geo g;
      st = st_geometry(n, dtype == FIF_F64, g) ? st_setup(p) : FIF_ERR_UNSUPPORTED_N;
    }
    if (st != FIF_OK) { free_plan(p); return st; }
    *out = p;
    return FIF_OK;
  }
  fif_status st = dtype == FIF_F64 ? upload_tables<double>(p) : upload_tables<float>(p);
  if (st != FIF_OK) { free_plan(p); return st; }
  const ResOps* ops = res_ops(dtype, p->NC);
  cudaError_t ce = ops->prepare();
  p->occ = ops->occupancy();
  p->block = ops->threads;
  p->smem = ops->smem;
  if (ce != cudaSuccess || p->occ < 1) {
    fprintf(stderr, "fif: kernel setup failed: %s (occ %d)\n", cudaGetErrorString(ce), p->occ);
    free_plan(p);
    return FIF_ERR_CUDA;
  }
  *out = p;
  return FIF_OK;
}

fif_status fif_plan_set_options(fif_plan_t p, fif_stop_rule stop, double gamma) {
  if (!p || (stop != FIF_STOP_SD && stop != FIF_STOP_N0) || !(gamma >= 0.0) || !(gamma < 1.0))
    return FIF_ERR_INVALID_ARG;
  if (p->regime == 3 && (stop != FIF_STOP_SD || gamma != 0.0)) return FIF_ERR_UNSUPPORTED_N;  // plain Alg. 2 only
  p->stop = (int32_t)stop;
  p->gamma = gamma;
  return FIF_OK;
}

fif_status fif_plan_set_mask_rule(fif_plan_t p, fif_mask_rule rule) {
  if (!p || (rule != FIF_MASK_EXTREMA && rule != FIF_MASK_SPECTRAL)) return FIF_ERR_INVALID_ARG;
  if (rule == FIF_MASK_SPECTRAL && (p->regime == 2 || p->regime == 3)) return FIF_ERR_UNSUPPORTED_N;
  if (rule == FIF_MASK_SPECTRAL && p->regime == 4) {
    // the cluster kernel has no spectral-peak search (its neighbouring bins live in other CTAs): the plan
    // becomes a streamed one, which computes the same decomposition (tests/test_gpu_cluster.py)
    if (cudaDeviceSynchronize() != cudaSuccess) return FIF_ERR_CUDA;
    st::Geo g;
    if (!st_geometry(p->n, p->dtype == FIF_F64, g)) return FIF_ERR_UNSUPPORTED_N;
    cl_free(p);
    p->d_cl_scr = nullptr;
    p->cl_P = p->cl_clusters = 0;
    cudaFree(p->d_Eh);
    cudaFree(p->d_El);
    cudaFree(p->d_tw);
    p->d_Eh = p->d_El = p->d_tw = nullptr;
    p->regime = 1;
    fif_status st = st_setup(p);
    if (st != FIF_OK) return st;
  }
  const int32_t old = p->mask;
  p->mask = (int32_t)rule;
  if (p->regime == 1 && old != p->mask) {  // the power array lives in the workspace: re-carve it
    fif_status s = FIF_ERR_INVALID_ARG;
    if (!p->d_ws_user || p->ws_user_bytes >= st_workspace_bytes(p))
      s = st_bind_workspace(p, p->d_ws_user, p->ws_user_bytes);
    if (s != FIF_OK) {
      p->mask = old;
      return s;
    }
  }
  return FIF_OK;
}

fif_status fif_plan_set_eigen_table(fif_plan_t p, int32_t enable) {
  if (!p) return FIF_ERR_INVALID_ARG;
  if (p->regime != 0) return enable ? FIF_ERR_UNSUPPORTED_N : FIF_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return FIF_ERR_CUDA;
  if (!enable) {
    cudaFree(p->d_wtab);
    p->d_wtab = nullptr;
    return FIF_OK;
  }
  if (p->d_wtab) return FIF_OK;
  const int nL = (int)((p->n - 1) / 4) - 1;  // L = 2 .. floor((n-1)/4) (reading A3)
  // per bin a Real pair {w_hat, a^(max_inner-1)} (fif_wtab_kernel)
  const size_t es = 2 * (p->dtype == FIF_F64 ? sizeof(double) : sizeof(float));
  if (cudaMalloc(&p->d_wtab, (size_t)nL * (size_t)(p->NC + 1) * es) != cudaSuccess) {
    p->d_wtab = nullptr;
    return FIF_ERR_OOM;
  }
  res_ops(p->dtype, p->NC)->fill_wtab(p, p->d_wtab, nL, 0);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p->d_wtab);
    p->d_wtab = nullptr;
    return FIF_ERR_CUDA;
  }
  return FIF_OK;
}

fif_status fif_plan_workspace_bytes(fif_plan_t p, size_t* bytes) {
  if (!p || !bytes) return FIF_ERR_INVALID_ARG;
  *bytes = p->regime == 1 ? st_workspace_bytes(p) : 0;
  return FIF_OK;
}

fif_status fif_plan_set_workspace(fif_plan_t p, void* d_ws, size_t bytes) {
  if (!p || ((uintptr_t)d_ws & 255u)) return FIF_ERR_INVALID_ARG;
  if (p->regime == 2) return d_ws ? FIF_ERR_INVALID_ARG : FIF_OK;  // distributed: plan-owned, peer-mappable
  if (p->regime != 1) return FIF_OK;                                 // resident / iterative: no workspace
  if (d_ws) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, d_ws) != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != p->device) {
      cudaGetLastError();
      return FIF_ERR_INVALID_ARG;
    }
  }
  return st_bind_workspace(p, d_ws, bytes);
}

fif_status fif_nccl_unique_id(void* out128) {
  if (!out128) return FIF_ERR_INVALID_ARG;
  return nccl_unique_id(out128);
}

static fif_status create_dist(fif_plan_t* out, int64_t n, fif_dtype dtype, fif_window window, double xi,
                              double delta, int32_t max_inner, int32_t max_imfs, const void* uid, int32_t rank,
                              int32_t nranks, int emulated) {
  if (!out) return FIF_ERR_INVALID_ARG;
  *out = nullptr;
  if (n < 9 || !(xi > 0.0) || !isfinite(xi) || !(delta > 0.0) || !isfinite(delta) || max_inner < 1 || max_imfs < 1 ||
      (dtype != FIF_F64 && dtype != FIF_F32) || (window != FIF_WINDOW_TRI_SQ && window != FIF_WINDOW_TRI_SQ_WIDE) ||
      nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || (!emulated && nranks > 1 && !uid))
    return FIF_ERR_INVALID_ARG;
  if (n % 2 || (n / 2) % ((int64_t)nranks * nranks)) return FIF_ERR_UNSUPPORTED_N;
  st::Geo g;
  if (!st_geometry(n / nranks, dtype == FIF_F64, g)) return FIF_ERR_UNSUPPORTED_N;
  fif_plan_s* p = new fif_plan_s();
  p->n = n; p->batch = 1; p->dtype = dtype; p->window = window; p->xi = xi; p->delta = delta;
  p->max_inner = max_inner; p->max_imfs = max_imfs; p->regime = 2;
  if (const char* gc = getenv("FIF_GRID_CAP")) p->grid_cap = atoi(gc) > 0 ? atoi(gc) : 0;
  if (cudaGetDevice(&p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) {
    free_plan(p);
    return FIF_ERR_CUDA;
  }
  fif_status st = dist_create(p, uid, rank, nranks, emulated);
  if (st != FIF_OK) { free_plan(p); return st; }
  *out = p;
  return FIF_OK;
}
fif_status fif_plan_create_dist(fif_plan_t* out, int64_t n_global, fif_dtype dtype, fif_window window, double xi,
                                double delta, int32_t max_inner, int32_t max_imfs, const void* nccl_unique_id,
                                int32_t rank, int32_t nranks) {
  return create_dist(out, n_global, dtype, window, xi, delta, max_inner, max_imfs, nccl_unique_id, rank, nranks, 0);
}
fif_status fif_plan_create_dist_emulated(fif_plan_t* out, int64_t n_global, fif_dtype dtype, fif_window window,
                                         double xi, double delta, int32_t max_inner, int32_t max_imfs,
                                         int32_t nranks) {
  return create_dist(out, n_global, dtype, window, xi, delta, max_inner, max_imfs, nullptr, 0, nranks, 1);
}

fif_status fif_decompose(fif_plan_t p, const void* d_signals, void* d_imfs, int32_t* d_imf_count,
                         int32_t* d_filter_len, int32_t* d_iters, void* stream) {
  if (!p) return FIF_ERR_INVALID_ARG;
  if (p->batch == 0) return FIF_OK;
  if (!d_signals || !d_imfs || !d_imf_count || !d_filter_len || !d_iters) return FIF_ERR_INVALID_ARG;
  if (((uintptr_t)d_signals | (uintptr_t)d_imfs) & 15) return FIF_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  Nvtx range(p->regime == 2 ? "fif_decompose/distributed"
             : p->regime == 1 ? "fif_decompose/streamed"
             : p->regime == 3 ? "fif_decompose/iterative"
             : p->regime == 4 ? "fif_decompose/cluster" : "fif_decompose/resident");
  if (p->regime == 2) {
    fif_status st = dist_decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, s);
    if (st != FIF_OK) return st;
    return launch_status();
  }
  if (p->regime == 1) {
    if (!p->d_X || !p->d_ctl) return FIF_ERR_INVALID_ARG;  // no workspace bound
    st_decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, 0, s);
    return launch_status();
  }
  if (p->regime == 3) {
    it_decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
    return launch_status();
  }
  if (p->regime == 4) {
    cl_decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
    return launch_status();
  }
  res_ops(p->dtype, p->NC)->decompose(p, d_signals, d_imfs, d_imf_count, d_filter_len, d_iters, p->batch, s);
  return launch_status();
}

fif_status fif_decompose_host(fif_plan_t p, const void* h_signals, void* h_imfs, int32_t* h_imf_count,
                              int32_t* h_filter_len, int32_t* h_iters, void* stream) {
  if (!p) return FIF_ERR_INVALID_ARG;
  if (p->batch == 0) return FIF_OK;
  if (!h_signals || !h_imfs || !h_imf_count || !h_filter_len || !h_iters) return FIF_ERR_INVALID_ARG;
  if (p->regime == 2) return FIF_ERR_INVALID_ARG;  // distributed plans take device buffers
  if (p->regime == 1 && (!p->d_X || !p->d_ctl)) return FIF_ERR_INVALID_ARG;  // no workspace bound
  Nvtx range("fif_decompose_host");
  const size_t es = elem_size(p->dtype);
  const size_t in_sig = (size_t)p->n * es, out_sig = in_sig * (size_t)(p->max_imfs + 1);
  const size_t meta_sig = (size_t)(1 + 2 * p->max_imfs);
  if (p->nstages == 0) {
    // chunks of ~1/8 of the batch (>= one full wave of CTAs when possible), 3 stages in flight.
    // Allocated into locals: p->nstages / p->chunk are committed only when every stage exists.
    int64_t chunk = (p->batch + 7) / 8;
    const int64_t wave = (int64_t)p->num_sms * (p->occ > 0 ? p->occ : 1);
    if (chunk < wave) chunk = wave < p->batch ? wave : p->batch;
    const int ns = (int)((p->batch + chunk - 1) / chunk < FIF_MAX_STAGES ? (p->batch + chunk - 1) / chunk
                                                                          : FIF_MAX_STAGES);
    Staging tmp[FIF_MAX_STAGES];
    fif_status err = FIF_OK;
    for (int i = 0; i < ns && err == FIF_OK; ++i) {
      Staging& S = tmp[i];
      if (cudaMalloc(&S.d_in, in_sig * chunk) != cudaSuccess || cudaMalloc(&S.d_out, out_sig * chunk) != cudaSuccess ||
          cudaMalloc(&S.d_meta, sizeof(int32_t) * meta_sig * chunk) != cudaSuccess)
        err = FIF_ERR_OOM;
      else if (cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking) != cudaSuccess ||
               cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming) != cudaSuccess)
        err = FIF_ERR_CUDA;
    }
    if (err != FIF_OK) {
      for (int i = 0; i < ns; ++i) {
        cudaFree(tmp[i].d_in);
        cudaFree(tmp[i].d_out);
        cudaFree(tmp[i].d_meta);
        if (tmp[i].stream) cudaStreamDestroy(tmp[i].stream);
        if (tmp[i].done) cudaEventDestroy(tmp[i].done);
      }
      cudaGetLastError();
      return err;
    }
    for (int i = 0; i < ns; ++i) p->st[i] = tmp[i];
    p->chunk = chunk;
    p->nstages = ns;
  }
  cudaStream_t user = (cudaStream_t)stream;
  cudaEvent_t start;
  if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) != cudaSuccess) return FIF_ERR_CUDA;
  bool ok = cudaEventRecord(start, user) == cudaSuccess;
  for (int i = 0; i < p->nstages && ok; ++i) ok = cudaStreamWaitEvent(p->st[i].stream, start, 0) == cudaSuccess;
  const int64_t nchunks = (p->batch + p->chunk - 1) / p->chunk;
  for (int64_t c = 0; c < nchunks && ok; ++c) {
    Staging& S = p->st[c % p->nstages];
    const int64_t b0 = c * p->chunk, nb = (b0 + p->chunk <= p->batch) ? p->chunk : p->batch - b0;
    int32_t* d_cnt = S.d_meta;
    int32_t* d_len = S.d_meta + nb;
    int32_t* d_it = d_len + nb * p->max_imfs;
    ok = cudaMemcpyAsync(S.d_in, (const char*)h_signals + b0 * in_sig, nb * in_sig, cudaMemcpyHostToDevice,
                         S.stream) == cudaSuccess;
    if (!ok) break;
    if (p->regime == 1) {
      // disjoint plan work buffers per chunk (chunks run concurrently on the staging streams)
      st_decompose(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, b0, S.stream);
    } else if (p->regime == 3) {
      it_decompose(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
    } else if (p->regime == 4) {
      cl_decompose(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
    } else {
      res_ops(p->dtype, p->NC)->decompose(p, S.d_in, S.d_out, d_cnt, d_len, d_it, nb, S.stream);
    }
    ok = cudaMemcpyAsync((char*)h_imfs + b0 * out_sig, S.d_out, nb * out_sig, cudaMemcpyDeviceToHost, S.stream) ==
             cudaSuccess &&
         cudaMemcpyAsync(h_imf_count + b0, d_cnt, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, S.stream) ==
             cudaSuccess &&
         cudaMemcpyAsync(h_filter_len + b0 * p->max_imfs, d_len, sizeof(int32_t) * nb * p->max_imfs,
                         cudaMemcpyDeviceToHost, S.stream) == cudaSuccess &&
         cudaMemcpyAsync(h_iters + b0 * p->max_imfs, d_it, sizeof(int32_t) * nb * p->max_imfs, cudaMemcpyDeviceToHost,
                         S.stream) == cudaSuccess;
  }
  // the user stream waits for every stage whatever happened, so no staged work outlives the call unseen
  for (int i = 0; i < p->nstages; ++i) {
    cudaEventRecord(p->st[i].done, p->st[i].stream);
    cudaStreamWaitEvent(user, p->st[i].done, 0);
  }
  cudaEventDestroy(start);
  if (!ok) {
    fprintf(stderr, "fif: host-path copy or event failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaStreamSynchronize(user);
    return FIF_ERR_CUDA;
  }
  fif_status st = launch_status();
  if (st != FIF_OK) return st;
  if (cudaStreamSynchronize(user) != cudaSuccess) return FIF_ERR_CUDA;
  return FIF_OK;
}

fif_status fif_destroy(fif_plan_t p) {
  if (!p) return FIF_OK;
  cudaDeviceSynchronize();
  free_plan(p);
  return FIF_OK;
}

int32_t fif_plan_kernels_per_call(fif_plan_t p) {
  if (!p || p->batch == 0) return 0;
  if (p->regime == 2) return dist_kernels_per_call(p);
  return p->regime == 1 ? st_kernels_per_call(p) : 1;
}

const char* fif_plan_regime(fif_plan_t p) {
  if (!p) return "none";
  if (p->regime == 3) return "iterative";
  if (p->regime == 4) return "cluster";
  return p->regime == 2 ? "distributed" : (p->regime == 1 ? "streamed" : "resident");
}

fif_status fif_plan_launch_config(fif_plan_t p, int32_t* grid, int32_t* block, int32_t* smem_bytes) {
  if (!p) return FIF_ERR_INVALID_ARG;
  const int64_t cap = p->regime == 1 ? (int64_t)p->st_grid
                      : p->regime == 4 ? (int64_t)p->cl_clusters * p->cl_P : (int64_t)p->num_sms * p->occ;
  if (grid) *grid = (int32_t)(p->regime == 1 ? cap
                             : p->regime == 4 ? (p->batch < p->cl_clusters ? p->batch * p->cl_P : cap)
                                              : (p->batch < cap ? p->batch : cap));
  if (block) *block = p->block;
  if (smem_bytes) *smem_bytes = (int32_t)p->smem;
  return FIF_OK;
}

// ---------------------------------------------------------------- test hooks
#define HOOK_SYNC(s)                                       \
  do {                                                     \
    fif_status st_ = launch_status();                      \
    if (st_ != FIF_OK) return st_;                         \
    if (cudaStreamSynchronize(s) != cudaSuccess) return FIF_ERR_CUDA; \
    return FIF_OK;                                         \
  } while (0)

fif_status fif_test_rfft(fif_plan_t p, int64_t batch, const void* d_in, void* d_out, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_out))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  res_ops(p->dtype, p->NC)->test_rfft(p, d_in, d_out, batch, s);
  HOOK_SYNC(s);
}

fif_status fif_test_irfft(fif_plan_t p, int64_t batch, const void* d_in, void* d_out, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_out))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  res_ops(p->dtype, p->NC)->test_irfft(p, d_in, d_out, batch, s);
  HOOK_SYNC(s);
}

fif_status fif_test_extrema(fif_plan_t p, int64_t batch, const void* d_in, int32_t* d_k, void* stream) {
  if (!p || batch < 0 || (batch && (!d_in || !d_k))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  res_ops(p->dtype, p->NC)->test_extrema(p, d_in, d_k, batch, s);
  HOOK_SYNC(s);
}

fif_status fif_test_window_spectrum(fif_plan_t p, int32_t L, void* d_out, void* stream) {
  if (!p || L < 1 || !d_out) return FIF_ERR_INVALID_ARG;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;
  cudaStream_t s = (cudaStream_t)stream;
  res_ops(p->dtype, p->NC)->test_window(p, L, d_out, s);
  HOOK_SYNC(s);
}

fif_status fif_test_inner(fif_plan_t p, int64_t batch, int32_t L, const void* d_in, void* d_imf, int32_t* d_N,
                          void* stream) {
  if (!p || batch < 0 || L < 1 || (batch && (!d_in || !d_imf || !d_N))) return FIF_ERR_INVALID_ARG;
  if (!batch) return FIF_OK;
  if (p->regime != 0) return FIF_ERR_UNSUPPORTED_N;  // hooks exercise the resident kernels
  cudaStream_t s = (cudaStream_t)stream;
  res_ops(p->dtype, p->NC)->test_inner(p, L, d_in, d_imf, d_N, batch, s);
  HOOK_SYNC(s);
}

}  // extern "C"
