// extern "C" entry points (include/nld_b200.h).  Each converts C++ errors
// into the status codes that the Python shim maps back onto the reference's
// exception classes (errors.py:4-45).
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nld_internal.cuh"

namespace nld {

static thread_local std::string g_last_error;

void set_error(int code, const std::string& msg) {
  (void)code;
  g_last_error = msg;
}

int fail(int code, const std::string& msg) {
  set_error(code, msg);
  return code;
}

void comm_host(nld_operator* op, void* buf, int64_t count, int dtype, int red) {
  if (!op->comm || count <= 0) return;
  if (op->comm(op->comm_ctx, buf, count, dtype, red, 0, nullptr) != 0)
    throw Error(NLD_ERR_CUDA, "allreduce callback failed (host buffer)");
}

void comm_device(nld_operator* op, double* buf, int64_t count, cudaStream_t st) {
  if (!op->comm || count <= 0) return;
  if (op->comm(op->comm_ctx, buf, count, RED_F64, RED_OP_SUM, 1, st) != 0)
    throw Error(NLD_ERR_CUDA, "allreduce callback failed (device buffer)");
}

}  // namespace nld

using nld::Error;

namespace {

// select the device that owns `ptr` (torch may have set another device on the
// calling thread; this library's runtime keeps its own current device)
void select_device_of(const void* ptr, int fallback) {
  int dev = fallback;
  if (ptr) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, ptr) == cudaSuccess &&
        attr.type == cudaMemoryTypeDevice)
      dev = attr.device;
    else
      cudaGetLastError();
  }
  NLD_CUDA(cudaSetDevice(dev));
}

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return NLD_OK;
  } catch (const Error& e) {
    return nld::fail(e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return nld::fail(NLD_ERR_CUDA, "host allocation failed");
  } catch (...) {
    return nld::fail(NLD_ERR_CUDA, "unknown failure");
  }
}

void ensure_built(nld_operator* op, int which, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(op->build_mu);
  if (op->params.mode == 1 || op->built[which]) return;
  nld::build_planset(op, which, st);
  op->built[which] = true;
}

const double* ensure_degree(nld_operator* op, int which, cudaStream_t st) {
  if (op->eta[which]) return op->eta[which];
  ensure_built(op, which, st);
  double* eta = nullptr;
  NLD_CUDA(cudaMalloc(&eta, sizeof(double) * op->N));
  double* ones = nullptr;
  NLD_CUDA(cudaMallocAsync(&ones, sizeof(double) * op->N, st));
  std::vector<double> h(op->N, 1.0);
  NLD_CUDA(cudaMemcpyAsync(ones, h.data(), sizeof(double) * op->N, cudaMemcpyHostToDevice, st));
  if (op->params.mode == 1)
    nld::dense_apply(op, which, NLD_APPLY_GAMMA, ones, eta, 1, op->N, nullptr, nullptr, st);
  else
    nld::apply_op(op, which, NLD_APPLY_GAMMA, ones, eta, 1, op->N, nullptr, nullptr, st);
  cudaFreeAsync(ones, st);
  NLD_CUDA(cudaStreamSynchronize(st));
  op->eta[which] = eta;
  return eta;
}

}  // namespace

extern "C" {

const char* nld_last_error(void) { return nld::g_last_error.c_str(); }

#ifdef NLD_AB_BUILD
int nld_abi_version(void) { return 1000 + NLD_ABI_VERSION; }   // test build: never the product
#else
int nld_abi_version(void) { return NLD_ABI_VERSION; }
#endif

int nld_op_create(const double* features_dev, int64_t n, int32_t n_features,
                  const int32_t* window_index, const int32_t* window_offset,
                  int32_t n_windows, double sigma, const nld_params* params, void* stream,
                  nld_operator** out) {
  return guarded([&] {
    if (!out) throw Error(NLD_ERR_VALUE, "null output handle");
    *out = nullptr;
    if (n <= 0) throw Error(NLD_ERR_DIMENSION, "at least one node is required");
    if (n_features <= 0) throw Error(NLD_ERR_DIMENSION, "features must be a 2-d array");
    if (!(sigma > 0)) throw Error(NLD_ERR_VALUE, "kernel width sigma must be positive");
    if (n_windows <= 0) throw Error(NLD_ERR_VALUE, "at least one feature window is required");
    if (!params) throw Error(NLD_ERR_VALUE, "null params");
    if (params->mode != 0 && params->mode != 1) throw Error(NLD_ERR_VALUE, "unknown mode");
    for (int w = 0; w < n_windows; ++w) {
      int sz = window_offset[w + 1] - window_offset[w];
      if (sz <= 0 || sz > 3)
        throw Error(NLD_ERR_WINDOW, "windows must have one to three feature dimensions");
      for (int k = window_offset[w]; k < window_offset[w + 1]; ++k)
        if (window_index[k] < 0 || window_index[k] >= n_features)
          throw Error(NLD_ERR_DIMENSION, "window index out of range");
    }
    if (params->mode == 0) {
      if (params->cutoff < 1 || params->cutoff > 8)
        throw Error(NLD_ERR_VALUE, "window cutoff must lie in [1, 8]");
      if (params->oversampling < 1.25)
        throw Error(NLD_ERR_VALUE, "oversampling factor must be >= 1.25");
      if (!(params->rmax > 0 && params->rmax <= 0.25))
        throw Error(NLD_ERR_VALUE, "rmax must lie in (0, 1/4]");
      if (params->n_expansion > 0 && params->n_expansion % 2)
        throw Error(NLD_ERR_VALUE, "expansion degree must be even");
    }
    if (n * (int64_t)n_windows >= (int64_t)INT32_MAX)
      throw Error(NLD_ERR_VALUE, "too many nodes for 32-bit node indices");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    select_device_of(features_dev, 0);
    {
      // keep stream-ordered temporaries cached instead of returning them to
      // the OS at every synchronisation
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
    }
    auto* op = new nld_operator();
    try {
      NLD_CUDA(cudaGetDevice(&op->device));
      op->N = n;
      op->N_global = n;
      op->D = n_features;
      op->L = n_windows;
      op->sigma = sigma;
      op->params = *params;
      op->win_offset.assign(window_offset, window_offset + n_windows + 1);
      op->win_index.assign(window_index, window_index + window_offset[n_windows]);
      NLD_CUDA(cudaMalloc(&op->feats, sizeof(double) * n * n_features));
      NLD_CUDA(cudaMemcpyAsync(op->feats, features_dev, sizeof(double) * n * n_features,
                               cudaMemcpyDeviceToDevice, st));
      NLD_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFree(op->feats);
      delete op;
      throw;
    }
    *out = op;
  });
}

int nld_op_destroy(nld_operator* op) {
  if (!op) return NLD_OK;
  return guarded([&] {
    cudaSetDevice(op->device);
    cudaDeviceSynchronize();
    for (int k = 0; k < 2; ++k) {
      if (op->built[k]) nld::free_planset(op->sets[k]);
      cudaFree(op->eta[k]);
    }
    nld::free_workspace(op->ws);
    cudaFree(op->feats);
    if (op->events)
      for (auto& e : op->ev) cudaEventDestroy(e);
    if (op->aux) {
      for (int w = 0; w < op->aux_windows; ++w) {
        cudaEventDestroy(op->ev_spread[w]);
        cudaEventDestroy(op->ev_conv[w]);
      }
      cudaEventDestroy(op->ev_fork);
      cudaEventDestroy(op->ev_join);
      cudaStreamDestroy(op->aux);
      if (op->aux2) cudaStreamDestroy(op->aux2);
    }
    delete op;
  });
}

int nld_op_set_comm(nld_operator* op, nld_allreduce_fn fn, void* ctx, int64_t global_n) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    if (op->built[0] || op->built[1])
      throw Error(NLD_ERR_VALUE, "set_comm must precede the first product");
    if (global_n < op->N) throw Error(NLD_ERR_DIMENSION, "global_n smaller than local n");
    if (op->params.mode == 1 && fn)
      throw Error(NLD_ERR_VALUE, "exact mode cannot be sharded");
    op->comm = fn;
    op->comm_ctx = ctx;
    op->N_global = global_n;
  });
}

int nld_op_set_timing(nld_operator* op, int32_t enabled) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    NLD_CUDA(cudaSetDevice(op->device));
    if (enabled && !op->events) {
      for (auto& e : op->ev) NLD_CUDA(cudaEventCreate(&e));
      op->events = true;
    }
    op->timing = enabled;
  });
}

int nld_op_debug_poison(nld_operator* op) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    NLD_CUDA(cudaSetDevice(op->device));
    NLD_CUDA(cudaDeviceSynchronize());
    nld::Workspace& ws = op->ws;
    const int64_t cap = std::max(ws.nrhs_cap, 1);
    const int64_t gt = std::max<int64_t>(1, ws.grid_total) * cap;
    auto fill = [](void* p, size_t bytes) {
      if (p && bytes) NLD_CUDA(cudaMemset(p, 0xFF, bytes));
    };
    fill(ws.blocks, sizeof(double) * std::max<int64_t>(1, ws.blocks_total) * cap);
    fill(ws.grid_in, sizeof(double) * (gt + cap));
    fill(ws.grid_out, sizeof(double) * gt);
    fill(ws.cbuf0, sizeof(double2) * gt);
    fill(ws.cbuf1, sizeof(double2) * gt);
    fill(ws.wout, sizeof(double) * std::max<int64_t>(1, op->N * op->L) * cap);
    fill(ws.vt, sizeof(double) * std::max<int64_t>(1, op->N) * cap);
    fill(ws.asm_y2, sizeof(double) * (ws.asm_cap / 8 + 1));
    fill(ws.asm_y2b, sizeof(double) * (ws.asm_cap / 8 + 1));
    fill(ws.cbuf2, sizeof(double2) * gt);
    fill(ws.cbuf3, sizeof(double2) * gt);
    if (ws.gdig) fill(ws.gdig, (size_t)nld::gather_gdig_bytes() * ws.gdig_cells * (cap / 16));
    fill(ws.cg, sizeof(double) * 6 * ws.cg_cap);
    NLD_CUDA(cudaDeviceSynchronize());
  });
}

int nld_op_apply(nld_operator* op, int32_t kind, const double* v, double* out, int32_t nrhs,
                 int64_t ld, const double* coef_host, void* stream) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    if (nrhs <= 0) throw Error(NLD_ERR_DIMENSION, "nrhs must be positive");
    if (ld < op->N) throw Error(NLD_ERR_DIMENSION, "leading dimension smaller than n");
    const int pm = (kind & NLD_LAYOUT_PIXEL_MAJOR) ? 1 : 0;
    kind &= ~NLD_LAYOUT_PIXEL_MAJOR;
    if (pm && nrhs > 256) throw Error(NLD_ERR_VALUE, "pixel-major batches hold at most 256 rhs");
    if (kind < 0 || kind > NLD_APPLY_WINDOW_SUM) throw Error(NLD_ERR_VALUE, "unknown kind");
    NLD_CUDA(cudaSetDevice(op->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int which = kind == NLD_APPLY_GAMMA_SQUARED ? 1 : 0;
    ensure_built(op, which, st);
    const double* eta = nullptr;
    if (kind == NLD_APPLY_SYSTEM || kind == NLD_APPLY_LAPLACIAN) eta = ensure_degree(op, 0, st);
    if (op->params.mode == 0) nld::ensure_workspace(op, op->sets[which], nrhs);
    double* coef = nullptr;
    if (kind == NLD_APPLY_SYSTEM) {
      if (!coef_host) throw Error(NLD_ERR_VALUE, "system apply needs (lam, mu) per rhs");
      NLD_CUDA(cudaMallocAsync(&coef, sizeof(double) * 2 * nrhs, st));
      NLD_CUDA(cudaMemcpyAsync(coef, coef_host, sizeof(double) * 2 * nrhs,
                               cudaMemcpyHostToDevice, st));
    }
    if (op->params.mode == 1) {
      if (kind == NLD_APPLY_WINDOW_SUM) throw Error(NLD_ERR_VALUE, "window sums need fast mode");
      nld::dense_apply(op, which, kind, v, out, nrhs, ld, coef, eta, st, pm);
    } else {
      nld::apply_op(op, which, kind, v, out, nrhs, ld, coef, eta, st, pm);
    }
    if (coef) cudaFreeAsync(coef, st);
    if (op->timing && op->events && op->params.mode == 0) {
      NLD_CUDA(cudaEventSynchronize(op->ev[5]));
      float t[5];
      for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&t[k], op->ev[k], op->ev[k + 1]);
      op->stats.spread_ms = t[0];
      op->stats.assemble_ms = t[1];
      op->stats.conv_ms = t[2];
      op->stats.gather_ms = t[3];
      op->stats.epilogue_ms = t[4];
      cudaEventElapsedTime(&op->stats.total_ms, op->ev[0], op->ev[5]);
    }
    NLD_CUDA(cudaGetLastError());
  });
}

int nld_op_degree(nld_operator* op, int32_t squared, double* eta_out, void* stream) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    NLD_CUDA(cudaSetDevice(op->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int which = squared ? 1 : 0;
    const double* eta = ensure_degree(op, which, st);
    if (eta_out) {
      if (squared)  // degree_squared = apply_squared(1) * L (kernel.py:148-154)
        nld::dev_axpby((double)op->L, eta, 0.0, eta, eta_out, op->N, st);
      else
        NLD_CUDA(cudaMemcpyAsync(eta_out, eta, sizeof(double) * op->N,
                                 cudaMemcpyDeviceToDevice, st));
    }
  });
}

int nld_op_assemble_dense(nld_operator* op, int32_t squared, double* out, void* stream) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    NLD_CUDA(cudaSetDevice(op->device));
    nld::dense_assemble(op, squared ? 1 : 0, out, static_cast<cudaStream_t>(stream));
  });
}

int nld_op_window_info(const nld_operator* op, int32_t window, nld_window_info* out) {
  return guarded([&] {
    if (!op || !out) throw Error(NLD_ERR_VALUE, "null argument");
    if (window < 0 || window >= op->L) throw Error(NLD_ERR_DIMENSION, "window out of range");
    std::memset(out, 0, sizeof(*out));
    if (!op->built[0]) throw Error(NLD_ERR_VALUE, "plans not built yet (apply first)");
    const nld::WinPlan& wp = op->sets[0].win[window];
    out->dim = wp.d;
    out->bandwidth = wp.M;
    out->grid = wp.n;
    out->cutoff = wp.m;
    for (int s = 0; s < 3; ++s) {
      out->center[s] = wp.center[s];
      out->box_lo[s] = wp.box_lo[s];
      out->box_w[s] = wp.box_w[s];
    }
    out->scale = wp.scale;
    out->sig_scaled = wp.sig_scaled;
    out->n_cells = wp.n_cells;
    out->n_subproblems = wp.n_subs;
    out->n_edge = wp.n_edge;
  });
}

int nld_op_stats(const nld_operator* op, nld_stats* out) {
  return guarded([&] {
    if (!op || !out) throw Error(NLD_ERR_VALUE, "null argument");
    *out = op->stats;
  });
}

int nld_cg_solve(nld_operator* op, const double* f, double* u, int32_t nrhs, int64_t ld,
                 const double* lam, const double* mu, int32_t precond, int32_t deflate,
                 double tol, int32_t maxit, int32_t warm_start, int32_t* iterations,
                 double* relres, int32_t* converged, double* history, int32_t history_cap,
                 void* stream) {
  return guarded([&] {
    if (!op) throw Error(NLD_ERR_VALUE, "null operator");
    if (nrhs <= 0) throw Error(NLD_ERR_DIMENSION, "nrhs must be positive");
    if (ld < op->N) throw Error(NLD_ERR_DIMENSION, "leading dimension smaller than n");
    if (precond < 0 || precond > 2) throw Error(NLD_ERR_VALUE, "unknown preconditioner");
    NLD_CUDA(cudaSetDevice(op->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ensure_built(op, 0, st);
    if (precond == NLD_PREC_L2) ensure_built(op, 1, st);
    nld::cg_solve(op, f, u, nrhs, ld, lam, mu, precond, deflate, tol, maxit, warm_start,
                  iterations, relres, converged, history, history_cap, st);
  });
}

int nld_basis_apply(const double* v, const double* x, double* out, int64_t n, int32_t adjoint,
                    void* stream) {
  return guarded([&] {
    if (n < 2) throw Error(NLD_ERR_DIMENSION, "basis needs at least two entries");
    select_device_of(v, 0);
    nld::dev_basis(v, x, out, n, adjoint, static_cast<cudaStream_t>(stream));
  });
}

int nld_scs(const double* x, double* out, int64_t n, int32_t down, void* stream) {
  return guarded([&] {
    if (n < 1) throw Error(NLD_ERR_DIMENSION, "empty vector");
    select_device_of(x, 0);
    nld::dev_scs(x, out, n, down, static_cast<cudaStream_t>(stream));
  });
}

int nld_axpby(double a, const double* x, double b, const double* y, double* out, int64_t n,
              void* stream) {
  return guarded([&] {
    select_device_of(x, 0);
    nld::dev_axpby(a, x, b, y, out, n, static_cast<cudaStream_t>(stream));
  });
}

int nld_dot(const double* x, const double* y, int64_t n, double* result, void* stream) {
  return guarded([&] {
    select_device_of(x, 0);
    *result = nld::dev_dot(x, y, n, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
