// Internal declarations shared by the nld_b200 translation units.
//
// Data layout in HBM (one operator, one plan set = one Gaussian width):
//   rows    : per window, the sorted node table.  Node e of window w has a
//             row of S*d fp64 principal Kaiser-Bessel weights (S = 2m, the
//             stencil offsets i = 1..2m of node_tables, transform.py:147-170),
//             dimension-major: [w_dim0(S)][w_dim1(S)][w_dim2(S)].
//   pix     : per window, int32 original pixel of sorted node e.
//   key     : per window, int32 flattened cell coordinate (sort key).
//   cells   : occupied stencil cells (all windows), with their subproblems.
//   subs    : work items: <= kSubMax nodes of one cell (grouped by dim).
//   grids   : per window the support box of the oversampled grid, real fp64,
//             [nrhs][sum of box sizes].
//   K       : per window the separable convolution kernel K(delta),
//             delta = 0..n-1, complex fp64 (FFT -> x coeffs -> FFT, fused).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/nld_b200.h"

namespace nld {

// Nodes per subproblem: between kSubMin and kSubMax, chosen per window so that
// every SM still gets several items (sub_cap).  Upper bound: the sliced spread
// sums K products of magnitude <= 2^14 per digit pair, six pairs per
// diagonal, in int32 (K <= 16384).  Large items amortise the per-item costs
// (spread accumulator drain, G digit load); small windows keep 2048 so the
// persistent kernels' snake deal stays balanced.
constexpr int kSubMin = 2048;
#ifndef NLD_SUB_MAX
#define NLD_SUB_MAX 8192
#endif
constexpr int kSubMax = NLD_SUB_MAX;
static_assert(kSubMax <= 16384 && kSubMax >= kSubMin, "subproblem size cap");
inline int sub_cap(long long nodes, int sms) {
  const long long per = nodes / ((long long)sms * 8);     // >= ~8 full items per SM
  long long cap = per < kSubMin ? kSubMin : (per > kSubMax ? kSubMax : per);
  return (int)((cap + 127) & ~127LL);
}
// A cell's subproblems: nsub = ceil(cnt / kSubMax) near-equal parts, sized in
// whole 128-node gather tiles -- no small remainder item paying the per-item
// costs (spread accumulator drain, G digit load) for a few nodes.
__host__ __device__ inline int sub_size(int cnt, int nsub) {
  const int per = (cnt + nsub - 1) / nsub;
  const int per128 = (per + 127) & ~127;
  return ((int64_t)(nsub - 1) * per128 < cnt) ? per128 : per;
}
constexpr int kMaxDim = 3;

struct Status {
  int code = NLD_OK;
  std::string msg;
};

void set_error(int code, const std::string& msg);
int fail(int code, const std::string& msg);

#define NLD_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) {                                               \
      throw ::nld::Error(NLD_ERR_CUDA, std::string(#call) + ": " +         \
                                           cudaGetErrorString(_e));        \
    }                                                                      \
  } while (0)

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

// Device-visible description of one window of one plan set.
struct WinDev {
  int d;             // window dimension 1..3
  int n;             // oversampled grid size per dimension
  int S;             // 2m principal stencil width
  int wrap;          // 1: box is the whole torus (positions mod n)
  int box_w[3];      // support box extents (unused dims = 1)
  int box_lo[3];
  int64_t box_size;  // prod box_w
  int64_t grid_off;  // offset of this window's box in a per-rhs grid buffer
  int64_t kern_off;  // offset (complex entries) into the K table
  int64_t cellmap_off;
  int64_t node_off;  // offset (nodes) into pix/key of this window = w*N
  int64_t row_off;   // offset (doubles) into rows
  int fast;          // 1: block path (templated kernels), 0: generic path
  int pad;
};

struct SubDev {
  int64_t start;     // absolute node index (w*N + sorted position)
  int64_t block;     // offset (doubles) of its partial block in the scratch
  int32_t count;
  int32_t cell;      // global cell index
  int32_t win;
  int32_t pad;
};

struct CellDev {
  int32_t cc[3];     // cell coordinate in box units (first principal point)
  int32_t win;
  int64_t block0;    // offset (doubles) of its first subproblem block
  int32_t nsub;
  int32_t blk;       // block size S^d
};

struct EdgeDev {     // node with a nonzero weight at i = 0 or i = 2m+1
  int32_t pix;
  int32_t win;
  int32_t cc[3];
  int32_t pad;
  double w[3][18];   // full width W = 2m+2 weights, m <= 8
};

// Host-side plan of one window.
struct WinPlan {
  int d = 0;
  int cols[3] = {0, 0, 0};
  double center[3] = {0, 0, 0};
  double scale = 1.0, sig_scaled = 0.0;
  int M = 0, n = 0, m = 0;
  double b = 0.0;
  int box_lo[3] = {0, 0, 0}, box_w[3] = {1, 1, 1};
  int wrap = 0;
  int64_t n_cells = 0, n_subs = 0, n_edge = 0;
  int64_t sub_off = 0;           // first subproblem in its dimension group
  int64_t edge_off = 0;          // first edge node in the edge list
};

// One Gaussian width (sigbar = 1/sigma^2 or 2/sigma^2) with its tables.
struct PlanSet {
  double sigbar = 0.0;
  std::vector<WinPlan> win;
  std::vector<WinDev> wdev_h;
  WinDev* wdev = nullptr;        // device copy
  double* rows = nullptr;
  int32_t* pix = nullptr;
  int32_t* key = nullptr;
  int32_t* cellmap = nullptr;
  int2* cellinfo = nullptr;      // per box key: (block offset / blk, nsub)
  double2* K = nullptr;
  CellDev* cells = nullptr;
  int64_t n_cells = 0;
  SubDev* subs[kMaxDim + 1] = {nullptr, nullptr, nullptr, nullptr};
  int64_t n_subs[kMaxDim + 1] = {0, 0, 0, 0};
  int64_t blocks_total = 0;      // doubles per rhs of block scratch
  EdgeDev* edges = nullptr;
  int64_t n_edges = 0;
  int64_t grid_total = 0;        // sum of box sizes
  int64_t generic_nodes = 0;     // nodes in windows on the generic path
  int16_t* sub_exp = nullptr;    // sliced spread: per 3-D subproblem eA/eB/eC
  int32_t* sub_order = nullptr;  // per window: its 3-D subproblems by descending size
  bool oz_ok = false;            // integer-sliced spread/gather enabled (no_sliced knob)
  std::vector<int64_t> gcell_lo, gcell_n;   // per window: its cells' global range
  int shares_tables_with = -1;   // index of the plan set whose tables we use
  bool owns_tables = true;
};

struct Workspace {
  int nrhs_cap = 0;
  double* blocks = nullptr;      // [blocks_total][nrhs]
  double* grid_in = nullptr;     // [nrhs][grid_total]
  double* grid_out = nullptr;
  double2* cbuf0 = nullptr;
  double2* cbuf1 = nullptr;
  double2* cbuf2 = nullptr;      // second aux stream's convolution scratch
  double2* cbuf3 = nullptr;
  double* wout = nullptr;        // [L][N][nrhs] per-window gathers
  double* vt = nullptr;          // [N][nrhs] pixel-major rhs
  double* coef = nullptr;        // [nrhs][2]
  int64_t grid_total = 0, blocks_total = 0;
  // separable assemble scratch (3-D windows): Y2 [box][8][nrhs] = asm_cap / 8
  double* asm_y2 = nullptr;
  double* asm_y2b = nullptr;     // second aux stream's assemble scratch
  int64_t asm_cap = 0;
  unsigned long long* vmax = nullptr;   // [nrhs_cap] sliced spread: max |v| bits
  uint8_t* gdig = nullptr;       // sliced gather: per (cell, 16-rhs group) G digits + exponents
  int64_t gdig_cells = 0;
  bool gdig_on_aux = false;      // this product's G digits were cut on the aux stream
  // persistent CG vectors (x, r, p, q, b, t): [6][cg_cap]
  double* cg = nullptr;
  int64_t cg_cap = 0;
};

}  // namespace nld

struct nld_operator {
  int64_t N = 0;                 // local nodes (this shard)
  int64_t N_global = 0;          // all shards
  nld_allreduce_fn comm = nullptr;
  void* comm_ctx = nullptr;
  int D = 0;
  int L = 0;
  double sigma = 0.0;
  nld_params params{};
  int device = 0;
  double* feats = nullptr;       // not owned (only used at plan build)
  std::vector<int> win_index, win_offset;
  nld::PlanSet sets[2];          // [0] sigbar, [1] squared
  bool built[2] = {false, false};
  double* eta[2] = {nullptr, nullptr};
  nld::Workspace ws;
  double* dense[2] = {nullptr, nullptr};
  int timing = 0;
  nld_stats stats{};
  cudaEvent_t ev[6] = {};
  bool events = false;
  cudaStream_t aux = nullptr;    // assemble/convolution streams (overlap): windows
  cudaStream_t aux2 = nullptr;   // alternate between them
  cudaEvent_t ev_spread[16] = {}, ev_conv[16] = {}, ev_fork = nullptr, ev_join = nullptr;
  int aux_windows = 0;
  std::mutex build_mu;           // lazy plan build (per operator: shards may
                                 // build concurrently in one process)
  // raw-torus plans (NFFT transform API): nodes used as given after the
  // affine map (p - raw_center) * raw_scale, no bounding-box scaling
  int raw = 0;
  int raw_check = 0;             // ScalingOverflowError if |q| >= 1/2
  double raw_center[3] = {0, 0, 0};
  double raw_scale = 1.0;
};

namespace nld {

void build_planset(nld_operator* op, int which, cudaStream_t st);
// integer-sliced tensor-core spread (nld_ozaki.cu)
bool use_ozaki();
int16_t* ozaki_exponents(PlanSet& ps, bool tables, cudaStream_t st);
void launch_spread_oz(const PlanSet& ps, const SubDev* subs, const int16_t* ex,
                      unsigned nsub, const unsigned long long* vmax,
                      const double* vt, int nrhs, double* blocks, cudaStream_t st,
                      const int32_t* order = nullptr);
void ozaki_vmax(const double* vt, int64_t n, int nrhs, unsigned long long* out, double* flag,
                cudaStream_t st);
void ozaki_poison(const double* flag, int nrhs, double* out, int64_t n, int64_t ld,
                  int pixel_major, cudaStream_t st);
void ozaki_prof_dump(const char* what, cudaStream_t st);
namespace mma { struct GatherEpi; }
void launch_gather_nm(const PlanSet& ps, const SubDev* subs, const int16_t* ex,
                      const int32_t* order, unsigned nsub, const double* grid, int64_t grid_ld,
                      double* out, int nrhs, const mma::GatherEpi& ep, cudaStream_t st,
                      uint8_t* gdig, int64_t cell_lo, int64_t ncell, bool gdig_ready = false);
void launch_gdig_nm(const PlanSet& ps, const double* grid, int64_t grid_ld, int nrhs,
                    uint8_t* gdig, int64_t cell_lo, int64_t ncell, cudaStream_t st);
// bytes per (cell, 16-rhs group) of precomputed gather G digits
int64_t gather_gdig_bytes();
void free_planset(PlanSet& ps);
void ensure_workspace(nld_operator* op, const PlanSet& ps, int nrhs);
void free_workspace(Workspace& ws);

// one fused operator application (all windows, nrhs right-hand sides)
void apply_op(nld_operator* op, int which, int kind, const double* v,
              double* out, int nrhs, int64_t ld, const double* coef_dev,
              const double* eta, cudaStream_t st, int pixel_major = 0,
              const unsigned long long* vmax_pre = nullptr, const double* flag_pre = nullptr);

// the two halves of a product, reused by the NFFT transform API
int spread_stage(nld_operator* op, const PlanSet& ps, const double* vt, int nrhs,
                 cudaStream_t st, bool flags = false);
int gather_stage(nld_operator* op, const PlanSet& ps, int nrhs, cudaStream_t st);

void dense_apply(nld_operator* op, int which, int kind, const double* v,
                 double* out, int nrhs, int64_t ld, const double* coef_dev,
                 const double* eta, cudaStream_t st, int pixel_major = 0);
// layout changes between rhs-major [nrhs][ld] and pixel-major [n][nrhs]
void to_pixel_major(const double* v, int64_t ldv, int64_t n, int nrhs, double* vt,
                    cudaStream_t st);
void to_rhs_major(const double* vt, int64_t n, int nrhs, double* out, int64_t ldo,
                  cudaStream_t st);
void dense_assemble(nld_operator* op, int which, double* out, cudaStream_t st);

void cg_solve(nld_operator* op, const double* f, double* u, int nrhs,
              int64_t ld, const double* lam, const double* mu, int prec,
              int deflate, double tol, int maxit, int warm, int* iters,
              double* relres, int* conv, double* hist, int hist_cap,
              cudaStream_t st);

// vector helpers (nld_vec.cu)
void dev_axpby(double a, const double* x, double b, const double* y,
               double* out, int64_t n, cudaStream_t st);
double dev_dot(const double* x, const double* y, int64_t n, cudaStream_t st);
void dev_scs(const double* x, double* out, int64_t n, int down,
             cudaStream_t st);
void dev_basis(const double* v, const double* x, double* out, int64_t n,
               int adjoint, cudaStream_t st);

int64_t expansion_degree(double sig_scaled, double eps);
void point_geometry(const double* F, int64_t N, int d, double rmax, double* center,
                    double* scale, cudaStream_t st);

// collective helpers (no-ops without a comm hook)
enum { RED_F64 = 0, RED_I32 = 1 };
enum { RED_OP_SUM = 0, RED_OP_MIN = 1, RED_OP_MAX = 2 };
void comm_host(nld_operator* op, void* buf, int64_t count, int dtype, int red);
void comm_device(nld_operator* op, double* buf, int64_t count, cudaStream_t st);

}  // namespace nld
