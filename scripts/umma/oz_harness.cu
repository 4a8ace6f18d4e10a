// Unit harness for the sliced spread kernel: one synthetic subproblem.
#include "../../paper_2407_06834_b200/csrc/nld_ozaki.cu"

extern "C" int oz_spread_one(const double* rows_h, const double* v_h, int K, double* blk_h,
                             int16_t* ex_h, int nsub) {
  using namespace nld;
  WinDev wd{};
  wd.row_off = 0;
  wd.node_off = 0;
  // nsub subproblems of K/nsub nodes (the last takes the rest), blocks 512 apart
  std::vector<SubDev> sds(nsub);
  for (int i = 0; i < nsub; ++i) {
    sds[i] = SubDev{};
    sds[i].start = (int64_t)i * (K / nsub);
    sds[i].count = i == nsub - 1 ? K - i * (K / nsub) : K / nsub;
    sds[i].block = 512 * i;
  }
  double *rows, *vt, *blk;
  int32_t* pix;
  WinDev* dw;
  SubDev* ds;
  int16_t* ex;
  cudaMalloc(&rows, K * 24 * 8); cudaMalloc(&vt, K * 16 * 8); cudaMalloc(&blk, 512 * 16 * 8 * nsub);
  cudaMalloc(&pix, K * 4); cudaMalloc(&dw, sizeof(WinDev)); cudaMalloc(&ds, sizeof(SubDev) * nsub);
  cudaMalloc(&ex, 24 * 2 * nsub);
  std::vector<int32_t> p(K);
  for (int i = 0; i < K; ++i) p[i] = i;
  cudaMemcpy(rows, rows_h, K * 24 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(vt, v_h, K * 16 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(pix, p.data(), K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, &wd, sizeof(WinDev), cudaMemcpyHostToDevice);
  cudaMemcpy(ds, sds.data(), sizeof(SubDev) * nsub, cudaMemcpyHostToDevice);
  oz::k_sub_exponents<<<nsub, 240>>>(ds, dw, rows, ex);
  PlanSet ps;
  ps.wdev = dw; ps.rows = rows; ps.pix = pix;
  unsigned long long* vm; cudaMalloc(&vm, 16 * 8); ozaki_vmax(vt, K, 16, vm, 0);
  launch_spread_oz(ps, ds, ex, nsub, vm, vt, 16, blk, 0);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(blk_h, blk, 512 * 16 * 8 * nsub, cudaMemcpyDeviceToHost);
  cudaMemcpy(ex_h, ex, 48 * nsub, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
