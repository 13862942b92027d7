// Tent-element transfers between the fine and the PML-coarsened grid.
//
// Reference: _prolong_1d / prolongation_matrix (twogrid.py:53-79) and the
// restriction h^d * P^T r (twogrid.py:153-154).  P is a tensor product of
// per-axis 1-D maps: 1 at coarse images, 1/2 at midpoints of merged cells,
// identity across uncoarsened PML cells (mesh.py:164-213).  Instead of a CSR
// matrix the device holds, per axis, for every coarse unknown the fine centre
// index and the two half-weights, and for every fine unknown its <= 2 coarse
// parents; both kernels are gathers (no atomics, deterministic).
//
// HBM bytes per fine DOF: restriction 16 (read r) + 16/2^d (write rc);
// prolongation 32 (read-modify-write u) + 16/2^d (read uc).

#include "hs_common.cuh"
#include "hs_transfer.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;

__global__ void k_restrict(TransferDesc t, const double2* __restrict__ r,
                           double2* __restrict__ rc, double scale) {
  const int64_t L2 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (L2 >= t.cr_cnt[2]) return;
  const int64_t row = blockIdx.y;
  const int64_t I0 = t.cr_lo[0] + row / t.cr_cnt[1];
  const int64_t I1 = t.cr_lo[1] + row % t.cr_cnt[1];
  const int64_t I2 = t.cr_lo[2] + L2;
  const int64_t nf = t.fw_cnt[0] * t.fw_cnt[1] * t.fw_cnt[2];
  const int64_t ncn = t.nc[0] * t.nc[1] * t.nc[2];
  r += (int64_t)blockIdx.z * nf;
  // fine centres, local to the window
  const int64_t c0 = t.ctr[0][I0] - t.fw_lo[0], c1 = t.ctr[1][I1] - t.fw_lo[1],
                c2 = t.ctr[2][I2] - t.fw_lo[2];
  double w0[3] = {t.wl[0][I0], 1.0, t.wr[0][I0]};
  double w1[3] = {t.wl[1][I1], 1.0, t.wr[1][I1]};
  double w2[3] = {t.wl[2][I2], 1.0, t.wr[2][I2]};
  double2 acc = czero();
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (w0[a] == 0.0) continue;
    const int64_t f0 = c0 + a - 1;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (w1[b] == 0.0) continue;
      const int64_t f1 = c1 + b - 1;
      const double w01 = w0[a] * w1[b];
      const double2* rrow = r + (f0 * t.fw_cnt[1] + f1) * t.fw_cnt[2];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (w2[c] == 0.0) continue;
        const double2 v = __ldg(rrow + c2 + c - 1);
        const double w = w01 * w2[c];
        acc.x = fma(w, v.x, acc.x);
        acc.y = fma(w, v.y, acc.y);
      }
    }
  }
  rc[(int64_t)blockIdx.z * ncn + (I0 * t.nc[1] + I1) * t.nc[2] + I2] = cscale(scale, acc);
}

__global__ void k_prolong(TransferDesc t, const double2* __restrict__ uc,
                          double2* __restrict__ u, int accumulate) {
  const int64_t l2 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (l2 >= t.fr_cnt[2]) return;
  const int64_t row = blockIdx.y;
  const int64_t f0 = t.fr_lo[0] + row / t.fr_cnt[1];     // global fine indices
  const int64_t f1 = t.fr_lo[1] + row % t.fr_cnt[1];
  const int64_t f2 = t.fr_lo[2] + l2;
  const int64_t nf = t.fw_cnt[0] * t.fw_cnt[1] * t.fw_cnt[2];
  const int64_t ncn = t.nc[0] * t.nc[1] * t.nc[2];
  uc += (int64_t)blockIdx.z * ncn;
  const int64_t i = (int64_t)blockIdx.z * nf +
                    ((f0 - t.fw_lo[0]) * t.fw_cnt[1] + (f1 - t.fw_lo[1])) * t.fw_cnt[2] +
                    (f2 - t.fw_lo[2]);
  double2 acc = czero();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int p0 = t.par[0][2 * f0 + a];
    if (p0 < 0) continue;
    const double w0 = t.pw[0][2 * f0 + a];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int p1 = t.par[1][2 * f1 + b];
      if (p1 < 0) continue;
      const double w01 = w0 * t.pw[1][2 * f1 + b];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int p2 = t.par[2][2 * f2 + c];
        if (p2 < 0) continue;
        const double w = w01 * t.pw[2][2 * f2 + c];
        const double2 v = __ldg(uc + ((int64_t)p0 * t.nc[1] + p1) * t.nc[2] + p2);
        acc.x = fma(w, v.x, acc.x);
        acc.y = fma(w, v.y, acc.y);
      }
    }
  }
  u[i] = accumulate ? cadd(u[i], acc) : acc;
}

}  // namespace

int transfer_restrict(Ctx* c, const Transfer* t, const double2* r, double2* rc, double scale,
                      int nrhs) {
  const TransferDesc& d = t->d;
  const int64_t rows = d.cr_cnt[0] * d.cr_cnt[1];
  if (rows == 0 || d.cr_cnt[2] == 0) return HS_OK;
  dim3 grid((unsigned)((d.cr_cnt[2] + kThreads - 1) / kThreads), (unsigned)rows,
            (unsigned)nrhs);
  const double ncomp = (double)rows * d.cr_cnt[2];
  ProfScope ps(c, K_RESTRICT, 16.0 * nrhs * (double)(d.nf[0] * d.nf[1] * d.nf[2]) *
                                  (ncomp / (double)(d.nc[0] * d.nc[1] * d.nc[2])) +
                                  16.0 * nrhs * ncomp);
  k_restrict<<<grid, kThreads, 0, c->stream>>>(d, r, rc, scale);
  HS_LAUNCH_CHECK(c, "restrict kernel");
  return HS_OK;
}

int transfer_prolong(Ctx* c, const Transfer* t, const double2* uc, double2* u, int accumulate,
                     int nrhs) {
  const TransferDesc& d = t->d;
  const int64_t rows = d.fr_cnt[0] * d.fr_cnt[1];
  if (rows == 0 || d.fr_cnt[2] == 0) return HS_OK;
  dim3 grid((unsigned)((d.fr_cnt[2] + kThreads - 1) / kThreads), (unsigned)rows,
            (unsigned)nrhs);
  const double ncomp = (double)rows * d.fr_cnt[2];
  ProfScope ps(c, K_PROLONG,
               16.0 * nrhs * ((accumulate ? 2 : 1) * ncomp +
                              (double)(d.nc[0] * d.nc[1] * d.nc[2]) *
                                  (ncomp / (double)(d.nf[0] * d.nf[1] * d.nf[2]))));
  k_prolong<<<grid, kThreads, 0, c->stream>>>(d, uc, u, accumulate);
  HS_LAUNCH_CHECK(c, "prolong kernel");
  return HS_OK;
}

// Build the per-axis tables on the host and upload them in one buffer.
int transfer_create(Ctx* c, int dim, const int64_t* fp_len, const int64_t* fp_concat,
                    const uint8_t* refined_concat, Transfer** out, const int64_t* window) {
  if (dim < 1 || dim > 3) return set_error(c, HS_E_SHAPE, "transfer dim must be 1..3");
  Transfer* t = new Transfer();
  t->dim = dim;
  // canonical axes: user axis a -> canonical axis (3 - dim + a)
  std::vector<int> ctr[3], par[3];
  std::vector<double> wl[3], wr[3], pw[3];
  const int64_t* fpp = fp_concat;
  const uint8_t* rp = refined_concat;
  for (int ca = 0; ca < 3; ++ca) {
    const int a = ca - (3 - dim);
    if (a < 0) {
      t->d.nf[ca] = t->d.nc[ca] = 1;
      ctr[ca] = {0};
      wl[ca] = {0.0};
      wr[ca] = {0.0};
      par[ca] = {0, -1};
      pw[ca] = {1.0, 0.0};
      continue;
    }
    const int64_t L = fp_len[a];  // coarse points 0..Nc
    const int64_t Nc = L - 1;
    const int64_t Nf = fpp[L - 1];
    if (L < 3) { delete t; return set_error(c, HS_E_SHAPE, "coarsening map too short"); }
    const int64_t nc = Nc - 1, nf = Nf - 1;
    t->d.nc[ca] = nc;
    t->d.nf[ca] = nf;
    ctr[ca].resize(nc);
    wl[ca].resize(nc);
    wr[ca].resize(nc);
    for (int64_t I = 0; I < nc; ++I) {
      const int64_t pnt = I + 1;
      ctr[ca][I] = (int)(fpp[pnt] - 1);
      wl[ca][I] = rp[pnt - 1] ? 0.5 : 0.0;
      wr[ca][I] = rp[pnt] ? 0.5 : 0.0;
    }
    par[ca].assign(2 * nf, -1);
    pw[ca].assign(2 * nf, 0.0);
    for (int64_t pnt = 1; pnt < Nc; ++pnt) {  // coarse images
      const int64_t fi = fpp[pnt] - 1;
      par[ca][2 * fi] = (int)(pnt - 1);
      pw[ca][2 * fi] = 1.0;
    }
    for (int64_t cell = 0; cell < Nc; ++cell) {  // midpoints of merged cells
      if (!rp[cell]) continue;
      const int64_t fi = fpp[cell];  // fine index of the midpoint (point fp+1)
      int slot = 0;
      for (int64_t cp = cell; cp <= cell + 1; ++cp) {
        if (cp >= 1 && cp <= Nc - 1) {
          par[ca][2 * fi + slot] = (int)(cp - 1);
          pw[ca][2 * fi + slot] = 0.5;
          ++slot;
        }
      }
    }
    fpp += L;
    rp += L - 1;
  }
  // identity window, or the shard window on the sweep axis
  for (int ca = 0; ca < 3; ++ca) {
    t->d.fw_lo[ca] = t->d.cr_lo[ca] = t->d.fr_lo[ca] = 0;
    t->d.fw_cnt[ca] = t->d.fr_cnt[ca] = t->d.nf[ca];
    t->d.cr_cnt[ca] = t->d.nc[ca];
  }
  if (window) {
    const int wa = 3 - dim;
    const int64_t fw_lo = window[0], fw_hi = window[1], cr_lo = window[2], cr_hi = window[3],
                  fr_lo = window[4], fr_hi = window[5];
    const int64_t nf = t->d.nf[wa], nc = t->d.nc[wa];
    bool ok = 0 <= fw_lo && fw_lo <= fw_hi && fw_hi <= nf && 0 <= cr_lo && cr_lo <= cr_hi &&
              cr_hi <= nc && fw_lo <= fr_lo && fr_lo <= fr_hi && fr_hi <= fw_hi;
    // every fine row a computed coarse row reads must lie inside the window
    for (int64_t I = cr_lo; ok && I < cr_hi; ++I) {
      const int64_t lo = ctr[wa][I] - (wl[wa][I] != 0.0), hi = ctr[wa][I] + (wr[wa][I] != 0.0);
      ok = lo >= fw_lo && hi < fw_hi;
    }
    if (!ok) {
      delete t;
      return set_error(c, HS_E_SHAPE, "transfer window does not cover the restriction stencil "
                                      "of its coarse rows (shard map)");
    }
    t->d.fw_lo[wa] = fw_lo;
    t->d.fw_cnt[wa] = fw_hi - fw_lo;
    t->d.cr_lo[wa] = cr_lo;
    t->d.cr_cnt[wa] = cr_hi - cr_lo;
    t->d.fr_lo[wa] = fr_lo;
    t->d.fr_cnt[wa] = fr_hi - fr_lo;
  }
  // pack: ints then doubles
  size_t ni = 0, nd = 0;
  for (int ca = 0; ca < 3; ++ca) {
    ni += ctr[ca].size() + par[ca].size();
    nd += wl[ca].size() + wr[ca].size() + pw[ca].size();
  }
  const size_t bytes = nd * sizeof(double) + ni * sizeof(int) + 64;
  std::vector<char> host(bytes, 0);
  char* base = nullptr;
  cudaError_t e = cudaMalloc((void**)&base, bytes);
  if (e != cudaSuccess) { delete t; return check_cuda(c, e, "transfer alloc"); }
  t->buf = base;
  size_t off = 0;
  auto put_d = [&](std::vector<double>& v) -> const double* {
    memcpy(host.data() + off, v.data(), v.size() * sizeof(double));
    const double* p = (const double*)(base + off);
    off += v.size() * sizeof(double);
    return p;
  };
  for (int ca = 0; ca < 3; ++ca) {
    t->d.wl[ca] = put_d(wl[ca]);
    t->d.wr[ca] = put_d(wr[ca]);
    t->d.pw[ca] = put_d(pw[ca]);
  }
  auto put_i = [&](std::vector<int>& v) -> const int* {
    memcpy(host.data() + off, v.data(), v.size() * sizeof(int));
    const int* p = (const int*)(base + off);
    off += v.size() * sizeof(int);
    return p;
  };
  for (int ca = 0; ca < 3; ++ca) {
    t->d.ctr[ca] = put_i(ctr[ca]);
    t->d.par[ca] = put_i(par[ca]);
  }
  e = cudaMemcpy(base, host.data(), off, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(base); delete t; return check_cuda(c, e, "transfer upload"); }
  *out = t;
  return HS_OK;
}

void transfer_destroy(Transfer* t) {
  if (!t) return;
  if (t->buf) cudaFree(t->buf);
  delete t;
}

}  // namespace hs
