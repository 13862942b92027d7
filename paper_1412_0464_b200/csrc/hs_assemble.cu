// Operator assembly on the device: the fine-level
// second-order FD operator with PML stretching / sponge damping and the FE
// engine of the coarse level and of every slab (added-PML slab operators),
// written straight into the [S][n] coefficient layout the stencil and sweep
// kernels consume -- no host arrays, no upload of S x n coefficients.
//
// Reference: _assemble_fd / assemble_fine / assemble_sponge
// (discretize.py:191-253), opt_coeffs / fe_constants / _assemble_fe
// (discretize.py:307-323, 413-506), subdomain_fe_operator (:685-723).
// The host computes only the per-axis 1-D arrays (stretching factors, cell
// widths, damping profiles: O(N) per axis, numpy, the reference's own
// expressions) and the row maps of the slab wavenumbers; every per-node
// product runs here in the reference's operation order, with the complex
// arithmetic written out the way numpy evaluates it (no fused multiply-add,
// Smith division), so the coefficients agree with the host assembly to the
// last bit or within an ulp (tests/test_gpu_parity.py: <= 1e-15 relative).
//
// HBM-bound streaming kernels: one thread per node writes S coefficients
// (2-D FE 9 x 16 B, 3-D 27 x 16 B) from a few per-node reads.

#include "hs_common.cuh"

#include <algorithm>
#include <vector>

namespace hs {

namespace {

constexpr int kThreads = 256;

// numpy's complex128 arithmetic, no contraction
__device__ __forceinline__ double2 nmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 nadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 nsub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 nrmul(double r, double2 b) {   // float64 array * complex128 array
  return nmul(make_double2(r, 0.0), b);
}
__device__ __forceinline__ double2 ndiv(double2 a, double2 b) {   // Smith, as numpy's loops
  const double br = fabs(b.x), bi = fabs(b.y);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return make_double2(a.x / br, a.y / br);
    const double rat = __ddiv_rn(b.y, b.x);
    const double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                        __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  const double rat = __ddiv_rn(b.x, b.y);
  const double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}
__device__ __forceinline__ double2 nneg(double2 a) { return make_double2(-a.x, -a.y); }

// canonical node index -> user-axis indices (dim <= 3, canonical axes 3-dim..2)
struct Grid {
  int dim;
  int64_t n[3];        // canonical node counts
  int64_t n_total;
};

__device__ __forceinline__ void node_index(const Grid& g, int64_t i, int idx[3]) {
  const int64_t i2 = i % g.n[2];
  const int64_t r = i / g.n[2];
  const int64_t i1 = r % g.n[1];
  const int64_t i0 = r / g.n[1];
  const int64_t c[3] = {i0, i1, i2};
  for (int a = 0; a < g.dim; ++a) idx[a] = (int)c[3 - g.dim + a];
}

// ---------------------------------------------------------------------------
// FD (discretize.py _fd_operator): per-axis alpha at cell midpoints / nodes
struct FdArgs {
  Grid g;
  double h2;
  const double2* ahalf[3];   // [N_a]
  const double2* anode[3];   // [N_a - 1]
  const double* gam[3];      // [N_a - 1] sponge gamma at nodes (per axis) or null
  int sponge;                // k^2 (1 + i gamma) instead of (k + 0i)^2
  const double* k;           // [n] wavenumber at the unknowns
  int slot_m[3], slot_p[3], slot_d;
  double2* out;              // [S][n]
};

__global__ void __launch_bounds__(kThreads) k_assemble_fd(FdArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= a.g.n_total) return;
  int idx[3];
  node_index(a.g, i, idx);
  const int dim = a.g.dim;
  double2 np_ = make_double2(1.0, 0.0);
  for (int ax = 0; ax < dim; ++ax) np_ = nmul(np_, a.anode[ax][idx[ax]]);
  const double kv = a.k[i];
  double2 k2;
  if (a.sponge) {
    double gsum = 0.0;
    for (int ax = 0; ax < dim; ++ax)
      if (a.gam[ax]) gsum = __dadd_rn(gsum, a.gam[ax][idx[ax]]);
    k2 = nrmul(__dmul_rn(kv, kv), make_double2(1.0, gsum));
  } else {
    k2 = nmul(make_double2(kv, 0.0), make_double2(kv, 0.0));
  }
  double2 diag = ndiv(nneg(k2), np_);
  const int64_t n = a.g.n_total;
  for (int ax = 0; ax < dim; ++ax) {
    const double2 tr = ndiv(np_, a.anode[ax][idx[ax]]);
    const double2 left = a.ahalf[ax][idx[ax]], right = a.ahalf[ax][idx[ax] + 1];
    const double2 ht = nrmul(a.h2, tr);
    a.out[(int64_t)a.slot_m[ax] * n + i] = ndiv(nneg(left), ht);
    a.out[(int64_t)a.slot_p[ax] * n + i] = ndiv(nneg(right), ht);
    diag = nadd(diag, ndiv(nadd(left, right), ht));
  }
  a.out[(int64_t)a.slot_d * n + i] = diag;
}

// ---------------------------------------------------------------------------
// FE (discretize.py _fe_operator, k per cell) with the optimized-table weights
constexpr int kMaxTab = 64;
constexpr int kMaxCoef = 5;

struct FeArgs {
  Grid g;                    // nodes of the operator (local for a slab)
  const double2* woa[3];     // [N_a] widths / alpha
  const double2* aow[3];     // [N_a] alpha / widths
  const double2* cw[3];      // [N_a] widths * (1 / alpha)
  const double* gc[3];       // [N_a] gamma at cell midpoints (per axis) or null
  int any_gamma;
  // wavenumbers: global arrays, axis-0 rows mapped local -> global by clamp
  const double* kn;          // nodes [rows][kn_ld]
  const double* kc;          // cells [rows][kc_ld]
  int64_t kn_ld, kc_ld;
  int nrow0, nlo, nhi;       // node row r -> clamp(nrow0 + r, nlo, nhi)
  int crow0, clo, chi;       // cell row r -> clamp(crow0 + r, clo, chi)
  int64_t cn[3];             // canonical cell counts of the local grid (n + 1 per axis)
  double h_ref;
  int ntab, ncoef;
  double tab_x[kMaxTab];
  double tab_c[kMaxTab * kMaxCoef];   // [ntab][ncoef]
  double2* out;              // [3^dim][n]
};

// np.interp(x, xp, fp) for one table column
__device__ double interp(const FeArgs& a, double x, int col) {
  const int n = a.ntab;
  if (!(x >= a.tab_x[0])) return a.tab_c[col];                  // below (or nan -> left)
  if (x >= a.tab_x[n - 1]) return a.tab_c[(n - 1) * a.ncoef + col];
  int j = 0;
  while (j + 1 < n - 1 && a.tab_x[j + 1] <= x) ++j;
  const double f0 = a.tab_c[j * a.ncoef + col], f1 = a.tab_c[(j + 1) * a.ncoef + col];
  const double slope = __ddiv_rn(__dsub_rn(f1, f0), __dsub_rn(a.tab_x[j + 1], a.tab_x[j]));
  return __dadd_rn(__dmul_rn(slope, __dsub_rn(x, a.tab_x[j])), f0);
}

__global__ void __launch_bounds__(kThreads) k_assemble_fe(FeArgs a) {
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= a.g.n_total) return;
  const int dim = a.g.dim;
  int idx[3];
  node_index(a.g, i, idx);
  // wavenumber at the node (axis-0 row map) -> table weights i_w, j_w
  const int64_t nrest = i % (a.g.n_total / a.g.n[3 - dim]);   // offset inside the axis-0 row
  const int grow = min(max(a.nrow0 + idx[0], a.nlo), a.nhi);
  const double kv = a.kn[(int64_t)grow * a.kn_ld + nrest];
  const double inv_g = __ddiv_rn(__dmul_rn(a.h_ref, kv), 6.283185307179586);
  double c[kMaxCoef];
  for (int j = 0; j < a.ncoef; ++j) c[j] = interp(a, inv_g, j);
  double iw[4], jw[3];
  if (dim == 2) {
    iw[0] = __ddiv_rn(c[0], 4.0);
    iw[1] = __ddiv_rn(c[1], 8.0);
    iw[2] = __ddiv_rn(__dsub_rn(__dsub_rn(1.0, c[0]), c[1]), 4.0);
    jw[0] = __ddiv_rn(c[2], 2.0);
    jw[1] = __ddiv_rn(__dsub_rn(1.0, c[2]), 2.0);
  } else {
    iw[0] = __ddiv_rn(c[0], 8.0);
    iw[1] = __ddiv_rn(c[1], 24.0);
    iw[2] = __ddiv_rn(c[2], 24.0);
    iw[3] = __ddiv_rn(__dsub_rn(__dsub_rn(__dsub_rn(1.0, c[0]), c[1]), c[2]), 8.0);
    jw[0] = __ddiv_rn(c[3], 4.0);
    jw[1] = __ddiv_rn(c[4], 8.0);
    jw[2] = __ddiv_rn(__dsub_rn(__dsub_rn(1.0, c[3]), c[4]), 4.0);
  }
  // cells around the node: per axis left = idx, right = idx + 1 (local cell index)
  const int cgrow[2] = {min(max(a.crow0 + idx[0], a.clo), a.chi),
                        min(max(a.crow0 + idx[0] + 1, a.clo), a.chi)};
  // k^2 (1 + i gamma) at the 2^dim cells around the node, index bits = axis sides
  double2 k2c[8];
  for (int q = 0; q < (1 << dim); ++q) {
    int64_t off = 0;
    double gsum = 0.0;
    for (int ax = 1; ax < dim; ++ax) {   // transverse cell offset inside the row
      const int ci = idx[ax] + ((q >> (dim - 1 - ax)) & 1);
      int64_t stride = 1;
      for (int b = ax + 1; b < dim; ++b) stride *= a.cn[3 - dim + b];
      off += (int64_t)ci * stride;
    }
    const int side0 = (q >> (dim - 1)) & 1;
    const double kv2 = a.kc[(int64_t)cgrow[side0] * a.kc_ld + off];
    if (a.any_gamma) {
      for (int ax = 0; ax < dim; ++ax) {
        if (!a.gc[ax]) continue;
        const int ci = idx[ax] + ((q >> (dim - 1 - ax)) & 1);
        gsum = __dadd_rn(gsum, a.gc[ax][ci]);
      }
    }
    k2c[q] = nrmul(__dmul_rn(kv2, kv2), make_double2(1.0, gsum));
  }
  const int64_t n = a.g.n_total;
  int slot = 0;
  // offsets in itertools.product((-1, 0, 1), repeat=dim) order (= sorted)
  const int noff = dim == 2 ? 9 : 27;
  for (int s = 0; s < noff; ++s, ++slot) {
    int o[3];
    {
      int t = s;
      for (int ax = dim - 1; ax >= 0; --ax) {
        o[ax] = t % 3 - 1;
        t /= 3;
      }
    }
    int nz = 0;
    for (int ax = 0; ax < dim; ++ax) nz += o[ax] != 0;
    // mass: sum over the cells picked per axis (-1: left, 0: left then right, +1: right)
    double2 mass = make_double2(0.0, 0.0);
    const int lo0 = o[0] > 0 ? 1 : 0, hi0 = o[0] < 0 ? 0 : 1;
    const int lo1 = dim > 1 ? (o[1] > 0 ? 1 : 0) : 0, hi1 = dim > 1 ? (o[1] < 0 ? 0 : 1) : 0;
    const int lo2 = dim > 2 ? (o[2] > 0 ? 1 : 0) : 0, hi2 = dim > 2 ? (o[2] < 0 ? 0 : 1) : 0;
    for (int s0 = lo0; s0 <= hi0; ++s0)
      for (int s1 = lo1; s1 <= hi1; ++s1)
        for (int s2 = lo2; s2 <= hi2; ++s2) {
          const int sides[3] = {s0, s1, s2};
          int q = 0;
          for (int ax = 0; ax < dim; ++ax) q = (q << 1) | sides[ax];
          double2 term = k2c[q];
          for (int ax = 0; ax < dim; ++ax) term = nmul(term, a.cw[ax][idx[ax] + sides[ax]]);
          mass = nadd(mass, term);
        }
    mass = nmul(mass, make_double2(iw[nz], 0.0));
    double2 entry = nneg(mass);
    for (int l = 0; l < dim; ++l) {
      const double2* d = a.aow[l];
      const int il = idx[l];
      const double2 sd = o[l] == 0 ? nneg(nadd(d[il], d[il + 1])) : (o[l] < 0 ? d[il] : d[il + 1]);
      double2 term = nmul(sd, make_double2(jw[nz - (o[l] != 0)], 0.0));
      for (int m = 0; m < dim; ++m) {
        if (m == l) continue;
        const double2* w = a.woa[m];
        const int im = idx[m];
        const double2 mw = o[m] == 0 ? nadd(w[im], w[im + 1]) : (o[m] < 0 ? w[im] : w[im + 1]);
        term = nmul(term, mw);
      }
      entry = nsub(entry, term);
    }
    a.out[(int64_t)slot * n + i] = entry;
  }
}

// 1 / diagonal and the first zero-diagonal node
__global__ void k_finish(const double2* __restrict__ dg, double2* __restrict__ invd, int64_t n,
                         unsigned long long* first_zero) {
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const double2 v = dg[i];
  if (v.x == 0.0 && v.y == 0.0) {
    atomicMin(first_zero, (unsigned long long)i);
    invd[i] = make_double2(0.0, 0.0);
    return;
  }
  const double d = 1.0 / (v.x * v.x + v.y * v.y);   // the host formula of hs_stencil_create
  invd[i] = make_double2(v.x * d, -v.y * d);
}

unsigned blocks_for(int64_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

// per-axis host arrays -> one device buffer
struct Staging {
  std::vector<char> host;
  char* dev = nullptr;
  template <class T>
  size_t add(const T* p, size_t count) {
    const size_t off = (host.size() + 15) & ~(size_t)15;
    host.resize(off + count * sizeof(T));
    memcpy(host.data() + off, p, count * sizeof(T));
    return off;
  }
  template <class T>
  const T* at(size_t off) const { return (const T*)(dev + off); }
};

int upload(Ctx* c, Staging& st) {
  HS_CUDA(c, cudaMalloc((void**)&st.dev, std::max<size_t>(st.host.size(), 16)), "assembly staging");
  HS_CUDA(c, cudaMemcpyAsync(st.dev, st.host.data(), st.host.size(), cudaMemcpyHostToDevice,
                             c->stream), "assembly staging upload");
  return HS_OK;
}

Grid make_grid(int dim, const int64_t* shape) {
  Grid g{};
  g.dim = dim;
  g.n[0] = g.n[1] = g.n[2] = 1;
  g.n_total = 1;
  for (int a = 0; a < dim; ++a) {
    g.n[3 - dim + a] = shape[a];
    g.n_total *= shape[a];
  }
  return g;
}

}  // namespace

int stencil_finish_device(Ctx* c, Stencil* op) {
  op->d.coeffs = op->coeffs;
  op->d.invd = nullptr;
  if (op->d.diag < 0) return HS_OK;
  const int64_t n = op->d.n;
  unsigned long long* fz = nullptr;
  HS_CUDA(c, cudaMalloc((void**)&op->invd, (size_t)n * sizeof(double2)), "invd alloc");
  HS_CUDA(c, cudaMalloc((void**)&fz, sizeof(unsigned long long)), "flag alloc");
  HS_CUDA(c, cudaMemsetAsync(fz, 0xff, sizeof(unsigned long long), c->stream), "flag init");
  k_finish<<<blocks_for(n), kThreads, 0, c->stream>>>(op->coeffs + (int64_t)op->d.diag * n,
                                                       op->invd, n, fz);
  HS_LAUNCH_CHECK(c, "finish kernel");
  unsigned long long first = ~0ull;
  cudaError_t e = cudaMemcpyAsync(&first, fz, sizeof first, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(fz);
  if (e != cudaSuccess) return check_cuda(c, e, "zero-diagonal scan");
  if (first != ~0ull) {
    op->has_zero_diag = 1;
    op->zero_diag_node = (long long)first;
  } else {
    op->d.invd = op->invd;
  }
  return HS_OK;
}

}  // namespace hs

using namespace hs;

extern "C" {

// declared in include/hsweep.h
int hs_assemble_fd(hs_ctx* cx, int dim, const int64_t* shape, double h,
                   const double* a_half, const double* a_node, const double* gamma_nodes,
                   const void* k_dev, hs_stencil** out) {
  Ctx* c = cx;
  if (!c || !shape || !a_half || !a_node || !k_dev || !out) return HS_E_ARG;
  if (dim < 1 || dim > 3) return set_error(c, HS_E_SHAPE, "assembly dim must be 1..3");
  // offsets sorted like the host (DeviceStencil.from_host): e_m(a), e_p(a), 0
  std::vector<std::vector<int8_t>> offs;
  for (int a = 0; a < dim; ++a)
    for (int sgn = -1; sgn <= 1; sgn += 2) {
      std::vector<int8_t> o(dim, 0);
      o[a] = (int8_t)sgn;
      offs.push_back(o);
    }
  offs.push_back(std::vector<int8_t>(dim, 0));
  std::sort(offs.begin(), offs.end());
  const int S = (int)offs.size();
  std::vector<int8_t> flat;
  for (auto& o : offs) flat.insert(flat.end(), o.begin(), o.end());
  hs_stencil* op = new hs_stencil();
  if (int r = stencil_init_desc(c, dim, shape, S, flat.data(), op)) {
    delete op;
    return r;
  }
  FdArgs args{};
  args.g = make_grid(dim, shape);
  args.h2 = h * h;
  for (int a = 0; a < dim; ++a) {
    for (int s = 0; s < S; ++s) {
      bool m = true, p = true;
      for (int b = 0; b < dim; ++b) {
        m = m && offs[s][b] == (b == a ? -1 : 0);
        p = p && offs[s][b] == (b == a ? 1 : 0);
      }
      if (m) args.slot_m[a] = s;
      if (p) args.slot_p[a] = s;
    }
  }
  args.slot_d = op->d.diag;
  Staging st;
  size_t oh[3], on[3], og[3];
  {
    size_t ph = 0, pn = 0;
    for (int a = 0; a < dim; ++a) {
      const int64_t N = shape[a] + 1;   // cells
      oh[a] = st.add((const double2*)a_half + ph, (size_t)N);
      on[a] = st.add((const double2*)a_node + pn, (size_t)(N - 1));
      if (gamma_nodes) og[a] = st.add(gamma_nodes + pn, (size_t)(N - 1));
      ph += N;
      pn += N - 1;
    }
  }
  if (int r = upload(c, st)) {
    delete op;
    return r;
  }
  for (int a = 0; a < dim; ++a) {
    args.ahalf[a] = st.at<double2>(oh[a]);
    args.anode[a] = st.at<double2>(on[a]);
    args.gam[a] = gamma_nodes ? st.at<double>(og[a]) : nullptr;
  }
  args.sponge = gamma_nodes != nullptr;
  args.k = (const double*)k_dev;
  cudaError_t e = cudaMalloc((void**)&op->coeffs, (size_t)S * op->d.n * sizeof(double2));
  if (e != cudaSuccess) {
    cudaFree(st.dev);
    delete op;
    return check_cuda(c, e, "assembly alloc");
  }
  args.out = op->coeffs;
  {
    ProfScope ps(c, K_SETUP, (double)op->d.n * (S * 16.0 + 8.0));
    k_assemble_fd<<<blocks_for(op->d.n), kThreads, 0, c->stream>>>(args);
  }
  c->launches++;
  e = cudaGetLastError();
  int r = e == cudaSuccess ? stencil_finish_device(c, op) : check_cuda(c, e, "assemble_fd");
  cudaFree(st.dev);   // (stream-ordered after the kernel: finish synchronised)
  if (r) {
    cudaFree(op->coeffs);
    cudaFree(op->invd);
    delete op;
    return r;
  }
  *out = op;
  return HS_OK;
}

int hs_assemble_fe(hs_ctx* cx, int dim, const int64_t* shape, const double* woa,
                   const double* aow, const double* cw, const double* gamma_cells,
                   const void* k_nodes_dev, int64_t kn_ld, const void* k_cells_dev,
                   int64_t kc_ld, const int32_t* rowmap, double h_ref, int ntab, int ncoef,
                   const double* tab_x, const double* tab_c, hs_stencil** out) {
  Ctx* c = cx;
  if (!c || !shape || !woa || !aow || !cw || !k_nodes_dev || !k_cells_dev || !rowmap ||
      !tab_x || !tab_c || !out)
    return HS_E_ARG;
  if (dim != 2 && dim != 3) return set_error(c, HS_E_SHAPE, "FE assembly needs dim 2 or 3");
  if (ntab < 2 || ntab > kMaxTab || ncoef != (dim == 2 ? 3 : 5))
    return set_error(c, HS_E_SHAPE, "optimized-coefficient table does not match the dimension");
  const int S = dim == 2 ? 9 : 27;
  std::vector<int8_t> flat;
  for (int s = 0; s < S; ++s) {
    int t = s;
    int8_t o[3];
    for (int a = dim - 1; a >= 0; --a) {
      o[a] = (int8_t)(t % 3 - 1);
      t /= 3;
    }
    flat.insert(flat.end(), o, o + dim);
  }
  hs_stencil* op = new hs_stencil();
  if (int r = stencil_init_desc(c, dim, shape, S, flat.data(), op)) {
    delete op;
    return r;
  }
  FeArgs args{};
  args.g = make_grid(dim, shape);
  args.cn[0] = args.cn[1] = args.cn[2] = 1;
  for (int a = 0; a < dim; ++a) args.cn[3 - dim + a] = shape[a] + 1;
  Staging st;
  size_t o1[3], o2[3], o3[3], o4[3];
  {
    size_t p = 0;
    for (int a = 0; a < dim; ++a) {
      const size_t N = (size_t)shape[a] + 1;
      o1[a] = st.add((const double2*)woa + p, N);
      o2[a] = st.add((const double2*)aow + p, N);
      o3[a] = st.add((const double2*)cw + p, N);
      if (gamma_cells) o4[a] = st.add(gamma_cells + p, N);
      p += N;
    }
  }
  if (int r = upload(c, st)) {
    delete op;
    return r;
  }
  for (int a = 0; a < dim; ++a) {
    args.woa[a] = st.at<double2>(o1[a]);
    args.aow[a] = st.at<double2>(o2[a]);
    args.cw[a] = st.at<double2>(o3[a]);
    args.gc[a] = gamma_cells ? st.at<double>(o4[a]) : nullptr;
  }
  args.any_gamma = gamma_cells != nullptr;
  args.kn = (const double*)k_nodes_dev;
  args.kc = (const double*)k_cells_dev;
  args.kn_ld = kn_ld;
  args.kc_ld = kc_ld;
  args.nrow0 = rowmap[0]; args.nlo = rowmap[1]; args.nhi = rowmap[2];
  args.crow0 = rowmap[3]; args.clo = rowmap[4]; args.chi = rowmap[5];
  args.h_ref = h_ref;
  args.ntab = ntab;
  args.ncoef = ncoef;
  for (int j = 0; j < ntab; ++j) args.tab_x[j] = tab_x[j];
  for (int j = 0; j < ntab * ncoef; ++j) args.tab_c[j] = tab_c[j];
  cudaError_t e = cudaMalloc((void**)&op->coeffs, (size_t)S * op->d.n * sizeof(double2));
  if (e != cudaSuccess) {
    cudaFree(st.dev);
    delete op;
    return check_cuda(c, e, "assembly alloc");
  }
  args.out = op->coeffs;
  {
    ProfScope ps(c, K_SETUP, (double)op->d.n * (S * 16.0 + 16.0));
    k_assemble_fe<<<blocks_for(op->d.n), kThreads, 0, c->stream>>>(args);
  }
  c->launches++;
  e = cudaGetLastError();
  int r = e == cudaSuccess ? stencil_finish_device(c, op) : check_cuda(c, e, "assemble_fe");
  cudaFree(st.dev);
  if (r) {
    cudaFree(op->coeffs);
    cudaFree(op->invd);
    delete op;
    return r;
  }
  *out = op;
  return HS_OK;
}

}  // extern "C"
