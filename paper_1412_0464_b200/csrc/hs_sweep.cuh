#pragma once
#include "hs_common.cuh"

namespace hs {

// One slab solve of a schedule (subdom_solve, sweepdd.py:236-268).
struct SweepTask {
  int slab;        // 0-based slab index j-1
  int lo;          // first grid point of the slab (1-based)
  int T;           // thickness (layers)
  int a, b;        // f rows [a, b) restricted into the slab (global 0-based rows)
  int ta, tb;      // u rows [ta, tb) scattered back
  int tin1, row1;  // forward transmission in: producer trace buffer, slab-local row of point p
  int tin3, row3;  // backward transmission in
  int out2, orow2; // forward trace out (trace buffer), slab-local row of the trace point
  int out4, orow4; // backward trace out
  int dst;         // 0: pass-1 solution u, 1: pass-2 buffer u2 (summed at the end)
};

constexpr int kMaxFront = 16;   // concurrent fronts (clusters) of one solve launch

struct SweepLaunch {
  enum Kind { kCombine, kSolve, kResidual } kind;
  int src;                  // solve: right-hand side 0 = f, 1 = g (mid-sweep residual)
  int nfront;
  int ffirst[kMaxFront], fcount[kMaxFront];   // front task ranges (global task indices)
  double bytes;             // algorithmic HBM bytes of the launch (profiler)
};

struct Sweep3;   // 3-D levels (hs_sweep3.cu)

// Per-application scratch of a sweep: traces, mid-sweep residual, pass-2
// contributions.  The Sweep owns one; a cycle lane owns another so that
// applications on different streams can run concurrently (2-D levels).
struct SweepWork {
  int nrhs = 1;                 // right-hand sides the buffers hold (each array nrhs copies)
  double2* trace = nullptr;     // [ntrace][2][M]
  double2* g = nullptr;         // [n0*M]
  double2* u2 = nullptr;        // [n0*M]
  // two-level partition exchange (G > 1): level-2 right-hand sides and their
  // arrival counters (see SolveArgs); xcount = the counters' value at the
  // next launch per front slot (host-side, monotone)
  double2* xbuf = nullptr;      // [kMaxFront][2][8][2][32]
  unsigned* xflag = nullptr;    // [kMaxFront][2][8]
  unsigned xcount[16] = {};
};

// Partitioned slab factors of every slab (see hs_sweep.cu).
struct Sweep {
  int J = 0, M = 0, n0 = 0;
  int tm = 16;                  // padded block size (16 or 32)
  int C = 1;                    // chunks per face segment = CTAs per cluster
  int G = 1;                    // face segments = clusters per front (two-level partition)
  int max_fronts = 16;          // fronts per solve launch (co-resident clusters / G)
  int max_nr = 1;               // widest slab-solve kernel (right-hand sides per chain: 1, 2 or 4)
  SweepWork batch;              // work set of the multi-right-hand-side applications (lazy)
  int L = 0;                    // local cyclic-reduction levels before the dense top
  int q = 1;                    // blocks left per chunk after L levels (dense inverse)
  int mmax = 0;                 // largest chunk (face points)
  int y0s[65] = {};             // chunk boundaries (G * C + 1 entries)
  int kstride = 0;              // kept-block records per chunk
  const Stencil* coarse = nullptr;
  double2* ef = nullptr;        // [J][M][tm^2]          Dinv at each block's elimination level
  double2* eb = nullptr;        // [J][M][2][tm^2]       Dinv L, Dinv U (back substitution)
  double2* kr = nullptr;        // [J][C][kstride][2][tm^2] alpha, gamma of kept blocks
  double2* sp = nullptr;        // [J][M][2][tm^2]       spikes W, V of every block
  double2* rk = nullptr;        // [J][C][2(C-1)][2 tm^2] rows of the reduced-system inverse
  double2* qd = nullptr;        // [J][C][q][q][tm^2]    inverse of the level-L reduced chunk system
  double2* x2 = nullptr;        // [J][GC][xstride][tm^2] level-2 blocks (packing only)
  double2* stream = nullptr;    // [J][C][nbs][tm^2]     all of the above in solve order (setup frees the rest)
  long long nbs = 0;            // blocks per (slab, chunk) stream
  uint32_t* ptab = nullptr;     // [C][plan words] solve-kernel item / chunk tables
  int nr = 0;                   // rows per restricted update (0: full updates)
  int cpl0 = 0;                 // level-0 kept updates from sparse couplings (cpl)
  double2* cpl = nullptr;       // [J][M][2][3][tm] level-0 thin-axis couplings
  int* rows = nullptr;          // [J][nr] solution rows the chain reads (outputs, traces)
  double2* ebr = nullptr;       // [J][M][tm^2] Dinv L, Dinv U restricted to those rows (packing only)
  double2* spr = nullptr;       // [J][M][tm^2] W, V restricted to those rows (packing only)
  double2* trace = nullptr;     // [ntrace][2][M] interface traces
  double2* g = nullptr;         // [n0*M] mid-sweep residual
  double2* u2 = nullptr;        // [n0*M] second-pass contributions
  SweepWork own;                // this sweep's own work set (trace/g/u2 + level-2 exchange)
  SweepTask* d_tasks = nullptr;
  std::vector<SweepTask> tasks;
  // launch plans by variant id: HS_VARIANT_UD, HS_VARIANT_X, then one per NX
  // cell grouping (sweep_plan_nx); an empty plan = variant not available
  std::vector<std::vector<SweepLaunch>> plan = std::vector<std::vector<SweepLaunch>>(2);
  bool has_plan(int v) const { return v >= 0 && v < (int)plan.size() && !plan[v].empty(); }
  // host copies of the partition geometry (NX plans are built after setup)
  std::vector<int64_t> hbeta, hbt, hlo, hhi;
  std::vector<int> hrows;       // [J][kNR] restricted-update rows (nr != 0)
  double rec_bytes = 0;         // streamed factor bytes per 2-D slab solve (profiler)
  long long factor_bytes = 0;
  int ntrace = 0;               // trace buffers of the schedules
  Sweep3* s3 = nullptr;         // 3-D level: block LU slabs, host-driven tasks
  Stencil* view = nullptr;      // exact solver: owned 3-axis view of the operator
};

int sweep_create(Ctx* c, const Stencil* coarse, int J, const int64_t* beta, const int64_t* bt,
                 const int64_t* lo, const int64_t* hi, const Stencil* const* slabs, Sweep** out);
void sweep_destroy(Sweep* s);
// launches [first, last) of the variant's plan (last < 0: to the end)
int sweep_apply(Ctx* c, Sweep* s, int variant, const double2* f, double2* u,
                const SweepWork* w = nullptr, int first = 0, int last = -1);
// nrhs right-hand sides f + r * stride -> u + r * stride through ONE chain of
// slab solves per group of up to max_nr (every factor block streamed once
// per group); per right-hand side bitwise the single application
int sweep_apply_many(Ctx* c, Sweep* s, int variant, int nrhs, const double2* f, double2* u,
                     int64_t stride, const SweepWork* w = nullptr);
// allocate / free a SweepWork sized for s (2-D levels only)
// NX schedule (prec_nx, sweepdd.py:403-437) for one cell grouping: j_cell
// (ncell + 1 entries, sentinels -1 and J + 1) and j_mid (ncell entries);
// returns the plan's variant id in *variant
int sweep_plan_nx(Ctx* c, Sweep* s, int ncell, const int64_t* j_cell, const int64_t* j_mid,
                  int* variant);
// one slab solve outside a schedule (subdom_solve); u rows [ta, tb) accumulated
int sweep_solve_one(Ctx* c, Sweep* s, int j, int64_t a, int64_t b, int64_t ta, int64_t tb,
                    const double2* B1, const double2* B3, double2* out2, double2* out4,
                    const double2* f, double2* u);
int sweep_work_create(Ctx* c, const Sweep* s, SweepWork* w, int nrhs = 1, bool batch = false);
void sweep_work_destroy(SweepWork* w);

// general sparse matrix rows (device CSR) for the exact solver's blocks
struct CsrSource {
  const int64_t* indptr = nullptr;
  const int64_t* indices = nullptr;
  const double2* vals = nullptr;
  int64_t n = 0;
};
int sweep3_create(Ctx* c, Sweep* s, const Stencil* coarse, const Stencil* const* slabs,
                  const int64_t* lo, const int64_t* hi, const CsrSource* csr);
int sweep3_task(Ctx* c, Sweep* s, const SweepTask& t, const double2* src, double2* const* u,
                const double2* coarse_coeffs, int64_t coarse_n);
// several right-hand sides through the 3-D chains: element strides between
// the right-hand sides' vectors (src, the two u destinations, trace buffers)
struct Sweep3Rhs {
  int nr;
  int64_t vs_src, vs_u[2], ts;
  double2* trace;
};
// one or two independent slab solves (two sweep fronts) in one chain launch
int sweep3_tasks(Ctx* c, Sweep* s, const SweepTask* const* ts, int nt, const double2* src,
                 double2* const* u, const double2* coarse_coeffs, int64_t coarse_n,
                 const Sweep3Rhs* mr = nullptr);
void sweep3_destroy(Sweep3* s3);
// Exact solver of a whole operator (ExactCoarseSolver / factorize,
// twogrid.py:99-105, sparselin.py:40-68): the operator as ONE block-LU slab
// (hs_sweep3.cu) behind the sweep interface -- plan HS_VARIANT_UD is a single
// slab solve over every row.
int exact_create(Ctx* c, const Stencil* op, Sweep** out);
// X plan cut at sweep-axis shard boundaries (relay emulation; hs_sweep.cu)
int sweep_plan_relay(Ctx* c, Sweep* s, int shards, int* variant);
// the same for a general sparse matrix in host CSR with block size NB >= its
// bandwidth (factorize(scipy matrix)); vectors hold ceil(n / NB) * NB entries
int exact_create_csr(Ctx* c, int64_t n, int64_t nnz, const int64_t* indptr, const int64_t* indices,
                     const double2* vals, int NB, Sweep** out);

}  // namespace hs
