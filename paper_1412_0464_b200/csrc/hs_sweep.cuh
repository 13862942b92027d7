#pragma once
#include "hs_common.cuh"

namespace hs {

// Slab solve geometry: every slab is a block-tridiagonal system along the face
// axis y (M blocks) whose blocks are tm x tm (thin sweep-axis layers padded to
// tm = 16 or 32; see Geo<TM> in hs_sweep.cu for the record layouts).

// One slab solve of a schedule (subdom_solve, sweepdd.py:236-268).
struct SweepTask {
  int slab;        // 0-based slab index j-1
  int lo;          // first grid point of the slab (1-based)
  int T;           // thickness (layers)
  int a, b;        // f rows [a, b) restricted into the slab (global 0-based rows)
  int ta, tb;      // u rows [ta, tb) scattered back
  int fdslot;      // row of the gathered right-hand side in this pass
  int tin1, row1;  // forward transmission in (buffer, slab-local row) or -1
  int tin3, row3;  // backward transmission in
  int out2, orow2; // forward trace out -> consumer's tin buffer, slab-local trace row
  int out4, orow4; // backward trace out
  int dst;         // 0: pass-1 solution u, 1: pass-2 buffer u2 (summed at the end)
};

struct SweepLaunch {
  enum Kind { kCombine, kGather, kFront, kResidual } kind;
  int src;                  // gather: 0 = f, 1 = g
  int first, count;         // task range (gather: all tasks of the pass)
  int nfront;
  int ffirst[2], fcount[2]; // front task ranges (global task indices)
  double bytes;             // algorithmic HBM bytes of the launch (profiler)
};

struct Sweep {
  int J = 0, M = 0, n0 = 0;
  int tm = 16;                  // padded block size (16 or 32)
  const Stencil* coarse = nullptr;
  double2* fwd_rec = nullptr;   // [J][M][FREC]
  double2* bwd_rec = nullptr;   // [J][M][BREC]
  double2* fdpre = nullptr;     // [max pass tasks][M][tm]
  double2* tin = nullptr;       // [ntin][M][2]
  double2* zs = nullptr;        // [2][M][tm]
  double2* g = nullptr;         // [n0*M] mid-sweep residual
  double2* u2 = nullptr;        // [n0*M] second-pass contributions
  SweepTask* d_tasks = nullptr;
  std::vector<SweepTask> tasks;
  std::vector<SweepLaunch> plan[2];   // by variant (UD, X)
  bool has_plan[2] = {false, false};
  long long factor_bytes = 0;
};

int sweep_create(Ctx* c, const Stencil* coarse, int J, const int64_t* beta, const int64_t* bt,
                 const int64_t* lo, const int64_t* hi, const Stencil* const* slabs, Sweep** out);
void sweep_destroy(Sweep* s);
int sweep_apply(Ctx* c, Sweep* s, int variant, const double2* f, double2* u);

}  // namespace hs
