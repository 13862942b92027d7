#pragma once
#include "hs_common.cuh"

namespace hs {

// Per-axis tent-transfer tables (canonical 3 axes, fastest last).
struct TransferDesc {
  int64_t nf[3], nc[3];   // global fine / coarse extents
  // Shard window along the sweep axis (canonical axis 3 - dim; the identity
  // window elsewhere): the fine buffer holds global rows [fw_lo, fw_lo +
  // fw_cnt); restriction computes coarse rows [cr_lo, cr_lo + cr_cnt) of a
  // full-size coarse vector; prolongation computes fine rows [fr_lo, fr_lo +
  // fr_cnt) of the windowed buffer from a full-size coarse vector.
  int64_t fw_lo[3], fw_cnt[3], cr_lo[3], cr_cnt[3], fr_lo[3], fr_cnt[3];
  const int* ctr[3];      // [nc]  fine centre index of coarse unknown I
  const double* wl[3];    // [nc]  weight of fine centre-1 (0 or 1/2)
  const double* wr[3];    // [nc]  weight of fine centre+1 (0 or 1/2)
  const int* par[3];      // [2*nf] coarse parents of fine unknown (or -1)
  const double* pw[3];    // [2*nf] parent weights
};

struct Transfer {
  int dim = 0;
  TransferDesc d{};
  char* buf = nullptr;
};

int transfer_create(Ctx* c, int dim, const int64_t* fp_len, const int64_t* fp_concat,
                    const uint8_t* refined_concat, Transfer** out,
                    const int64_t* window = nullptr /* fw_lo fw_hi cr_lo cr_hi fr_lo fr_hi */);
void transfer_destroy(Transfer* t);
int transfer_restrict(Ctx* c, const Transfer* t, const double2* r, double2* rc, double scale,
                      int nrhs);
int transfer_prolong(Ctx* c, const Transfer* t, const double2* uc, double2* u, int accumulate,
                     int nrhs);

}  // namespace hs
