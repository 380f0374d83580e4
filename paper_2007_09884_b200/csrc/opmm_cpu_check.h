// opmm_cpu_check.h -- host serial re-score of one OPC (Fig. 4 CPU_check).
#pragma once
#include "opmm.h"

namespace opmm {
// Serial fp64 RK4 re-score of one OPC against the host recorded trace
// (n_steps+1 samples); metric 0 = L1 sum, 1 = RMS.  PAPER.md:352.
double cpu_check_score(const double opc[OPMM_NPARAM], const double* rec, const opmm_control* ctl,
                       int metric);
}  // namespace opmm
