// dist_solve.cuh — preconditioner and Krylov solve on a row-partitioned hierarchy.
#pragma once

#include "dist_hierarchy.cuh"
#include "krylov.cuh"

namespace aggmg_b200 {

// z = M r on the calling rank's rows (z needs room for the level-0 halo: see dist_solve).
void dist_apply_preconditioner(DistHierarchy& h, const CycleCfg& cfg, const double* r, double* z);
// PCG (cfg.method == 1) or FGMRES over the ranks' rows; b, x are this rank's owned entries.
SolveOut dist_solve(DistHierarchy& h, const DistCsr& A, const CycleCfg& cyc, const SolverCfg& cfg,
                    const double* b, double* x);

}  // namespace aggmg_b200
