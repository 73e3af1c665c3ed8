// sparse.cu — persistent sm_100a solver for CSR / ELL MDPs (placeholder until
// the sparse kernel lands; dense problems are served by dense.cu).
#include "internal.h"

namespace rmb {

rmb_status sparse_solve(Problem&, const SolveRequest&, double*, int64_t, long long*, int64_t, SolveResult*)
{
    set_error("sparse solver not built yet");
    return RMB_ERR_UNSUPPORTED;
}

}  // namespace rmb
