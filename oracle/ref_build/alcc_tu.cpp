// TEST INFRASTRUCTURE ONLY. Translation unit that compiles the reference's
// proj/core/src/alcc.cpp unmodified, from where it lies (path given by
// -DCVXREG_REF_ALCC_CPP). alcc.cpp:200-203 (alcc_solve) calls alcc_core with
// two trailing `nullptr` arguments that alcc.hpp:130-134 does not declare, so
// the file does not compile on its own. The overload below is declared first
// and forwards to the 12-argument alcc_core of alcc.hpp; nothing else changes.
#include <cstddef>

#include "cvxreg/alcc.hpp"

namespace cvxreg {
inline AlccResult alcc_core(const ConstraintRows& rows, const VectorXd& center_y,
                            const VectorXd& center_xi, double gamma, double Bbar_y,
                            double Bbar_xi, double sigma_A1, double sigma_A2,
                            const AlccConfig& cfg, double target_subopt,
                            const VectorXd& warm_y, const VectorXd& warm_xi,
                            std::nullptr_t, std::nullptr_t) {
  return alcc_core(rows, center_y, center_xi, gamma, Bbar_y, Bbar_xi, sigma_A1,
                   sigma_A2, cfg, target_subopt, warm_y, warm_xi);
}
}  // namespace cvxreg

#include CVXREG_REF_ALCC_CPP
