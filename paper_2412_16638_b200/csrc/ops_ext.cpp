// North-star extensions without a reference counterpart: block-Jacobi
// preconditioner with per-block storage precision, CSR SpMV with
// fp16/fp32/fp64 value storage (accessor-style: storage precision is
// independent of the compute precision).
#include "ops.hpp"

namespace mprkb {

std::unique_ptr<Op> make_block_jacobi(int, const Problem&, double, double, int, int) {
  MPRKB_THROW(1, "block-Jacobi preconditioner: not built yet");
}

std::unique_ptr<Op> make_csr(int, int, const int*, const int*, const void*, int) {
  MPRKB_THROW(1, "CSR operator: not built yet");
}

std::unique_ptr<Op> make_csr_stencil(int, const StencilSpec&, int) {
  MPRKB_THROW(1, "CSR operator: not built yet");
}

}  // namespace mprkb
