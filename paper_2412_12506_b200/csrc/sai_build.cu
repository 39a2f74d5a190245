// GPU SAI build (placeholder until the batched least-squares path lands).
#include "mg.hpp"
namespace ldgmg_b200 {
SaiResult build_sai_gpu(Ctx&, const Bsr&, int, int, int, double, bool) {
    fail(LDGMG_ERR_LOGIC, "build_sai: GPU least-squares build not available in this build");
}
}  // namespace ldgmg_b200
