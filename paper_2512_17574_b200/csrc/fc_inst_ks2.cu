// fc_inst_ks2.cu -- instances of the fused kernel with KSH = 2 (H window
// of 64 source pixels per 8 outputs) and KSV = 1..4.  Split by KSH so the
// instances compile in parallel.
#include "fc_fused.cuh"

namespace fc {

void instances_ksh2(Instance* out) {
  out[0] = FC_INST(2, 1);
  out[1] = FC_INST(2, 2);
  out[2] = FC_INST(2, 3);
  out[3] = FC_INST(2, 4);
}

}  // namespace fc
