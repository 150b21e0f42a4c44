// fc_inst_ks1.cu -- instances of the fused kernel with KSH = 1 (H window
// of 32 source pixels per 8 outputs) and KSV = 1..4.  Split by KSH so the
// instances compile in parallel.
#include "fc_fused.cuh"

namespace fc {

void instances_ksh1(Instance* out) {
  out[0] = FC_INST(1, 1);
  out[1] = FC_INST(1, 2);
  out[2] = FC_INST(1, 3);
  out[3] = FC_INST(1, 4);
}

}  // namespace fc
