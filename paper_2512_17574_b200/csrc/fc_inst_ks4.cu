// fc_inst_ks4.cu -- instances of the fused kernel with KSH = 4 (H window
// of 128 source pixels per 8 outputs) and KSV = 1..4.  Split by KSH so the
// instances compile in parallel.
#include "fc_fused.cuh"

namespace fc {

void instances_ksh4(Instance* out) {
  out[0] = FC_INST(4, 1);
  out[1] = FC_INST(4, 2);
  out[2] = FC_INST(4, 3);
  out[3] = FC_INST(4, 4);
}

}  // namespace fc
