// fc_inst_ks3.cu -- instances of the fused kernel with KSH = 3 (H window
// of 96 source pixels per 8 outputs) and KSV = 1..4.  Split by KSH so the
// instances compile in parallel.
#include "fc_fused.cuh"

namespace fc {

void instances_ksh3(Instance* out) {
  out[0] = FC_INST(3, 1);
  out[1] = FC_INST(3, 2);
  out[2] = FC_INST(3, 3);
  out[3] = FC_INST(3, 4);
}

}  // namespace fc
