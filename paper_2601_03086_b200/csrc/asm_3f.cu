// asm_3f.cu — instantiation of the element kernels for dim=3, float.
#include "launch.cuh"

namespace pfem {
template pfem_status run_assemble<3, float>(const Call&);
}  // namespace pfem
