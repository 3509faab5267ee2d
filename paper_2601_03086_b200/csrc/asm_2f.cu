// asm_2f.cu — instantiation of the element kernels for dim=2, float.
#include "launch.cuh"

namespace pfem {
template pfem_status run_assemble<2, float>(const Call&);
}  // namespace pfem
