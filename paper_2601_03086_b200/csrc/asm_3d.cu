// asm_3d.cu — instantiation of the element kernels for dim=3, double.
#include "launch.cuh"

namespace pfem {
template pfem_status run_assemble<3, double>(const Call&);
}  // namespace pfem
