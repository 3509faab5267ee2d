// asm_2d.cu — instantiation of the element kernels for dim=2, double.
#include "launch.cuh"

namespace pfem {
template pfem_status run_assemble<2, double>(const Call&);
}  // namespace pfem
