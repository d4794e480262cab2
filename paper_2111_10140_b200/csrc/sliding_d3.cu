// v2 sliding-window spread/gather instantiations, d=3 windows.
#include "sliding_impl.cuh"

namespace afs {
AFS_SLIDING_INSTANTIATE(3)
}  // namespace afs
