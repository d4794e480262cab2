// v2 sliding-window spread/gather instantiations, d=2 windows.
#include "sliding_impl.cuh"

namespace afs {
AFS_SLIDING_INSTANTIATE(2)
}  // namespace afs
