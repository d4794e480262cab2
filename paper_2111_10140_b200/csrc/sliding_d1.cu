// v2 sliding-window spread/gather instantiations, d=1 windows.
#include "sliding_impl.cuh"

namespace afs {
AFS_SLIDING_INSTANTIATE(1)
}  // namespace afs
