// Instantiation set 1 of the look-ahead tiled update (update_kern.cuh): MathExact, normalize=false.
#include "update_kern.cuh"

namespace plnmf {
namespace upd {
template void launch_pl<MathExact, false>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
}  // namespace upd
}  // namespace plnmf
