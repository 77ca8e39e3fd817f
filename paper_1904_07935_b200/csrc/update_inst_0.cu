// Instantiation set 0 of the look-ahead tiled update (update_kern.cuh): MathExact, normalize=true.
#include "update_kern.cuh"

namespace plnmf {
namespace upd {
template void launch_pl<MathExact, true>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
}  // namespace upd
}  // namespace plnmf
