// Instantiation set 2 of the look-ahead tiled update (update_kern.cuh): MathFused, normalize=true.
#include "update_kern.cuh"

namespace plnmf {
namespace upd {
template void launch_pl<MathFused, true>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
}  // namespace upd
}  // namespace plnmf
