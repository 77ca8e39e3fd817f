// Instantiation set 3 of the look-ahead tiled update (update_kern.cuh): MathFused, normalize=false.
#include "update_kern.cuh"

namespace plnmf {
namespace upd {
template void launch_pl<MathFused, false>(cudaStream_t, const kern::PhaseBPlan&, LookArgs&);
}  // namespace upd
}  // namespace plnmf
