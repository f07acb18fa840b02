#include "model_ops.cuh"
namespace gato {
ModelOps gato_ops_double_integrator(int dims) {
  if (dims == 1) return make_ops<DoubleIntegratorModel<1>>();
  if (dims == 2) return make_ops<DoubleIntegratorModel<2>>();
  return make_ops<DoubleIntegratorModel<7>>();
}
}  // namespace gato
