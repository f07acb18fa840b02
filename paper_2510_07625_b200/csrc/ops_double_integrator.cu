#include "model_ops.cuh"
namespace gato {
// dynamics.py:145-163: point masses in `dims` dimensions, instantiated for dims = 1..7
ModelOps gato_ops_double_integrator(int dims) {
  switch (dims) {
    case 1: return make_ops<DoubleIntegratorModel<1>>();
    case 2: return make_ops<DoubleIntegratorModel<2>>();
    case 3: return make_ops<DoubleIntegratorModel<3>>();
    case 4: return make_ops<DoubleIntegratorModel<4>>();
    case 5: return make_ops<DoubleIntegratorModel<5>>();
    case 6: return make_ops<DoubleIntegratorModel<6>>();
    default: return make_ops<DoubleIntegratorModel<7>>();
  }
}
}  // namespace gato
