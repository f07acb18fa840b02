#include "model_ops.cuh"
namespace gato {
ModelOps gato_ops_pendulum() { return make_ops<PendulumModel>(); }
}  // namespace gato
