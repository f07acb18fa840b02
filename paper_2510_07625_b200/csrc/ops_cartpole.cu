#include "model_ops.cuh"
namespace gato {
ModelOps gato_ops_cartpole() { return make_ops<CartpoleModel>(); }
}  // namespace gato
