#include "model_ops.cuh"
namespace gato {
ModelOps gato_ops_iiwa14() { return make_ops<Iiwa14Model>(); }
}  // namespace gato
