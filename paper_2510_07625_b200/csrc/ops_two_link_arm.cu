#include "model_ops.cuh"
namespace gato {
ModelOps gato_ops_two_link_arm() { return make_ops<TwoLinkArmModel>(); }
}  // namespace gato
