// Temporary: kernel families not yet implemented report SFK_EUNSUPPORTED.
#include "sfk_internal.cuh"
namespace sfk {
int launch_hex_colloc_action(const sfk_plan*, int64_t, double*, const double*, const double*,
                             const double*, cudaStream_t) {
  return fail(SFK_EUNSUPPORTED, "collocated hex action: not implemented yet");
}
int launch_quad_action(const sfk_plan*, const sfk_plan*, int64_t, double*, double*, const double*,
                       const double*, cudaStream_t) {
  return fail(SFK_EUNSUPPORTED, "quad action: not implemented yet");
}
int launch_hex_matrix(const sfk_plan*, int64_t, double*, const double*, cudaStream_t) {
  return fail(SFK_EUNSUPPORTED, "hex matrix: not implemented yet");
}
int launch_hex_neohookean(const sfk_plan*, int64_t, double*, const double*, const double*,
                          cudaStream_t) {
  return fail(SFK_EUNSUPPORTED, "neo-Hookean: not implemented yet");
}
}  // namespace sfk
