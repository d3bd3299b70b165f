/* quota_b200.hpp -- C++ drop-in surface of the B200 QUOTA path.
 *
 * The reference C++ API itself (proj/include/quota/model.hpp,
 * selector.hpp, recipe.hpp -- unmodified) IS the surface: link
 * libquota_b200_cxx.so ahead of the reference library (or LD_PRELOAD it) and
 * quota::forward_prefill / quota::decode_step / quota::make_recipe_hook run on
 * the B200 (paper_2604_17320_b200/cxx/quota_backend.cpp, over the C ABI in
 * quota_b200.h).  This header adds the two helpers the drop-in needs.
 */
#ifndef QUOTA_B200_HPP
#define QUOTA_B200_HPP

#include "quota/model.hpp"

namespace quota_b200 {

/* prepare_quant_env (model.cpp:212-237) with one weight scale per OUTPUT
 * channel (GroupAxis::PerColumn) -- the axis an int32-accumulator W4A4 GEMM
 * applies in its epilogue.  The reference's own prepare_quant_env scales per
 * input channel (GroupAxis::PerRow), which the device path rejects. */
quota::QuantEnv prepare_quant_env_per_channel(const quota::Model& model, const quota::QuantConfig& config,
                                              const quota::ActScales& act);

/* Drop every device engine and session (frees HBM). */
void release_device_sessions();

}  // namespace quota_b200

#endif
