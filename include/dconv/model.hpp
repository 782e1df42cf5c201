// dconv/model.hpp -- the part of the reference's model.hpp that crosses the
// operator API (BlockingParams, model.hpp:54-61).  The CPU machine model and
// autotuner (model.hpp:28-109) are out of scope for the GPU path; on the GPU
// c_ob / c_ib select the blocked layout and the CUDA tile selector replaces
// the register model.
#pragma once

namespace dconv {

struct BlockingParams {
  int c_ob = 1;  ///< output-channel block of the layout
  int w_ob = 1;  ///< CPU register-tile width (accepted, unused on the GPU)
  int c_ib = 1;  ///< input-channel block of the layout
  friend bool operator==(const BlockingParams&, const BlockingParams&) = default;
};

}  // namespace dconv
