// dconv/shape.hpp -- drop-in for the reference header of the same name
// (/root/reference/proj/core/include/dconv/shape.hpp:29-45).  Same type, same
// fields, same validation (std::invalid_argument "ConvShape: ...").
#pragma once

namespace dconv {

/// Geometry of one valid (unpadded) convolution: (row y, column x)
/// coordinates, h_o = (h_i - h_f) / stride + 1; inexact strides are rejected.
struct ConvShape {
  int c_i;
  int c_o;
  int h_i;
  int w_i;
  int h_f;
  int w_f;
  int stride;
  int h_o;  ///< derived
  int w_o;  ///< derived

  ConvShape(int ci, int co, int hi, int wi, int hf, int wf, int s = 1);

  friend bool operator==(const ConvShape&, const ConvShape&) = default;
};

}  // namespace dconv
