// polyargmax/errors.hpp — exception types of the drop-in C++ API.
//
// Interface-compatible with the reference's error hierarchy
// (/root/reference/proj/include/polyargmax/errors.hpp:9-87): same namespace,
// class names, base class (std::runtime_error) and constructor signatures, so
// reference-side code that catches these types keeps working.  Each class
// also carries the pam_status code it is raised for (include/pam_c_api.h).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace polyargmax {

/// Root of every error raised by the library (errors.hpp:9).
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
  explicit Error(const char* what) : std::runtime_error(what) {}
};

// Plain subclasses: a message, nothing else.  The macro keeps the list short;
// each line names the SPEC clause that raises it.
#define POLYARGMAX_PLAIN_ERROR(NAME)                                  \
  class NAME : public Error {                                         \
   public:                                                            \
    explicit NAME(const std::string& what) : Error(what) {}           \
    explicit NAME(const char* what) : Error(what) {}                  \
  }

POLYARGMAX_PLAIN_ERROR(DegenerateInputError);  // s^2 < eps_var
POLYARGMAX_PLAIN_ERROR(InvalidParamsError);    // CutMaxParams invariants
POLYARGMAX_PLAIN_ERROR(RangeError);            // approximation domain
POLYARGMAX_PLAIN_ERROR(DomainError);           // u in {0,1}, p,q outside (0,1)
POLYARGMAX_PLAIN_ERROR(WidthMismatchError);    // hesim (out of scope here)
POLYARGMAX_PLAIN_ERROR(BadRotationError);      // hesim (out of scope here)
POLYARGMAX_PLAIN_ERROR(RangeProofViolation);   // encargmax (out of scope here)
POLYARGMAX_PLAIN_ERROR(SingularityError);      // grad (out of scope here)
POLYARGMAX_PLAIN_ERROR(BadSpecError);          // cli (out of scope here)

#undef POLYARGMAX_PLAIN_ERROR

/// Malformed input file; remembers where.
class FormatError : public Error {
 public:
  FormatError(const std::string& what, std::size_t byte_offset)
      : Error(what + " (byte offset " + std::to_string(byte_offset) + ")"), byte_offset_(byte_offset) {}
  std::size_t byte_offset() const { return byte_offset_; }

 private:
  std::size_t byte_offset_;
};

/// A vector (row) containing NaN/Inf; remembers which one.
class NonFiniteError : public Error {
 public:
  NonFiniteError(const std::string& what, std::size_t vector_index)
      : Error(what + " (vector " + std::to_string(vector_index) + ")"), vector_index_(vector_index) {}
  std::size_t vector_index() const { return vector_index_; }

 private:
  std::size_t vector_index_;
};

}  // namespace polyargmax
