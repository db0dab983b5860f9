// TEST INFRASTRUCTURE (oracle): link-time stand-ins for reference functions
// that container.cpp references but that lie outside the hot path and need
// more of Eigen than the shim provides (binary-factor, rotation and toy-model
// code).  The uniform / f32 container paths never call them; if they are
// called, the checker fails loudly.
#include <stdexcept>

#include "ocw/binfact.hpp"
#include "ocw/model.hpp"
#include "ocw/preprocess.hpp"

namespace ocw {
namespace {
[[noreturn]] void outside() { throw std::logic_error("oracle: outside the hot path"); }
}  // namespace
Matrix dequantize_binfact(const DbfMatrix&) { outside(); }
Matrix dequantize_binfact(const MdbfMatrix&) { outside(); }
size_t dbf_storage_bytes(const DbfMatrix&) { outside(); }
size_t mdbf_storage_bytes(const MdbfMatrix&) { outside(); }
Rotation Rotation::random_orthogonal(size_t, size_t) { outside(); }
Rotation Rotation::hadamard(size_t) { outside(); }
void ToyModelConfig::validate() const { outside(); }
}  // namespace ocw
