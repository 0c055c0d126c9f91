// tsdict/errors.hpp -- drop-in for the reference error model
// (/root/reference/proj/include/tsdict/errors.hpp:13-68): one exception type
// carrying a stable code; what() is prefixed by the code name. The ordinal
// order of errc is part of the C ABI (status = 1 + ordinal, tsdict_cuda.h).
#ifndef TSDICT_B200_ERRORS_HPP
#define TSDICT_B200_ERRORS_HPP

#include <stdexcept>
#include <string>

#include "tsdict_cuda.h"

namespace tsdict {

enum class errc {
  window_too_small,
  window_too_large,
  non_finite_input,
  length_mismatch,
  series_too_short,
  iteration_cap_exceeded,
  source_mismatch,
  window_mismatch,
  empty_dictionary,
  empty_profile,
  degenerate_labels,
  parse_error,
  version_error,
  schema_error,
  io_error,
  invalid_argument,
};

// names come from the C library so both sides of the boundary agree
inline const char* errc_name(errc c) { return tsd_status_name(static_cast<int>(c) + 1); }

class error : public std::runtime_error {
 public:
  error(errc code, const std::string& message)
      : std::runtime_error(std::string(errc_name(code)) + ": " + message), code_(code) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

// A device failure has no errc counterpart; it surfaces as std::runtime_error.
class device_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {

// Maps a C ABI status to the reference exception (message already carries
// the code-name prefix, so it is stripped before re-wrapping).
inline void raise_status(int st) {
  if (st == TSD_OK) return;
  std::string msg = tsd_last_error();
  if (st == TSD_CUDA_ERROR || st < 1 || st > 16) throw device_error(msg);
  const errc code = static_cast<errc>(st - 1);
  const std::string prefix = std::string(errc_name(code)) + ": ";
  if (msg.compare(0, prefix.size(), prefix) == 0) msg = msg.substr(prefix.size());
  throw error(code, msg);
}

}  // namespace detail
}  // namespace tsdict

#endif
