// ddm-b200: exception taxonomy of the reference library (`proj/core/include/ddm/errors.hpp`),
// kept name- and hierarchy-compatible so callers' catch clauses keep working. The C-ABI
// maps them to status codes 1 (InputError), 2 (PlanError / bad_alloc), 3 (IoError).
#ifndef DDM_B200_ERRORS_HPP
#define DDM_B200_ERRORS_HPP

#include <stdexcept>
#include <string>

namespace ddm {

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

/// Bad arguments, malformed headers, corrupt or inconsistent partial files.
class InputError : public Error {
public:
    using Error::Error;
};

/// The budget (host `memory_bytes`, or device memory / kernel limits) cannot hold the job.
class PlanError : public Error {
public:
    using Error::Error;
};

/// Filesystem failures.
class IoError : public Error {
public:
    using Error::Error;
};

/// Device failures (no reference counterpart; status 4 at the C-ABI).
class DeviceError : public Error {
public:
    using Error::Error;
};

} // namespace ddm

#endif
