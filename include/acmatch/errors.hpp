// Exception types of the acmatch API. Names and the is-a relation to
// acmatch::Error match the reference (/root/reference/proj/include/acmatch/
// errors.hpp:9-48) so callers' catch clauses keep working; DeviceError is new
// and reports CUDA-side failures of the GPU scan. Each C-ABI status code of
// include/acg.h maps to one of these (aho_corasick.hpp: detail::throw_acg).
#pragma once

#include <stdexcept>
#include <string>

namespace acmatch {

struct Error : std::runtime_error {
    explicit Error(const std::string& what_arg) : std::runtime_error(what_arg) {}
};

#define ACMATCH_DERIVED_ERROR(kind) \
    struct kind : Error {           \
        using Error::Error;         \
    }

ACMATCH_DERIVED_ERROR(EmptyPatternError);        // ACG_ERR_EMPTY_PATTERN
ACMATCH_DERIVED_ERROR(EmptyDictionaryError);     // ACG_ERR_EMPTY_DICTIONARY
ACMATCH_DERIVED_ERROR(InvalidWorkerCountError);  // ACG_ERR_INVALID_WORKER_COUNT
ACMATCH_DERIVED_ERROR(ZeroTimeError);            // reference bench API (out of scope here)
ACMATCH_DERIVED_ERROR(InfeasiblePlantError);     // reference corpus API (out of scope here)
ACMATCH_DERIVED_ERROR(IoError);                  // ACG_ERR_IO (io.hpp drop-in: acg_load_input / acg_load_patterns)
ACMATCH_DERIVED_ERROR(DeviceError);              // ACG_ERR_CUDA / _OUT_OF_MEMORY / _NO_DEVICE

#undef ACMATCH_DERIVED_ERROR

}  // namespace acmatch
