// Host-side internals shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "plnmf_gpu.h"

namespace plnmf {

void set_last_error(const std::string& msg);
void validate_config(const plnmf_config& c);
void init_factors_host(int64_t v, int64_t d, const plnmf_config& cfg, double* w, double* ht);
// parsed Matrix Market file (mm.cpp)
const std::vector<int64_t>& mm_rows(const plnmf_mm* m);
const std::vector<int64_t>& mm_cols(const plnmf_mm* m);
const std::vector<double>& mm_values(const plnmf_mm* m);
bool mm_coordinate(const plnmf_mm* m);
int64_t mm_nrows(const plnmf_mm* m);
int64_t mm_ncols(const plnmf_mm* m);
void synth_csr(int64_t rows, int64_t cols, double density, uint64_t seed, int64_t* row_ptr,
               int64_t* col_idx, double* values, int64_t* nnz);

// Matrix Market parse failure (proj/include/plnmf/matrix_market.hpp:12-19):
// "source:line: what", a std::runtime_error.
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& source, int64_t line, const std::string& what);
    int64_t line() const { return line_; }

private:
    int64_t line_ = 0;
};

// Non-finite objective (proj/src/solver.cpp:96-98 throws std::runtime_error).
struct NonFinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// ||A|| == 0 (proj/src/metrics.cpp:84,101 throw std::domain_error).
struct DomainError : std::domain_error {
    using std::domain_error::domain_error;
};
// A CUDA runtime failure, re-thrown by the engine with its message.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Runs f, mapping the reference's exception types onto status codes.
template <class F>
plnmf_status guarded(F&& f) {
    try {
        f();
        return PLNMF_OK;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return PLNMF_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        set_last_error(e.what());
        return PLNMF_DOMAIN;
    } catch (const ParseError& e) {
        set_last_error(e.what());
        return PLNMF_PARSE;
    } catch (const DeviceError& e) {
        set_last_error(e.what());
        return PLNMF_CUDA;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return PLNMF_RUNTIME;
    } catch (const std::runtime_error& e) {
        set_last_error(e.what());
        return PLNMF_RUNTIME;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PLNMF_RUNTIME;
    }
}

}  // namespace plnmf
