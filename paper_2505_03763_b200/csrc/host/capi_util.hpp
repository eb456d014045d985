// Exception -> status-code translation for the C-ABI (errors.hpp taxonomy ->
// SW_E* codes, see include/splitwise.h).
#pragma once

#include <exception>
#include <string>

#include "../../../include/splitwise.h"
#include "base.hpp"

namespace sw {

extern thread_local std::string g_last_error;
char* dup_text(const std::string& s);

// Raised by CUDA call checks; maps to SW_ECUDA.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return SW_OK;
    } catch (const ConfigError& e) {
        g_last_error = std::string("ConfigError: ") + e.what();
        return SW_ECONFIG;
    } catch (const ParseError& e) {
        g_last_error = std::string("ParseError: ") + e.what();
        return SW_ECONFIG;
    } catch (const IoError& e) {
        g_last_error = std::string("IoError: ") + e.what();
        return SW_EIO;
    } catch (const ContractViolation& e) {
        g_last_error = std::string("ContractViolation: ") + e.what();
        return SW_ECONTRACT;
    } catch (const CudaError& e) {
        g_last_error = std::string("CudaError: ") + e.what();
        return SW_ECUDA;
    } catch (const std::exception& e) {
        g_last_error = std::string("error: ") + e.what();
        return SW_ECONTRACT;
    }
}

}  // namespace sw
