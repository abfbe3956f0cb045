// blockmask/device.hpp — glue between the drop-in C++ API and libbbm's C ABI (bbm_capi.h).
//
// Not part of the reference's interface. Maps bbm_status onto the reference's error convention
// (require() -> std::invalid_argument, matrix.hpp:47-49) and owns the device-side MaskPrep.
// Link with -L<repo>/paper_2409_15097_b200 -lbbm.
#pragma once

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>

#include "../bbm_capi.h"

namespace blockmask {
namespace device {

/// Device a prep is built on when the caller does not choose one (BBM_DEVICE, default 0).
inline int default_device() {
    static const int dev = [] {
        const char* s = std::getenv("BBM_DEVICE");
        return s ? std::atoi(s) : 0;
    }();
    return dev;
}

/// Invalid arguments become std::invalid_argument exactly as the reference's require() throws;
/// a kernel-side limitation (head dim, d_v != d_k) is also an invalid argument for this engine.
/// CUDA failures (including "no device": there is no CPU fallback) are std::runtime_error.
inline void check(bbm_status st, const char* what) {
    if (st == BBM_OK) return;
    const std::string msg = std::string(bbm_last_error());
    if (st == BBM_ERR_INVALID || st == BBM_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(std::string(what) + ": " + msg);
}

/// Shared owner of a bbm_prep (device metadata), so MaskPrep / BlockSums stay cheap to copy.
class PrepHandle {
public:
    explicit PrepHandle(bbm_prep h) : h_(h) {}
    ~PrepHandle() { if (h_) bbm_prep_destroy(h_); }
    PrepHandle(const PrepHandle&) = delete;
    PrepHandle& operator=(const PrepHandle&) = delete;
    bbm_prep get() const { return h_; }

private:
    bbm_prep h_ = nullptr;
};

using PrepPtr = std::shared_ptr<PrepHandle>;

}  // namespace device
}  // namespace blockmask
