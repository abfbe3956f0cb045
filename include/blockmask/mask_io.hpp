// blockmask/mask_io.hpp — drop-in for the reference's mask files (proj/include/blockmask/
// mask_io.hpp:14-207): the "BBMK" mask file and the "BBLK" occupancy sidecar, same byte layout,
// 4M-token cap and MaskIoError kinds, through libbbm (bbm_capi.h). Extension:
// preprocess_mask_file() uploads a file's byte rows as-is and unpacks them on the device.
#pragma once

#include <cstdint>
#include <filesystem>
#include <stdexcept>
#include <string>

#include "blockmask/device.hpp"
#include "blockmask/engine.hpp"
#include "blockmask/mask.hpp"

namespace blockmask {

class MaskIoError : public std::runtime_error {
public:
    enum class Kind { io_failure, bad_magic, bad_version, dimension_overflow, truncated, trailing_data };
    MaskIoError(Kind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    Kind kind() const { return kind_; }

private:
    Kind kind_;
};

namespace detail {
inline void io_check(bbm_status st, const char* what) {
    if (st >= BBM_ERR_IO_FAILURE && st <= BBM_ERR_IO_TRAILING_DATA)
        throw MaskIoError(static_cast<MaskIoError::Kind>(st - BBM_ERR_IO_FAILURE), bbm_last_error());
    device::check(st, what);
}
}  // namespace detail

inline void write_mask(const Mask& mask, const std::filesystem::path& path) {
    detail::io_check(bbm_write_mask_file(path.c_str(), mask.words(), mask.size()), "write_mask");
}

inline Mask read_mask(const std::filesystem::path& path) {
    std::uint64_t n = 0;
    detail::io_check(bbm_read_mask_file(path.c_str(), &n, nullptr), "read_mask");
    Mask m(n);
    detail::io_check(bbm_read_mask_file(path.c_str(), &n, m.words()), "read_mask");
    return m;
}

struct OccupancyFile {
    std::uint64_t n_tokens = 0;
    BlockSpec spec;
    BlockOccupancy occupancy;
};

inline void write_occupancy(const BlockOccupancy& occ, std::size_t n_tokens, BlockSpec spec,
                            const std::filesystem::path& path) {
    std::vector<std::uint8_t> v(occ.rows() * occ.cols());
    for (std::size_t p = 0; p < occ.rows(); ++p)
        for (std::size_t q = 0; q < occ.cols(); ++q) v[p * occ.cols() + q] = occ.at(p, q) ? 1 : 0;
    detail::io_check(bbm_write_occupancy_file(path.c_str(), v.data(), n_tokens, spec.block_i, spec.block_j),
                     "write_occupancy");
}

inline OccupancyFile read_occupancy(const std::filesystem::path& path) {
    std::uint64_t n = 0, bi = 0, bj = 0;
    detail::io_check(bbm_read_occupancy_file(path.c_str(), &n, &bi, &bj, nullptr), "read_occupancy");
    OccupancyFile f;
    f.n_tokens = n;
    f.spec = BlockSpec{bi, bj};
    f.occupancy = BlockOccupancy((n + bi - 1) / bi, (n + bj - 1) / bj);
    detail::io_check(bbm_read_occupancy_file(path.c_str(), &n, &bi, &bj, f.occupancy.data()), "read_occupancy");
    return f;
}

/// read_mask + preprocess_mask, the file's byte rows unpacked on the device.
inline MaskPrep preprocess_mask_file(const std::filesystem::path& path, BlockSpec spec) {
    spec.validate();
    bbm_prep h = nullptr;
    detail::io_check(bbm_preprocess_mask_file(path.c_str(), spec.block_i, spec.block_j,
                                              device::default_device(), &h),
                     "preprocess_mask_file");
    MaskPrep prep = detail::prep_from_handle(h, spec);
    return prep;
}

}  // namespace blockmask
