// socfield/pinned.hpp — additive (no counterpart in the reference, whose state never leaves host memory).
//
// The engine copies a SimState's dense arrays (occupancy, the four strength images) to the device and
// back on every Engine::run / tick.  From pageable memory that copy bounces through the driver's staging
// buffers; from page-locked memory it is one DMA at PCIe rate.  HostPin page-locks the storage of an
// array for exactly as long as that storage lives.  The owning class spells out its special members so that
//   copy construct   the copy has fresh storage: not locked
//   copy assign      the owner's storage may be reallocated: unlocked first
//   move             the lock travels with the buffer
//   destroy          unlocked before the buffer is freed
// and `ensure` re-checks (address, size) before every use, so a buffer replaced through raw_mut() is noticed.
#pragma once

#include <cstddef>

namespace socfield::detail {

class HostPin {
public:
    HostPin() = default;
    HostPin(const HostPin&) noexcept {}
    HostPin& operator=(const HostPin&) noexcept {
        release();
        return *this;
    }
    HostPin(HostPin&& other) noexcept : ptr_(other.ptr_), bytes_(other.bytes_) {
        other.ptr_ = nullptr;
        other.bytes_ = 0;
    }
    HostPin& operator=(HostPin&& other) noexcept {
        if (this != &other) {
            release();
            ptr_ = other.ptr_;
            bytes_ = other.bytes_;
            other.ptr_ = nullptr;
            other.bytes_ = 0;
        }
        return *this;
    }
    ~HostPin() { release(); }

    // Page-locks [p, p + bytes) unless it already is; arrays under 1 MiB are left alone.  Failure to lock is
    // not an error: the copy then takes the staged path.
    void ensure(const void* p, std::size_t bytes) noexcept;
    void release() noexcept;
    bool locked() const noexcept { return ptr_ != nullptr; }

private:
    const void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

} // namespace socfield::detail
