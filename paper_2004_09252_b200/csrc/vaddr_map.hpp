// vaddr_map.hpp -- the page store's per-client index (store.inc): a flat
// open-addressing hash map vaddr -> slot.  Header-only and CUDA-free so the
// CPU tests can compile it against std::unordered_map (tests/test_vaddr_map.py).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace pc {

// vaddr -> slot of one client: open addressing with linear probing and
// backward-shift deletion (no tombstones), load factor <= 1/2.  A node-based
// std::unordered_map cost as much host time per batch as the PCIe transfer
// (26 vs 53 GB/s, tools/store_probe.py); flat arrays do not.  Keys are
// page-aligned vaddrs, so ~0 (never aligned) marks an empty cell.
class VaddrMap {
 public:
  size_t size() const { return size_; }
  bool empty() const { return size_ == 0; }
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap > keys_.size()) rehash(cap);
  }
  const uint32_t *find(uint64_t k) const {
    if (keys_.empty() || k == kEmpty) return nullptr;
    for (size_t i = home(k);; i = (i + 1) & mask_) {
      if (keys_[i] == k) return &vals_[i];
      if (keys_[i] == kEmpty) return nullptr;
    }
  }
  bool count(uint64_t k) const { return find(k) != nullptr; }
  // false (and no change) when k is already present
  bool insert(uint64_t k, uint32_t v) {
    reserve(size_ + 1);
    size_t i = home(k);
    for (; keys_[i] != kEmpty; i = (i + 1) & mask_)
      if (keys_[i] == k) return false;
    keys_[i] = k;
    vals_[i] = v;
    ++size_;
    return true;
  }
  bool erase(uint64_t k) {
    if (keys_.empty() || k == kEmpty) return false;
    size_t i = home(k);
    for (; keys_[i] != k; i = (i + 1) & mask_)
      if (keys_[i] == kEmpty) return false;
    // backward shift: pull later members of the probe run into the hole
    for (size_t j = (i + 1) & mask_; keys_[j] != kEmpty; j = (j + 1) & mask_) {
      const size_t h = home(keys_[j]);
      if (((j - h) & mask_) >= ((j - i) & mask_)) {
        keys_[i] = keys_[j];
        vals_[i] = vals_[j];
        i = j;
      }
    }
    keys_[i] = kEmpty;
    --size_;
    return true;
  }
  template <typename F>
  void for_each(F f) const {
    for (size_t i = 0; i < keys_.size(); ++i)
      if (keys_[i] != kEmpty) f(keys_[i], vals_[i]);
  }

 private:
  static constexpr uint64_t kEmpty = ~0ull;
  size_t home(uint64_t k) const { return static_cast<size_t>(((k >> 12) * 0x9E3779B97F4A7C15ull) >> shift_); }
  void rehash(size_t cap) {
    std::vector<uint64_t> ok;
    std::vector<uint32_t> ov;
    ok.swap(keys_);
    ov.swap(vals_);
    keys_.assign(cap, kEmpty);
    vals_.assign(cap, 0);
    mask_ = cap - 1;
    shift_ = 64;
    for (size_t c = cap; c > 1; c >>= 1) --shift_;
    size_ = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != kEmpty) insert(ok[i], ov[i]);
  }
  std::vector<uint64_t> keys_;
  std::vector<uint32_t> vals_;
  size_t size_ = 0, mask_ = 0;
  int shift_ = 64;
};

} // namespace pc
