"""CPU test of the page store's native index (csrc/vaddr_map.hpp: open
addressing, backward-shift deletion): a C++ driver replays random
insert / erase / find / iterate sequences -- clustered keys, growth and
wrap-around included -- against std::unordered_map."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DRIVER = r"""
#include <cstdio>
#include <random>
#include <unordered_map>
#include "vaddr_map.hpp"

int main() {
  std::mt19937_64 rng(12345);
  for (int round = 0; round < 40; ++round) {
    pc::VaddrMap m;
    std::unordered_map<uint64_t, uint32_t> ref;
    // few distinct pages -> long probe runs and many erase shifts
    const uint64_t span = 8 + rng() % (round < 20 ? 64 : 20000);
    const uint64_t base = (rng() & 0xffffffffff000ull) | 0xfff0000000000000ull * (round % 3 == 0);
    for (int op = 0; op < 20000; ++op) {
      const uint64_t k = base + 4096ull * (rng() % span);
      const uint32_t v = static_cast<uint32_t>(rng());
      switch (rng() % 4) {
        case 0: case 1: {
          const bool a = m.insert(k, v), b = ref.emplace(k, v).second;
          if (a != b) { printf("insert mismatch\n"); return 1; }
          break;
        }
        case 2: {
          const bool a = m.erase(k), b = ref.erase(k) > 0;
          if (a != b) { printf("erase mismatch\n"); return 2; }
          break;
        }
        default: {
          const uint32_t *f = m.find(k);
          auto it = ref.find(k);
          if ((f == nullptr) != (it == ref.end()) || (f && *f != it->second)) { printf("find mismatch\n"); return 3; }
        }
      }
      if (m.size() != ref.size()) { printf("size mismatch\n"); return 4; }
    }
    size_t seen = 0;
    bool ok = true;
    m.for_each([&](uint64_t k, uint32_t v) { ++seen; auto it = ref.find(k); ok &= it != ref.end() && it->second == v; });
    if (!ok || seen != ref.size()) { printf("iterate mismatch\n"); return 5; }
    if (m.find(~0ull) || m.erase(~0ull)) { printf("empty marker leaked\n"); return 6; }
  }
  printf("ok\n");
  return 0;
}
"""


def test_vaddr_map_matches_unordered_map(tmp_path):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no C++ compiler")
    src = tmp_path / "vm.cpp"
    src.write_text(DRIVER)
    exe = tmp_path / "vm"
    subprocess.run([gxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I",
                    os.path.join(ROOT, "paper_2004_09252_b200", "csrc"), str(src), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout)
