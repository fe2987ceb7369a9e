// numa.hpp -- host placement for a GPU's staging ("a per-GPU
// pinned staging ring and streams on a NUMA-local host thread").
//
// On a two-socket 8-GPU host, half of the GPUs hang off each socket's PCIe
// root.  Bounce copies and pinned staging on the far socket cross the socket
// link twice per page, so each engine binds its runner and bounce threads to
// the CPUs local to its GPU and allocates its pinned buffers with a
// preferred-node memory policy while bound.  Everything here is read from
// sysfs (/sys/bus/pci/devices/<bus id>/{numa_node,local_cpulist}); when the
// platform does not report a node (numa_node == -1, e.g. a single-socket VM)
// the placement is a no-op.
#pragma once
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>

namespace pc {

struct DevicePlacement {
  int node = -1;          // NUMA node of the GPU's PCIe root, -1 = unknown
  bool has_cpus = false;  // cpus holds the GPU-local CPUs
  cpu_set_t cpus;
};

// Parse a kernel cpulist ("0-15,32-47") into a cpu_set_t.
inline bool parse_cpulist(const char *s, cpu_set_t *set) {
  CPU_ZERO(set);
  bool any = false;
  while (*s) {
    while (*s == ',' || isspace(static_cast<unsigned char>(*s))) ++s;
    if (!isdigit(static_cast<unsigned char>(*s))) break;
    char *end = nullptr;
    long lo = strtol(s, &end, 10), hi = lo;
    s = end;
    if (*s == '-') {
      hi = strtol(s + 1, &end, 10);
      s = end;
    }
    for (long c = lo; c <= hi && c < CPU_SETSIZE; ++c) {
      CPU_SET(static_cast<int>(c), set);
      any = true;
    }
  }
  return any;
}

inline DevicePlacement device_placement(int device) {
  DevicePlacement p;
  CPU_ZERO(&p.cpus);
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return p;
  }
  for (char *c = bus; *c; ++c) *c = static_cast<char>(tolower(static_cast<unsigned char>(*c)));
  const std::string dir = std::string("/sys/bus/pci/devices/") + bus + "/";
  if (FILE *f = fopen((dir + "numa_node").c_str(), "r")) {
    if (fscanf(f, "%d", &p.node) != 1) p.node = -1;
    fclose(f);
  }
  if (p.node < 0) return p; // no locality reported: leave placement to the OS
  if (FILE *f = fopen((dir + "local_cpulist").c_str(), "r")) {
    char buf[4096] = {0};
    if (fgets(buf, sizeof buf, f)) p.has_cpus = parse_cpulist(buf, &p.cpus);
    fclose(f);
  }
  return p;
}

// Bind the calling thread to the placement's CPUs (no-op when unknown).
inline void bind_thread(const DevicePlacement &p) {
  if (p.has_cpus) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), &p.cpus);
}

// Scoped: the calling thread runs on the GPU-local CPUs and allocates from
// the GPU's node (MPOL_PREFERRED) so pinned buffers created inside the scope
// are first touched there; both are restored on exit.
class NodeScope {
 public:
  explicit NodeScope(const DevicePlacement &p) {
    if (p.node < 0) return;
    active_ = pthread_getaffinity_np(pthread_self(), sizeof(cpu_set_t), &saved_) == 0;
    if (active_) bind_thread(p);
    unsigned long mask[16] = {0};
    if (p.node < static_cast<int>(8 * sizeof mask)) {
      mask[p.node / (8 * sizeof(unsigned long))] |= 1ul << (p.node % (8 * sizeof(unsigned long)));
      constexpr int kMpolPreferred = 1;
      policy_ = syscall(SYS_set_mempolicy, kMpolPreferred, mask, 8 * sizeof mask) == 0;
    }
  }
  ~NodeScope() {
    if (policy_) syscall(SYS_set_mempolicy, 0 /* MPOL_DEFAULT */, nullptr, 0);
    if (active_) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), &saved_);
  }
  NodeScope(const NodeScope &) = delete;
  NodeScope &operator=(const NodeScope &) = delete;

 private:
  bool active_ = false, policy_ = false;
  cpu_set_t saved_;
};

} // namespace pc
