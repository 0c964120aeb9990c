// NUMA placement of a GPU's host-side snapshot work (B200-side addition).
//
// On a multi-socket 8-GPU node each GPU's PCIe link hangs off one socket.
// D2H into pinned memory / file pages on the other socket crosses the socket
// interconnect. The engine therefore binds its threads (copier, completer,
// workers: they first-touch file pages and hash them) to the GPU's node and
// allocates the pinned pool with that node preferred. No libnuma: sysfs +
// raw syscalls. A no-op on single-node hosts or when sysfs says -1.
#pragma once

#include <sched.h>

#include <string>

namespace tsb {

struct numa_place {
  int node = -1;      // GPU's NUMA node, -1 = unknown / single node
  cpu_set_t cpus;     // that node's CPUs ∩ this process's allowed set
  bool valid = false;
};

// Node of `device` from /sys/bus/pci/devices/<bus id>/numa_node, when the host
// has more than one node.
numa_place numa_for_device(int device);
// Parses a sysfs cpulist ("0-3,8,10-11") into a set; false on garbage.
bool parse_cpulist(const std::string& s, cpu_set_t* out);
// Binds the calling thread (CPU affinity + preferred memory node).
void numa_bind_thread(const numa_place& p);
// RAII: prefer `p.node` for allocations made by this thread while alive.
class numa_prefer_scope {
 public:
  explicit numa_prefer_scope(const numa_place& p);
  ~numa_prefer_scope();

 private:
  bool active_ = false;
  int old_mode_ = 0;
  unsigned long old_mask_[16] = {};
};

}  // namespace tsb
