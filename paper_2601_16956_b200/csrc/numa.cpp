// NUMA placement (see numa.hpp).
#include "numa.hpp"

#include <cuda_runtime.h>
#include <pthread.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>

namespace tsb {

namespace {
constexpr int kMpolDefault = 0, kMpolPreferred = 1;
constexpr unsigned long kMaxNode = 16 * 8 * sizeof(unsigned long);

std::string read_line(const std::string& path) {
  std::ifstream f(path);
  std::string s;
  if (f) std::getline(f, s);
  return s;
}

int node_count() {
  const std::string s = read_line("/sys/devices/system/node/online");  // e.g. "0-1"
  if (s.empty()) return 1;
  cpu_set_t set;  // reuse the list parser: a node list has the same syntax
  if (!parse_cpulist(s, &set)) return 1;
  return CPU_COUNT(&set);
}

long set_mempolicy(int mode, const unsigned long* mask, unsigned long maxnode) {
  return syscall(SYS_set_mempolicy, mode, mask, maxnode);
}
long get_mempolicy(int* mode, unsigned long* mask, unsigned long maxnode) {
  return syscall(SYS_get_mempolicy, mode, mask, maxnode, nullptr, 0ul);
}
}  // namespace

bool parse_cpulist(const std::string& s, cpu_set_t* out) {
  CPU_ZERO(out);
  size_t i = 0;
  bool any = false;
  while (i < s.size()) {
    if (s[i] == ',' || std::isspace(static_cast<unsigned char>(s[i]))) {
      ++i;
      continue;
    }
    if (!std::isdigit(static_cast<unsigned char>(s[i]))) return false;
    long a = 0;
    while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) a = a * 10 + (s[i++] - '0');
    long b = a;
    if (i < s.size() && s[i] == '-') {
      ++i;
      if (i >= s.size() || !std::isdigit(static_cast<unsigned char>(s[i]))) return false;
      b = 0;
      while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) b = b * 10 + (s[i++] - '0');
    }
    if (b < a || b >= CPU_SETSIZE) return false;
    for (long c = a; c <= b; ++c) CPU_SET(static_cast<int>(c), out);
    any = true;
  }
  return any;
}

numa_place numa_for_device(int device) {
  numa_place p;
  CPU_ZERO(&p.cpus);
  if (std::getenv("TS_NO_NUMA") || node_count() < 2) return p;
  char bus[32] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return p;
  }
  std::string id(bus);
  for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  const std::string nn = read_line("/sys/bus/pci/devices/" + id + "/numa_node");
  if (nn.empty()) return p;
  const int node = std::atoi(nn.c_str());
  if (node < 0 || static_cast<unsigned long>(node) >= kMaxNode) return p;
  cpu_set_t node_cpus, allowed;
  if (!parse_cpulist(read_line("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"), &node_cpus))
    return p;
  if (sched_getaffinity(0, sizeof allowed, &allowed) != 0) return p;
  CPU_AND(&p.cpus, &node_cpus, &allowed);
  if (CPU_COUNT(&p.cpus) == 0) return p;  // the process may not run there (cpuset)
  p.node = node;
  p.valid = true;
  return p;
}

void numa_bind_thread(const numa_place& p) {
  if (!p.valid) return;
  pthread_setaffinity_np(pthread_self(), sizeof p.cpus, &p.cpus);  // best effort
  unsigned long mask[16] = {};
  mask[p.node / (8 * sizeof(unsigned long))] |= 1ul << (p.node % (8 * sizeof(unsigned long)));
  set_mempolicy(kMpolPreferred, mask, kMaxNode);
}

numa_prefer_scope::numa_prefer_scope(const numa_place& p) {
  if (!p.valid) return;
  if (get_mempolicy(&old_mode_, old_mask_, kMaxNode) != 0) return;
  unsigned long mask[16] = {};
  mask[p.node / (8 * sizeof(unsigned long))] |= 1ul << (p.node % (8 * sizeof(unsigned long)));
  active_ = set_mempolicy(kMpolPreferred, mask, kMaxNode) == 0;
}

numa_prefer_scope::~numa_prefer_scope() {
  if (!active_) return;
  if (old_mode_ == kMpolDefault) set_mempolicy(kMpolDefault, nullptr, 0);
  else set_mempolicy(old_mode_, old_mask_, kMaxNode);
}

}  // namespace tsb
