// CPU self-test of the raw-syscall io_uring wrapper (csrc/uring.cpp): writes
// a file through uring_pwrite in 4 KiB..1 MiB pieces, reads it back through
// uring_pread, compares with the source, and checks the short-read contract
// at end of file. Prints "ok <ops>" or "skip" (no io_uring here).
#include <fcntl.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "uring.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  if (!tsb::uring_available()) {
    std::puts("skip");
    return 0;
  }
  const size_t n = (24u << 20) + 12345;
  std::vector<unsigned char> src(n), dst(n + 8192, 0xee);
  for (size_t i = 0; i < n; ++i) src[i] = static_cast<unsigned char>((i * 2654435761u) >> 11);
  const int fd = ::open(argv[1], O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return 3;
  for (uint64_t piece : {4096ull, 65536ull, 1ull << 20}) {
    if (tsb::uring_pwrite(fd, src.data(), n, 0, piece) != static_cast<int64_t>(n)) return 4;
    std::memset(dst.data(), 0, dst.size());
    if (tsb::uring_pread(fd, dst.data(), n, 0, piece) != static_cast<int64_t>(n)) return 5;
    if (std::memcmp(src.data(), dst.data(), n) != 0) return 6;
    // a read past the end is short, in order from the start
    if (tsb::uring_pread(fd, dst.data(), n + 8192, 0, piece) != static_cast<int64_t>(n)) return 7;
    // an offset write lands where it should
    if (tsb::uring_pwrite(fd, src.data() + 100, 5000, 7, piece) != 5000) return 8;
    if (::pread(fd, dst.data(), 5000, 7) != 5000 || std::memcmp(dst.data(), src.data() + 100, 5000) != 0) return 9;
    if (tsb::uring_pwrite(fd, src.data() + 7, 5000, 7, piece) != 5000) return 10;  // restore
  }
  ::close(fd);
  ::unlink(argv[1]);
  std::printf("ok %llu\n", static_cast<unsigned long long>(tsb::uring_ops()));
  return 0;
}
