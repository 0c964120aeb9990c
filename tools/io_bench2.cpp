// Variant of io_bench: several files written concurrently through shared mappings.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/dev/shm";
  const size_t per = (argc > 2 ? std::stoul(argv[2]) : 4ul) << 30, chunk = 64 << 20;
  const int nf = 2;
  std::vector<char> src(per);
  std::memset(src.data(), 7, per);
  for (int variant = 0; variant < 4; ++variant) {
    for (int T : {4, 8, 16}) {
      std::vector<int> fds(nf);
      std::vector<char*> maps(nf);
      for (int f = 0; f < nf; ++f) {
        fds[f] = open((dir + "/iob2_" + std::to_string(f)).c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
        if (ftruncate(fds[f], per)) return 1;
        int flags = MAP_SHARED | (variant == 1 ? MAP_POPULATE : 0);
        maps[f] = static_cast<char*>(mmap(nullptr, per, PROT_READ | PROT_WRITE, flags, fds[f], 0));
        if (variant == 3) madvise(maps[f], per, MADV_HUGEPAGE);
      }
      double t0 = now();
      std::vector<std::thread> th;
      for (int k = 0; k < T; ++k)
        th.emplace_back([&, k] {
          const int f = k % nf, kk = k / nf, TT = T / nf;
          for (size_t off = kk * chunk; off < per; off += TT * chunk) {
            if (variant == 2) madvise(maps[f] + off, chunk, MADV_POPULATE_WRITE);
            std::memcpy(maps[f] + off, src.data() + off, chunk);
          }
        });
      for (auto& x : th) x.join();
      const double t = now() - t0;
      const char* names[] = {"mmap", "mmap_populate(incl)", "madv_populate_write", "mmap_hugepage"};
      std::printf("{\"files\": %d, \"variant\": \"%s\", \"threads\": %d, \"GBps\": %.2f}\n", nf, names[variant], T,
                  nf * per / t / 1e9);
      std::fflush(stdout);
      for (int f = 0; f < nf; ++f) {
        munmap(maps[f], per);
        close(fds[f]);
        unlink((dir + "/iob2_" + std::to_string(f)).c_str());
      }
    }
  }
  return 0;
}
