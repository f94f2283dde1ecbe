// Host-side rank coordination for the replay engine: a one-box shared-memory
// coordinator (POSIX shm + per-rank epoch counters). Every operation is a
// collective call: all ranks invoke the same sequence. Waits spin briefly,
// then yield, and give up with Error(IoFailure) after the timeout so a dead
// rank can never hang the others.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>

#include "lagom/b200.hpp"
#include "lagom/error.hpp"

namespace lagom::b200 {

namespace {

constexpr int kMaxRanks = 8;
constexpr std::uint64_t kMagic = 0x4c41474f4d534831ull;  // "LAGOMSH1"
constexpr std::size_t kPayload = 1 << 20;                // per-rank mailbox bytes

struct alignas(128) Counter {
  std::atomic<std::uint64_t> v;
};

struct Segment {
  std::atomic<std::uint64_t> magic;
  std::int32_t nranks;
  Counter arrive[kMaxRanks];
  alignas(128) unsigned char mailbox[kMaxRanks][kPayload];
};

class SingleCoordinator final : public Coordinator {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  void barrier() override {}
  void broadcast(void*, std::size_t, int) override {}
  void allgather(const void* in, std::size_t bytes, void* out) override {
    if (out != in) std::memcpy(out, in, bytes);
  }
  void allreduce_max(double*, std::size_t) override {}
};

class ShmCoordinator final : public Coordinator {
 public:
  ShmCoordinator(const std::string& name, int rank, int size, double timeout_s)
      : name_(name[0] == '/' ? name : "/" + name), rank_(rank), size_(size), timeout_s_(timeout_s) {
    if (size < 1 || size > kMaxRanks || rank < 0 || rank >= size)
      throw Error(ErrorCode::InvalidInput, "coordinator", "rank/size out of range");
    const std::size_t bytes = sizeof(Segment);
    const auto t0 = std::chrono::steady_clock::now();
    int fd = -1;
    if (rank == 0) {
      shm_unlink(name_.c_str());
      fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, static_cast<off_t>(bytes)) != 0)
        throw Error(ErrorCode::IoFailure, name_, "cannot create shared-memory segment");
    } else {
      for (;;) {
        fd = shm_open(name_.c_str(), O_RDWR, 0600);
        if (fd >= 0) {
          struct stat st{};
          if (fstat(fd, &st) == 0 && static_cast<std::size_t>(st.st_size) >= bytes) break;
          close(fd);
          fd = -1;
        }
        check_deadline(t0, "attach");
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(ErrorCode::IoFailure, name_, "mmap failed");
    seg_ = static_cast<Segment*>(p);
    if (rank == 0) {
      seg_->nranks = size;
      for (auto& c : seg_->arrive) c.v.store(0, std::memory_order_relaxed);
      seg_->magic.store(kMagic, std::memory_order_release);
    } else {
      while (seg_->magic.load(std::memory_order_acquire) != kMagic) {
        check_deadline(t0, "attach");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (seg_->nranks != size) throw Error(ErrorCode::InvalidInput, name_, "rank count mismatch");
    }
    barrier();
    if (rank == 0) shm_unlink(name_.c_str());  // everyone is attached
  }

  ~ShmCoordinator() override {
    if (seg_) munmap(seg_, sizeof(Segment));
  }

  int rank() const override { return rank_; }
  int size() const override { return size_; }

  void barrier() override {
    const std::uint64_t e = ++epoch_;
    seg_->arrive[rank_].v.store(e, std::memory_order_release);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < size_; ++r) {
      unsigned spins = 0;
      while (seg_->arrive[r].v.load(std::memory_order_acquire) < e) {
        if (++spins < 4096) {
          __builtin_ia32_pause();
        } else {
          sched_yield();
          if ((spins & 1023) == 0) check_deadline(t0, "barrier");
        }
      }
    }
  }

  void broadcast(void* buf, std::size_t bytes, int root) override {
    check_size(bytes);
    barrier();  // previous readers of the root's mailbox are done
    if (rank_ == root) std::memcpy(seg_->mailbox[root], buf, bytes);
    barrier();
    if (rank_ != root) std::memcpy(buf, seg_->mailbox[root], bytes);
  }

  void allgather(const void* in, std::size_t bytes, void* out) override {
    check_size(bytes);
    barrier();
    std::memcpy(seg_->mailbox[rank_], in, bytes);
    barrier();
    for (int r = 0; r < size_; ++r)
      std::memcpy(static_cast<unsigned char*>(out) + r * bytes, seg_->mailbox[r], bytes);
  }

  void allreduce_max(double* v, std::size_t n) override {
    const std::size_t bytes = n * sizeof(double);
    check_size(bytes);
    barrier();
    std::memcpy(seg_->mailbox[rank_], v, bytes);
    barrier();
    for (int r = 0; r < size_; ++r) {
      const double* other = reinterpret_cast<const double*>(seg_->mailbox[r]);
      for (std::size_t i = 0; i < n; ++i) v[i] = other[i] > v[i] ? other[i] : v[i];
    }
  }

 private:
  void check_size(std::size_t bytes) const {
    if (bytes > kPayload) throw Error(ErrorCode::InvalidInput, "coordinator", "payload too large");
  }
  void check_deadline(std::chrono::steady_clock::time_point t0, const char* what) const {
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (s > timeout_s_)
      throw Error(ErrorCode::IoFailure, name_, std::string("coordinator timeout in ") + what);
  }

  std::string name_;
  int rank_, size_;
  double timeout_s_;
  Segment* seg_ = nullptr;
  std::uint64_t epoch_ = 0;
};

}  // namespace

std::unique_ptr<Coordinator> make_single_coordinator() { return std::make_unique<SingleCoordinator>(); }

std::unique_ptr<Coordinator> make_shm_coordinator(const std::string& name, int rank, int size,
                                                  double timeout_s) {
  if (size == 1) return make_single_coordinator();
  return std::make_unique<ShmCoordinator>(name, rank, size, timeout_s);
}

}  // namespace lagom::b200
