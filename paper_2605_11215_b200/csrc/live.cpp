// librcv.so — node-local liveness for the real-kill commit (host code).
//
// Every rank maps one POSIX shared-memory segment.  A native thread per rank
// stamps the rank's heartbeat slot every period (CLOCK_MONOTONIC, shared by
// every process of the node) and declares a peer dead when its stamp is
// older than the deadline or its process is gone: the peer's bit is OR-ed
// into the segment's dead word.  The segment is registered with CUDA as
// mapped host memory, so the barrier kernels of every GPU read that word
// while they wait and stop waiting for a dead peer within microseconds of
// the declaration — detection is bounded by the deadline (milliseconds), not
// by a barrier timeout.
//
// Agreement (comm.py:129-172's "every survivor repairs the same membership"):
// the replicated control plane polls at fixed points of its step; poll `seq`
// is decided by the first rank that reaches it, which compare-and-swaps the
// dead word's current value into the segment's decision ring.  Every rank
// that reaches `seq` later adopts that value, so all survivors act on the same
// failed set at the same point of the protocol without waiting for each other.

#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <signal.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <string>
#include <thread>

#include "../../include/rcv.h"

extern "C" int rcv_set_error(int code, const char *msg);

namespace {

constexpr uint64_t kMagic = 0x7263762d6c697665ull;  // "rcv-live"
constexpr int kMaxRanks = 32;
constexpr int kRing = 256;

struct alignas(64) Slot {
  std::atomic<uint64_t> beat_ns;      // last heartbeat
  std::atomic<uint64_t> dead_ns;      // when a watcher first declared it dead
  std::atomic<uint64_t> kill_ns;      // benchmark: when it killed itself
  std::atomic<int32_t> pid;
};

struct Segment {
  std::atomic<uint64_t> magic;
  std::atomic<uint32_t> world;
  alignas(64) std::atomic<uint32_t> dead;  // the device-visible dead word
  alignas(64) Slot slot[kMaxRanks];
  std::atomic<uint64_t> decision[kRing];     // (seq << 32) | mask
  std::atomic<uint64_t> decision_ns[kRing];  // when it was decided
};

uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

bool pid_gone(int32_t pid) {
  if (pid <= 0) return false;
  if (kill(pid, 0) == -1 && errno == ESRCH) return true;
  // a SIGKILLed child is a zombie until its parent reaps it
  char path[64];
  snprintf(path, sizeof path, "/proc/%d/stat", pid);
  FILE *f = fopen(path, "r");
  if (!f) return true;
  char buf[256];
  const size_t n = fread(buf, 1, sizeof buf - 1, f);
  fclose(f);
  buf[n] = 0;
  const char *rp = strrchr(buf, ')');
  return rp && rp[1] == ' ' && (rp[2] == 'Z' || rp[2] == 'X');
}

int err(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return rcv_set_error(code, buf);
}

}  // namespace

struct rcv_liveness {
  Segment *seg = nullptr;
  size_t bytes = 0;
  std::string name;
  int rank = 0, world = 0;
  uint64_t period_ns = 0, deadline_ns = 0;
  uint32_t *dev_dead = nullptr;
  bool registered = false;
  std::atomic<bool> stop{false};
  std::thread th;

  void watch() {
    uint64_t pid_check_at = 0;
    while (!stop.load(std::memory_order_relaxed)) {
      const uint64_t t = now_ns();
      seg->slot[rank].beat_ns.store(t, std::memory_order_release);
      const bool check_pids = t >= pid_check_at;
      if (check_pids) pid_check_at = t + 4 * period_ns;
      const uint32_t dead = seg->dead.load(std::memory_order_acquire);
      for (int r = 0; r < world; ++r) {
        if (r == rank || ((dead >> r) & 1u)) continue;
        const uint64_t b = seg->slot[r].beat_ns.load(std::memory_order_acquire);
        const bool stale = b != 0 && t > b && t - b > deadline_ns;
        if (stale || (check_pids && pid_gone(seg->slot[r].pid.load()))) {
          uint64_t zero = 0;
          seg->slot[r].dead_ns.compare_exchange_strong(zero, t);
          seg->dead.fetch_or(1u << r, std::memory_order_acq_rel);
        }
      }
      timespec ts{(time_t)(period_ns / 1000000000ull), (long)(period_ns % 1000000000ull)};
      nanosleep(&ts, nullptr);
    }
  }
};

extern "C" {

int rcv_liveness_create(const char *name, int rank, int world, uint64_t period_ns,
                        uint64_t deadline_ns, rcv_liveness **out) {
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return err(RCV_ERANGE, "liveness: rank %d of %d (at most %d ranks)", rank, world, kMaxRanks);
  if (!name || name[0] != '/') return err(RCV_EINVAL, "liveness: shm name must start with '/'");
  if (period_ns == 0 || deadline_ns < 2 * period_ns)
    return err(RCV_EINVAL, "liveness: deadline must be at least two periods");
  const long page = sysconf(_SC_PAGESIZE);
  const size_t bytes = (sizeof(Segment) + page - 1) / page * page;
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return err(RCV_EINVAL, "liveness: shm_open(%s): %s", name, strerror(errno));
  if (ftruncate(fd, (off_t)bytes) != 0) {
    close(fd);
    return err(RCV_EINVAL, "liveness: ftruncate: %s", strerror(errno));
  }
  void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return err(RCV_EINVAL, "liveness: mmap: %s", strerror(errno));
  rcv_liveness *lv = new rcv_liveness();
  lv->seg = (Segment *)p;
  lv->bytes = bytes;
  lv->name = name;
  lv->rank = rank;
  lv->world = world;
  lv->period_ns = period_ns;
  lv->deadline_ns = deadline_ns;
  // a fresh segment is zero-filled; the first rank stamps it
  uint64_t zero = 0;
  lv->seg->magic.compare_exchange_strong(zero, kMagic);
  lv->seg->world.store((uint32_t)world);
  lv->seg->slot[rank].pid.store((int32_t)getpid());
  lv->seg->slot[rank].beat_ns.store(now_ns());
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess) {
    cudaGetLastError();
    n_dev = 0;
  }
  if (n_dev == 0) {  // host-only (the CPU test box): heartbeat and agreement, no device word
    lv->th = std::thread([lv]() { lv->watch(); });
    *out = lv;
    return RCV_OK;
  }
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    delete lv;
    return err(RCV_ECUDA, "liveness: cudaHostRegister: %s", cudaGetErrorString(e));
  }
  lv->registered = true;
  void *dp = nullptr;
  e = cudaHostGetDevicePointer(&dp, (void *)&lv->seg->dead, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaHostUnregister(p);
    munmap(p, bytes);
    delete lv;
    return err(RCV_ECUDA, "liveness: cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  }
  lv->dev_dead = (uint32_t *)dp;
  lv->th = std::thread([lv]() { lv->watch(); });
  *out = lv;
  return RCV_OK;
}

int rcv_liveness_dead_word(rcv_liveness *lv, const uint32_t **device_ptr, uint32_t *now) {
  if (device_ptr) *device_ptr = lv->dev_dead;
  if (now) *now = lv->seg->dead.load(std::memory_order_acquire);
  return RCV_OK;
}

int rcv_liveness_decide(rcv_liveness *lv, uint64_t seq, uint32_t *mask_out, uint64_t *decided_ns) {
  if (seq == 0 || seq >= (1ull << 32)) return err(RCV_ERANGE, "liveness: poll sequence %llu", (unsigned long long)seq);
  std::atomic<uint64_t> &d = lv->seg->decision[seq % kRing];
  uint64_t cur = d.load(std::memory_order_acquire);
  for (;;) {
    if ((cur >> 32) == seq) break;
    if ((cur >> 32) > seq)
      return err(RCV_EINVAL, "liveness: poll %llu was overtaken (ranks drifted %d polls apart)",
                 (unsigned long long)seq, kRing);
    const uint64_t want = (seq << 32) | lv->seg->dead.load(std::memory_order_acquire);
    if (d.compare_exchange_weak(cur, want, std::memory_order_acq_rel)) {
      lv->seg->decision_ns[seq % kRing].store(now_ns(), std::memory_order_release);
      cur = want;
      break;
    }
  }
  *mask_out = (uint32_t)(cur & 0xffffffffu);
  if (decided_ns) *decided_ns = lv->seg->decision_ns[seq % kRing].load(std::memory_order_acquire);
  return RCV_OK;
}

int rcv_liveness_stats(rcv_liveness *lv, int rank, uint64_t *beat_ns, uint64_t *dead_ns,
                       uint64_t *kill_ns, uint64_t *now) {
  if (rank < 0 || rank >= lv->world) return err(RCV_ERANGE, "liveness: rank %d", rank);
  const Slot &s = lv->seg->slot[rank];
  if (beat_ns) *beat_ns = s.beat_ns.load();
  if (dead_ns) *dead_ns = s.dead_ns.load();
  if (kill_ns) *kill_ns = s.kill_ns.load();
  if (now) *now = now_ns();
  return RCV_OK;
}

int rcv_liveness_note_kill(rcv_liveness *lv) {
  lv->seg->slot[lv->rank].kill_ns.store(now_ns(), std::memory_order_release);
  return RCV_OK;
}

int rcv_liveness_destroy(rcv_liveness *lv, int unlink_name) {
  if (!lv) return RCV_OK;
  lv->stop.store(true);
  if (lv->th.joinable()) lv->th.join();
  if (lv->registered) cudaHostUnregister(lv->seg);
  munmap(lv->seg, lv->bytes);
  if (unlink_name) shm_unlink(lv->name.c_str());
  delete lv;
  return RCV_OK;
}

}  // extern "C"
