// DIVUQ1 container ingest / egress (io.py:43-134).
//
// Layout (io.py:3-5): one ASCII header line
//   "DIVUQ1 <nx> <ny> <dx> <dy> <n_members>\n"
// then n_members blocks, each the u-plane then the v-plane as nx*ny
// little-endian float32, row-major.  That payload IS the (M, 2, N) member-major
// fp32 layout the ensemble kernels read, so ingest is a straight copy:
// file -> pinned staging (double-buffered) -> HBM, with the read of chunk i+1
// overlapping the host->device copy of chunk i.  Header reals are written with
// Python repr's shortest round-trip rules so files are byte-identical to the
// reference's writer (io.py:38-55).
#pragma once

#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <condition_variable>
#include <functional>
#include <thread>
#include <vector>

namespace divuq {
namespace io {

constexpr int kFormatError = -20;   // io.FormatError
constexpr int kLengthError = -21;   // io.LengthError
constexpr int kOsError = -22;       // OSError
constexpr int kDataError = -23;     // io.DataError (non-finite payload)

// Python repr(float) (shortest round-trip digits; exponent form when the
// decimal exponent is < -4 or >= 16), and io.py:38-40's integer shortcut.
inline std::string py_repr(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x < 0 ? "-inf" : "inf";
  if (x == std::floor(x) && std::fabs(x) < 9007199254740992.0) {  // io._fmt: repr(int(x))
    char b[32];
    std::snprintf(b, sizeof b, "%lld", static_cast<long long>(x));
    return b;
  }
  char buf[64];
  int p = 1;
  for (; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*e", p - 1, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  // buf = [-]d[.ddd]e[+-]XX
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const size_t e = s.find('e');
  std::string digits = s.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int ex = std::atoi(s.c_str() + e + 1);
  std::string out;
  if (ex >= -4 && ex < 16) {
    const int decpt = ex + 1;
    if (decpt <= 0) {
      out = "0." + std::string(size_t(-decpt), '0') + digits;
    } else if (decpt >= int(digits.size())) {
      out = digits + std::string(size_t(decpt - int(digits.size())), '0') + ".0";
    } else {
      out = digits.substr(0, size_t(decpt)) + "." + digits.substr(size_t(decpt));
    }
  } else {
    out = digits.substr(0, 1);
    if (digits.size() > 1) out += "." + digits.substr(1);
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return neg ? "-" + out : out;
}

struct Header {
  int64_t nx, ny, members;
  double dx, dy;
  int64_t offset;  // payload byte offset
};

// Python int()/float() accept single underscores between digits ("1_000")
inline bool strip_underscores(const std::string& t, std::string* out) {
  out->clear();
  for (size_t i = 0; i < t.size(); ++i) {
    if (t[i] != '_') { out->push_back(t[i]); continue; }
    if (i == 0 || i + 1 == t.size() || !std::isdigit((unsigned char)t[i - 1]) ||
        !std::isdigit((unsigned char)t[i + 1]))
      return false;
  }
  return true;
}

inline bool parse_int(const std::string& tok, int64_t* v) {
  std::string t;
  if (tok.empty() || !strip_underscores(tok, &t)) return false;
  char* end = nullptr;
  errno = 0;
  const long long x = std::strtoll(t.c_str(), &end, 10);
  if (errno || *end) return false;
  *v = x;
  return true;
}

inline bool parse_real(const std::string& tok, double* v) {
  // Python float() takes no hex literals and no nan payloads
  std::string t;
  if (tok.empty() || tok.find_first_of("xX(") != std::string::npos || !strip_underscores(tok, &t))
    return false;
  char* end = nullptr;
  const double x = std::strtod(t.c_str(), &end);
  if (*end) return false;
  *v = x;
  return true;
}

// io.py:58-86: header parse + validation + payload length check
inline int read_header(const char* path, Header* h) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return kOsError;
  std::string line;
  int c;
  while ((c = std::fgetc(f)) != EOF) {
    line.push_back(char(c));
    if (c == '\n') break;
  }
  h->offset = int64_t(line.size());
  if (std::fseek(f, 0, SEEK_END) != 0) { std::fclose(f); return kOsError; }
  const long long total = std::ftell(f);
  std::fclose(f);
  std::vector<std::string> parts;
  std::string cur;
  for (char ch : line) {
    if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f') {
      if (!cur.empty()) parts.push_back(cur), cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  if (!cur.empty()) parts.push_back(cur);
  if (parts.size() != 6 || parts[0] != "DIVUQ1") return kFormatError;
  if (!parse_int(parts[1], &h->nx) || !parse_int(parts[2], &h->ny) || !parse_real(parts[3], &h->dx) ||
      !parse_real(parts[4], &h->dy) || !parse_int(parts[5], &h->members))
    return kFormatError;
  if (h->members < 1) return kFormatError;
  if (h->nx < 2 || h->ny < 2 || !(h->dx > 0) || !(h->dy > 0)) return kFormatError;  // UniformGrid2
  long long expected = 0;  // members * 2 * nx * ny * 4; an overflowing header cannot match any file
  if (__builtin_mul_overflow(h->members, h->nx, &expected) ||
      __builtin_mul_overflow(expected, h->ny, &expected) ||
      __builtin_mul_overflow(expected, 8LL, &expected) || total - h->offset != expected)
    return kLengthError;
  return 0;
}

// Process-wide ring of pinned staging buffers for the HBM ingest (portable
// across devices).  Pinning is paid once, not per file.
struct Staging {
  static constexpr int kBuffers = 3;
  static constexpr int64_t kChunk = int64_t(32) << 20;  // bytes per buffer
  std::mutex mu;
  char* buf[kBuffers] = {};
  int ensure() {
    for (auto& p : buf)
      if (!p) {
        const cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), size_t(kChunk),
                                            cudaHostAllocPortable);
        if (e != cudaSuccess) { p = nullptr; return int(e); }
      }
    return 0;
  }
};
inline Staging& staging() {
  static Staging* s = new Staging();  // never destroyed: no CUDA calls at static teardown
  return *s;
}

// Persistent host workers for the parallel page-cache reads and staging
// copies: spawning 16 std::threads per 32 MB chunk cost ~0.3 ms per chunk.
// run(n, fn) executes fn(0..n-1) spread over the caller and the workers and
// returns when all are done; calls are serialised.  Workers are never joined (detached at
// process exit with the pool, which is never destroyed).
class HostPool {
 public:
  static constexpr int kMax = 16;
  static HostPool& get() {
    // a fork()ed child has none of the parent's workers: it builds its own
    // pool (the parent's copy is leaked), so run() never waits on ghosts
    static std::mutex mu;
    static HostPool* p = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (!p || owner != ::getpid()) {
      p = new HostPool();
      owner = ::getpid();
    }
    return *p;
  }
  int size() const { return n_; }
  template <typename F>
  void run(int n, F&& fn) {
    if (n <= 1 || n_ == 1) {
      for (int t = 0; t < n; ++t) fn(t);
      return;
    }
    std::lock_guard<std::mutex> serial(call_mu_);
    const int workers = std::min(n, n_);
    // worker w runs tasks w, w + workers, ... so any n is covered
    std::function<void(int)> task = [&, workers](int w) {
      for (int t = w; t < n; t += workers) fn(t);
    };
    {
      std::lock_guard<std::mutex> lk(mu_);
      task_ = &task;
      ntask_ = workers;
      pending_ = workers - 1;
      ++gen_;
    }
    cv_.notify_all();
    task(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    task_ = nullptr;
  }

 private:
  HostPool() {
    n_ = int(std::min<unsigned>(kMax, std::max(1u, std::thread::hardware_concurrency())));
    for (int id = 1; id < n_; ++id) std::thread([this, id] { loop(id); }).detach();
  }
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* task;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= ntask_) continue;
        task = task_;
      }
      (*task)(id);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_ = 1;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  int ntask_ = 0, pending_ = 0;
  const std::function<void(int)>* task_ = nullptr;
};

// read len bytes at file offset off into dst with up to 16 concurrent
// pread()s, one per host core (page-cache copies are per-thread memcpy-bound)
inline bool pread_span(int fd, char* dst, int64_t len, int64_t off) {
  while (len > 0) {
    const ssize_t r = ::pread(fd, dst, size_t(len), off_t(off));
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      return false;
    }
    dst += r; off += r; len -= r;
  }
  return true;
}

inline int io_threads() {   // DIVUQ_IO_THREADS (1..16, default 16)
  static const int v = [] {
    const char* e = std::getenv("DIVUQ_IO_THREADS");
    const int n = e ? std::atoi(e) : 16;
    return n < 1 ? 1 : (n > 16 ? 16 : n);
  }();
  return v;
}

inline bool pread_parallel(int fd, char* dst, int64_t len, int64_t off) {
  constexpr int kMaxThreads = 16;
  const int64_t kSlice = int64_t(1) << 20;
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<int64_t>(std::min<int64_t>(io_threads(), hw), (len + kSlice - 1) / kSlice));
  if (nt <= 1) return pread_span(fd, dst, len, off);
  const int64_t per = (len + nt - 1) / nt;
  bool ok[kMaxThreads] = {};
  HostPool::get().run(nt, [&](int t) {
    const int64_t a = t * per, n = std::min(per, len - a);
    ok[t] = n <= 0 || pread_span(fd, dst + a, n, off + a);
  });
  bool all = true;
  for (int t = 0; t < nt; ++t) all = all && ok[t];
  return all;
}

}  // namespace io
}  // namespace divuq
