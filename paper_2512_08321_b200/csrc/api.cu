// api.cu — the C-ABI (include/crtg.h): argument checks, workspace planning and the
// stream-ordered launch sequence of the complex Ozaki-II pipeline.
//
// Pipeline of crtg_gemm_complex (reference emulate.py:193-240):
//   K1   scaling: fast (row pairwise / column sequential sums of squares) or
//        accurate (bound operands + tcgen05 bound GEMM + row/col maxima)
//   K2   quantize + residues of A, packed for tcgen05 (once)
//   for each column block of B (n_block, bitwise-neutral working-set bound):
//     K2 quantize + residues of the B block (transposed into K-major tiles)
//     K3 Karatsuba INT8 GEMMs for all N moduli, modular epilogue -> int8 planes
//     K4 CRT + inverse scaling -> C block
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/crtg.h"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

using namespace crtg;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_check(int err, const char* where) {
  if (err == 0) return CRTG_OK;
  return fail(CRTG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(cudaError_t(err)));
}

#define CRTG_TRY(expr, where)                    \
  do {                                           \
    const int _e = (expr);                       \
    if (_e) return cuda_check(_e, where);        \
  } while (0)

// ---- instrumentation: launch counter and per-stage CUDA-event timers ----
std::atomic<uint64_t> g_launches{0};
}  // namespace

void crtg::note_launches(int n) { g_launches += uint64_t(n); }

bool crtg::pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("CRTG_PDL");
    return !(v && *v && std::atoi(v) == 0);
  }();
  return on;
}

namespace {
std::mutex g_prof_mu;
bool g_prof_on = false;
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};
std::vector<ProfRec> g_prof;

struct StageTimer {
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  StageTimer(int st, cudaStream_t str) : stage(st), s(str) {
    if (g_prof_on) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~StageTimer() {
    if (a) {
      cudaEventRecord(b, s);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof.push_back({stage, a, b});
    }
  }
};

int sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n <= 0) n = 148;
  cache[dev] = n;
  return n;
}

// Wide 256 x 256 Karatsuba tiles for large products; the 128 x 256
// double-buffered kernel for short K loops (k < 8192) over fewer than 1024 wide
// tiles, where its TMEM double buffer hides the epilogue and its twice-as-many
// tiles fill the 148 SMs better (fast, N=14: 4096^3 3.15 vs 3.31 ms, 6144^3 8.73 vs
// 8.93, 8192^3 19.6 vs 19.4, 16384^3 162 vs 136; tools/small_ab.py).
// CRTG_GEMM=wide / one forces either kernel; all are bitwise identical.
bool wide_enabled(const GemmArgs& g) {
  static const int force = [] {
    const char* v = std::getenv("CRTG_GEMM");
    if (!v) return -1;
    const std::string s(v);
    return s == "wide" ? 1 : s == "one" ? 0 : -1;
  }();
  if (force >= 0) return force == 1;
  return int64_t(g.kb) * 128 >= 8192 || int64_t(g.mt / 2) * g.nt >= 1024;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// CRTG_GROUP_M: raster experiment knob (default 16 row tiles per column
// sweep; 8 / 32 read 20-30% more DRAM, profiles/r01_gemm_raster_experiment.json)
int run_gemm(int mode, const GemmArgs& g0, cudaStream_t s) {
  GemmArgs g = g0;
  static const int group_m = env_int("CRTG_GROUP_M", 0);
  g.group_m = group_m;
  if (wide_enabled(g) && (mode == EPI_KARATSUBA || mode == EPI_REAL) && (g.mt % 2) == 0 &&
      (g.mt0 % 2) == 0)
    return launch_gemm_wide(mode, g, sm_count(), s);
  return launch_gemm(mode, g, sm_count(), s);
}

// B's chain runs on the caller's stream (a side stream co-running with the
// power-capped GEMM lowered its clock: 190 vs 163 ms)
cudaStream_t side_stream(cudaStream_t s) { return s; }

// Small products (one column block, output 1024^2..4096^2) leave most SMs
// idle in the latency-bound statistics and residue kernels, so B's column
// statistics and residues run on a forked per-thread stream beside A's (joined
// before the GEMM).  Bitwise neutral: the two chains are independent.  Fast,
// N=14: 1024^3 245 -> 229 us, 2048^3 639 -> 620 us, 4096^3 3.08 -> 3.02 ms;
// below 1024^2 the extra events cost more than the overlap gains, at 8192^2
// it is noise (profiles/r01_fork_ab.jsonl).  CRTG_FORK=0 disables it.
cudaStream_t fork_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local std::map<int, cudaStream_t> streams;
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  // highest priority: B's chain (column statistics -> residues of B) is the
  // longer of the two and the block scheduler should not queue it behind A's
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t st = nullptr;
  cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi);
  streams[dev] = st;
  return st;
}

// graphed: the launch sequence is being captured (replays pay nothing for the
// extra events, so the fork pays below 1024^2 too)
bool fork_wanted(int64_t m_pad, int64_t n_pad, int64_t n, int64_t nb, bool graphed) {
  static const bool on = env_int("CRTG_FORK", 1) != 0;
  const int64_t out = m_pad * n_pad;
  return on && nb >= n && (graphed || out >= int64_t(1024) * 1024) &&
         out <= int64_t(4096) * 4096;
}

struct Events {
  std::vector<cudaEvent_t> ev;
  cudaEvent_t get() {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ev.push_back(e);
    return e;
  }
  ~Events() {
    for (auto e : ev) cudaEventDestroy(e);  // released once they complete
  }
};

int check_consts(const crtg_consts* K, int* n_out) {
  if (!K) return fail(CRTG_ERR_CONFIG, "modulus constants are required");
  const int n = K->num_moduli;
  if (n < 1 || n > CRTG_MAX_MODULI) return fail(CRTG_ERR_CONFIG, "num_moduli must be in 1..20");
  for (int l = 0; l < n; ++l)
    if (K->moduli[l] < 2 || K->moduli[l] > 256)
      return fail(CRTG_ERR_CONFIG, "modulus outside [2, 256]");
  *n_out = n;
  return CRTG_OK;
}

ModConst make_mod(int p) {
  ModConst c{};
  c.p = p;
  c.is_pow2 = (p & (p - 1)) == 0;
  int sh = 0;
  while ((2 << sh) <= p) ++sh;  // floor(log2 p)
  c.shift = sh;
  if (!c.is_pow2) {
    const unsigned __int128 num = (unsigned __int128)1 << (32 + sh);
    c.magic = uint32_t((num + p - 1) / p);
  }
  c.half = (p + 1) / 2;
  c.c16 = uint32_t((1u << 16) % p);
  c.c32 = uint32_t((uint64_t(1) << 32) % p);
  const int64_t q = ((int64_t(1) << 30) + p - 1) / p;
  c.bias = int32_t(q * p);
  c.neg_p = uint32_t(-p);
  c.h = uint32_t(p / 2);
  c.bias_h = uint32_t(c.bias) + c.h;
  c.nphase = 3;
  return c;
}

// smallest j in [1, p) with j^2 == -1 (mod p), or 0.  Exists iff p is odd (or
// 2) and every prime factor of p is 1 mod 4: then Z[i]/p splits and a complex
// product mod p is two independent products (U U', V V') instead of three.
int sqrt_minus_one(int p) {
  if (p % 2 == 0) return 0;
  for (int j = 1; j < p; ++j)
    if ((j * j + 1) % p == 0) return j;
  return 0;
}

int inv_mod(int a, int p) {
  for (int x = 1; x < p; ++x)
    if ((a * x) % p == 1) return x;
  return 0;
}

// CRTG_SPLIT=0 forces the 3-product Karatsuba form for every modulus (A/B
// experiments; the results are bit-identical either way)
bool split_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("CRTG_SPLIT");
    return !(v && v[0] == '0');
  }();
  return on;
}

// switch modulus l of the pipeline constants to the split (2-product) form
void make_split(ModConst& mc, ResConst& rc, int p) {
  const int j = sqrt_minus_one(p);
  if (j == 0) return;
  mc.nphase = 2;
  mc.inv2 = uint32_t(inv_mod(2, p));
  mc.inv2j = uint32_t(inv_mod((2 * j) % p, p));
  const int off = int(rc.off) % p;
  rc.split = 1;
  rc.gj = uint32_t(j);
  rc.gjn = uint32_t(p - j);
  rc.gku = uint32_t((p - (j * off) % p) % p);
  rc.gkv = uint32_t((p - ((p - j) * off) % p) % p);
  // direct U / V tables (residue.cu: res_uv)
  auto bytes_of = [&](uint32_t w, int i) { return (w >> (8 * i)) & 0xFFu; };
  auto scale_tab = [&](uint32_t w, int n, int jj) {
    uint32_t o = 0;
    for (int i = 0; i < n; ++i) o |= ((uint32_t(jj) * bytes_of(w, i)) % uint32_t(p)) << (8 * i);
    return o;
  };
  rc.uw0123 = scale_tab(rc.dw0123, 4, j);
  rc.uw45 = scale_tab(rc.dw45, 2, j);
  rc.vw0123 = scale_tab(rc.dw0123, 4, p - j);
  rc.vw45 = scale_tab(rc.dw45, 2, p - j);
  auto pow2_mod = [&](int e) {
    uint64_t t = 1 % uint64_t(p);
    for (int i = 0; i < e; ++i) t = (t * 2) % uint64_t(p);
    return int64_t(t);
  };
  auto kk = [&](int jj, int e) {  // (off - (1 + jj) 2^e) mod p
    const int64_t v = (int64_t(off) - (1 + jj) * pow2_mod(e)) % p;
    return uint32_t(v < 0 ? v + p : v);
  };
  rc.ku31 = kk(j, 31);
  rc.ku63 = kk(j, 63);
  rc.kuw = kk(j, 90);
  rc.kv31 = kk(p - j, 31);
  rc.kv63 = kk(p - j, 63);
  rc.kvw = kk(p - j, 90);
}

// residue-kernel constants of modulus p for the stored representative t - off
ResConst make_res(int p, uint32_t off) {
  ResConst rc{};
  const uint64_t P = uint64_t(p);
  const bool pow2 = (p & (p - 1)) == 0;
  int sh = 0;
  while ((2 << sh) <= p) ++sh;  // floor(log2 p)
  if (pow2) {
    rc.magic = uint32_t(uint64_t(1) << (32 - sh));  // umulhi(u, 2^(32-s)) = u >> s
    rc.shift = 0;
  } else {
    const unsigned __int128 num = (unsigned __int128)1 << (32 + sh);
    rc.magic = uint32_t((num + P - 1) / P);
    rc.shift = sh;
  }
  rc.neg_p = uint32_t(-p);
  rc.off = off;
  uint32_t cw[6];
  uint64_t c = 1 % P;
  for (int i = 0; i < 6; ++i) {
    cw[i] = uint32_t(c);  // < p <= 256
    c = (c << 16) % P;
  }
  rc.dw0123 = cw[0] | (cw[1] << 8) | (cw[2] << 16) | (cw[3] << 24);
  rc.dw45 = cw[4] | (cw[5] << 8);
  auto pow2_mod = [&](int e) {
    uint64_t t = 1 % P;
    for (int i = 0; i < e; ++i) t = (t * 2) % P;
    return t;
  };
  const uint64_t o = off % P;
  rc.k31 = uint32_t((o + P - pow2_mod(31)) % P);
  rc.k63 = uint32_t((o + P - pow2_mod(63)) % P);
  rc.kw = uint32_t((o + P - pow2_mod(90)) % P);
  rc.sum_k = uint32_t((P - o) % P);
  return rc;
}

// split = true: moduli with a square root of -1 use the 2-product form (the
// production pipeline); false keeps the reference's [re, im, re+im] planes for
// every modulus (the crtg_residues parity hook unpacks them)
DevConsts make_dev_uncached(const crtg_consts& K, bool split, bool uns);

// The complex pipeline's residues as UNSIGNED bytes t in [0, p) with u8 x u8
// tcgen05 products (instead of the signed t - 128): same e-planes, but the
// tensor cores draw less power on them (ZGEMM 16384^3: K3 -1.7%, DESIGN.md
// section 3).  The epilogue's single biased reduction needs every product below
// 2^30, i.e. (p - 1)^2 k_pad < 2^30: k_pad <= 16384; longer K keeps the signed
// encoding (|product| <= 128^2 k <= 2^30 up to k = 65536).  CRTG_U8=0 disables.
bool unsigned_residues(int64_t k) {
  static const bool on = env_int("CRTG_U8", 1) != 0;
  return on && round_up(k, 128) <= 16384;
}

// the constant tables take ~0.1 ms of host integer arithmetic to build (modular
// inverses, powers, square roots of -1); small calls would pay that every time,
// so the last few (constants, split) pairs are cached per thread
DevConsts make_dev(const crtg_consts& K, bool split = true, bool uns = false) {
  struct Entry {
    crtg_consts key;
    bool split, uns;
    DevConsts val;
  };
  static thread_local std::vector<Entry> cache;
  for (const auto& e : cache)
    if (e.split == split && e.uns == uns && std::memcmp(&e.key, &K, sizeof(K)) == 0) return e.val;
  if (cache.size() >= 8) cache.erase(cache.begin());
  cache.push_back({K, split, uns, make_dev_uncached(K, split, uns)});
  return cache.back().val;
}

DevConsts make_dev_uncached(const crtg_consts& K, bool split, bool uns) {
  DevConsts d{};
  d.n = K.num_moduli;
  d.uns = uns ? 1 : 0;
  for (int l = 0; l < d.n; ++l) {
    const int p = K.moduli[l];
    d.mc[l] = make_mod(p);
    const ModConst& mc = d.mc[l];
    d.rc[l] = make_res(p, uint32_t(p / 2));
    d.rx[l] = make_res(p, uns ? 0u : 128u);
    d.rx[l].xor_mask = uns ? 0u : 0x80808080u;
    if (split && split_enabled()) {
      make_split(d.mc[l], d.rc[l], p);
      make_split(d.mc[l], d.rx[l], p);
    }
    d.coeff_hi[l] = K.coeff_hi[l];
    d.coeff_lo[l] = K.coeff_lo[l];
  }
  d.p_hi = K.p_hi;
  d.p_lo = K.p_lo;
  // S1 grid: every coeff_hi is a multiple of 2^g (crt.py:72-86); take the
  // largest common power of two and split the integer quotients into limbs.
  int g = 1100;
  for (int l = 0; l < d.n; ++l) {
    if (K.coeff_hi[l] == 0.0) continue;
    int e;
    const double fr = std::frexp(K.coeff_hi[l], &e);
    // coeff_hi = fr * 2^e; lowest set bit of the 53-bit significand
    const uint64_t mant = uint64_t(std::ldexp(fr, 53));
    g = std::min(g, e - 53 + __builtin_ctzll(mant));
  }
  if (g == 1100) g = 0;
  bool limbs_ok = true;
  for (int l = 0; l < d.n; ++l) {
    const double q = std::ldexp(K.coeff_hi[l], -g);
    if (q >= 281474976710656.0) limbs_ok = false;  // 2^48
    const uint64_t H = uint64_t(q);
    d.hi_limb[l][0] = int32_t(H & 0xFFFF);
    d.hi_limb[l][1] = int32_t((H >> 16) & 0xFFFF);
    d.hi_limb[l][2] = int32_t(H >> 32);
  }
  d.hi_scale = limbs_ok ? std::ldexp(1.0, g) : 0.0;  // 0 -> kernel keeps the f64 S1 sum
  for (int l = 0; l < d.n; l += 2)
    for (int t = 0; t < 3; ++t)
      d.limb_pair[l / 2][t] = uint32_t(d.hi_limb[l][t]) |
                              (l + 1 < d.n ? uint32_t(d.hi_limb[l + 1][t]) << 16 : 0u);
  {
    const double c = 134217729.0 * d.p_hi;
    d.p_split_hi = c - (c - d.p_hi);
    d.p_split_lo = d.p_hi - d.p_split_hi;
  }
  d.inv_p = 1.0 / d.p_hi;
  d.p_fast = K.p_fast;
  d.p_accu = K.p_accu;
  d.delta = K.delta;
  return d;
}

// ---- numpy pairwise-sum tree of one row (see kernels.cuh PwTree) ----
struct HostTree {
  std::vector<int2> leaves;
  std::vector<int2> nodes;  // sorted by height
  std::vector<int> level_start;
};

const HostTree& pairwise_tree(int64_t n) {
  static std::mutex mu;
  static std::map<int64_t, HostTree> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  HostTree t;
  struct Raw {
    int left, right, height;  // child ids: >= 0 leaf index, < 0 -> ~node index
  };
  std::vector<Raw> raw;
  // returns id: leaf index >= 0, or ~node index
  struct Rec {
    HostTree& t;
    std::vector<Raw>& raw;
    int go(int64_t start, int64_t len, int* height) {
      if (len <= 128) {
        t.leaves.push_back(make_int2(int(start), int(len)));
        *height = 0;
        return int(t.leaves.size()) - 1;
      }
      int64_t h = len / 2;
      h -= h % 8;
      int hl, hr;
      const int l = go(start, h, &hl);
      const int r = go(start + h, len - h, &hr);
      *height = std::max(hl, hr) + 1;
      raw.push_back({l, r, *height});
      return ~int(raw.size() - 1);
    }
  } rec{t, raw};
  int hroot = 0;
  rec.go(0, n, &hroot);
  const int nl = int(t.leaves.size());
  // order nodes by height; slot of node = nl + sorted position
  std::vector<int> order(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) order[i] = int(i);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return raw[a].height < raw[b].height; });
  std::vector<int> pos(raw.size());
  for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = int(i);
  auto slot = [&](int id) { return id >= 0 ? id : nl + pos[~id]; };
  for (int idx : order) t.nodes.push_back(make_int2(slot(raw[idx].left), slot(raw[idx].right)));
  t.level_start.push_back(0);
  for (int h = 1; h <= hroot; ++h) {
    int cnt = 0;
    for (auto& r : raw) cnt += r.height == h;
    t.level_start.push_back(t.level_start.back() + cnt);
  }
  return cache.emplace(n, std::move(t)).first->second;
}

// the same tree in device memory, uploaded once per (device, k) and kept: the
// per-call pageable uploads cost ~10 us each on small products
int device_tree(int64_t k, PwTree& out) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, PwTree> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, k});
  if (it != cache.end()) {
    out = it->second;
    return CRTG_OK;
  }
  const HostTree& ht = pairwise_tree(k);
  const size_t lb = ht.leaves.size() * sizeof(int2), nb = ht.nodes.size() * sizeof(int2),
               sb = ht.level_start.size() * sizeof(int);
  char* tb = nullptr;
  CRTG_TRY(cudaMalloc(&tb, lb + nb + sb + 16), "tree alloc");
  CRTG_TRY(cudaMemcpy(tb, ht.leaves.data(), lb, cudaMemcpyHostToDevice), "tree copy");
  if (nb) CRTG_TRY(cudaMemcpy(tb + lb, ht.nodes.data(), nb, cudaMemcpyHostToDevice), "tree copy");
  CRTG_TRY(cudaMemcpy(tb + lb + nb, ht.level_start.data(), sb, cudaMemcpyHostToDevice), "tree copy");
  PwTree t{int(ht.leaves.size()), int(ht.nodes.size()), int(ht.level_start.size()) - 1,
           reinterpret_cast<const int2*>(tb), reinterpret_cast<const int2*>(tb + lb),
           reinterpret_cast<const int*>(tb + lb + nb)};
  cache[{dev, k}] = t;
  out = t;
  return CRTG_OK;
}

size_t tree_bytes(int64_t k) { return size_t(16) * (k / 64 + 4) + 4 * 64 + 256; }

// ---- workspace plan ----
struct Region {
  size_t off = 0, bytes = 0;
};
struct Plan {
  int64_t m, n, k, N, nb, m_pad, n_pad, nb_pad, k_pad;
  Region diag, mu, nu, rowabs, colabs, colsq, tree, bar_mu, bar_nu, rowmax, colmax, a_pack,
      b_pack, e_re, e_im, a_bars, b_bars, rowsq;
  size_t total = 0;
};

void add(Plan& p, Region& r, size_t bytes) {
  r.off = p.total;
  r.bytes = bytes;
  p.total += (bytes + 255) & ~size_t(255);
}

Plan make_plan(int mode, int64_t m, int64_t n, int64_t k, int64_t N, int64_t n_block,
               bool real = false) {
  Plan p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.N = N;
  p.m_pad = round_up(std::max<int64_t>(m, 1), 256);  // even 128-row tiles (CTA pairs)
  p.n_pad = round_up(std::max<int64_t>(n, 1), 256);
  p.k_pad = round_up(std::max<int64_t>(k, 1), 128);
  int64_t nb = n_block < 1 ? n : n_block;
  nb = std::min(round_up(nb, 256), p.n_pad);
  p.nb = nb;
  p.nb_pad = nb;
  add(p, p.diag, 8 * CRTG_DIAG_LEN);
  add(p, p.mu, 4 * p.m_pad);
  add(p, p.nu, 4 * p.n_pad);
  add(p, p.rowabs, 8 * p.m_pad);
  add(p, p.colabs, 8 * p.n_pad);
  add(p, p.colsq, 16 * p.n_pad);
  add(p, p.tree, tree_bytes(k));
  add(p, p.a_pack, size_t(real ? N : 3 * N) * p.m_pad * p.k_pad);
  const int nbuf = 1;
  const int ppm = real ? 1 : 3;  // planes per modulus
  add(p, p.b_pack, size_t(nbuf) * size_t(ppm * N) * p.nb_pad * p.k_pad);
  add(p, p.e_re, size_t(nbuf) * size_t(N) * m * p.nb_pad);
  add(p, p.e_im, real ? 0 : size_t(nbuf) * size_t(N) * m * p.nb_pad);
  add(p, p.rowsq, real ? 16 * p.m_pad : 0);
  if (mode == CRTG_ACCURATE) {
    add(p, p.bar_mu, 4 * p.m_pad);
    add(p, p.bar_nu, 4 * p.n_pad);
    add(p, p.rowmax, 4 * p.m_pad);
    add(p, p.colmax, 4 * p.n_pad);
    add(p, p.a_bars, size_t(3) * p.m_pad * p.k_pad);
    add(p, p.b_bars, size_t(3) * p.n_pad * p.k_pad);
  }
  return p;
}

template <typename T>
T* at(void* ws, const Region& r) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + r.off);
}

int check_dims(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc,
               int64_t max_k = 65536) {
  if (m < 1 || n < 1 || k < 1) return fail(CRTG_ERR_DIMENSION, "m, n, k must be positive");
  if (k > max_k)
    return fail(CRTG_ERR_DIMENSION,
                "inner dimension " + std::to_string(k) + " exceeds " + std::to_string(max_k));
  if (lda < k || ldb < n || ldc < n) return fail(CRTG_ERR_DIMENSION, "leading dimension too small");
  if (m > (int64_t(1) << 31) || n > (int64_t(1) << 31))
    return fail(CRTG_ERR_DIMENSION, "dimension too large");
  return CRTG_OK;
}

// accurate mode, the local part (scaling.py:229-258): absmax, bars, bound
// operands and the tcgen05 bound GEMM -> row / column maxima in the plan
int accurate_partial(const Plan& P, int precision, const void* A, int64_t lda, const void* B,
                     int64_t ldb, const DevConsts& dc, void* ws, unsigned long long* diag,
                     cudaStream_t s) {
  const bool single = (precision & CRTG_IN_C64) != 0;
  double* rowabs = at<double>(ws, P.rowabs);
  double* colabs = at<double>(ws, P.colabs);
  int32_t* bar_mu = at<int32_t>(ws, P.bar_mu);
  int32_t* bar_nu = at<int32_t>(ws, P.bar_nu);
  int32_t* rowmax = at<int32_t>(ws, P.rowmax);
  int32_t* colmax = at<int32_t>(ws, P.colmax);
  CRTG_TRY(cudaMemsetAsync(colabs, 0, P.colabs.bytes, s), "memset");
  CRTG_TRY(cudaMemsetAsync(rowmax, 0, P.rowmax.bytes, s), "memset");
  CRTG_TRY(cudaMemsetAsync(colmax, 0, P.colmax.bytes, s), "memset");
  StageTimer timer(CRTG_STAGE_SCALING, s);
  PwTree tree{};
  CRTG_TRY(launch_row_stats(single ? E_C64 : E_C128, false, A, lda, P.m, P.k, tree, dc.p_fast, dc.delta, nullptr,
                            rowabs, diag, s),
           "row absmax");
  CRTG_TRY(launch_bar(rowabs, P.m, bar_mu, s), "bar");
  CRTG_TRY(launch_col_absmax(single ? E_C64 : E_C128, B, ldb, P.k, P.n, colabs, diag, s), "col absmax");
  CRTG_TRY(launch_bar(colabs, P.n, bar_nu, s), "bar");
  const int64_t a_plane = P.m_pad * P.k_pad, b_plane = P.n_pad * P.k_pad;
  int8_t* abars = at<int8_t>(ws, P.a_bars);
  int8_t* bbars = at<int8_t>(ws, P.b_bars);
  CRTG_TRY(launch_pack(single ? E_C64 : E_C128, 0, PACK_BARS, A, lda, P.m, P.k, 0, bar_mu, dc, abars, a_plane,
                       P.m_pad / 128, diag + CRTG_DIAG_OVERFLOW_A, s),
           "bars A");
  CRTG_TRY(launch_pack(single ? E_C64 : E_C128, 1, PACK_BARS, B, ldb, P.n, P.k, 0, bar_nu, dc, bbars, b_plane,
                       P.n_pad / 128, diag + CRTG_DIAG_OVERFLOW_B, s),
           "bars B");
  GemmArgs g{};
  g.a = abars;
  g.b = bbars;
  g.a_plane = a_plane;
  g.b_plane = b_plane;
  g.a_rb = int(P.m_pad / 128);
  g.b_rb = int(P.n_pad / 128);
  g.mt = int(P.m_pad / 128);
  g.nt = int(P.n_pad / 256);
  g.kb = int(P.k_pad / 128);
  g.nl = 1;
  g.planes_per_l = 3;
  g.nphase = 3;
  g.m = int(P.m);
  g.n = int(P.n);
  g.row_max = rowmax;
  g.col_max = colmax;
  CRTG_TRY(launch_gemm(EPI_BOUND, g, sm_count(), s), "bound gemm");
  return CRTG_OK;
}

// exponents (fast or accurate) into mu / nu of the plan
// Fast mode: A's row statistics on `s`, B's column statistics on `side`
// (independent; both streams must already be ordered after the inputs).
// Accurate mode: everything on `s`.
int run_scaling(const Plan& P, int precision, int mode, const void* A, int64_t lda,
                const void* B, int64_t ldb, const DevConsts& dc, void* ws,
                unsigned long long* diag, cudaStream_t s, cudaStream_t side) {
  const bool single = (precision & CRTG_IN_C64) != 0;  // input element type
  int32_t* mu = at<int32_t>(ws, P.mu);
  int32_t* nu = at<int32_t>(ws, P.nu);
  double* rowabs = at<double>(ws, P.rowabs);
  double* colabs = at<double>(ws, P.colabs);
  PwTree tree{};
  if (mode == CRTG_FAST) {
    if (int e = device_tree(P.k, tree)) return e;
    // B's column statistics first: on a forked stream they head the longer
    // chain (statistics -> residues of B), and launched after A's row
    // statistics their few CTAs found every SM taken (1024^3: started 12 us late)
    {
      StageTimer timer(CRTG_STAGE_SCALING, side);
      CRTG_TRY(launch_col_fast(single ? E_C64 : E_C128, B, ldb, P.k, P.n, colabs,
                               at<double>(ws, P.colsq), dc.p_fast, dc.delta, nu, diag, side),
               "col sumsq");
    }
    StageTimer timer(CRTG_STAGE_SCALING, s);
    CRTG_TRY(launch_row_stats(single ? E_C64 : E_C128, true, A, lda, P.m, P.k, tree, dc.p_fast,
                              dc.delta, mu, rowabs, diag, s),
             "row stats");
    return CRTG_OK;
  }
  // accurate mode (scaling.py:229-274)
  if (int e = accurate_partial(P, precision, A, lda, B, ldb, dc, ws, diag, s)) return e;
  StageTimer timer(CRTG_STAGE_SCALING, s);
  CRTG_TRY(launch_accurate_exps(at<int32_t>(ws, P.rowmax), rowabs, at<int32_t>(ws, P.bar_mu), P.m,
                                dc.p_accu, dc.delta, mu, diag + CRTG_DIAG_CLAMPED_MU, s),
           "accurate mu");
  CRTG_TRY(launch_accurate_exps(at<int32_t>(ws, P.colmax), colabs, at<int32_t>(ws, P.bar_nu), P.n,
                                dc.p_accu, dc.delta, nu, diag + CRTG_DIAG_CLAMPED_NU, s),
           "accurate nu");
  return CRTG_OK;
}

// K2..K4 with exponents already in device memory (mu: m, nu: n).  A's residues
// and the GEMMs run on `s`; B's residues and the CRT run on `side`, double
// buffered per column block so that, while GEMM_j runs, the side stream does
// CRT_{j-1} and the residues of block j+2 (launched with one CTA per SM so they
// co-reside with the persistent GEMM CTAs).  `side` must already be ordered
// after nu; `s` after mu.  On return `s` is ordered after everything.
int run_pipeline(const Plan& P, int precision, const void* A, int64_t lda, const void* B,
                 int64_t ldb, void* C, int64_t ldc, const DevConsts& dc, const int32_t* mu,
                 const int32_t* nu, void* ws, unsigned long long* dg, cudaStream_t s,
                 cudaStream_t side, Events& E, cudaStream_t first_b = nullptr) {
  const int64_t m = P.m, n = P.n, k = P.k;
  const int N = int(P.N);
  const bool in32 = (precision & CRTG_IN_C64) != 0;
  const bool single = (precision & CRTG_SINGLE) != 0;  // result type / CRT path
  // co-resident launch width for side-stream kernels (overlap mode only)
  const int nsm = side != s ? sm_count() : 0;
  const int nbuf = (side != s && P.nb < n) ? 2 : 1;
  // K2: residues of A (once)
  const int64_t a_plane = P.m_pad * P.k_pad;
  int8_t* apack = at<int8_t>(ws, P.a_pack);
  {
    StageTimer timer(CRTG_STAGE_RESIDUE_A, s);
    CRTG_TRY(launch_pack(in32 ? E_C64 : E_C128, 0, PACK_RESIDUE, A, lda, m, k, 0, mu, dc, apack, a_plane,
                         P.m_pad / 128, dg + CRTG_DIAG_OVERFLOW_A, s),
             "residues A");
  }
  const int64_t nblk = (n + P.nb - 1) / P.nb;
  const size_t bbuf = size_t(3 * N) * P.nb_pad * P.k_pad;
  const size_t ebuf = size_t(N) * m * P.nb_pad;
  const size_t csz = single ? 8 : 16;
  std::vector<cudaEvent_t> ev_r(nblk), ev_g(nblk), ev_c(nblk);
  auto bpack = [&](int64_t j) { return at<int8_t>(ws, P.b_pack) + (j % nbuf) * bbuf; };
  auto ere = [&](int64_t j) { return at<int8_t>(ws, P.e_re) + (j % nbuf) * ebuf; };
  auto eim = [&](int64_t j) { return at<int8_t>(ws, P.e_im) + (j % nbuf) * ebuf; };
  auto residues_b = [&](int64_t j, int max_ctas) -> int {
    const int64_t j0 = j * P.nb, w = std::min(P.nb, n - j0), w_pad = round_up(w, 256);
    // block 0 may go to the caller's fork stream (small products)
    cudaStream_t rs = (j == 0 && first_b) ? first_b : side;
    StageTimer timer(CRTG_STAGE_RESIDUE_B, rs);
    CRTG_TRY(launch_pack(in32 ? E_C64 : E_C128, 1, PACK_RESIDUE, B, ldb, w, k, j0, nu + j0, dc, bpack(j),
                         w_pad * P.k_pad, w_pad / 128, dg + CRTG_DIAG_OVERFLOW_B, rs, max_ctas),
             "residues B");
    ev_r[j] = E.get();
    return int(cudaEventRecord(ev_r[j], rs));
  };
  CRTG_TRY(residues_b(0, 0), "event");
  if (nblk > 1 && nbuf == 2) CRTG_TRY(residues_b(1, nsm), "event");
  for (int64_t j = 0; j < nblk; ++j) {
    const int64_t j0 = j * P.nb, w = std::min(P.nb, n - j0), w_pad = round_up(w, 256);
    CRTG_TRY(cudaStreamWaitEvent(s, ev_r[j], 0), "wait");
    if (j >= nbuf) CRTG_TRY(cudaStreamWaitEvent(s, ev_c[j - nbuf], 0), "wait");
    GemmArgs g{};
    g.a = apack;
    g.b = bpack(j);
    g.a_plane = a_plane;
    g.b_plane = w_pad * P.k_pad;
    g.a_rb = int(P.m_pad / 128);
    g.b_rb = int(w_pad / 128);
    g.mt = int(P.m_pad / 128);
    g.nt = int(w_pad / 256);
    g.kb = int(P.k_pad / 128);
    g.nl = N;
    g.planes_per_l = 3;
    g.nphase = 3;
    g.m = int(m);
    g.n = int(w);
    g.e_re = ere(j);
    g.e_im = eim(j);
    g.e_ld = P.nb_pad;
    g.e_plane = m * P.nb_pad;
    for (int l = 0; l < N; ++l) g.mc[l] = dc.mc[l];
    g.uns = dc.uns;
    {
      StageTimer timer(CRTG_STAGE_GEMM, s);
      CRTG_TRY(run_gemm(EPI_KARATSUBA, g, s), "karatsuba gemm");
    }
    ev_g[j] = E.get();
    CRTG_TRY(cudaEventRecord(ev_g[j], s), "record");
    CRTG_TRY(cudaStreamWaitEvent(side, ev_g[j], 0), "wait");
    {
      StageTimer timer(CRTG_STAGE_CRT, side);
      CRTG_TRY(launch_crt(single, false, m, w, ere(j), eim(j), g.e_plane, g.e_ld, mu, nu + j0, dc,
                          static_cast<char*>(C) + j0 * csz, ldc, side,
                          j + 1 < nblk ? nsm : 0),
               "crt");
    }
    ev_c[j] = E.get();
    CRTG_TRY(cudaEventRecord(ev_c[j], side), "record");
    if (nbuf == 2 && j + 2 < nblk) CRTG_TRY(residues_b(j + 2, nsm), "event");
    if (nbuf == 1 && j + 1 < nblk) CRTG_TRY(residues_b(j + 1, 0), "event");
  }
  CRTG_TRY(cudaStreamWaitEvent(s, ev_c[nblk - 1], 0), "wait");
  return CRTG_OK;
}

// Read back the device counters of a synchronous call.  The destination is
// page-locked, one per host thread (a pageable one is a staged copy); only
// synchronous calls write it, each right before its own stream synchronisation.
int eval_diag(const volatile unsigned long long* hd);

int check_diag(const unsigned long long* diag_dev, cudaStream_t s) {
  thread_local unsigned long long* h = [] {
    void* p = nullptr;
    if (cudaHostAlloc(&p, 8 * CRTG_DIAG_LEN, cudaHostAllocPortable) != cudaSuccess) p = nullptr;
    return static_cast<unsigned long long*>(p);
  }();
  unsigned long long hs[CRTG_DIAG_LEN];
  unsigned long long* hd = h ? h : hs;
  CRTG_TRY(cudaMemcpyAsync(hd, diag_dev, 8 * CRTG_DIAG_LEN, cudaMemcpyDeviceToHost, s),
           "diag copy");
  CRTG_TRY(cudaStreamSynchronize(s), "sync");
  return eval_diag(hd);
}

// Synchronous small products replay a graph that ends with k_diag_out, which
// stores the counters straight into this page-locked, device-mapped buffer of
// the calling thread (no separate copy after the graph).  Only synchronous
// calls write it, each followed by its own stream synchronisation.
struct MappedDiag {
  unsigned long long* h = nullptr;
  unsigned long long* d = nullptr;
};
MappedDiag mapped_diag() {
  thread_local MappedDiag m = [] {
    MappedDiag r;
    void* p = nullptr;
    if (cudaHostAlloc(&p, 8 * CRTG_DIAG_LEN, cudaHostAllocPortable | cudaHostAllocMapped) ==
        cudaSuccess) {
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, p, 0) == cudaSuccess) {
        r.h = static_cast<unsigned long long*>(p);
        r.d = static_cast<unsigned long long*>(dp);
      } else {
        cudaFreeHost(p);
      }
    }
    return r;
  }();
  return m;
}

__global__ void k_diag_out(const unsigned long long* __restrict__ dg,
                           unsigned long long* __restrict__ out) {
  if (threadIdx.x < CRTG_DIAG_LEN) out[threadIdx.x] = dg[threadIdx.x];
}

int eval_diag(const volatile unsigned long long* hd) {
  if (hd[CRTG_DIAG_NONFINITE_A]) return fail(CRTG_ERR_DOMAIN, "A contains non-finite entries");
  if (hd[CRTG_DIAG_NONFINITE_B]) return fail(CRTG_ERR_DOMAIN, "B contains non-finite entries");
  if (hd[CRTG_DIAG_OVERFLOW_A] || hd[CRTG_DIAG_OVERFLOW_B])
    return fail(CRTG_ERR_DOMAIN, "scaled magnitudes exceed the quantization budget");
  if (hd[CRTG_DIAG_INT32_OVERFLOW])
    return fail(CRTG_ERR_ARITH, "dot product exceeds the 32-bit accumulator");
  return CRTG_OK;
}

}  // namespace

extern "C" {

const char* crtg_version(void) { return "crtg 0.1.0 (sm_100a tcgen05 int8)"; }

const char* crtg_last_error(void) { return g_last_error.c_str(); }

int crtg_device_check(int device) {
  cudaDeviceProp prop;
  const cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_check(int(e), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(CRTG_ERR_CUDA, std::string("device is sm_") + std::to_string(prop.major) +
                                   std::to_string(prop.minor) + ", kernels are built for sm_100a");
  return CRTG_OK;
}

size_t crtg_workspace_size(int precision, int mode, int64_t m, int64_t n, int64_t k,
                           int num_moduli, int64_t n_block) {
  (void)precision;
  return make_plan(mode, m, n, k, num_moduli, n_block).total;
}

int crtg_scaling(int precision, int mode, int64_t m, int64_t n, int64_t k, const void* A,
                 int64_t lda, const void* B, int64_t ldb, const crtg_consts* K, void* ws,
                 size_t ws_bytes, int32_t* mu_out, int32_t* nu_out, uint64_t* diag,
                 void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if (mode != CRTG_FAST && mode != CRTG_ACCURATE) return fail(CRTG_ERR_CONFIG, "bad mode");
  // fast_scaling itself has no k cap (scaling.py:198-213); the bound product does
  if (int e = check_dims(m, n, k, lda, ldb, n, mode == CRTG_FAST ? (int64_t(1) << 18) : 65536))
    return e;
  const Plan P = make_plan(mode, m, n, k, N, n);
  if (ws_bytes < P.total) return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* dg = diag ? reinterpret_cast<unsigned long long*>(diag)
                                : at<unsigned long long>(ws, P.diag);
  CRTG_TRY(cudaMemsetAsync(dg, 0, 8 * CRTG_DIAG_LEN, s), "memset");
  const DevConsts dc = make_dev(*K);
  Events E;
  cudaStream_t side = side_stream(s);
  cudaEvent_t ev0 = E.get();
  CRTG_TRY(cudaEventRecord(ev0, s), "record");
  CRTG_TRY(cudaStreamWaitEvent(side, ev0, 0), "wait");
  if (int e = run_scaling(P, precision, mode, A, lda, B, ldb, dc, ws, dg, s, side)) return e;
  cudaEvent_t ev1 = E.get();
  CRTG_TRY(cudaEventRecord(ev1, side), "record");
  CRTG_TRY(cudaStreamWaitEvent(s, ev1, 0), "wait");
  if (mu_out)
    CRTG_TRY(cudaMemcpyAsync(mu_out, at<int32_t>(ws, P.mu), 4 * m, cudaMemcpyDeviceToDevice, s), "copy");
  if (nu_out)
    CRTG_TRY(cudaMemcpyAsync(nu_out, at<int32_t>(ws, P.nu), 4 * n, cudaMemcpyDeviceToDevice, s), "copy");
  return CRTG_OK;
}

}  // extern "C"

namespace {

// the launch sequence of one complex product (scaling, residues, GEMMs, CRT);
// every launch is stream-ordered on s (plus the forked B chain joined back)
int enqueue_complex(const Plan& P, int precision, int mode, const void* A, int64_t lda,
                    const void* B, int64_t ldb, void* C, int64_t ldc, const DevConsts& dc,
                    void* ws, int32_t* mu_out, int32_t* nu_out, unsigned long long* dg,
                    cudaStream_t s, bool graphed = false) {
  CRTG_TRY(cudaMemsetAsync(dg, 0, 8 * CRTG_DIAG_LEN, s), "memset");
  Events E;
  cudaStream_t side = side_stream(s);
  // B's chain (column statistics, residues of block 0) on `aux`
  const bool forked = side == s && fork_wanted(P.m_pad, P.n_pad, P.n, P.nb, graphed);
  cudaStream_t aux = forked ? fork_stream() : side;
  cudaEvent_t ev0 = E.get();
  CRTG_TRY(cudaEventRecord(ev0, s), "record");
  CRTG_TRY(cudaStreamWaitEvent(aux, ev0, 0), "wait");
  if (int e = run_scaling(P, precision, mode, A, lda, B, ldb, dc, ws, dg, s, aux)) return e;
  if (mode == CRTG_ACCURATE) {  // exponents were produced on s
    cudaEvent_t ev1 = E.get();
    CRTG_TRY(cudaEventRecord(ev1, s), "record");
    CRTG_TRY(cudaStreamWaitEvent(aux, ev1, 0), "wait");
  }
  int32_t* mu = at<int32_t>(ws, P.mu);
  int32_t* nu = at<int32_t>(ws, P.nu);
  if (int e = run_pipeline(P, precision, A, lda, B, ldb, C, ldc, dc, mu, nu, ws, dg, s, side, E,
                           forked ? aux : nullptr))
    return e;
  if (mu_out) CRTG_TRY(cudaMemcpyAsync(mu_out, mu, 4 * P.m, cudaMemcpyDeviceToDevice, s), "copy");
  if (nu_out) CRTG_TRY(cudaMemcpyAsync(nu_out, nu, 4 * P.n, cudaMemcpyDeviceToDevice, s), "copy");
  return CRTG_OK;
}

// Small products are launch-bound: ~10 kernels, a dozen events and two streams
// per call cost more host time than the GPU work below ~2048^3.  The second
// call with identical arguments (pointers, shape, constants) captures the
// launch sequence into a CUDA graph; later calls replay it with one
// cudaGraphLaunch.  Replays run the same kernels on the same buffers, so the
// results are bitwise those of the eager path.  Per host thread, at most
// kGraphCache graphs are kept (least recently used evicted).
struct GraphKey {
  int precision, mode, dev;
  int64_t m, n, k, lda, ldb, ldc, n_block;
  const void *A, *B;
  void *C, *ws;
  size_t ws_bytes;
  int32_t *mu_out, *nu_out;
  unsigned long long* dg;
  int sync;  // synchronous: the graph ends with k_diag_out into mapped_diag()
  crtg_consts K;
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};
struct GraphEntry {
  GraphKey key;
  int seen = 0;
  int kernels = 0;
  cudaGraphExec_t exec = nullptr;
  uint64_t used = 0;
};
constexpr size_t kGraphCache = 16;

cudaStream_t capture_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local std::map<int, cudaStream_t> streams;
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  streams[dev] = st;
  return st;
}

bool graph_wanted(const Plan& P, cudaStream_t s) {
  static const bool on = env_int("CRTG_GRAPHS", 1) != 0;
  if (!on || g_prof_on || P.nb < P.n) return false;
  if (double(P.m) * double(P.n) * double(P.k) > 8.6e9) return false;  // above ~2048^3
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone)
    return false;  // the caller is capturing: stay in its graph
  return true;
}

}  // namespace

extern "C" {

int crtg_gemm_complex(int precision, int mode, int64_t m, int64_t n, int64_t k, const void* A,
                      int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                      const crtg_consts* K, int64_t n_block, void* ws, size_t ws_bytes,
                      int32_t* mu_out, int32_t* nu_out, uint64_t* diag, int sync_check,
                      void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if ((precision & ~(CRTG_SINGLE | CRTG_IN_C64)) != 0)
    return fail(CRTG_ERR_CONFIG, "precision must be double or single");
  if (mode != CRTG_FAST && mode != CRTG_ACCURATE) return fail(CRTG_ERR_CONFIG, "bad mode");
  if (int e = check_dims(m, n, k, lda, ldb, ldc)) return e;
  const Plan P = make_plan(mode, m, n, k, N, n_block);
  if (!ws || ws_bytes < P.total)
    return fail(CRTG_ERR_WORKSPACE, "workspace too small: need " + std::to_string(P.total));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* dg = diag ? reinterpret_cast<unsigned long long*>(diag)
                                : at<unsigned long long>(ws, P.diag);
  const DevConsts dc = make_dev(*K, true, unsigned_residues(k));
  if (!graph_wanted(P, s)) {
    if (int e = enqueue_complex(P, precision, mode, A, lda, B, ldb, C, ldc, dc, ws, mu_out, nu_out,
                                dg, s))
      return e;
    return sync_check ? check_diag(dg, s) : CRTG_OK;
  }
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.precision = precision;
  key.mode = mode;
  cudaGetDevice(&key.dev);
  key.m = m; key.n = n; key.k = k; key.lda = lda; key.ldb = ldb; key.ldc = ldc;
  key.n_block = n_block;
  key.A = A; key.B = B; key.C = C; key.ws = ws; key.ws_bytes = ws_bytes;
  key.mu_out = mu_out; key.nu_out = nu_out; key.dg = dg;
  const MappedDiag md = sync_check ? mapped_diag() : MappedDiag{};
  key.sync = md.d ? 1 : 0;
  std::memcpy(&key.K, K, sizeof(crtg_consts));
  static thread_local std::vector<GraphEntry> cache;
  static thread_local uint64_t tick = 0;
  GraphEntry* hit = nullptr;
  for (auto& g : cache)
    if (g.key == key) hit = &g;
  if (!hit) {
    if (cache.size() >= kGraphCache) {
      auto lru = std::min_element(cache.begin(), cache.end(), [](const GraphEntry& a,
                                                                 const GraphEntry& b) {
        return a.used < b.used;
      });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      cache.erase(lru);
    }
    cache.push_back(GraphEntry{key});
    hit = &cache.back();
  }
  hit->used = ++tick;
  if (!hit->exec && ++hit->seen >= 2) {
    // second identical call: capture the launch sequence (the first one ran
    // eagerly and created every lazily initialised resource)
    // captured on a private stream: the caller's may be the legacy default
    // stream, which cannot be captured; the graph is then launched on s
    const uint64_t before = crtg_launch_count();
    cudaStream_t cs = capture_stream();
    CRTG_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture");
    int e = enqueue_complex(P, precision, mode, A, lda, B, ldb, C, ldc, dc, ws, mu_out, nu_out,
                            dg, cs, true);
    if (!e && key.sync) {
      k_diag_out<<<1, 32, 0, cs>>>(dg, md.d);
      e = cuda_check(launched(1), "diag out");
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    if (e) {
      if (graph) cudaGraphDestroy(graph);
      return e;
    }
    CRTG_TRY(int(ec), "end capture");
    const cudaError_t ei =
        cudaGraphInstantiate(&hit->exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    CRTG_TRY(int(ei), "graph instantiate");
    hit->kernels = int(crtg_launch_count() - before);
    note_launches(-hit->kernels);  // counted when replayed below
  }
  if (hit->exec) {
    CRTG_TRY(cudaGraphLaunch(hit->exec, s), "graph launch");
    note_launches(hit->kernels);
    if (key.sync) {
      CRTG_TRY(cudaStreamSynchronize(s), "sync");
      return eval_diag(md.h);
    }
  } else if (int e = enqueue_complex(P, precision, mode, A, lda, B, ldb, C, ldc, dc, ws, mu_out,
                                     nu_out, dg, s)) {
    return e;
  }
  return sync_check ? check_diag(dg, s) : CRTG_OK;
}

int crtg_residues(int precision, int operand, int64_t rows, int64_t kdim, const void* X,
                  int64_t ldx, const int32_t* exps, const crtg_consts* K, int8_t* out, void* ws,
                  size_t ws_bytes, uint64_t* diag, void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if (rows < 1 || kdim < 1) return fail(CRTG_ERR_DIMENSION, "empty operand");
  const int64_t r_pad = round_up(rows, 256), k_pad = round_up(kdim, 128);
  const int64_t plane = r_pad * k_pad;
  if (ws_bytes < size_t(3 * N) * plane) return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevConsts dc = make_dev(*K, false);
  dc.sym = 1;  // the reference's symmetric residues (crt.py:136-151)
  int8_t* packed = static_cast<int8_t*>(ws);
  unsigned long long* ovf = reinterpret_cast<unsigned long long*>(diag) +
                            (operand == 0 ? CRTG_DIAG_OVERFLOW_A : CRTG_DIAG_OVERFLOW_B);
  CRTG_TRY(launch_pack((precision & CRTG_IN_C64) ? E_C64 : E_C128, operand, PACK_RESIDUE, X, ldx, rows, kdim, 0,
                       exps, dc, packed, plane, r_pad / 128, ovf, s),
           "residues");
  for (int q = 0; q < 3 * N; ++q)
    CRTG_TRY(launch_unpack_i8(packed + q * plane, rows, kdim, r_pad / 128, out + q * rows * kdim, s),
             "unpack");
  return CRTG_OK;
}

size_t crtg_i8_workspace_size(int64_t m, int64_t n, int64_t k, int nplanes) {
  const int64_t m_pad = round_up(m, 256), n_pad = round_up(n, 256), k_pad = round_up(k, 128);
  size_t t = 0;
  t += round_up(size_t(nplanes) * m_pad * k_pad, 256);
  t += round_up(size_t(nplanes) * n_pad * k_pad, 256);
  t += round_up(size_t(m) * n_pad * 4, 256);
  t += round_up(size_t(m) * n_pad * 2, 256);
  // Karatsuba sums, or the split-modulus U and V planes
  t += 2 * round_up(size_t(m_pad) * k_pad + size_t(n_pad) * k_pad, 256);
  return t;
}

int crtg_gemm_i8_i32(int64_t m, int64_t n, int64_t k, const int8_t* A, const int8_t* B, int32_t* C,
                     void* ws, size_t ws_bytes, void* stream) {
  if (m < 1 || n < 1 || k < 1) return fail(CRTG_ERR_DIMENSION, "m, n, k must be positive");
  // k * 128^2 <= 2^30: no int32 wrap is possible (larger k: two calls, int64 sum)
  if (k > 65536) return fail(CRTG_ERR_DIMENSION, "inner dimension exceeds 65536");
  if (ws_bytes < crtg_i8_workspace_size(m, n, k, 1))
    return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t m_pad = round_up(m, 256), n_pad = round_up(n, 256), k_pad = round_up(k, 128);
  int8_t* ap = static_cast<int8_t*>(ws);
  int8_t* bp = ap + round_up(m_pad * k_pad, 256);
  int32_t* raw = reinterpret_cast<int32_t*>(bp + round_up(n_pad * k_pad, 256));
  CRTG_TRY(launch_pack_i8(A, 0, m, k, ap, m_pad / 128, s), "pack A");
  CRTG_TRY(launch_pack_i8(B, 1, n, k, bp, n_pad / 128, s), "pack B");
  GemmArgs g{};
  g.a = ap;
  g.b = bp;
  g.a_plane = m_pad * k_pad;
  g.b_plane = n_pad * k_pad;
  g.a_rb = int(m_pad / 128);
  g.b_rb = int(n_pad / 128);
  g.mt = int(m_pad / 128);
  g.nt = int(n_pad / 256);
  g.kb = int(k_pad / 128);
  g.nl = 1;
  g.planes_per_l = 1;
  g.nphase = 1;
  g.m = int(m);
  g.n = int(n);
  g.raw = raw;
  g.raw_ld = n_pad;
  g.raw_plane = m * n_pad;
  CRTG_TRY(run_gemm(EPI_RAW, g, s), "i8 gemm");
  CRTG_TRY(cudaMemcpy2DAsync(C, n * 4, raw, n_pad * 4, n * 4, m, cudaMemcpyDeviceToDevice, s),
           "copy out");
  return CRTG_OK;
}

}  // extern "C"

namespace {
__global__ void k_mod_sum(const int8_t* __restrict__ x, const int8_t* __restrict__ y, int64_t count,
                          ModConst mc, int8_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t r = mod_i32(int32_t(x[i]) + int32_t(y[i]), mc);
  out[i] = int8_t(to_sym(r, mc));
}

// split-modulus planes x + c y (U: c = j, V: c = p - j) in the 128-offset
// representative ((v + 128) mod p) - 128 in [-128, p - 129] (signed operands:
// crtg_complex_gemm_mod's GEMM runs with g.uns = 0)
__global__ void k_mod_lin(const int8_t* __restrict__ x, const int8_t* __restrict__ y, int c,
                          int64_t count, ModConst mc, int8_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t r = mod_i32(int32_t(x[i]) + c * int32_t(y[i]) + 128, mc);
  out[i] = int8_t(int32_t(r) - 128);
}
}  // namespace

extern "C" int crtg_complex_gemm_mod(int64_t m, int64_t n, int64_t k, const int8_t* ar,
                                     const int8_t* ai, const int8_t* br, const int8_t* bi, int p,
                                     int8_t* e_re, int8_t* e_im, void* ws, size_t ws_bytes,
                                     void* stream) {
  if (m < 1 || n < 1 || k < 1) return fail(CRTG_ERR_DIMENSION, "m, n, k must be positive");
  if (k > 65536) return fail(CRTG_ERR_DIMENSION, "inner dimension exceeds 65536");
  if (p < 2 || p > 256) return fail(CRTG_ERR_DOMAIN, "modulus outside [2, 256]");
  if (ws_bytes < crtg_i8_workspace_size(m, n, k, 3))
    return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t m_pad = round_up(m, 256), n_pad = round_up(n, 256), k_pad = round_up(k, 128);
  const int64_t a_plane = m_pad * k_pad, b_plane = n_pad * k_pad;
  int8_t* ap = static_cast<int8_t*>(ws);
  int8_t* bp = ap + round_up(3 * a_plane, 256);
  int8_t* eo = bp + round_up(3 * b_plane, 256);  // [2][m][n_pad]
  int8_t* sums = eo + round_up(m * n_pad * 4, 256);
  ModConst mc = make_mod(p);
  const int j = split_enabled() ? sqrt_minus_one(p) : 0;
  const unsigned ga = unsigned((m * k + 255) / 256), gb = unsigned((k * n + 255) / 256);
  if (j) {
    // split modulus: U = sym(re + j im), V = sym(re - j im), two products
    ResConst unused{};
    make_split(mc, unused, p);
    int8_t* u = sums;                   // [U_a | U_b]
    int8_t* v = sums + m * k + k * n;   // [V_a | V_b]
    k_mod_lin<<<ga, 256, 0, s>>>(ar, ai, j, m * k, mc, u);
    k_mod_lin<<<gb, 256, 0, s>>>(br, bi, j, k * n, mc, u + m * k);
    k_mod_lin<<<ga, 256, 0, s>>>(ar, ai, p - j, m * k, mc, v);
    k_mod_lin<<<gb, 256, 0, s>>>(br, bi, p - j, k * n, mc, v + m * k);
    CRTG_TRY(launched(4), "split planes");
    CRTG_TRY(launch_pack_i8(u, 0, m, k, ap, m_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(v, 0, m, k, ap + a_plane, m_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(u + m * k, 1, n, k, bp, n_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(v + m * k, 1, n, k, bp + b_plane, n_pad / 128, s), "pack");
  } else {
    // Karatsuba operand sums sa = sym(ar + ai), sb = sym(br + bi)  (kernel.py:101-103)
    k_mod_sum<<<ga, 256, 0, s>>>(ar, ai, m * k, mc, sums);
    k_mod_sum<<<gb, 256, 0, s>>>(br, bi, k * n, mc, sums + m * k);
    CRTG_TRY(launched(2), "mod sum");
    CRTG_TRY(launch_pack_i8(ar, 0, m, k, ap, m_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(ai, 0, m, k, ap + a_plane, m_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(sums, 0, m, k, ap + 2 * a_plane, m_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(br, 1, n, k, bp, n_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(bi, 1, n, k, bp + b_plane, n_pad / 128, s), "pack");
    CRTG_TRY(launch_pack_i8(sums + m * k, 1, n, k, bp + 2 * b_plane, n_pad / 128, s), "pack");
  }
  GemmArgs g{};
  g.a = ap;
  g.b = bp;
  g.a_plane = a_plane;
  g.b_plane = b_plane;
  g.a_rb = int(m_pad / 128);
  g.b_rb = int(n_pad / 128);
  g.mt = int(m_pad / 128);
  g.nt = int(n_pad / 256);
  g.kb = int(k_pad / 128);
  g.nl = 1;
  g.planes_per_l = 3;
  g.nphase = 3;
  g.m = int(m);
  g.n = int(n);
  g.e_re = eo;
  g.e_im = eo + m * n_pad;
  g.e_ld = n_pad;
  g.e_plane = 0;
  g.mc[0] = mc;
  CRTG_TRY(run_gemm(EPI_KARATSUBA, g, s), "karatsuba gemm");
  CRTG_TRY(cudaMemcpy2DAsync(e_re, n, g.e_re, n_pad, n, m, cudaMemcpyDeviceToDevice, s), "copy");
  CRTG_TRY(cudaMemcpy2DAsync(e_im, n, g.e_im, n_pad, n, m, cudaMemcpyDeviceToDevice, s), "copy");
  return CRTG_OK;
}

extern "C" int crtg_crt_reconstruct(int precision, int64_t m, int64_t n, const int8_t* e_re,
                                    const int8_t* e_im, const int32_t* mu, const int32_t* nu,
                                    const crtg_consts* K, void* C, int64_t ldc, void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if (m < 1 || n < 1 || ldc < n) return fail(CRTG_ERR_DIMENSION, "bad shape");
  const DevConsts dc = make_dev(*K);
  CRTG_TRY(launch_crt((precision & CRTG_SINGLE) != 0, false, m, n, e_re, e_im, m * n, n, mu, nu, dc, C, ldc,
                      static_cast<cudaStream_t>(stream)),
           "crt");
  return CRTG_OK;
}

extern "C" uint64_t crtg_launch_count(void) { return g_launches.load(); }

extern "C" int crtg_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return CRTG_OK;
}

extern "C" int crtg_profile_read(double* ms, uint64_t* launches) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    recs.swap(g_prof);
  }
  for (int i = 0; i < CRTG_STAGE_COUNT; ++i) {
    if (ms) ms[i] = 0.0;
    if (launches) launches[i] = 0;
  }
  int status = CRTG_OK;
  for (auto& r : recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
      status = fail(CRTG_ERR_CUDA, "profile event failure");
    if (r.stage >= 0 && r.stage < CRTG_STAGE_COUNT) {
      if (ms) ms[r.stage] += t;
      if (launches) launches[r.stage] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  return status;
}

extern "C" int crtg_gemm_complex_exps(int precision, int64_t m, int64_t n, int64_t k,
                                      const void* A, int64_t lda, const void* B, int64_t ldb,
                                      void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                                      const int32_t* mu, const int32_t* nu, void* ws,
                                      size_t ws_bytes, uint64_t* diag, int sync_check,
                                      void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if ((precision & ~(CRTG_SINGLE | CRTG_IN_C64)) != 0)
    return fail(CRTG_ERR_CONFIG, "precision must be double or single");
  if (!mu || !nu) return fail(CRTG_ERR_CONFIG, "exponent vectors are required");
  if (int e = check_dims(m, n, k, lda, ldb, ldc)) return e;
  const Plan P = make_plan(CRTG_FAST, m, n, k, N, n_block);
  if (!ws || ws_bytes < P.total)
    return fail(CRTG_ERR_WORKSPACE, "workspace too small: need " + std::to_string(P.total));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* dg = diag ? reinterpret_cast<unsigned long long*>(diag)
                                : at<unsigned long long>(ws, P.diag);
  CRTG_TRY(cudaMemsetAsync(dg, 0, 8 * CRTG_DIAG_LEN, s), "memset");
  const DevConsts dc = make_dev(*K, true, unsigned_residues(k));
  Events E;
  cudaStream_t side = side_stream(s);
  cudaEvent_t ev0 = E.get();
  CRTG_TRY(cudaEventRecord(ev0, s), "record");
  CRTG_TRY(cudaStreamWaitEvent(side, ev0, 0), "wait");
  if (int e = run_pipeline(P, precision, A, lda, B, ldb, C, ldc, dc, mu, nu, ws, dg, s, side, E))
    return e;
  if (sync_check) return check_diag(dg, s);
  return CRTG_OK;
}

extern "C" int crtg_accurate_partial(int precision, int64_t m, int64_t n, int64_t k,
                                     const void* A, int64_t lda, const void* B, int64_t ldb,
                                     const crtg_consts* K, void* ws, size_t ws_bytes,
                                     int32_t* row_max, int32_t* col_max, int32_t* bar_mu,
                                     int32_t* bar_nu, double* row_abs, double* col_abs,
                                     uint64_t* diag, void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if (int e = check_dims(m, n, k, lda, ldb, n)) return e;
  const Plan P = make_plan(CRTG_ACCURATE, m, n, k, N, n);
  if (!ws || ws_bytes < P.total) return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  if (!diag) return fail(CRTG_ERR_CONFIG, "diag is required");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* dg = reinterpret_cast<unsigned long long*>(diag);
  const DevConsts dc = make_dev(*K);
  if (int e = accurate_partial(P, precision, A, lda, B, ldb, dc, ws, dg, s)) return e;
  auto copy = [&](void* dst, const Region& r, size_t bytes) {
    return dst ? int(cudaMemcpyAsync(dst, static_cast<char*>(ws) + r.off, bytes,
                                     cudaMemcpyDeviceToDevice, s))
               : 0;
  };
  CRTG_TRY(copy(row_max, P.rowmax, 4 * m), "copy");
  CRTG_TRY(copy(col_max, P.colmax, 4 * n), "copy");
  CRTG_TRY(copy(bar_mu, P.bar_mu, 4 * m), "copy");
  CRTG_TRY(copy(bar_nu, P.bar_nu, 4 * n), "copy");
  CRTG_TRY(copy(row_abs, P.rowabs, 8 * m), "copy");
  CRTG_TRY(copy(col_abs, P.colabs, 8 * n), "copy");
  return CRTG_OK;
}

extern "C" int crtg_accurate_exponents(int64_t count, const int32_t* maxb, const double* absval,
                                       const int32_t* bar, const crtg_consts* K, int32_t* out,
                                       uint64_t* clamp_counter, void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if (count < 1) return fail(CRTG_ERR_DIMENSION, "empty exponent vector");
  CRTG_TRY(launch_accurate_exps(maxb, absval, bar, count, K->p_accu, K->delta, out,
                                reinterpret_cast<unsigned long long*>(clamp_counter),
                                static_cast<cudaStream_t>(stream)),
           "accurate exponents");
  return CRTG_OK;
}

namespace {
// per-thread, per-device copy-engine streams for the host-buffer entry
cudaStream_t copy_stream(int which) {
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local std::map<int, cudaStream_t> streams[2];
  auto it = streams[which].find(dev);
  if (it != streams[which].end()) return it->second;
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  streams[which][dev] = st;
  return st;
}
}  // namespace

// host-entry pieces: A in row chunks, B in column blocks (multiples of 256)
struct HostChunks {
  int64_t rows;  // rows per A chunk
  int64_t cols;  // columns per B block
};

// Staircase streaming: A in row chunks and B in column blocks of about 1/16 of
// the matrix each, transferred interleaved (A0 B0 A1 B1 ...).  Every piece that
// lands releases a whole strip of output tiles (A_t: rows of chunk t x blocks
// 0..t-1; B_t: chunks 0..t x block t), computed as ONE GEMM launch over the
// strip.  With f of both operands resident only f^2 of the product can run, so
// the wall time is bounded below by max_f [f T_x + (1 - f^2) T_c]; finer pieces
// approach that bound (8 -> 16 pieces: ~5 ms at 16384^3, tools/e2e_profile.py).
HostChunks host_chunks(const Plan& P) {
  static const int npieces = std::max(1, env_int("CRTG_HOST_PIECES", 16));
  auto piece = [](int64_t x) {
    return x >= 4096 ? round_up((x + npieces - 1) / npieces, 256) : round_up(x, 256);
  };
  return HostChunks{piece(P.m), piece(P.n)};
}

// one plan over the whole product: B's packed planes and the e-planes span all n
Plan host_plan(int mode, int64_t m, int64_t n, int64_t k, int N, int64_t n_block) {
  (void)n_block;  // the strips bound the working set; results are bitwise invariant
  return make_plan(mode, m, n, k, N, round_up(std::max<int64_t>(n, 1), 256));
}

namespace {
int load_tree(const Plan& P, void* ws, cudaStream_t s, PwTree& tree);  // below
}  // namespace

namespace {
// false only for plain pageable host memory (the staged path); page-locked,
// device or managed memory goes to the copy engine directly
bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type != cudaMemoryTypeUnregistered;
}

// Pageable host operands: pieces are gathered by host threads (OpenMP) into a
// ring of pinned staging slots and copied from there on the copy engine, so a
// plain numpy caller gets full-rate PCIe without page-locking its arrays (which
// costs ~0.33 s per 4 GiB plus the unlock).  The CPU runs at most kSlots pieces
// ahead of the copy engine.
struct HostStager {
  static constexpr int kSlots = 3;
  char* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  bool pending[kSlots] = {};
  size_t bytes = 0;
  int next = 0;
  int ensure(size_t need) {
    if (need <= bytes) return 0;
    for (int i = 0; i < kSlots; ++i) {
      if (pending[i]) cudaEventSynchronize(done[i]);
      pending[i] = false;
      if (slot[i]) cudaFreeHost(slot[i]);
      slot[i] = nullptr;
    }
    bytes = 0;
    for (int i = 0; i < kSlots; ++i) {
      if (int e = int(cudaHostAlloc(reinterpret_cast<void**>(&slot[i]), need, cudaHostAllocPortable)))
        return e;
      if (!done[i])
        if (int e = int(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming))) return e;
    }
    bytes = need;
    return 0;
  }
  // next free slot (waits for the copy that last read it)
  char* acquire(int& s) {
    s = next;
    next = (next + 1) % kSlots;
    if (pending[s]) cudaEventSynchronize(done[s]);
    pending[s] = false;
    return slot[s];
  }
  int release(int s, cudaStream_t st) {
    pending[s] = true;
    return int(cudaEventRecord(done[s], st));
  }
  void free_all() {
    for (int i = 0; i < kSlots; ++i) {
      if (pending[i]) cudaEventSynchronize(done[i]);
      pending[i] = false;
      if (slot[i]) cudaFreeHost(slot[i]);
      slot[i] = nullptr;
      if (done[i]) cudaEventDestroy(done[i]);
      done[i] = nullptr;
    }
    bytes = 0;
    next = 0;
  }
  ~HostStager() { free_all(); }  // thread exit
};

HostStager& host_stager() {
  static thread_local HostStager st;
  return st;
}

HostStager& host_out_stager() {
  static thread_local HostStager st;
  return st;
}
}  // namespace

extern "C" void crtg_release_host_staging(void) {
  host_stager().free_all();
  host_out_stager().free_all();
}

namespace {

// rows of src (row_bytes each, contiguous) -> dst at dst_pitch, host threads
void scatter_rows(char* dst, const char* src, int64_t rows, size_t row_bytes, size_t dst_pitch) {
  const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(rows, 64));
#pragma omp parallel for num_threads(16) schedule(static)
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t r0 = rows * b / nblk, r1 = rows * (b + 1) / nblk;
    for (int64_t r = r0; r < r1; ++r)
      std::memcpy(dst + size_t(r) * dst_pitch, src + size_t(r) * row_bytes, row_bytes);
  }
}

// dst (contiguous rows of row_bytes) <- rows of src at src_pitch, host threads
void gather_rows(char* dst, const char* src, int64_t rows, size_t row_bytes, size_t src_pitch) {
  const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(rows, 64));
#pragma omp parallel for num_threads(16) schedule(static)
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t r0 = rows * b / nblk, r1 = rows * (b + 1) / nblk;
    if (src_pitch == row_bytes) {
      std::memcpy(dst + size_t(r0) * row_bytes, src + size_t(r0) * src_pitch,
                  size_t(r1 - r0) * row_bytes);
    } else {
      for (int64_t r = r0; r < r1; ++r)
        std::memcpy(dst + size_t(r) * row_bytes, src + size_t(r) * src_pitch, row_bytes);
    }
  }
}
}  // namespace

extern "C" size_t crtg_host_workspace_size(int precision, int mode, int64_t m, int64_t n,
                                           int64_t k, int num_moduli, int64_t n_block) {
  const Plan P = host_plan(mode, m, n, k, num_moduli, n_block);
  const size_t esz = (precision & CRTG_IN_C64) ? 8 : 16;
  const size_t csz = (precision & CRTG_SINGLE) ? 8 : 16;
  auto r = [](size_t x) { return (x + 255) & ~size_t(255); };
  return P.total + r(size_t(m) * k * esz) + r(size_t(k) * n * esz) + r(size_t(m) * n * csz);
}

// End-to-end entry on HOST buffers (pinned for full overlap).  Transfers run
// A_0, B_0, A_1, B_1, ... on a copy-engine stream; each landed piece gets its
// statistics (fast mode) and residues, then the strip of output tiles it
// completes runs as one GEMM + CRT, and the strip of C goes back on a second
// copy stream while the next strip computes.  Accurate mode needs every bound
// maximum first and so waits for all inputs before its exponents.
extern "C" int crtg_gemm_complex_host(int precision, int mode, int64_t m, int64_t n, int64_t k,
                                      const void* A, int64_t lda, const void* B, int64_t ldb,
                                      void* C, int64_t ldc, const crtg_consts* K, int64_t n_block,
                                      void* ws, size_t ws_bytes, uint64_t* diag, int sync_check,
                                      void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if ((precision & ~(CRTG_SINGLE | CRTG_IN_C64)) != 0)
    return fail(CRTG_ERR_CONFIG, "precision must be double or single");
  if (mode != CRTG_FAST && mode != CRTG_ACCURATE) return fail(CRTG_ERR_CONFIG, "bad mode");
  if (int e = check_dims(m, n, k, lda, ldb, ldc)) return e;
  const Plan P = host_plan(mode, m, n, k, N, n_block);
  const HostChunks hc = host_chunks(P);
  if (!ws || ws_bytes < crtg_host_workspace_size(precision, mode, m, n, k, N, n_block))
    return fail(CRTG_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t h2d = copy_stream(0), d2h = copy_stream(1);
  const bool in32 = (precision & CRTG_IN_C64) != 0;
  const bool single = (precision & CRTG_SINGLE) != 0;
  const int elem = in32 ? E_C64 : E_C128;
  const size_t esz = in32 ? 8 : 16, csz = single ? 8 : 16;
  auto r = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* dA = static_cast<char*>(ws) + P.total;
  char* dB = dA + r(size_t(m) * k * esz);
  char* dC = dB + r(size_t(k) * n * esz);  // m x n, row-major (ld n)
  unsigned long long* dg = diag ? reinterpret_cast<unsigned long long*>(diag)
                                : at<unsigned long long>(ws, P.diag);
  const DevConsts dc = make_dev(*K, true, unsigned_residues(k));
  Events E;
  cudaEvent_t ev0 = E.get();
  CRTG_TRY(cudaMemsetAsync(dg, 0, 8 * CRTG_DIAG_LEN, s), "memset");
  CRTG_TRY(cudaMemsetAsync(at<double>(ws, P.colabs), 0, P.colabs.bytes, s), "memset");
  CRTG_TRY(cudaEventRecord(ev0, s), "record");
  CRTG_TRY(cudaStreamWaitEvent(h2d, ev0, 0), "wait");
  CRTG_TRY(cudaStreamWaitEvent(d2h, ev0, 0), "wait");

  // CRTG_HOST_TRACE=1: print a timeline (ms after the call starts) of every
  // piece landing and every strip's GEMM start / end (diagnostics only)
  static const bool trace = env_int("CRTG_HOST_TRACE", 0) != 0;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  cudaEvent_t t0ev = nullptr;
  auto mark = [&](const std::string& what, cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.push_back({what, e});
  };
  if (trace) {
    cudaEventCreate(&t0ev);
    cudaEventRecord(t0ev, s);
  }
  const int64_t nrc = (m + hc.rows - 1) / hc.rows;
  const int64_t ncb = (n + hc.cols - 1) / hc.cols;
  std::vector<cudaEvent_t> evA(nrc), evB(ncb);
  // pageable operands go through pinned staging slots (HostStager)
  const bool stage_a = !host_pinned(A), stage_b = !host_pinned(B);
  HostStager& stager = host_stager();
  if (stage_a || stage_b) {
    const size_t need = std::max(size_t(hc.rows) * k * esz, size_t(hc.cols) * k * esz);
    CRTG_TRY(stager.ensure(need), "pinned staging");
  }
  auto copy_a = [&](int64_t i) -> int {
    const int64_t i0 = i * hc.rows, h = std::min(hc.rows, m - i0);
    const char* src = static_cast<const char*>(A) + size_t(i0) * lda * esz;
    if (stage_a) {
      int sl = 0;
      char* buf = stager.acquire(sl);
      gather_rows(buf, src, h, size_t(k) * esz, size_t(lda) * esz);
      CRTG_TRY(cudaMemcpyAsync(dA + size_t(i0) * k * esz, buf, size_t(h) * k * esz,
                               cudaMemcpyHostToDevice, h2d),
               "H2D A");
      CRTG_TRY(stager.release(sl, h2d), "record");
    } else {
      CRTG_TRY(cudaMemcpy2DAsync(dA + size_t(i0) * k * esz, k * esz, src, lda * esz, k * esz, h,
                                 cudaMemcpyHostToDevice, h2d),
               "H2D A");
    }
    evA[i] = E.get();
    mark("A" + std::to_string(i) + " landed", h2d);
    return int(cudaEventRecord(evA[i], h2d));
  };
  auto copy_b = [&](int64_t j) -> int {
    const int64_t j0 = j * hc.cols, w = std::min(hc.cols, n - j0);
    const char* src = static_cast<const char*>(B) + j0 * esz;
    if (stage_b) {
      int sl = 0;
      char* buf = stager.acquire(sl);
      gather_rows(buf, src, k, size_t(w) * esz, size_t(ldb) * esz);
      CRTG_TRY(cudaMemcpy2DAsync(dB + j0 * esz, n * esz, buf, w * esz, w * esz, k,
                                 cudaMemcpyHostToDevice, h2d),
               "H2D B");
      CRTG_TRY(stager.release(sl, h2d), "record");
    } else {
      CRTG_TRY(cudaMemcpy2DAsync(dB + j0 * esz, n * esz, src, ldb * esz, w * esz, k,
                                 cudaMemcpyHostToDevice, h2d),
               "H2D B");
    }
    evB[j] = E.get();
    mark("B" + std::to_string(j) + " landed", h2d);
    return int(cudaEventRecord(evB[j], h2d));
  };
  // transfer order: A0 B0 A1 B1 ... (the longer list's tail last).  Fast mode
  // enqueues each copy right before the strip it releases (a staged copy blocks
  // the CPU until a slot is free, and the strips must already be queued behind
  // the copies); accurate mode needs every piece before its exponents.
  const int64_t npieces = std::max(nrc, ncb);
  if (mode == CRTG_ACCURATE) {
    for (int64_t t = 0; t < npieces; ++t) {
      if (t < nrc) CRTG_TRY(copy_a(t), "record");
      if (t < ncb) CRTG_TRY(copy_b(t), "record");
    }
  }

  int32_t* mu = at<int32_t>(ws, P.mu);
  int32_t* nu = at<int32_t>(ws, P.nu);
  PwTree tree{};
  if (mode == CRTG_ACCURATE) {
    CRTG_TRY(cudaStreamWaitEvent(s, evA[nrc - 1], 0), "wait");
    CRTG_TRY(cudaStreamWaitEvent(s, evB[ncb - 1], 0), "wait");
    if (int e = run_scaling(P, precision, mode, dA, k, dB, n, dc, ws, dg, s, s)) return e;
  } else {
    if (int e = load_tree(P, ws, s, tree)) return e;
  }
  const int64_t a_plane = P.m_pad * P.k_pad, b_plane = P.n_pad * P.k_pad;
  int8_t* apack = at<int8_t>(ws, P.a_pack);
  int8_t* bpack = at<int8_t>(ws, P.b_pack);
  int8_t* ere = at<int8_t>(ws, P.e_re);
  int8_t* eim = at<int8_t>(ws, P.e_im);

  auto piece_a = [&](int64_t i) -> int {  // A chunk i: statistics (fast) and residues
    const int64_t i0 = i * hc.rows, h = std::min(hc.rows, m - i0);
    CRTG_TRY(cudaStreamWaitEvent(s, evA[i], 0), "wait");
    const char* Ai = dA + size_t(i0) * k * esz;
    if (mode == CRTG_FAST) {
      StageTimer timer(CRTG_STAGE_SCALING, s);
      CRTG_TRY(launch_row_stats(elem, true, Ai, k, h, k, tree, dc.p_fast, dc.delta, mu + i0,
                                at<double>(ws, P.rowabs) + i0, dg, s),
               "row stats");
    }
    StageTimer timer(CRTG_STAGE_RESIDUE_A, s);
    CRTG_TRY(launch_pack(elem, 0, PACK_RESIDUE, Ai, k, h, k, 0, mu + i0, dc, apack, a_plane,
                         P.m_pad / 128, dg + CRTG_DIAG_OVERFLOW_A, s, 0, i0,
                         i == nrc - 1 ? P.m_pad - i0 : h),
             "residues A");
    return CRTG_OK;
  };
  auto piece_b = [&](int64_t j) -> int {  // B block j: statistics (fast) and residues
    const int64_t j0 = j * hc.cols, w = std::min(hc.cols, n - j0);
    CRTG_TRY(cudaStreamWaitEvent(s, evB[j], 0), "wait");
    if (mode == CRTG_FAST) {
      StageTimer timer(CRTG_STAGE_SCALING, s);
      CRTG_TRY(launch_col_fast(elem, dB + j0 * esz, n, k, w, at<double>(ws, P.colabs) + j0,
                               at<double>(ws, P.colsq) + 2 * j0, dc.p_fast, dc.delta, nu + j0,
                               dg, s),
               "col stats");
    }
    StageTimer timer(CRTG_STAGE_RESIDUE_B, s);
    CRTG_TRY(launch_pack(elem, 1, PACK_RESIDUE, dB, n, w, k, j0, nu + j0, dc, bpack, b_plane,
                         P.n_pad / 128, dg + CRTG_DIAG_OVERFLOW_B, s, 0, j0,
                         j == ncb - 1 ? P.n_pad - j0 : w),
             "residues B");
    return CRTG_OK;
  };
  // output strip rows [r0, r1) x columns [c0, c1): one GEMM launch, one CRT, one D2H
  // PCIe is full duplex but not free: with C copied back while inputs stream in,
  // H2D drops from 55.6 to ~46 GB/s (tools/pcie_2d.py duplex).  The input
  // transfer is the critical path, so the copy-back of finished strips is held
  // back until a fraction CRTG_D2H_GATE (default 0.6) of the input pieces has
  // been queued (the d2h stream then also waits for that piece to land); the
  // backlog drains beside the last pieces and the final strips.
  static const double d2h_gate = [] {
    const char* v = std::getenv("CRTG_D2H_GATE");
    return v && *v ? std::atof(v) : 0.6;
  }();
  const int64_t total_pieces = nrc + ncb;
  const int64_t gate_piece =
      std::min<int64_t>(total_pieces - 1, int64_t(d2h_gate * double(total_pieces)));
  int64_t pieces_queued = 0;
  bool gate_open = gate_piece <= 0;
  struct PendingD2H {
    int64_t r0, r1, c0, c1;
    cudaEvent_t ready;
  };
  std::vector<PendingD2H> pending_d2h;
  // pageable C: strips come back through a second ring of pinned slots and host
  // threads scatter them into C (serviced between pieces and drained at the end)
  const bool stage_c = !host_pinned(C);
  HostStager& ostager = host_out_stager();
  struct OutCopy {
    int slot;
    int64_t r0, r1, c0, c1;
  };
  std::vector<OutCopy> out_q;  // FIFO of staged strips not yet in C
  if (stage_c) {
    const size_t need = std::max(size_t(hc.rows) * n, size_t(m) * hc.cols) * csz;
    CRTG_TRY(ostager.ensure(need), "pinned staging");
  }
  auto finish_out = [&](const OutCopy& o) {  // slot's copy has landed (waited by the caller)
    scatter_rows(static_cast<char*>(C) + (size_t(o.r0) * ldc + o.c0) * csz, ostager.slot[o.slot],
                 o.r1 - o.r0, size_t(o.c1 - o.c0) * csz, size_t(ldc) * csz);
  };
  auto service_out = [&](bool drain) -> int {
    while (!out_q.empty()) {
      const OutCopy& o = out_q.front();
      if (!drain) {
        const cudaError_t q = cudaEventQuery(ostager.done[o.slot]);
        if (q == cudaErrorNotReady) break;
        CRTG_TRY(int(q), "event");
      } else {
        CRTG_TRY(cudaEventSynchronize(ostager.done[o.slot]), "sync");
      }
      finish_out(o);
      ostager.pending[o.slot] = false;
      out_q.erase(out_q.begin());
    }
    return CRTG_OK;
  };
  auto enqueue_d2h = [&](const PendingD2H& x) -> int {
    CRTG_TRY(cudaStreamWaitEvent(d2h, x.ready, 0), "wait");
    if (!stage_c)
      return int(cudaMemcpy2DAsync(static_cast<char*>(C) + (size_t(x.r0) * ldc + x.c0) * csz,
                                   ldc * csz, dC + (size_t(x.r0) * n + x.c0) * csz, n * csz,
                                   (x.c1 - x.c0) * csz, x.r1 - x.r0, cudaMemcpyDeviceToHost, d2h));
    // the next slot must be empty: it is held by the oldest staged strip (slots
    // are used round-robin), so finish that one
    const int sl = ostager.next;
    if (ostager.pending[sl] && !out_q.empty()) {
      const OutCopy o = out_q.front();
      CRTG_TRY(cudaEventSynchronize(ostager.done[o.slot]), "sync");
      finish_out(o);
      ostager.pending[o.slot] = false;
      out_q.erase(out_q.begin());
    }
    int got = 0;
    char* buf = ostager.acquire(got);
    CRTG_TRY(cudaMemcpy2DAsync(buf, (x.c1 - x.c0) * csz, dC + (size_t(x.r0) * n + x.c0) * csz,
                               n * csz, (x.c1 - x.c0) * csz, x.r1 - x.r0, cudaMemcpyDeviceToHost,
                               d2h),
             "D2H C");
    CRTG_TRY(ostager.release(got, d2h), "record");
    out_q.push_back({got, x.r0, x.r1, x.c0, x.c1});
    return CRTG_OK;
  };
  // called after every queued input piece (ev = its landing event)
  auto piece_queued = [&](cudaEvent_t ev) -> int {
    ++pieces_queued;
    if (stage_c) CRTG_TRY(service_out(false), "D2H C");
    if (!gate_open && pieces_queued > gate_piece) {
      gate_open = true;
      CRTG_TRY(cudaStreamWaitEvent(d2h, ev, 0), "wait");
      for (const auto& x : pending_d2h) CRTG_TRY(enqueue_d2h(x), "D2H C");
      pending_d2h.clear();
    }
    return CRTG_OK;
  };
  auto strip = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
    mark("strip " + std::to_string(r0) + ":" + std::to_string(r1) + " x " + std::to_string(c0) +
             ":" + std::to_string(c1) + " start", s);
    GemmArgs g{};
    g.a = apack;
    g.b = bpack;
    g.a_plane = a_plane;
    g.b_plane = b_plane;
    g.a_rb = int(P.m_pad / 128);
    g.b_rb = int(P.n_pad / 128);
    g.mt0 = int(r0 / 128);
    g.mt = int((std::min(round_up(r1, 256), P.m_pad) - r0) / 128);
    g.nt0 = int(c0 / 256);
    g.nt = int((std::min(round_up(c1, 256), P.n_pad) - c0) / 256);
    g.kb = int(P.k_pad / 128);
    g.nl = N;
    g.planes_per_l = 3;
    g.nphase = 3;
    g.m = int(r1);
    g.n = int(c1);
    g.e_re = ere;
    g.e_im = eim;
    g.e_ld = P.n_pad;
    g.e_plane = m * P.n_pad;
    for (int l = 0; l < N; ++l) g.mc[l] = dc.mc[l];
    g.uns = dc.uns;
    {
      StageTimer timer(CRTG_STAGE_GEMM, s);
      CRTG_TRY(run_gemm(EPI_KARATSUBA, g, s), "karatsuba gemm");
    }
    char* cst = dC + (size_t(r0) * n + c0) * csz;
    {
      StageTimer timer(CRTG_STAGE_CRT, s);
      CRTG_TRY(launch_crt(single, false, r1 - r0, c1 - c0, ere + r0 * P.n_pad + c0,
                          eim + r0 * P.n_pad + c0, g.e_plane, g.e_ld, mu + r0, nu + c0, dc, cst, n,
                          s),
               "crt");
    }
    cudaEvent_t evC = E.get();
    CRTG_TRY(cudaEventRecord(evC, s), "record");
    mark("  strip end", s);
    (void)cst;
    const PendingD2H x{r0, r1, c0, c1, evC};
    if (gate_open) {
      CRTG_TRY(enqueue_d2h(x), "D2H C");
    } else {
      pending_d2h.push_back(x);
    }
    return CRTG_OK;
  };
  for (int64_t t = 0; t < npieces; ++t) {
    if (t < nrc) {  // A_t: rows of chunk t x every block already resident
      if (mode == CRTG_FAST) CRTG_TRY(copy_a(t), "record");
      CRTG_TRY(piece_queued(evA[t]), "gate");
      CRTG_TRY(piece_a(t), "piece A");
      const int64_t jb = std::min(t, ncb);
      if (jb > 0)
        CRTG_TRY(strip(t * hc.rows, std::min((t + 1) * hc.rows, m), 0, std::min(jb * hc.cols, n)),
                 "strip");
    }
    if (t < ncb) {  // B_t: every resident chunk x block t
      if (mode == CRTG_FAST) CRTG_TRY(copy_b(t), "record");
      CRTG_TRY(piece_queued(evB[t]), "gate");
      CRTG_TRY(piece_b(t), "piece B");
      const int64_t ib = std::min(t + 1, nrc);
      const int64_t c0 = t * hc.cols, c1 = std::min((t + 1) * hc.cols, n);
      if (t == npieces - 1 && ib >= 8) {
        // the last strip in four row parts: the D2H of each part overlaps the
        // next part's GEMM, so only a quarter of the final copy-back is exposed
        const int64_t per = (ib + 3) / 4;
        for (int64_t i = 0; i < ib; i += per)
          CRTG_TRY(strip(i * hc.rows, std::min(std::min(i + per, ib) * hc.rows, m), c0, c1),
                   "strip");
      } else {
        CRTG_TRY(strip(0, std::min(ib * hc.rows, m), c0, c1), "strip");
      }
    }
  }
  for (const auto& x : pending_d2h) CRTG_TRY(enqueue_d2h(x), "D2H C");
  pending_d2h.clear();
  if (stage_c) CRTG_TRY(service_out(true), "D2H C");  // C complete on return
  cudaEvent_t evD = E.get();
  CRTG_TRY(cudaEventRecord(evD, d2h), "record");
  CRTG_TRY(cudaStreamWaitEvent(s, evD, 0), "wait");
  if (trace) {
    mark("done", s);
    cudaStreamSynchronize(s);
    std::vector<std::pair<float, std::string>> tl;
    for (auto& mk : marks) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, t0ev, mk.second) == cudaSuccess) tl.push_back({ms, mk.first});
    }
    std::sort(tl.begin(), tl.end());
    for (auto& x : tl) std::fprintf(stderr, "[crtg trace] %8.2f ms  %s\n", x.first, x.second.c_str());
    for (auto& mk : marks) cudaEventDestroy(mk.second);
    cudaEventDestroy(t0ev);
  }
  if (sync_check) return check_diag(dg, s);
  return CRTG_OK;
}

// ---------------------------------------------------------------------------
// Real domain (emulate_gemm_real, emulate.py:169-190).
// The reference keeps the caller's memory layout for real operands, so numpy
// sums the squares pairwise along the contiguous axis and sequentially along the
// strided one; an operand stored column-major is therefore processed as the
// transpose of a row-major matrix by the "other" kernel family, which yields
// exactly that order.
// ---------------------------------------------------------------------------
namespace {
int load_tree(const Plan& P, void* ws, cudaStream_t s, PwTree& tree) {
  (void)ws;
  (void)s;
  return device_tree(P.k, tree);
}
}  // namespace

extern "C" size_t crtg_real_workspace_size(int precision, int mode, int64_t m, int64_t n,
                                           int64_t k, int num_moduli, int64_t n_block) {
  (void)precision;
  return make_plan(mode, m, n, k, num_moduli, n_block, true).total;
}

extern "C" int crtg_gemm_real(int precision, int mode, int64_t m, int64_t n, int64_t k,
                              const void* A, int64_t lda, int a_colmajor, const void* B,
                              int64_t ldb, int b_colmajor, void* C, int64_t ldc,
                              const crtg_consts* K, int64_t n_block, void* ws, size_t ws_bytes,
                              int32_t* mu_out, int32_t* nu_out, uint64_t* diag, int sync_check,
                              void* stream) {
  int N = 0;
  if (int e = check_consts(K, &N)) return e;
  if ((precision & ~(CRTG_SINGLE | CRTG_IN_F32)) != 0)
    return fail(CRTG_ERR_CONFIG, "precision must be double or single");
  if (mode != CRTG_FAST && mode != CRTG_ACCURATE) return fail(CRTG_ERR_CONFIG, "bad mode");
  // k cap: 2^17 in fast mode, 2^16 in accurate mode (emulate.py:179-182)
  const int64_t kcap = mode == CRTG_FAST ? (int64_t(1) << 17) : (int64_t(1) << 16);
  if (m < 1 || n < 1 || k < 1) return fail(CRTG_ERR_DIMENSION, "m, n, k must be positive");
  if (k > kcap)
    return fail(CRTG_ERR_DIMENSION,
                "inner dimension " + std::to_string(k) + " exceeds " + std::to_string(kcap));
  if ((a_colmajor ? lda < m : lda < k) || (b_colmajor ? ldb < k : ldb < n) || ldc < n)
    return fail(CRTG_ERR_DIMENSION, "leading dimension too small");
  const Plan P = make_plan(mode, m, n, k, N, n_block, true);
  if (!ws || ws_bytes < P.total)
    return fail(CRTG_ERR_WORKSPACE, "workspace too small: need " + std::to_string(P.total));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int elem = (precision & CRTG_IN_F32) ? E_F32 : E_F64;
  const size_t esz = (precision & CRTG_IN_F32) ? 4 : 8;
  const bool single = (precision & CRTG_SINGLE) != 0;
  unsigned long long* dg = diag ? reinterpret_cast<unsigned long long*>(diag)
                                : at<unsigned long long>(ws, P.diag);
  const DevConsts dc = make_dev(*K, true, unsigned_residues(k));
  int32_t* mu = at<int32_t>(ws, P.mu);
  int32_t* nu = at<int32_t>(ws, P.nu);
  double* rowabs = at<double>(ws, P.rowabs);
  double* colabs = at<double>(ws, P.colabs);
  CRTG_TRY(cudaMemsetAsync(dg, 0, 8 * CRTG_DIAG_LEN, s), "memset");
  CRTG_TRY(cudaMemsetAsync(rowabs, 0, P.rowabs.bytes, s), "memset");
  CRTG_TRY(cudaMemsetAsync(colabs, 0, P.colabs.bytes, s), "memset");
  // operand A rows: row-major -> row kernels; column-major -> column kernels on A^T.
  // operand B columns: row-major -> column kernels; column-major -> row kernels on B^T.
  // diag offsets: the row kernels report into (NONFINITE_A, CLAMPED_MU), the column
  // kernels into (NONFINITE_B, CLAMPED_NU); +-1 re-targets them to the other operand.
  {
    StageTimer timer(CRTG_STAGE_SCALING, s);
    PwTree tree{};
    if (mode == CRTG_FAST) {
      if (int e = load_tree(P, ws, s, tree)) return e;
      if (!a_colmajor) {
        CRTG_TRY(launch_row_stats(elem, true, A, lda, m, k, tree, dc.p_fast, dc.delta, mu, rowabs,
                                  dg, s), "row stats");
      } else {
        CRTG_TRY(launch_col_fast(elem, A, lda, k, m, rowabs, at<double>(ws, P.rowsq), dc.p_fast,
                                 dc.delta, mu, dg - 1, s), "col sumsq");
      }
      if (!b_colmajor) {
        CRTG_TRY(launch_col_fast(elem, B, ldb, k, n, colabs, at<double>(ws, P.colsq), dc.p_fast,
                                 dc.delta, nu, dg, s), "col sumsq");
      } else {
        CRTG_TRY(launch_row_stats(elem, true, B, ldb, n, k, tree, dc.p_fast, dc.delta, nu, colabs,
                                  dg + 1, s), "row stats");
      }
    } else {
      // accurate: absmax -> bars -> bound operands -> tcgen05 bound GEMM -> exponents
      if (!a_colmajor)
        CRTG_TRY(launch_row_stats(elem, false, A, lda, m, k, tree, dc.p_fast, dc.delta, nullptr,
                                  rowabs, dg, s), "row absmax");
      else
        CRTG_TRY(launch_col_absmax(elem, A, lda, k, m, rowabs, dg - 1, s), "col absmax");
      if (!b_colmajor)
        CRTG_TRY(launch_col_absmax(elem, B, ldb, k, n, colabs, dg, s), "col absmax");
      else
        CRTG_TRY(launch_row_stats(elem, false, B, ldb, n, k, tree, dc.p_fast, dc.delta, nullptr,
                                  colabs, dg + 1, s), "row absmax");
      int32_t* bar_mu = at<int32_t>(ws, P.bar_mu);
      int32_t* bar_nu = at<int32_t>(ws, P.bar_nu);
      int32_t* rowmax = at<int32_t>(ws, P.rowmax);
      int32_t* colmax = at<int32_t>(ws, P.colmax);
      CRTG_TRY(cudaMemsetAsync(rowmax, 0, P.rowmax.bytes, s), "memset");
      CRTG_TRY(cudaMemsetAsync(colmax, 0, P.colmax.bytes, s), "memset");
      CRTG_TRY(launch_bar(rowabs, m, bar_mu, s), "bar");
      CRTG_TRY(launch_bar(colabs, n, bar_nu, s), "bar");
      const int64_t a_plane = P.m_pad * P.k_pad, b_plane = P.n_pad * P.k_pad;
      int8_t* abars = at<int8_t>(ws, P.a_bars);
      int8_t* bbars = at<int8_t>(ws, P.b_bars);
      // bars of a real operand: sum and difference planes are both A, so the
      // complex bound (X + |D|)/2 reduces to the real bound A*B (scaling.py:257-258)
      CRTG_TRY(launch_pack(elem, a_colmajor ? 1 : 0, PACK_BARS, A, lda, m, k, 0, bar_mu, dc, abars,
                           a_plane, P.m_pad / 128, dg + CRTG_DIAG_OVERFLOW_A, s), "bars A");
      CRTG_TRY(launch_pack(elem, b_colmajor ? 0 : 1, PACK_BARS, B, ldb, n, k, 0, bar_nu, dc, bbars,
                           b_plane, P.n_pad / 128, dg + CRTG_DIAG_OVERFLOW_B, s), "bars B");
      GemmArgs g{};
      g.a = abars;
      g.b = bbars;
      g.a_plane = a_plane;
      g.b_plane = b_plane;
      g.a_rb = int(P.m_pad / 128);
      g.b_rb = int(P.n_pad / 128);
      g.mt = int(P.m_pad / 128);
      g.nt = int(P.n_pad / 256);
      g.kb = int(P.k_pad / 128);
      g.nl = 1;
      g.planes_per_l = 3;
      g.nphase = 3;
      g.m = int(m);
      g.n = int(n);
      g.row_max = rowmax;
      g.col_max = colmax;
      CRTG_TRY(launch_gemm(EPI_BOUND, g, sm_count(), s), "bound gemm");
      CRTG_TRY(launch_accurate_exps(rowmax, rowabs, bar_mu, m, dc.p_accu, dc.delta, mu,
                                    dg + CRTG_DIAG_CLAMPED_MU, s), "accurate mu");
      CRTG_TRY(launch_accurate_exps(colmax, colabs, bar_nu, n, dc.p_accu, dc.delta, nu,
                                    dg + CRTG_DIAG_CLAMPED_NU, s), "accurate nu");
    }
  }
  // residues of A: one plane per modulus
  const int64_t a_plane = P.m_pad * P.k_pad;
  int8_t* apack = at<int8_t>(ws, P.a_pack);
  {
    StageTimer timer(CRTG_STAGE_RESIDUE_A, s);
    CRTG_TRY(launch_pack(elem, a_colmajor ? 1 : 0, PACK_RESIDUE, A, lda, m, k, 0, mu, dc, apack,
                         a_plane, P.m_pad / 128, dg + CRTG_DIAG_OVERFLOW_A, s), "residues A");
  }
  int8_t* bpack = at<int8_t>(ws, P.b_pack);
  int8_t* ere = at<int8_t>(ws, P.e_re);
  const size_t csz = single ? 4 : 8;
  for (int64_t j0 = 0; j0 < n; j0 += P.nb) {
    const int64_t w = std::min(P.nb, n - j0), w_pad = round_up(w, 256);
    {
      StageTimer timer(CRTG_STAGE_RESIDUE_B, s);
      if (!b_colmajor)
        CRTG_TRY(launch_pack(elem, 1, PACK_RESIDUE, B, ldb, w, k, j0, nu + j0, dc, bpack,
                             w_pad * P.k_pad, w_pad / 128, dg + CRTG_DIAG_OVERFLOW_B, s),
                 "residues B");
      else
        CRTG_TRY(launch_pack(elem, 0, PACK_RESIDUE, static_cast<const char*>(B) + j0 * ldb * esz,
                             ldb, w, k, 0, nu + j0, dc, bpack, w_pad * P.k_pad, w_pad / 128,
                             dg + CRTG_DIAG_OVERFLOW_B, s),
                 "residues B");
    }
    GemmArgs g{};
    g.a = apack;
    g.b = bpack;
    g.a_plane = a_plane;
    g.b_plane = w_pad * P.k_pad;
    g.a_rb = int(P.m_pad / 128);
    g.b_rb = int(w_pad / 128);
    g.mt = int(P.m_pad / 128);
    g.nt = int(w_pad / 256);
    g.kb = int(P.k_pad / 128);
    g.nl = N;
    g.planes_per_l = 1;
    g.nphase = 1;
    g.m = int(m);
    g.n = int(w);
    g.e_re = ere;
    g.e_ld = P.nb_pad;
    g.e_plane = m * P.nb_pad;
    g.overflow = dg + CRTG_DIAG_INT32_OVERFLOW;
    for (int l = 0; l < N; ++l) g.mc[l] = dc.mc[l];
    g.uns = dc.uns;
    {
      StageTimer timer(CRTG_STAGE_GEMM, s);
      CRTG_TRY(run_gemm(EPI_REAL, g, s), "real gemm");
    }
    {
      StageTimer timer(CRTG_STAGE_CRT, s);
      CRTG_TRY(launch_crt(single, true, m, w, ere, nullptr, g.e_plane, g.e_ld, mu, nu + j0, dc,
                          static_cast<char*>(C) + j0 * csz, ldc, s),
               "crt");
    }
  }
  if (mu_out) CRTG_TRY(cudaMemcpyAsync(mu_out, mu, 4 * m, cudaMemcpyDeviceToDevice, s), "copy");
  if (nu_out) CRTG_TRY(cudaMemcpyAsync(nu_out, nu, 4 * n, cudaMemcpyDeviceToDevice, s), "copy");
  if (sync_check) return check_diag(dg, s);
  return CRTG_OK;
}

// ---------------------------------------------------------------------------
// Accuracy harness: reference_gemm_dd + max_relative_error
// ---------------------------------------------------------------------------
extern "C" int crtg_dd_gemm(int is_complex, int64_t m, int64_t n, int64_t k, const void* A,
                            int64_t lda, const void* B, int64_t ldb, void* hi, void* lo,
                            int64_t ldo, void* stream) {
  if (m < 1 || n < 1 || k < 1) return fail(CRTG_ERR_DIMENSION, "m, n, k must be positive");
  if (lda < k || ldb < n || ldo < n) return fail(CRTG_ERR_DIMENSION, "leading dimension too small");
  CRTG_TRY(launch_dd_gemm(is_complex != 0, m, n, k, static_cast<const double*>(A), lda,
                          static_cast<const double*>(B), ldb, static_cast<double*>(hi),
                          static_cast<double*>(lo), ldo, static_cast<cudaStream_t>(stream)),
           "dd gemm");
  return CRTG_OK;
}

extern "C" int crtg_max_relative_error(int is_complex, int64_t m, int64_t n, const void* approx,
                                       int approx_single, int64_t ld_approx, const void* hi,
                                       const void* lo, int64_t ldo, uint64_t* max_bits,
                                       uint64_t* zero_count, void* stream) {
  if (m < 1 || n < 1) return fail(CRTG_ERR_DIMENSION, "empty matrix");
  CRTG_TRY(launch_max_rel_err(is_complex != 0, m, n, approx, approx_single != 0, ld_approx,
                              static_cast<const double*>(hi), static_cast<const double*>(lo), ldo,
                              reinterpret_cast<unsigned long long*>(max_bits),
                              reinterpret_cast<unsigned long long*>(zero_count),
                              static_cast<cudaStream_t>(stream)),
           "max relative error");
  return CRTG_OK;
}

// ---------------------------------------------------------------------------
// stage-level API (include/crtg.h "stage-level entry points")
// ---------------------------------------------------------------------------
namespace {
int stage_flags(uint64_t* flags, int n, cudaStream_t s) {
  if (!flags) return fail(CRTG_ERR_CONFIG, "a device flags array is required");
  CRTG_TRY(cudaMemsetAsync(flags, 0, 8 * size_t(n), s), "memset");
  return CRTG_OK;
}

int stage_read_flags(const uint64_t* flags, int n, unsigned long long* h, cudaStream_t s) {
  CRTG_TRY(cudaMemcpyAsync(h, flags, 8 * size_t(n), cudaMemcpyDeviceToHost, s), "flags copy");
  CRTG_TRY(cudaStreamSynchronize(s), "sync");
  return CRTG_OK;
}
}  // namespace

extern "C" {

int crtg_log2_upper(const double* x, int64_t n, float* out, uint64_t* flags, int sync_check,
                    void* stream) {
  if (n < 0) return fail(CRTG_ERR_DIMENSION, "negative length");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int e = stage_flags(flags, 1, s)) return e;
  auto* f = reinterpret_cast<unsigned long long*>(flags);
  CRTG_TRY(launch_log2_upper(x, n, out, f, s), "log2_upper");
  if (!sync_check) return CRTG_OK;
  unsigned long long h[1];
  if (int e = stage_read_flags(flags, 1, h, s)) return e;
  if (h[0]) return fail(CRTG_ERR_DOMAIN, "log2_upper requires positive finite input");
  return CRTG_OK;
}

int crtg_quantize(const double* x, int64_t rows, int64_t cols, int64_t ldx, const int64_t* exps,
                  int axis, double* out, int64_t ldo, uint64_t* flags, int sync_check,
                  void* stream) {
  if (rows < 0 || cols < 0) return fail(CRTG_ERR_DIMENSION, "negative extent");
  if (axis != 0 && axis != 1) return fail(CRTG_ERR_CONFIG, "axis must be 0 (rows) or 1 (columns)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int e = stage_flags(flags, 1, s)) return e;
  auto* f = reinterpret_cast<unsigned long long*>(flags);
  CRTG_TRY(launch_quantize(x, rows, cols, ldx, exps, axis, out, ldo, f, s), "quantize");
  if (!sync_check) return CRTG_OK;
  unsigned long long h[1];
  if (int e = stage_read_flags(flags, 1, h, s)) return e;
  if (h[0]) return fail(CRTG_ERR_DOMAIN, "scaled magnitudes exceed the quantization budget");
  return CRTG_OK;
}

int crtg_symmetric_mod(int kind, const void* x, int64_t count, const int32_t* moduli, int nmod,
                       int8_t* out, uint64_t* flags, int sync_check, void* stream) {
  if ((kind & ~8) < 0 || (kind & ~8) > 2)
    return fail(CRTG_ERR_CONFIG, "kind must be 0 (f64), 1 (i64) or 2 (i32), plus 8 for strict");
  if (nmod < 1 || nmod > CRTG_MAX_MODULI) return fail(CRTG_ERR_CONFIG, "need 1..20 moduli");
  if (count < 0) return fail(CRTG_ERR_DIMENSION, "negative length");
  SymModuli mods{};
  mods.n = nmod;
  for (int l = 0; l < nmod; ++l) {
    if (moduli[l] < 2 || moduli[l] > 256)
      return fail(CRTG_ERR_DOMAIN, "modulus must be in [2, 256]");
    mods.p[l] = moduli[l];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (int e = stage_flags(flags, 3, s)) return e;
  auto* f = reinterpret_cast<unsigned long long*>(flags);
  CRTG_TRY(launch_sym_mod(kind, x, count, mods, out, f, s), "symmetric residues");
  if (!sync_check) return CRTG_OK;
  unsigned long long h[3];
  if (int e = stage_read_flags(flags, 3, h, s)) return e;
  if (h[0]) return fail(CRTG_ERR_DOMAIN, "matrix entries must be finite");
  if (h[1])
    return fail(CRTG_ERR_DOMAIN, (kind & 3) == 0 ? "matrix entries must be below 2^90"
                                                 : "integer entries must be below 2^61");
  if (h[2]) return fail(CRTG_ERR_DOMAIN, "matrix entries must be integer-valued");
  return CRTG_OK;
}

int crtg_crt_accumulate(const int8_t* e, int64_t count, const crtg_consts* K, int single,
                        double* s1, double* s2, void* stream) {
  int N = 0;
  if (int r = check_consts(K, &N)) return r;
  if (count < 0) return fail(CRTG_ERR_DIMENSION, "negative length");
  CrtCoeffs cf{};
  for (int l = 0; l < N; ++l) {
    cf.hi[l] = K->coeff_hi[l];
    cf.lo[l] = K->coeff_lo[l];
  }
  CRTG_TRY(launch_crt_accumulate(e, N, count, cf, single != 0, s1, s2,
                                 static_cast<cudaStream_t>(stream)),
           "crt_accumulate");
  return CRTG_OK;
}

int crtg_symmetric_mod_wide(const double* s_hi, const double* s_lo, int64_t count, double p_hi,
                            double p_lo, int use_dd, double* out, void* stream) {
  if (count < 0) return fail(CRTG_ERR_DIMENSION, "negative length");
  CRTG_TRY(launch_sym_mod_wide(s_hi, s_lo, count, p_hi, p_lo, use_dd != 0, out,
                               static_cast<cudaStream_t>(stream)),
           "symmetric_mod_wide");
  return CRTG_OK;
}

int crtg_inverse_scale(const double* c, int64_t rows, int64_t cols, int64_t ldc, const int64_t* mu,
                       const int64_t* nu, int out_f32, void* out, int64_t ldo, void* stream) {
  if (rows < 0 || cols < 0) return fail(CRTG_ERR_DIMENSION, "negative extent");
  CRTG_TRY(launch_inverse_scale(c, rows, cols, ldc, mu, nu, out_f32 != 0, out, ldo,
                                static_cast<cudaStream_t>(stream)),
           "inverse_scale");
  return CRTG_OK;
}

}  // extern "C"
