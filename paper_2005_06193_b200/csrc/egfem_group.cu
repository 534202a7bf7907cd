// Batched tensor action (step (2b), cfg5) by row groups with compiled-in sparsity (B200 / sm_100a).
//
//   R_{i,p} = Σ_{(j,k)} T_ijk U_{j,p} W_{k,p}       for p < batch
//
// Why groups.  For W = V forms row i of T lives on the square stencil N(i) × N(i) (the cell
// clique around i).  In a P2 (or any higher-order) space many rows' stencils are subsets of a
// neighbour's: every P2 edge-midpoint row i has N(i) ⊆ N(v) for both end vertices v.  Rows that
// share one stencil form a group (leader = the row with the widest stencil containing the
// member's, ties to the lowest index; cfg5: one vertex + the midpoints of its three
// "forward" edges).  A warp owns one group and 32·P pairs: it loads W at the group stencil into
// registers once (|N|·P values), then for each stencil point a (ascending j)
//     U_a (P values, one load)
//     X_{m,a} = Σ_b T_{m, N_a, N_b} W_b           for each member m with fiber (m, N_a)
//     R_m    += U_a X_{m,a}
// so each W value feeds every nonzero of the group in its column (≈ 18 FMAs per value for
// cfg5 instead of ≈ 8.6 per row), each U value every member's fiber at a (4 instead of 1),
// and each T value P FMAs (broadcast load, sequential in program order).
//
// Why compiled.  Register-resident W needs compile-time indices and skipping T's zeros
// without branches needs the pattern in the instruction stream: the builder hashes each
// group's pattern (stencil width, members, and per member the fibers and their k positions),
// and for the frequent pattern classes generates one straight-line kernel each (NVRTC, one
// program per tensor, sm_100a CUBIN, loaded with cudaLibraryLoadData).  The group's values are
// packed in exactly the kernel's FMA order, so the T stream is one contiguous sequential read.
// Rows of rare classes (boundary corners of small meshes, unstructured leftovers) run the
// per-row dense-block kernel (egfem_dense.cu, `launch_dense_rows`).
//
// Summation order: X_{m,a} over b ascending (k ascending), R_m over a ascending (j ascending):
// the fiber-factored canonical order of the row; fixed, so bitwise reproducible.
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <atomic>
#include <mutex>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include "egfem_internal.cuh"

namespace egfem {

// Kernel variants of a class: bit 0 = U and W are the same array (the u-slot values are the
// W registers already loaded: no U loads), bit 1 = batch is a multiple of 32·P (no pair guards),
// bit 2 = one pair per lane (batches below 64 or odd multiples of 32: a rank's shard of a
// sharded batch) instead of the plan's P, bit 3 = the symmetrized pattern (U == W only, below).
//
// Symmetrized pattern.  With U == W (the pairs (u, w = u) of the Burgers term (u·∇)u, PAPER.md
// L396) the row action is a quadratic form, R_{i,p} = Σ_{j,k} T_ijk u_j u_k, so it equals
//   R_{i,p} = Σ_j u_j Σ_{k ≥ j} S_ijk u_k,   S_ijk = T_ijk + T_ikj (k > j),  S_ijj = T_ijj,
// which needs one FMA per (j ≤ k) pair instead of one per nonzero: cfg5's 26.1 M FMAs per pair
// drop to ≈ 16 M.  The builder keeps, per class, the symmetrized pattern and S packed in its
// FMA order (rounded once); the generated kernel is the same straight-line form.  The sums
// run in a different order than the unsymmetrized kernel (graded by tolerance against the
// oracle, like every kernel); EGFEM_GROUP_SYM=0 disables it.
// Bit 4 = the symmetrized pattern at P = 4 pairs per lane (U == W, batch >= 128; P = 4 under a
// 168-register cap measured best there: cfg5 0.49 ms at P = 2 / 120 registers, 0.433 at P = 2 /
// 96, 0.428 at P = 4 / 168).
constexpr int kVariants = 32;

struct GroupClass {
  int n = 0;       // group stencil width |N(leader)|
  int g = 0;       // members (leader first)
  int nv = 0;      // value record stride (nonzeros rounded up to 16 bytes)
  int ncp = 0;     // column record stride (n rounded up to 4)
  int64_t ninst = 0;
  int32_t* cols = nullptr;  // ninst × ncp: global column of stencil point b
  int32_t* rows = nullptr;  // ninst × g: member rows
  void* vals = nullptr;     // ninst × nv, dtype: T values in FMA program order
  std::vector<int32_t> key; // the pattern (Pattern::key), kept to generate variants on demand
  std::vector<int32_t> skey;  // the symmetrized pattern (U == W), empty when disabled
  int snv = 0;                // its value record stride
  void* svals = nullptr;      // ninst × snv, dtype: S values in its FMA program order
  cudaKernel_t fn[kVariants] = {};
  int per_sm[kVariants] = {};     // resident CTAs per SM (registers), for the persistent grid
  size_t dyn_set[kVariants] = {};  // dynamic shared memory the kernel was opted in for
  int carve_set[kVariants] = {};
};

struct GroupPlan {
  int pairs_per_lane = 2;
  int run = 4;  // consecutive instances per CTA run
  int interleave = 4;  // fiber chains interleaved in the generated code
  int prefetch = 0;  // unstaged form: 1 = bulk L2 prefetch one CTA round ahead (measured slower on cfg5)
  bool persistent = false;  // grid = resident CTAs (else up to `cap` CTAs per SM of runs)
  int cap = 32;
  int carveout = -1;  // preferred shared-memory carveout in percent (-1: driver default)
  bool staged = false;    // full variants: W tiles by TMA bulk copies (kernel_source_staged; measured slower on cfg5)
  bool sym = false;       // symmetrized classes built (the U == W launches take them)
  int sym_P = 4;          // their pairs per lane for batches >= 128 (EGFEM_GROUP_SYM_P: 2 keeps the plan's P)
  bool f64 = true;
  std::vector<GroupClass> classes;
  std::vector<cudaLibrary_t> libs;
  std::mutex mu;         // guards the lazily compiled variants and the side streams
  std::mutex launch_mu;  // one enqueue at a time: the fork event and side streams are shared
  // side streams for the small classes and the fallback rows (fork-join around the big class)
  int side_dev = -1;
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_done;
  cudaEvent_t fork = nullptr;
  // rows outside the compiled classes: per stencil width (width, first entry, count)
  int32_t* fb_rows = nullptr;
  std::vector<std::array<int64_t, 3>> fb_classes;
  int64_t fb_count = 0;
  std::string info;
};

namespace {

// One group pattern: per member the fibers (a) and per fiber the k positions (b), all as
// positions in the leader's stencil.
struct Pattern {
  int n = 0;
  std::vector<std::vector<std::pair<int, std::vector<int>>>> members;
  std::vector<int32_t> key() const {
    std::vector<int32_t> s{n, (int)members.size()};
    for (const auto& m : members) {
      s.push_back((int)m.size());
      for (const auto& f : m) {
        s.push_back(f.first);
        s.push_back((int)f.second.size());
        s.insert(s.end(), f.second.begin(), f.second.end());
      }
    }
    return s;
  }
  int nnz() const {
    int c = 0;
    for (const auto& m : members)
      for (const auto& f : m) c += (int)f.second.size();
    return c;
  }
};

struct KeyHash {
  size_t operator()(const std::vector<int32_t>& v) const {
    uint64_t h = 1469598103934665603ull;
    for (int32_t x : v) {
      h ^= (uint32_t)x;
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

// Record strides of a class's packed arrays (16-byte aligned records for cp.async).
inline int cols_stride(int n) { return (n + 3) & ~3; }
inline int vals_stride(int nnz, int vs) { const int per16 = 16 / vs; return (nnz + per16 - 1) / per16 * per16; }

// Contiguous pair mapping (full variants): lane l owns pairs P·l .. P·l+P-1 of its 32·P chunk,
// so its values at one node are P consecutive elements: loaded / stored as 16-byte vectors.
std::string vec_load(const char* S, int P, const std::string& dst, const std::string& ptr) {
  std::string o;
  char b[256];
  const bool dbl = std::strcmp(S, "double") == 0;
  if (P == 1) {
    std::snprintf(b, sizeof(b), "const %s %s_0 = __ldg(%s);", S, dst.c_str(), ptr.c_str());
    return b;
  }
  const int per = dbl ? 2 : (P >= 4 ? 4 : 2);  // elements per vector load
  const char* V = dbl ? "double2" : (per == 4 ? "float4" : "float2");
  for (int v = 0; v < P / per; ++v) {
    std::snprintf(b, sizeof(b), "const %s %s_v%d = __ldg(reinterpret_cast<const %s*>(%s) + %d); ", V, dst.c_str(), v, V,
                  ptr.c_str(), v);
    o += b;
    const char* comp[4] = {"x", "y", "z", "w"};
    for (int e = 0; e < per; ++e) {
      std::snprintf(b, sizeof(b), "const %s %s_%d = %s_v%d.%s; ", S, dst.c_str(), v * per + e, dst.c_str(), v, comp[e]);
      o += b;
    }
  }
  return o;
}

std::string vec_store(const char* S, int P, const std::string& ptr, const std::string& src) {
  std::string o;
  char b[256];
  const bool dbl = std::strcmp(S, "double") == 0;
  if (P == 1) {
    std::snprintf(b, sizeof(b), "*(%s) = %s_0;", ptr.c_str(), src.c_str());
    return b;
  }
  const int per = dbl ? 2 : (P >= 4 ? 4 : 2);
  for (int v = 0; v < P / per; ++v) {
    if (dbl)
      std::snprintf(b, sizeof(b), "reinterpret_cast<double2*>(%s)[%d] = make_double2(%s_%d, %s_%d); ", ptr.c_str(), v,
                    src.c_str(), 2 * v, src.c_str(), 2 * v + 1);
    else if (per == 4)
      std::snprintf(b, sizeof(b), "reinterpret_cast<float4*>(%s)[%d] = make_float4(%s_%d, %s_%d, %s_%d, %s_%d); ",
                    ptr.c_str(), v, src.c_str(), 4 * v, src.c_str(), 4 * v + 1, src.c_str(), 4 * v + 2, src.c_str(),
                    4 * v + 3);
    else
      std::snprintf(b, sizeof(b), "reinterpret_cast<float2*>(%s)[%d] = make_float2(%s_%d, %s_%d); ", ptr.c_str(), v,
                    src.c_str(), 2 * v, src.c_str(), 2 * v + 1);
    o += b;
  }
  return o;
}

void emit_body(std::string& o, const Pattern& pt, const char* S, int P, bool same, bool full, int IL, int nv,
               const char* indent, bool contig = false,
               const std::function<std::string(int)>& lazy_w = std::function<std::string(int)>());

// Straight-line kernel source for one pattern class.  P pairs per lane (lane, lane+32, ...).
// A CTA walks runs of `run` consecutive instances (runs dealt round-robin, so the CTAs in flight
// cover one moving window of the mesh and consecutive instances of a run share most of their
// stencil in L1); each instance's column record and value record are staged in shared memory
// by cp.async one instance ahead (double buffer), and the CTA's warps take its 32·P-pair chunks.
// same: U == W (u_a is the register w_a); full: batch % (32·P) == 0 (no guards).
std::string kernel_source(const Pattern& pt, const std::string& name, const char* S, int P, bool same, bool full,
                          int IL, int maxreg = -1) {
  const int n = pt.n, g = (int)pt.members.size();
  const int vs = std::strcmp(S, "double") == 0 ? 8 : 4;
  const int nv = vals_stride(pt.nnz(), vs), ncp = cols_stride(n);
  std::string o;
  char buf[512];
  auto emit = [&](const char* fmt, auto... a) {
    std::snprintf(buf, sizeof(buf), fmt, a...);
    o += buf;
  };
  // register cap: 120 registers give 4 resident 128-thread CTAs (16 warps/SM) — the DFMA chains
  // and the W loads that start an instance need the extra warps (cfg5, P = 2: 130 → 120
  // registers, 12 → 16 warps, 0.673 → 0.639 ms, no spills).  Applied when the instance state
  // (W and the member accumulators, P doubles each) is small; EGFEM_GROUP_MAXREG overrides
  // (0 = no cap).
  static const int env_reg = std::getenv("EGFEM_GROUP_MAXREG") ? std::atoi(std::getenv("EGFEM_GROUP_MAXREG")) : -1;
  const int maxnreg = env_reg >= 0 ? env_reg : maxreg >= 0 ? maxreg : (2 * P * (n + g) <= 96 && P <= 2 ? 120 : 0);
  if (maxnreg > 0)
    emit("extern \"C\" __global__ void __maxnreg__(%d) %s(const int* __restrict__ gcols, "
         "const int* __restrict__ grows, const %s* __restrict__ gvals, long long ninst, int B, int run, int pf, "
         "const %s* __restrict__ U, const %s* __restrict__ W, %s* __restrict__ R) {\n",
         maxnreg, name.c_str(), S, S, S, S);
  else
    emit("extern \"C\" __global__ void __launch_bounds__(128) %s(const int* __restrict__ gcols, "
         "const int* __restrict__ grows, const %s* __restrict__ gvals, long long ninst, int B, int run, int pf, "
         "const %s* __restrict__ U, const %s* __restrict__ W, %s* __restrict__ R) {\n",
         name.c_str(), S, S, S, S);
  emit("  __shared__ __align__(16) %s s_v[2][%d];\n", S, nv);
  emit("  __shared__ __align__(16) int s_c[2][%d];\n", ncp);
  emit("  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;\n");
  emit("  const int nch = (B + %d) / %d;\n", 32 * P - 1, 32 * P);
  emit("  const long long gstride = (long long)gridDim.x * run;\n");
  emit("  auto gof = [&](int q) { const int r = q / run; return (long long)blockIdx.x * run + r * gstride + (q - r * run); };\n");
  emit("  auto stage = [&](long long gi, int b) {\n");
  emit("    if (gi >= ninst) return;\n");
  emit("    const char* vsrc = reinterpret_cast<const char*>(gvals + gi * %d);\n", nv);
  emit("    const char* csrc = reinterpret_cast<const char*>(gcols + gi * %d);\n", ncp);
  emit("    for (int x = threadIdx.x; x < %d; x += blockDim.x) {\n", nv * vs / 16 + ncp / 4);
  emit("      const bool isv = x < %d;\n", nv * vs / 16);
  emit("      char* dst = isv ? reinterpret_cast<char*>(s_v[b]) + 16 * x : reinterpret_cast<char*>(s_c[b]) + 16 * (x - %d);\n",
       nv * vs / 16);
  emit("      const char* src = isv ? vsrc + 16 * x : csrc + 16 * (x - %d);\n", nv * vs / 16);
  emit("      asm volatile(\"cp.async.cg.shared.global [%%0], [%%1], 16;\" :: \"r\"((unsigned)__cvta_generic_to_shared(dst)), \"l\"(src) : \"memory\");\n");
  emit("    }\n  };\n");
  // value / column records one instance ahead (double buffer)
  emit("  if (gof(0) >= ninst) return;\n");
  emit("  stage(gof(0), 0);\n");
  emit("  asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  emit("  for (int q = 0;; ++q) {\n");
  emit("    const long long gi = gof(q);\n");
  emit("    if (gi >= ninst) break;\n");
  emit("    stage(gof(q + 1), (q + 1) & 1);\n");
  emit("    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  // pf == 1: L2 bulk prefetch of the W (and U) node rows of the instance one CTA round ahead
  emit("    if (pf == 1 && threadIdx.x < %d) {\n", n);
  emit("      const long long ga = gi + gstride;\n");
  emit("      if (ga < ninst) {\n");
  emit("        const long long c = __ldg(gcols + ga * %d + threadIdx.x);\n", ncp);
  emit("        asm volatile(\"cp.async.bulk.prefetch.L2.global [%%0], %%1;\" :: \"l\"(W + c * B), \"r\"((unsigned)(B * %d)) : \"memory\");\n", vs);
  if (!same)
    emit("        asm volatile(\"cp.async.bulk.prefetch.L2.global [%%0], %%1;\" :: \"l\"(U + c * B), \"r\"((unsigned)(B * %d)) : \"memory\");\n", vs);
  emit("      }\n    }\n");
  emit("    asm volatile(\"cp.async.wait_group 1;\" ::: \"memory\");\n");
  emit("    __syncthreads();\n");
  emit("    const %s* sv = s_v[q & 1];\n", S);
  emit("    const int* sc = s_c[q & 1];\n");
  emit("    for (int ch = warp; ch < nch; ch += nw) {\n");
  if (full)
    emit("      const int p0 = ch * %d + %d * lane;\n", 32 * P, P);
  else
    emit("      const int p0 = ch * %d + lane;\n", 32 * P);
  emit("      const %s* Wp = W + p0;\n", S);
  if (!same) emit("      const %s* Up = U + p0;\n", S);
  if (!full)
    for (int q = 0; q < P; ++q) emit("      const bool ok%d = p0 + %d < B;\n", q, 32 * q);
  static const bool lazy = std::getenv("EGFEM_GROUP_LAZY") && std::getenv("EGFEM_GROUP_LAZY")[0] == '1';
  std::function<std::string(int)> lazy_w;
  if (full && lazy) {  // W loads emitted before their first use (the compiler hoists as registers allow)
    for (int b = 0; b < n; ++b)
      for (int q = 0; q < P; ++q) emit("      %s w%d_%d;\n", S, b, q);
    lazy_w = [&, S, P](int b) {
      std::string bs = std::to_string(b);
      std::string l = vec_load(S, P, "lw" + bs, "(Wp + (long long)sc[" + bs + "] * B)");
      std::string a = "{ " + l;
      for (int q = 0; q < P; ++q) a += " w" + bs + "_" + std::to_string(q) + " = lw" + bs + "_" + std::to_string(q) + ";";
      return a + " }";
    };
  } else {
    for (int b = 0; b < n; ++b) {
      emit("      const %s* wc%d = Wp + (long long)sc[%d] * B;\n", S, b, b);
      if (full) {
        o += "      " + vec_load(S, P, "w" + std::to_string(b), "wc" + std::to_string(b)) + "\n";
        continue;
      }
      for (int q = 0; q < P; ++q)
        emit("      const %s w%d_%d = ok%d ? __ldg(wc%d + %d) : (%s)0;\n", S, b, q, q, b, 32 * q, S);
    }
  }
  emit("      {\n");
  emit_body(o, pt, S, P, same, full, IL, nv, "        ", full, lazy_w);
  for (int m = 0; m < g; ++m) {
    emit("      { %s* rr = R + (long long)__ldg(grows + gi * %d + %d) * B + p0;\n", S, g, m);
    if (full) {
      o += "        " + vec_store(S, P, "rr", "r" + std::to_string(m)) + "\n";
    } else {
      for (int q = 0; q < P; ++q) emit("        if (ok%d) rr[%d] = r%d_%d;\n", q, 32 * q, m, q);
    }
    emit("      }\n");
  }
  emit("      }\n");
  emit("    }\n");
  emit("    __syncthreads();\n");
  emit("  }\n}\n");
  return o;
}

// The compute body shared by both kernel forms: register W (w<b>_<q>) is loaded; emits the
// u values, the interleaved fiber chains and the accumulators r<m>_<q>.  `uload(a, q)` gives
// the expression of U at stencil point a for pair slot q when U != W.
void emit_body(std::string& o, const Pattern& pt, const char* S, int P, bool same, bool full, int IL, int nv,
               const char* indent, bool contig, const std::function<std::string(int)>& lazy_w) {
  const int n = pt.n, g = (int)pt.members.size();
  char buf[512];
  auto emit = [&](const char* fmt, auto... a) {
    o += indent;
    std::snprintf(buf, sizeof(buf), fmt, a...);
    o += buf;
  };
  for (int x = 0; x < nv / 2; ++x) emit("%s2 t%d;\n", S, x);
  std::vector<char> r_live(g, 0), loaded(nv / 2 + 1, 0);
  for (int m = 0; m < g; ++m)
    for (int q = 0; q < P; ++q) emit("%s r%d_%d;\n", S, m, q);
  int e = 0;
  std::vector<char> w_done(n, 0);
  for (int a = 0; a < n; ++a) {
    bool any = false;
    for (int m = 0; m < g; ++m)
      for (const auto& f : pt.members[m]) any |= f.first == a;
    if (!any) continue;
    if (lazy_w) {  // W values first used at this stencil point: loaded here (shorter live ranges)
      std::vector<int> need;
      if (same) need.push_back(a);
      for (int m = 0; m < g; ++m)
        for (const auto& f : pt.members[m])
          if (f.first == a) need.insert(need.end(), f.second.begin(), f.second.end());
      for (int b : need)
        if (!w_done[b]) {
          w_done[b] = 1;
          o += indent;
          o += lazy_w(b) + "\n";
        }
    }
    emit("{\n");
    if (same) {
      for (int q = 0; q < P; ++q) emit("  const %s u%d = w%d_%d;\n", S, q, a, q);
    } else {
      emit("  const %s* uc = Up + (long long)sc[%d] * B;\n", S, a);
      if (full && contig) {
        o += indent;
        o += "  " + vec_load(S, P, "uu", "uc") + "\n";
        for (int q = 0; q < P; ++q) emit("  const %s u%d = uu_%d;\n", S, q, q);
      } else {
        for (int q = 0; q < P; ++q) {
          if (full)
            emit("  const %s u%d = __ldg(uc + %d);\n", S, q, 32 * q);
          else
            emit("  const %s u%d = ok%d ? __ldg(uc + %d) : (%s)0;\n", S, q, q, 32 * q, S);
        }
      }
    }
    struct Fib {
      int m;
      const std::vector<int>* bs;
      int e0;
    };
    std::vector<Fib> fa;
    for (int m = 0; m < g; ++m)
      for (const auto& f : pt.members[m])
        if (f.first == a) {
          fa.push_back({m, &f.second, e});
          e += (int)f.second.size();
        }
    for (size_t f0 = 0; f0 < fa.size(); f0 += IL) {
      const size_t f1 = std::min(fa.size(), f0 + (size_t)IL);
      emit("  {\n");
      size_t len = 0;
      for (size_t f = f0; f < f1; ++f) {
        len = std::max(len, fa[f].bs->size());
        for (int q = 0; q < P; ++q) emit("    %s x%d_%d;\n", S, (int)(f - f0), q);
      }
      for (size_t st = 0; st < len; ++st)
        for (size_t f = f0; f < f1; ++f) {
          if (st >= fa[f].bs->size()) continue;
          const int ee = fa[f].e0 + (int)st, b = (*fa[f].bs)[st];
          if (!loaded[ee >> 1]) {
            emit("    t%d = *reinterpret_cast<const %s2*>(sv + %d);\n", ee >> 1, S, ee & ~1);
            loaded[ee >> 1] = 1;
          }
          for (int q = 0; q < P; ++q) {
            if (st == 0)
              emit("    x%d_%d = t%d.%c * w%d_%d;\n", (int)(f - f0), q, ee >> 1, (ee & 1) ? 'y' : 'x', b, q);
            else
              emit("    x%d_%d = fma(t%d.%c, w%d_%d, x%d_%d);\n", (int)(f - f0), q, ee >> 1, (ee & 1) ? 'y' : 'x',
                   b, q, (int)(f - f0), q);
          }
        }
      for (size_t f = f0; f < f1; ++f) {
        const int m = fa[f].m;
        if (fa[f].bs->empty())
          for (int q = 0; q < P; ++q) emit("    x%d_%d = (%s)0;\n", (int)(f - f0), q, S);
        for (int q = 0; q < P; ++q) {
          if (r_live[m])
            emit("    r%d_%d = fma(u%d, x%d_%d, r%d_%d);\n", m, q, q, (int)(f - f0), q, m, q);
          else
            emit("    r%d_%d = u%d * x%d_%d;\n", m, q, q, (int)(f - f0), q);
        }
        r_live[m] = 1;
      }
      emit("  }\n");
    }
    emit("}\n");
  }
  for (int m = 0; m < g; ++m)
    if (!r_live[m])
      for (int q = 0; q < P; ++q) emit("r%d_%d = (%s)0;\n", m, q, S);
}

// Staged form (batch % (32·P) == 0): each warp's W tile (its 32·P pairs at the n stencil nodes,
// one contiguous row segment per node in the node-major layout) arrives by TMA 1D bulk copies
// (cp.async.bulk + mbarrier) one instance ahead, so the loads that start an instance are shared-
// memory loads; value and column records are staged by cp.async two instances ahead (triple
// buffer: the columns of the next instance address its W copies).  Pair blocks of nw·32·P pairs
// are the grid's y dimension.
std::string kernel_source_staged(const Pattern& pt, const std::string& name, const char* S, int P, bool same,
                                 int IL) {
  const int n = pt.n, g = (int)pt.members.size();
  const int vs = std::strcmp(S, "double") == 0 ? 8 : 4;
  const int nv = vals_stride(pt.nnz(), vs), ncp = cols_stride(n);
  const int PW = 32 * P;
  std::string o;
  char buf[640];
  auto emit = [&](const char* fmt, auto... a) {
    std::snprintf(buf, sizeof(buf), fmt, a...);
    o += buf;
  };
  emit("extern \"C\" __global__ void __launch_bounds__(128) %s(const int* __restrict__ gcols, "
       "const int* __restrict__ grows, const %s* __restrict__ gvals, long long ninst, int B, int run, int pf, "
       "const %s* __restrict__ U, const %s* __restrict__ W, %s* __restrict__ R) {\n",
       name.c_str(), S, S, S, S);
  emit("  extern __shared__ __align__(128) unsigned char s_dyn[];\n");
  emit("  __shared__ __align__(16) %s s_v[3][%d];\n", S, nv);
  emit("  __shared__ __align__(16) int s_c[3][%d];\n", ncp);
  emit("  __shared__ __align__(8) unsigned long long s_bar[4];\n");
  emit("  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;\n");
  emit("  %s* s_w = reinterpret_cast<%s*>(s_dyn) + (size_t)warp * %d;\n", S, S, n * PW);
  emit("  const int pw0 = blockIdx.y * nw * %d + warp * %d;\n", PW, PW);
  emit("  const int p0 = pw0 + lane;\n");
  emit("  const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar[warp]);\n");
  emit("  const long long gstride = (long long)gridDim.x * run;\n");
  emit("  auto gof = [&](long long q) { return (long long)blockIdx.x * run + (q / run) * gstride + (q %% run); };\n");
  emit("  auto stage = [&](long long gi, int b) {\n");
  emit("    if (gi >= ninst) return;\n");
  emit("    const char* vsrc = reinterpret_cast<const char*>(gvals + gi * %d);\n", nv);
  emit("    const char* csrc = reinterpret_cast<const char*>(gcols + gi * %d);\n", ncp);
  emit("    for (int x = threadIdx.x; x < %d; x += blockDim.x) {\n", nv * vs / 16 + ncp / 4);
  emit("      const bool isv = x < %d;\n", nv * vs / 16);
  emit("      char* dst = isv ? reinterpret_cast<char*>(s_v[b]) + 16 * x : reinterpret_cast<char*>(s_c[b]) + 16 * (x - %d);\n",
       nv * vs / 16);
  emit("      const char* src = isv ? vsrc + 16 * x : csrc + 16 * (x - %d);\n", nv * vs / 16);
  emit("      asm volatile(\"cp.async.cg.shared.global [%%0], [%%1], 16;\" :: \"r\"((unsigned)__cvta_generic_to_shared(dst)), \"l\"(src) : \"memory\");\n");
  emit("    }\n  };\n");
  emit("  auto issue_w = [&](long long gi, int cb) {\n");
  emit("    if (gi >= ninst) return;\n");
  emit("    if (lane == 0) asm volatile(\"mbarrier.arrive.expect_tx.shared::cta.b64 _, [%%0], %%1;\" :: \"r\"(bar), \"r\"(%d) : \"memory\");\n",
       n * PW * vs);
  emit("    __syncwarp();\n");
  emit("    if (lane < %d) {\n", n);
  emit("      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n");
  emit("      const %s* src = W + (long long)s_c[cb][lane] * B + pw0;\n", S);
  emit("      const unsigned dst = (unsigned)__cvta_generic_to_shared(s_w + lane * %d);\n", PW);
  emit("      asm volatile(\"cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%%0], [%%1], %%2, [%%3];\" :: \"r\"(dst), \"l\"(src), \"r\"(%d), \"r\"(bar) : \"memory\");\n",
       PW * vs);
  emit("    }\n  };\n");
  emit("  if (gof(0) >= ninst) return;\n");
  emit("  if (lane == 0) {\n");
  emit("    asm volatile(\"mbarrier.init.shared::cta.b64 [%%0], 1;\" :: \"r\"(bar) : \"memory\");\n");
  emit("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n");
  emit("  }\n");
  emit("  stage(gof(0), 0);\n");
  emit("  stage(gof(1), 1);\n");
  emit("  asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  emit("  asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n");
  emit("  __syncthreads();\n");
  emit("  issue_w(gof(0), 0);\n");
  emit("  int b0 = 0;\n");  // buffer of instance q (q % 3)
  emit("  for (long long q = 0;; ++q) {\n");
  emit("    const long long gi = gof(q);\n");
  emit("    if (gi >= ninst) break;\n");
  emit("    const int b1 = b0 == 2 ? 0 : b0 + 1, b2 = b1 == 2 ? 0 : b1 + 1;\n");
  emit("    stage(gof(q + 2), b2);\n");
  emit("    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  emit("    asm volatile(\"{\\n.reg .pred p;\\nWAIT_%%=:\\nmbarrier.try_wait.parity.shared::cta.b64 p, [%%0], %%1;\\n@!p bra WAIT_%%=;\\n}\\n\" :: \"r\"(bar), \"r\"((unsigned)(q & 1)) : \"memory\");\n");
  for (int b = 0; b < n; ++b)
    for (int q = 0; q < P; ++q) emit("    const %s w%d_%d = s_w[%d + lane];\n", S, b, q, b * PW + 32 * q);
  emit("    __syncwarp();\n");
  emit("    issue_w(gof(q + 1), b1);\n");
  emit("    const %s* sv = s_v[b0];\n", S);
  emit("    const int* sc = s_c[b0];\n");
  if (!same) emit("    const %s* Up = U + p0;\n", S);
  emit("    {\n");
  emit_body(o, pt, S, P, same, true, IL, nv, "      ");
  for (int m = 0; m < g; ++m) {
    emit("      { %s* rr = R + (long long)__ldg(grows + gi * %d + %d) * B + p0;\n", S, g, m);
    for (int q = 0; q < P; ++q) emit("        rr[%d] = r%d_%d;\n", 32 * q, m, q);
    emit("      }\n");
  }
  emit("    }\n");
  emit("    asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n");
  emit("    __syncthreads();\n");
  emit("    b0 = b1;\n");
  emit("  }\n}\n");
  return o;
}

Pattern pattern_from_key(const std::vector<int32_t>& key) {
  Pattern pt;
  size_t x = 0;
  pt.n = key[x++];
  const int g = key[x++];
  for (int m = 0; m < g; ++m) {
    const int nf = key[x++];
    std::vector<std::pair<int, std::vector<int>>> fibs;
    for (int f = 0; f < nf; ++f) {
      const int a = key[x++], c = key[x++];
      std::vector<int> bs(key.begin() + x, key.begin() + x + c);
      x += c;
      fibs.push_back({a, bs});
    }
    pt.members.push_back(fibs);
  }
  return pt;
}

// Process-wide cache of compiled programs (tests rebuild the same tensors many times).
std::mutex g_cache_mu;
std::unordered_map<std::string, std::vector<char>> g_cubins;

egfem_status compile_cubin(const std::string& src, std::vector<char>* cubin, std::string* log_out) {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cubins.find(src);
    if (it != g_cubins.end()) {
      *cubin = it->second;
      return EGFEM_OK;
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "egfem_group.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    set_error("nvrtcCreateProgram failed");
    return EGFEM_ERR_CUDA;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--ptxas-options=-v"};
  const nvrtcResult cr = nvrtcCompileProgram(prog, 4, opts);
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  std::string log(ls, '\0');
  if (ls) nvrtcGetProgramLog(prog, &log[0]);
  if (log_out) *log_out = log;
  if (const char* e = getenv("EGFEM_GROUP_LOG"))
    if (e[0] == '1') std::fprintf(stderr, "[egfem_group] NVRTC log:\n%s\n", log.c_str());
  if (cr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    set_error("NVRTC compile of the grouped batched kernels failed: " + log.substr(0, 2000));
    return EGFEM_ERR_CUDA;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cubins[src] = *cubin;
  return EGFEM_OK;
}

template <typename T>
egfem_status upload(T** d, const std::vector<T>& h) {
  EGFEM_CUDA_TRY(cudaMalloc(d, sizeof(T) * std::max<size_t>(h.size(), 1)));
  if (!h.empty()) EGFEM_CUDA_TRY(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return EGFEM_OK;
}

int g_sms_grp[64] = {0};

}  // namespace

void free_group_plan(GroupPlan* gp) {
  if (!gp) return;
  for (auto& c : gp->classes) {
    if (c.cols) cudaFree(c.cols);
    if (c.rows) cudaFree(c.rows);
    if (c.vals) cudaFree(c.vals);
    if (c.svals) cudaFree(c.svals);
  }
  if (gp->fb_rows) cudaFree(gp->fb_rows);
  for (cudaLibrary_t l : gp->libs) cudaLibraryUnload(l);
  for (cudaStream_t x : gp->side) cudaStreamDestroy(x);
  for (cudaEvent_t x : gp->side_done) cudaEventDestroy(x);
  if (gp->fork) cudaEventDestroy(gp->fork);
  delete gp;
}

const char* group_plan_info(const egfem_tensor* t) { return t->grp ? t->grp->info.c_str() : ""; }

// Offline: row groups, pattern classes, packed values and the compiled kernels (W = V tensors
// that have dense blocks).  EGFEM_GROUPS=0 disables the path; EGFEM_GROUP_P sets P (1, 2, 4).
egfem_status make_groups(egfem_tensor* t, const std::vector<int64_t>& hrf) {
  if (!t->blk || !t->w_is_v || t->n_u <= 0 || t->nnz <= 0) return EGFEM_OK;
  if (const char* e = getenv("EGFEM_GROUPS"))
    if (e[0] == '0') return EGFEM_OK;
  int P = 2;  // pairs per lane (measured on cfg5: P = 2 at 16 warps/SM beats P = 4 at 8)
  if (const char* e = getenv("EGFEM_GROUP_P")) P = std::max(1, std::min(4, atoi(e)));
  int run = 2;
  if (const char* e = getenv("EGFEM_GROUP_RUN")) run = std::max(1, atoi(e));
  const int64_t n_u = t->n_u, n_fib = t->n_fib, nnz = t->nnz;
  std::vector<int32_t> fj(n_fib);
  std::vector<uint32_t> fnz(n_fib + 1), nk(nnz);
  EGFEM_CUDA_TRY(cudaMemcpy(fj.data(), t->fib_j, 4 * n_fib, cudaMemcpyDeviceToHost));
  EGFEM_CUDA_TRY(cudaMemcpy(fnz.data(), t->fib_nz, 4 * (n_fib + 1), cudaMemcpyDeviceToHost));
  EGFEM_CUDA_TRY(cudaMemcpy(nk.data(), t->nz_k, 4 * nnz, cudaMemcpyDeviceToHost));
  const bool f64 = t->dtype == EGFEM_F64;
  const size_t vs = f64 ? 8 : 4;
  std::vector<unsigned char> hv(vs * nnz);
  EGFEM_CUDA_TRY(cudaMemcpy(hv.data(), t->nz_val, vs * nnz, cudaMemcpyDeviceToHost));
  const uint32_t km = t->kmask();
  auto sten = [&](int64_t i) { return std::make_pair(fj.data() + hrf[i], (int)(hrf[i + 1] - hrf[i])); };
  auto subset = [&](int64_t i, int64_t l) {  // N(i) ⊆ N(l), both ascending
    auto [a, na] = sten(i);
    auto [b, nb] = sten(l);
    return std::includes(b, b + nb, a, a + na);
  };
  // owner: the widest stencil containing N(i) (ties: lowest row); candidates lie in N(i).  A
  // partitioned handle addresses columns in its window: column c is local row c − doff
  const int64_t doff = t->row_begin - t->col_begin;
  std::vector<int32_t> owner(n_u);
  for (int64_t i = 0; i < n_u; ++i) {
    auto [a, na] = sten(i);
    int64_t best = i;
    for (int x = 0; x < na; ++x) {
      const int64_t l = a[x] - doff;
      if (l == i || l < 0 || l >= n_u) continue;
      const int nl = (int)(hrf[l + 1] - hrf[l]);
      const int nbst = (int)(hrf[best + 1] - hrf[best]);
      if ((nl > nbst || (nl == nbst && l < best)) && subset(i, l)) best = l;
    }
    owner[i] = (int32_t)best;
  }
  constexpr int kMaxMembers = 12;
  std::vector<std::vector<int32_t>> members(n_u);
  std::vector<int32_t> leaders;
  for (int64_t i = 0; i < n_u; ++i) {
    int64_t o = owner[i];
    if (owner[o] != o || (int)members[o].size() >= kMaxMembers) o = i;  // chains / overfull: own group
    if (o == i) {
      members[i].insert(members[i].begin(), (int32_t)i);
      leaders.push_back((int32_t)i);
    } else {
      members[o].push_back((int32_t)i);
    }
  }
  // Rows that joined a group before its leader was seen are fine (leader inserted first above
  // only for i == o; fix the order: leader first, members ascending).
  for (int32_t l : leaders) {
    auto& m = members[l];
    std::sort(m.begin(), m.end());
    auto it = std::find(m.begin(), m.end(), l);
    std::rotate(m.begin(), it, it + 1);
  }
  std::sort(leaders.begin(), leaders.end());
  // patterns
  std::unordered_map<std::vector<int32_t>, int, KeyHash> cls_of;
  std::vector<Pattern> cls_pat;
  std::vector<std::vector<int32_t>> cls_inst;
  for (int32_t l : leaders) {
    auto [lc, ln] = sten(l);
    Pattern pt;
    pt.n = ln;
    auto posof = [&](int32_t col) { return (int)(std::lower_bound(lc, lc + ln, col) - lc); };
    for (int32_t m : members[l]) {
      std::vector<std::pair<int, std::vector<int>>> fibs;
      for (int64_t f = hrf[m]; f < hrf[m + 1]; ++f) {
        std::vector<int> bs;
        for (uint32_t e = fnz[f]; e < fnz[f + 1]; ++e) bs.push_back(posof((int32_t)(nk[e] & km)));
        fibs.push_back({posof(fj[f]), bs});
      }
      pt.members.push_back(fibs);
    }
    auto key = pt.key();
    auto it = cls_of.find(key);
    int c;
    if (it == cls_of.end()) {
      c = (int)cls_pat.size();
      cls_of.emplace(key, c);
      cls_pat.push_back(pt);
      cls_inst.push_back({});
    } else {
      c = it->second;
    }
    cls_inst[c].push_back(l);
  }
  // compiled classes: frequent ones (≥ 8 instances), the 24 most frequent at most
  std::vector<int> order(cls_pat.size());
  for (size_t c = 0; c < order.size(); ++c) order[c] = (int)c;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cls_inst[x].size() > cls_inst[y].size(); });
  std::vector<int> chosen;
  for (int c : order)
    if (cls_inst[c].size() >= 8 && chosen.size() < 24) chosen.push_back(c);
  std::vector<char> in_fb(cls_pat.size(), 1);
  for (int c : chosen) in_fb[c] = 0;
  auto* gp = new GroupPlan();
  gp->pairs_per_lane = P;
  gp->run = run;
  gp->interleave = 4;
  if (const char* e = getenv("EGFEM_GROUP_IL")) gp->interleave = std::max(1, atoi(e));
  if (const char* e = getenv("EGFEM_GROUP_PF")) gp->prefetch = atoi(e);
  if (const char* e = getenv("EGFEM_GROUP_STAGED")) gp->staged = e[0] != '0';
  if (const char* e = getenv("EGFEM_GROUP_PERSIST")) gp->persistent = e[0] != '0';
  if (const char* e = getenv("EGFEM_GROUP_CAP")) gp->cap = std::max(1, atoi(e));
  if (const char* e = getenv("EGFEM_GROUP_CARVE")) gp->carveout = atoi(e);
  gp->sym = true;
  if (const char* e = getenv("EGFEM_GROUP_SYM")) gp->sym = e[0] != '0';
  if (const char* e = getenv("EGFEM_GROUP_SYM_P")) gp->sym_P = atoi(e) == 4 ? 4 : 2;
  gp->f64 = f64;
  for (size_t x = 0; x < chosen.size(); ++x) {
    GroupClass gc;
    const Pattern& pt = cls_pat[chosen[x]];
    gc.n = pt.n;
    gc.g = (int)pt.members.size();
    gc.nv = vals_stride(pt.nnz(), (int)vs);
    gc.ncp = cols_stride(pt.n);
    gc.ninst = (int64_t)cls_inst[chosen[x]].size();
    gc.key = pt.key();
    gp->classes.push_back(std::move(gc));
    gp->info += " [class " + std::to_string(x) + ": width " + std::to_string(pt.n) + ", " +
                std::to_string(pt.members.size()) + " rows, " + std::to_string(cls_inst[chosen[x]].size()) +
                " groups]";
  }
  // per-class device arrays: columns, member rows, values in program order
  int64_t fma_can = 0, fma_sym = 0;
  for (size_t x = 0; x < chosen.size(); ++x) {
    GroupClass& gc = gp->classes[x];
    const Pattern& pt = cls_pat[chosen[x]];
    const auto& inst = cls_inst[chosen[x]];
    std::vector<int32_t> hc((size_t)gc.ninst * gc.ncp, 0), hr((size_t)gc.ninst * gc.g);
    std::vector<unsigned char> hvals((size_t)gc.ninst * gc.nv * vs, 0);
    for (int64_t q = 0; q < gc.ninst; ++q) {
      const int32_t l = inst[q];
      auto [lc, ln] = sten(l);
      std::copy(lc, lc + ln, hc.begin() + q * gc.ncp);
      const auto& mem = members[l];
      for (int m = 0; m < gc.g; ++m) hr[q * gc.g + m] = mem[m];
      // program order: a ascending, members in order, then the fiber's nonzeros (k ascending)
      int e = 0;
      for (int a = 0; a < gc.n; ++a)
        for (int m = 0; m < gc.g; ++m) {
          const int32_t row = mem[m];
          for (int fi = 0; fi < (int)pt.members[m].size(); ++fi) {
            if (pt.members[m][fi].first != a) continue;
            const int64_t f = hrf[row] + fi;
            for (uint32_t z = fnz[f]; z < fnz[f + 1]; ++z, ++e)
              std::memcpy(&hvals[((size_t)q * gc.nv + e) * vs], &hv[(size_t)z * vs], vs);
          }
        }
    }
    egfem_status st;
    if ((st = upload(&gc.cols, hc)) || (st = upload(&gc.rows, hr))) {
      free_group_plan(gp);
      return st;
    }
    unsigned char* dv = nullptr;
    if ((st = upload(&dv, hvals))) {
      free_group_plan(gp);
      return st;
    }
    gc.vals = dv;
    if (!gp->sym) continue;
    // the symmetrized pattern (U == W): per member the (a ≤ b) pairs of T's (a, b) ∪ (b, a) nonzeros
    const int n = gc.n, g = gc.g;
    Pattern sp;
    sp.n = n;
    for (int m = 0; m < g; ++m) {
      std::vector<char> on((size_t)n * n, 0);
      for (const auto& f : pt.members[m])
        for (int b : f.second) on[(size_t)std::min(f.first, b) * n + std::max(f.first, b)] = 1;
      std::vector<std::pair<int, std::vector<int>>> fibs;
      for (int a = 0; a < n; ++a) {
        std::vector<int> bs;
        for (int b = a; b < n; ++b)
          if (on[(size_t)a * n + b]) bs.push_back(b);
        if (!bs.empty()) fibs.push_back({a, bs});
      }
      sp.members.push_back(fibs);
    }
    gc.skey = sp.key();
    gc.snv = vals_stride(sp.nnz(), (int)vs);
    auto fmas = [](const Pattern& x) {  // FMAs per pair and instance: one per nonzero, one per fiber
      int c = x.nnz();
      for (const auto& m : x.members) c += (int)m.size();
      return (int64_t)c;
    };
    fma_can += gc.ninst * fmas(pt);
    fma_sym += gc.ninst * fmas(sp);
    std::vector<unsigned char> hs((size_t)gc.ninst * gc.snv * vs, 0);
    std::vector<double> dense((size_t)g * n * n, 0.0);
    std::vector<size_t> touched;
    auto val = [&](size_t z) {
      if (f64) {
        double x;
        std::memcpy(&x, &hv[z * vs], 8);
        return x;
      }
      float x;
      std::memcpy(&x, &hv[z * vs], 4);
      return (double)x;
    };
    for (int64_t q = 0; q < gc.ninst; ++q) {
      const auto& mem = members[inst[q]];
      for (size_t z : touched) dense[z] = 0.0;
      touched.clear();
      for (int m = 0; m < g; ++m)
        for (int fi = 0; fi < (int)pt.members[m].size(); ++fi) {
          const int64_t f = hrf[mem[m]] + fi;
          const int a = pt.members[m][fi].first;
          const auto& bs = pt.members[m][fi].second;
          for (uint32_t z = fnz[f]; z < fnz[f + 1]; ++z) {
            const size_t at = ((size_t)m * n + a) * n + bs[z - fnz[f]];
            dense[at] = val(z);
            touched.push_back(at);
          }
        }
      // S in the kernel's program order: a ascending, members in order, b ascending
      int e = 0;
      for (int a = 0; a < n; ++a)
        for (int m = 0; m < g; ++m)
          for (const auto& f : sp.members[m]) {
            if (f.first != a) continue;
            for (int b : f.second) {
              const double x = a == b ? dense[((size_t)m * n + a) * n + a]
                                      : dense[((size_t)m * n + a) * n + b] + dense[((size_t)m * n + b) * n + a];
              unsigned char* dst = &hs[((size_t)q * gc.snv + e++) * vs];
              if (f64) {
                std::memcpy(dst, &x, 8);
              } else {
                const float xf = (float)x;
                std::memcpy(dst, &xf, 4);
              }
            }
          }
    }
    unsigned char* ds = nullptr;
    if ((st = upload(&ds, hs))) {
      free_group_plan(gp);
      return st;
    }
    gc.svals = ds;
  }
  if (gp->sym)
    gp->info += " [U == W: symmetrized patterns, S_ijk = T_ijk + T_ikj for k > j: " + std::to_string(fma_sym) +
                " instead of " + std::to_string(fma_can) + " FMAs per pair in the compiled classes]";
  // fallback rows (rare classes), grouped by stencil width, row order within a width
  std::vector<int32_t> fb;
  for (size_t c = 0; c < cls_pat.size(); ++c)
    if (in_fb[c])
      for (int32_t l : cls_inst[c])
        for (int32_t m : members[l]) fb.push_back(m);
  std::stable_sort(fb.begin(), fb.end(), [&](int32_t x, int32_t y) {
    const int64_t nx = hrf[x + 1] - hrf[x], ny = hrf[y + 1] - hrf[y];
    return nx != ny ? nx < ny : x < y;
  });
  for (size_t s = 0; s < fb.size();) {
    const int64_t w = hrf[fb[s] + 1] - hrf[fb[s]];
    size_t e = s;
    while (e < fb.size() && hrf[fb[e] + 1] - hrf[fb[e]] == w) ++e;
    gp->fb_classes.push_back({w, (int64_t)s, (int64_t)(e - s)});
    s = e;
  }
  gp->fb_count = (int64_t)fb.size();
  if (!fb.empty()) {
    egfem_status st = upload(&gp->fb_rows, fb);
    if (st) {
      free_group_plan(gp);
      return st;
    }
  }
  t->grp = gp;
  return EGFEM_OK;
}

// Diagnostic (no GPU needed): generate and NVRTC-compile the kernel of a pattern given by its
// serialized key (Pattern::key: n, g, then per member the fiber count and per fiber (a, count,
// b...)).  EGFEM_GROUP_DUMP=<prefix> writes <prefix>.cu and <prefix>.cubin.
egfem_status group_compile_key(const int32_t* key, int32_t len, int P, int f64, std::string* log) {
  Pattern pt;
  int x = 0;
  auto next = [&](int32_t* v) {
    if (x >= len) return false;
    *v = key[x++];
    return true;
  };
  int32_t n = 0, g = 0;
  if (!next(&n) || !next(&g) || n < 1 || n > 64 || g < 1 || g > 32) return EGFEM_ERR_INVALID_ARGUMENT;
  pt.n = n;
  for (int m = 0; m < g; ++m) {
    int32_t nf = 0;
    if (!next(&nf) || nf < 0 || nf > n) return EGFEM_ERR_INVALID_ARGUMENT;
    std::vector<std::pair<int, std::vector<int>>> fibs;
    for (int f = 0; f < nf; ++f) {
      int32_t a = 0, c = 0;
      if (!next(&a) || !next(&c) || a < 0 || a >= n || c < 0 || c > n) return EGFEM_ERR_INVALID_ARGUMENT;
      std::vector<int> bs(c);
      for (int q = 0; q < c; ++q) {
        int32_t b = 0;
        if (!next(&b) || b < 0 || b >= n) return EGFEM_ERR_INVALID_ARGUMENT;
        bs[q] = b;
      }
      fibs.push_back({a, bs});
    }
    pt.members.push_back(fibs);
  }
  if (x != len) return EGFEM_ERR_INVALID_ARGUMENT;
  const int v = std::getenv("EGFEM_GROUP_VARIANT") ? std::atoi(std::getenv("EGFEM_GROUP_VARIANT")) : 0;
  const int il = std::getenv("EGFEM_GROUP_IL") ? std::max(1, std::atoi(std::getenv("EGFEM_GROUP_IL"))) : 2;
  const bool stg = ((v >> 1) & 1) && !(std::getenv("EGFEM_GROUP_STAGED") && std::getenv("EGFEM_GROUP_STAGED")[0] == '0');
  const std::string src = stg ? kernel_source_staged(pt, "egfem_grp_test", f64 ? "double" : "float", P, v & 1, il)
                              : kernel_source(pt, "egfem_grp_test", f64 ? "double" : "float", P, v & 1, (v >> 1) & 1, il);
  std::vector<char> cubin;
  egfem_status st = compile_cubin(src, &cubin, log);
  if (const char* d = getenv("EGFEM_GROUP_DUMP")) {
    if (FILE* f = std::fopen((std::string(d) + ".cu").c_str(), "w")) {
      std::fwrite(src.data(), 1, src.size(), f);
      std::fclose(f);
    }
    if (!st)
      if (FILE* f = std::fopen((std::string(d) + ".cubin").c_str(), "wb")) {
        std::fwrite(cubin.data(), 1, cubin.size(), f);
        std::fclose(f);
      }
  }
  return st;
}

bool group_path_ok(const egfem_tensor* t, egfem_layout layout) {
  return t->grp != nullptr && layout == EGFEM_LAYOUT_NODE_MAJOR;
}

// Compile variant v of every class (one NVRTC program per class, compiled on parallel host
// threads; process-wide cache keyed by source), on first use.
egfem_status ensure_variant(GroupPlan* gp, int v) {
  std::lock_guard<std::mutex> lk(gp->mu);
  const size_t nc = gp->classes.size();
  bool all = true;
  for (const auto& gc : gp->classes) all &= gc.fn[v] != nullptr;
  if (all) return EGFEM_OK;
  const bool same = v & 1, full = (v >> 1) & 1;
  const int P = (v & 4) ? 1 : (v & 16) ? 4 : gp->pairs_per_lane;
  // register caps of the symmetrized kernels (measured on cfg5, see kVariants)
  const int maxreg = (v & 8) ? (P == 4 ? 168 : P == 2 ? 96 : -1) : -1;
  std::vector<std::string> names(nc), srcs(nc);
  std::vector<std::vector<char>> cubins(nc);
  std::vector<egfem_status> sts(nc, EGFEM_OK);
  for (size_t c = 0; c < nc; ++c) {
    names[c] = "egfem_grp_" + std::to_string(c) + "_v" + std::to_string(v);
    const Pattern pt = pattern_from_key((v & 8) ? gp->classes[c].skey : gp->classes[c].key);
    const char* S = gp->f64 ? "double" : "float";
    srcs[c] = full && gp->staged ? kernel_source_staged(pt, names[c], S, P, same, gp->interleave)
                                 : kernel_source(pt, names[c], S, P, same, full, gp->interleave, maxreg);
  }
  std::vector<std::thread> th;
  std::atomic<size_t> next{0};
  const unsigned nt = std::max(1u, std::min<unsigned>((unsigned)nc, std::thread::hardware_concurrency()));
  std::vector<std::string> errs(nc);
  for (unsigned w = 0; w < nt; ++w)
    th.emplace_back([&] {
      for (size_t c = next++; c < nc; c = next++) {
        std::string log;
        sts[c] = compile_cubin(srcs[c], &cubins[c], &log);
        if (sts[c]) errs[c] = egfem_last_error();
      }
    });
  for (auto& t : th) t.join();
  for (size_t c = 0; c < nc; ++c) {
    if (sts[c]) {
      set_error(errs[c]);
      return sts[c];
    }
    cudaLibrary_t lib = nullptr;
    cudaError_t ce = cudaLibraryLoadData(&lib, cubins[c].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (ce != cudaSuccess) {
      set_error(std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce));
      return EGFEM_ERR_CUDA;
    }
    gp->libs.push_back(lib);
    ce = cudaLibraryGetKernel(&gp->classes[c].fn[v], lib, names[c].c_str());
    if (ce != cudaSuccess) {
      set_error(std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(ce));
      return EGFEM_ERR_CUDA;
    }
  }
  return EGFEM_OK;
}

constexpr int kSideStreams = 4;

egfem_status ensure_side(GroupPlan* gp, int dev) {
  std::lock_guard<std::mutex> lk(gp->mu);
  if (gp->side_dev == dev) return EGFEM_OK;
  gp->side.resize(kSideStreams);
  gp->side_done.resize(kSideStreams);
  for (int k = 0; k < kSideStreams; ++k) {
    EGFEM_CUDA_TRY(cudaStreamCreateWithFlags(&gp->side[k], cudaStreamNonBlocking));
    EGFEM_CUDA_TRY(cudaEventCreateWithFlags(&gp->side_done[k], cudaEventDisableTiming));
  }
  EGFEM_CUDA_TRY(cudaEventCreateWithFlags(&gp->fork, cudaEventDisableTiming));
  gp->side_dev = dev;
  return EGFEM_OK;
}

// The largest class runs on the caller's stream; the other classes and the fallback rows run
// concurrently on side streams (fork / join by events, so the call stays stream-ordered and
// CUDA-graph capturable): their launches are small and latency-bound, serialized they cost
// ≈ 20 % of the cfg5 action.
egfem_status launch_groups(const egfem_tensor* t, int32_t batch, const void* U, const void* W, void* R,
                           cudaStream_t s) {
  GroupPlan* gp = t->grp;
  const int dev = t->device & 63;
  if (!g_sms_grp[dev]) EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_grp[dev], cudaDevAttrMultiProcessorCount, t->device));
  // pairs per lane: the plan's P, or 1 for batches narrower than one 32·P chunk (e.g. a rank's
  // 32-pair shard of the 256 cfg5 pairs: 0.221 -> 0.172 ms); wider batches keep P (B = 96 at
  // P = 1 measured slower than B = 128 at P = 2)
  const bool sym = U == W && gp->sym;
  int P = gp->pairs_per_lane;
  const bool p4 = sym && gp->sym_P == 4 && batch >= 128;
  if (p4) P = 4;
  else if (P > 1 && batch < 32 * P) P = 1;
  const int nch = (batch + 32 * P - 1) / (32 * P);
  const int v = (U == W ? 1 : 0) | (batch % (32 * P) == 0 ? 2 : 0) | (P == 1 && gp->pairs_per_lane != 1 ? 4 : 0) |
                (sym ? 8 : 0) | (p4 ? 16 : 0);
  egfem_status st = ensure_variant(gp, v);
  if (st) return st;
  const size_t nc = gp->classes.size();
  const bool fork = nc + (gp->fb_count > 0 ? 1 : 0) > 1;
  // concurrent callers (other host threads, other streams) enqueue one after the other: the
  // fork / join events and the side streams are per handle (results stay ordered per stream)
  std::lock_guard<std::mutex> lk(gp->launch_mu);
  if (fork) {
    if ((st = ensure_side(gp, t->device))) return st;
    EGFEM_CUDA_TRY(cudaEventRecord(gp->fork, s));
    for (int k = 0; k < kSideStreams; ++k) EGFEM_CUDA_TRY(cudaStreamWaitEvent(gp->side[k], gp->fork, 0));
  }
  const bool staged = gp->staged && (v & 2);
  const size_t vsz0 = gp->f64 ? 8 : 4;
  int nw = std::min(4, nch);
  if (staged) {  // warps per CTA: a divisor of the chunk count whose W tiles fit 48 KB
    int maxn = 1;
    for (const auto& gc : gp->classes) maxn = std::max(maxn, gc.n);
    nw = 1;
    for (int d = std::min(4, nch); d >= 1; --d)
      if (nch % d == 0 && (size_t)d * maxn * 32 * P * vsz0 <= 48 * 1024) {
        nw = d;
        break;
      }
  }
  const int threads = 32 * nw;
  const int pblocks = staged ? nch / nw : 1;
  int next_side = 0;
  // bulk L2 prefetch needs 16-byte rows and 16-byte aligned arrays
  const size_t vsz = gp->f64 ? 8 : 4;
  const int pf = gp->prefetch == 1 ? (((size_t)batch * vsz) % 16 == 0 && ((uintptr_t)U % 16) == 0 &&
                                       ((uintptr_t)W % 16) == 0)
                                    : gp->prefetch;
  auto launch_class = [&](size_t c, cudaStream_t str) -> egfem_status {
    GroupClass& gc = gp->classes[c];
    const int64_t runs = (gc.ninst + gp->run - 1) / gp->run;
    if (gc.per_sm[v] == 0) {  // persistent grid: the resident CTAs walk the runs round-robin
      cudaFuncAttributes fa{};
      int per = 1;
      if (cudaFuncGetAttributes(&fa, (const void*)gc.fn[v]) == cudaSuccess && fa.numRegs > 0)
        per = std::max(1, std::min(32, 65536 / (std::max(fa.numRegs, 1) * threads)));
      else
        cudaGetLastError();
      gc.per_sm[v] = per;
    }
    const int64_t ctas =
        std::max<int64_t>(1, std::min<int64_t>(runs, (int64_t)g_sms_grp[dev] * (gp->persistent ? gc.per_sm[v] : gp->cap)));
    long long ninst = gc.ninst;
    int B = batch, run = gp->run, pfl = pf;
    void* vals = (v & 8) ? gc.svals : gc.vals;
    void* args[] = {(void*)&gc.cols, (void*)&gc.rows, (void*)&vals, &ninst, &B, &run, &pfl, (void*)&U, (void*)&W, &R};
    const size_t dyn = staged ? (size_t)nw * gc.n * 32 * P * vsz0 : 0;
    if (!gc.carve_set[v]) {  // L1 over shared memory: consecutive instances of a run share stencil rows
      if (gp->carveout >= 0)
        cudaFuncSetAttribute((const void*)gc.fn[v], cudaFuncAttributePreferredSharedMemoryCarveout, gp->carveout);
      cudaGetLastError();
      gc.carve_set[v] = 1;
    }
    if (dyn > 0 && gc.dyn_set[v] < dyn) {
      cudaError_t ce = cudaFuncSetAttribute((const void*)gc.fn[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (ce != cudaSuccess) {
        set_error(std::string("cudaFuncSetAttribute(dynamic smem ") + std::to_string(dyn) + "): " + cudaGetErrorString(ce));
        return EGFEM_ERR_CUDA;
      }
      gc.dyn_set[v] = dyn;
    }
    cudaError_t ce = cudaLaunchKernel((const void*)gc.fn[v], dim3((unsigned)ctas, (unsigned)pblocks), dim3(threads), args,
                                      dyn, str);
    if (ce != cudaSuccess) {
      set_error(std::string("grouped batched kernel launch (grid ") + std::to_string(ctas) + "x" +
                std::to_string(pblocks) + ", block " + std::to_string(threads) + ", dyn smem " + std::to_string(dyn) +
                "): " + cudaGetErrorString(ce));
      return EGFEM_ERR_CUDA;
    }
    count_launch();
    return EGFEM_OK;
  };
  // side work first (its CTAs are placed before the big class fills the machine)
  for (size_t c = 1; c < nc; ++c) {
    if ((st = launch_class(c, gp->side[next_side]))) return st;
    next_side = (next_side + 1) % kSideStreams;
  }
  if (gp->fb_count > 0) {
    cudaStream_t fs = fork ? gp->side[next_side] : s;
    if ((st = launch_dense_rows(t, batch, gp->fb_rows, gp->fb_classes, U, W, R, fs))) return st;
  }
  if (nc > 0 && (st = launch_class(0, s))) return st;
  if (fork)
    for (int k = 0; k < kSideStreams; ++k) {
      EGFEM_CUDA_TRY(cudaEventRecord(gp->side_done[k], gp->side[k]));
      EGFEM_CUDA_TRY(cudaStreamWaitEvent(s, gp->side_done[k], 0));
    }
  return EGFEM_OK;
}

}  // namespace egfem
