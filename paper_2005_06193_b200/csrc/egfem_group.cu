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
// W registers already loaded: no U loads), bit 1 = batch is a multiple of 32·P (no pair guards).
constexpr int kVariants = 4;

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
  cudaKernel_t fn[kVariants] = {nullptr, nullptr, nullptr, nullptr};
};

struct GroupPlan {
  int pairs_per_lane = 2;
  int run = 4;  // consecutive instances per CTA run
  bool f64 = true;
  std::vector<GroupClass> classes;
  std::vector<cudaLibrary_t> libs;
  std::mutex mu;  // guards the lazily compiled variants
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

// Straight-line kernel source for one pattern class.  P pairs per lane (lane, lane+32, ...).
// A CTA walks runs of `run` consecutive instances (runs dealt round-robin, so the CTAs in flight
// cover one moving window of the mesh and consecutive instances of a run share most of their
// stencil in L1); each instance's column record and value record are staged in shared memory
// by cp.async one instance ahead (double buffer), and the CTA's warps take its 32·P-pair chunks.
// same: U == W (u_a is the register w_a); full: batch % (32·P) == 0 (no guards).
std::string kernel_source(const Pattern& pt, const std::string& name, const char* S, int P, bool same, bool full) {
  const int n = pt.n, g = (int)pt.members.size();
  const int vs = std::strcmp(S, "double") == 0 ? 8 : 4;
  const int nv = vals_stride(pt.nnz(), vs), ncp = cols_stride(n);
  std::string o;
  char buf[512];
  auto emit = [&](const char* fmt, auto... a) {
    std::snprintf(buf, sizeof(buf), fmt, a...);
    o += buf;
  };
  emit("extern \"C\" __global__ void __launch_bounds__(128) %s(const int* __restrict__ gcols, "
       "const int* __restrict__ grows, const %s* __restrict__ gvals, long long ninst, int B, int run, "
       "const %s* __restrict__ U, const %s* __restrict__ W, %s* __restrict__ R) {\n",
       name.c_str(), S, S, S, S);
  emit("  __shared__ __align__(16) %s s_v[2][%d];\n", S, nv);
  emit("  __shared__ __align__(16) int s_c[2][%d];\n", ncp);
  emit("  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;\n");
  emit("  const int nch = (B + %d) / %d;\n", 32 * P - 1, 32 * P);
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
  emit("  if (gof(0) >= ninst) return;\n");
  emit("  stage(gof(0), 0);\n");
  emit("  asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  emit("  for (long long q = 0;; ++q) {\n");
  emit("    const long long gi = gof(q);\n");
  emit("    if (gi >= ninst) break;\n");
  emit("    stage(gof(q + 1), (int)((q + 1) & 1));\n");
  emit("    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n");
  emit("    asm volatile(\"cp.async.wait_group 1;\" ::: \"memory\");\n");
  emit("    __syncthreads();\n");
  emit("    const %s* sv = s_v[q & 1];\n", S);
  emit("    const int* sc = s_c[q & 1];\n");
  emit("    for (int ch = warp; ch < nch; ch += nw) {\n");
  emit("      const int p0 = ch * %d + lane;\n", 32 * P);
  emit("      const %s* Wp = W + p0;\n", S);
  if (!same) emit("      const %s* Up = U + p0;\n", S);
  if (!full)
    for (int q = 0; q < P; ++q) emit("      const bool ok%d = p0 + %d < B;\n", q, 32 * q);
  for (int x = 0; x < nv / 2; ++x) emit("      %s2 t%d;\n", S, x);
  for (int b = 0; b < n; ++b) {
    emit("      const %s* wc%d = Wp + (long long)sc[%d] * B;\n", S, b, b);
    for (int q = 0; q < P; ++q) {
      if (full)
        emit("      const %s w%d_%d = __ldg(wc%d + %d);\n", S, b, q, b, 32 * q);
      else
        emit("      const %s w%d_%d = ok%d ? __ldg(wc%d + %d) : (%s)0;\n", S, b, q, q, b, 32 * q, S);
    }
  }
  // program order: stencil point a ascending; members in order; b ascending.  The first product
  // of every chain is a plain multiply (fma(a, b, 0) rounds identically), so no zero-fills.
  std::vector<char> r_live(g, 0);
  for (int m = 0; m < g; ++m)
    for (int q = 0; q < P; ++q) emit("      %s r%d_%d;\n", S, m, q);
  int e = 0;
  for (int a = 0; a < n; ++a) {
    bool any = false;
    for (int m = 0; m < g; ++m)
      for (const auto& f : pt.members[m]) any |= f.first == a;
    if (!any) continue;
    emit("      {\n");
    if (same) {
      for (int q = 0; q < P; ++q) emit("        const %s u%d = w%d_%d;\n", S, q, a, q);
    } else {
      emit("        const %s* uc = Up + (long long)sc[%d] * B;\n", S, a);
      for (int q = 0; q < P; ++q) {
        if (full)
          emit("        const %s u%d = __ldg(uc + %d);\n", S, q, 32 * q);
        else
          emit("        const %s u%d = ok%d ? __ldg(uc + %d) : (%s)0;\n", S, q, q, 32 * q, S);
      }
    }
    for (int m = 0; m < g; ++m)
      for (const auto& f : pt.members[m]) {
        if (f.first != a) continue;
        emit("        {\n");
        for (int q = 0; q < P; ++q) emit("          %s x%d;\n", S, q);
        bool first = true;
        for (int b : f.second) {
          if ((e & 1) == 0) emit("          t%d = *reinterpret_cast<const %s2*>(sv + %d);\n", e >> 1, S, e);
          for (int q = 0; q < P; ++q) {
            if (first)
              emit("          x%d = t%d.%c * w%d_%d;\n", q, e >> 1, (e & 1) ? 'y' : 'x', b, q);
            else
              emit("          x%d = fma(t%d.%c, w%d_%d, x%d);\n", q, e >> 1, (e & 1) ? 'y' : 'x', b, q, q);
          }
          first = false;
          ++e;
        }
        if (f.second.empty())
          for (int q = 0; q < P; ++q) emit("          x%d = (%s)0;\n", q, S);
        for (int q = 0; q < P; ++q) {
          if (r_live[m])
            emit("          r%d_%d = fma(u%d, x%d, r%d_%d);\n", m, q, q, q, m, q);
          else
            emit("          r%d_%d = u%d * x%d;\n", m, q, q, q);
        }
        r_live[m] = 1;
        emit("        }\n");
      }
    emit("      }\n");
  }
  for (int m = 0; m < g; ++m)
    if (!r_live[m])
      for (int q = 0; q < P; ++q) emit("      r%d_%d = (%s)0;\n", m, q, S);
  for (int m = 0; m < g; ++m) {
    emit("      { %s* rr = R + (long long)__ldg(grows + gi * %d + %d) * B + p0;\n", S, g, m);
    for (int q = 0; q < P; ++q) {
      if (full)
        emit("        rr[%d] = r%d_%d;\n", 32 * q, m, q);
      else
        emit("        if (ok%d) rr[%d] = r%d_%d;\n", q, 32 * q, m, q);
    }
    emit("      }\n");
  }
  emit("    }\n");
  emit("    __syncthreads();\n");
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
  }
  if (gp->fb_rows) cudaFree(gp->fb_rows);
  for (cudaLibrary_t l : gp->libs) cudaLibraryUnload(l);
  delete gp;
}

const char* group_plan_info(const egfem_tensor* t) { return t->grp ? t->grp->info.c_str() : ""; }

// Offline: row groups, pattern classes, packed values and the compiled kernels (W = V tensors
// that have dense blocks).  EGFEM_GROUPS=0 disables the path; EGFEM_GROUP_P sets P (1, 2, 4).
egfem_status make_groups(egfem_tensor* t, const std::vector<int64_t>& hrf) {
  if (!t->blk || !t->w_is_v || t->n_u <= 0 || t->nnz <= 0) return EGFEM_OK;
  if (const char* e = getenv("EGFEM_GROUPS"))
    if (e[0] == '0') return EGFEM_OK;
  int P = 2;
  if (const char* e = getenv("EGFEM_GROUP_P")) P = std::max(1, std::min(4, atoi(e)));
  int run = 4;
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
  // owner: the widest stencil containing N(i) (ties: lowest row); candidates lie in N(i)
  std::vector<int32_t> owner(n_u);
  for (int64_t i = 0; i < n_u; ++i) {
    auto [a, na] = sten(i);
    int64_t best = i;
    for (int x = 0; x < na; ++x) {
      const int64_t l = a[x];
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
  std::vector<int32_t> pos(0);
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
  }
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
  const std::string src = kernel_source(pt, "egfem_grp_test", f64 ? "double" : "float", P, v & 1, (v >> 1) & 1);
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
  std::vector<std::string> names(nc), srcs(nc);
  std::vector<std::vector<char>> cubins(nc);
  std::vector<egfem_status> sts(nc, EGFEM_OK);
  for (size_t c = 0; c < nc; ++c) {
    names[c] = "egfem_grp_" + std::to_string(c) + "_v" + std::to_string(v);
    srcs[c] = kernel_source(pattern_from_key(gp->classes[c].key), names[c], gp->f64 ? "double" : "float",
                            gp->pairs_per_lane, same, full);
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

egfem_status launch_groups(const egfem_tensor* t, int32_t batch, const void* U, const void* W, void* R,
                           cudaStream_t s) {
  GroupPlan* gp = t->grp;
  const int dev = t->device & 63;
  if (!g_sms_grp[dev]) EGFEM_CUDA_TRY(cudaDeviceGetAttribute(&g_sms_grp[dev], cudaDevAttrMultiProcessorCount, t->device));
  const int P = gp->pairs_per_lane;
  const int nch = (batch + 32 * P - 1) / (32 * P);
  const int v = (U == W ? 1 : 0) | (batch % (32 * P) == 0 ? 2 : 0);
  egfem_status st = ensure_variant(gp, v);
  if (st) return st;
  const int threads = 32 * std::min(4, nch);
  for (const auto& gc : gp->classes) {
    const int64_t runs = (gc.ninst + gp->run - 1) / gp->run;
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(runs, (int64_t)g_sms_grp[dev] * 32));
    long long ninst = gc.ninst;
    int B = batch, run = gp->run;
    void* args[] = {(void*)&gc.cols, (void*)&gc.rows, (void*)&gc.vals, &ninst, &B, &run, (void*)&U, (void*)&W, &R};
    EGFEM_CUDA_TRY(cudaLaunchKernel((const void*)gc.fn[v], dim3((unsigned)ctas), dim3(threads), args, 0, s));
    count_launch();
  }
  if (gp->fb_count > 0) {
    st = launch_dense_rows(t, batch, gp->fb_rows, gp->fb_classes, U, W, R, s);
    if (st) return st;
  }
  return EGFEM_OK;
}

}  // namespace egfem
