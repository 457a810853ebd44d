// cy_gemm.cu -- host side of the C ABI (include/cypress_b200.h): argument validation, TMA
// descriptor encoding (cached), config selection, cluster launch.  No torch, no libcuda link
// (the driver's cuTensorMapEncodeTiled is fetched through cudaGetDriverEntryPoint).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "cy_kernel.cuh"
#include "cypress_b200.h"

namespace {

using cy::Params;

// ------------------------------------------------------------------------------------------
// kernel menu
struct KDesc {
  int var, dt, cg, bn, stages, threads, smem, mc;  // bn = output tile width (TILE_N); mc = pairs sharing B
  int bn_cta;                                      // B columns per CTA per B slot (multiple of 64)
  int bk;                                          // K per stage (64 or 128)
  int mx;                                          // 1: 2 x 2 multicast cluster of 128 x bn CTA tiles
  const void* fn;
  int ct_m() const { return mx ? 256 : 128 * cg * mc; }  // cluster tile rows
  int ct_n() const { return mx ? 2 * bn : bn; }          // cluster tile columns
  int csize() const { return mx ? 4 : cg * mc; }         // CTAs per cluster (before split-K)
};

template <int DT, int CG, int BN, int ST, int VAR, int NSUB = 1, int MC = 1, int BK = 64, int MX = 0>
KDesc kdesc() {
  using C = cy::Cfg<DT, CG, BN, ST, VAR, NSUB, MC, BK, MX>;
  return KDesc{VAR, DT, CG, C::TILE_N, ST, C::THREADS, C::SMEM_BYTES, MC, C::BN_CTA, BK, MX,
               (const void*)&cy::cy_sm100_kernel<C>};
}

// Shapes (cta_group, tile N, pairs per cluster) offered per variant; the GEMM menu defines the
// public config ids.
struct Shape { int cg, bn, mc, bk, mx; };
// The narrow tiles (pair 256 x 128, single 128 x 64) stage K = 128 per k-block: with 24 KB stages
// the per-SM TMA op rate, not bandwidth, bounded them (measured, graph replay: 1024^3 7.8 -> 6.7 us on
// 128 x 64, 2048^3 22.1 -> 16.4 us on 256 x 128); the wide tiles keep K = 64 (K = 128 leaves them
// 2-3 stages: 8192^3 715 -> 810 us on 256 x 256).
// Experiment build only (CY_GEMM_MX): config 7, the 128 x 64 K = 128 tile in a 2 x 2 cluster that
// multicasts A along N and B along M, so each CTA issues half of its operand bytes.  Bit-exact on
// the whole GEMM suite, but not faster (graph replay: 1024^3 7.4 vs 7.0 us on config 4, 2048^3 and
// 4096^3 on par with config 4): the narrow tiles are bound by the latency of the bytes each SM
// receives, which multicast does not reduce.
constexpr Shape kGemmMenu[] = {{2, 256, 1, 64, 0}, {2, 128, 1, 128, 0}, {1, 256, 1, 64, 0}, {1, 128, 1, 64, 0},
                               {1, 64, 1, 128, 0}, {2, 512, 1, 64, 0}, {2, 512, 2, 64, 0}
#ifdef CY_GEMM_MX
                               , {1, 64, 1, 128, 1}
#endif
};
constexpr int kNumGemmCfg = sizeof(kGemmMenu) / sizeof(kGemmMenu[0]);

template <int DT>
void add_all(std::vector<KDesc>& v) {
  v.push_back(kdesc<DT, 2, 256, 6, cy::V_GEMM>());
  v.push_back(kdesc<DT, 2, 128, 4, cy::V_GEMM, 1, 1, 128>());
  v.push_back(kdesc<DT, 1, 256, 4, cy::V_GEMM>());
  v.push_back(kdesc<DT, 1, 128, 6, cy::V_GEMM>());
  v.push_back(kdesc<DT, 1, 64, 4, cy::V_GEMM, 1, 1, 128>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_GEMM, 2>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_GEMM, 2, 2>());
#ifdef CY_GEMM_MX
  v.push_back(kdesc<DT, 1, 64, 4, cy::V_GEMM, 1, 1, 128, 1>());
#endif
  v.push_back(kdesc<DT, 2, 256, 6, cy::V_ROWREDUCE>());
  v.push_back(kdesc<DT, 2, 128, 8, cy::V_ROWREDUCE>());
  v.push_back(kdesc<DT, 1, 128, 6, cy::V_ROWREDUCE>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_ROWREDUCE, 2>());
  v.push_back(kdesc<DT, 2, 128, 6, cy::V_DUAL_PAIR>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_DUAL_PAIR>());
  v.push_back(kdesc<DT, 1, 128, 4, cy::V_DUAL_PAIR>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_DUAL_SUM>());
  v.push_back(kdesc<DT, 2, 128, 6, cy::V_DUAL_SUM>());
  v.push_back(kdesc<DT, 1, 128, 4, cy::V_DUAL_SUM>());
  v.push_back(kdesc<DT, 2, 128, 6, cy::V_DUAL_GLU>());
  v.push_back(kdesc<DT, 2, 256, 4, cy::V_DUAL_GLU>());
  v.push_back(kdesc<DT, 1, 128, 4, cy::V_DUAL_GLU>());
}

const std::vector<KDesc>& menu() {
  static const std::vector<KDesc> v = [] {
    std::vector<KDesc> r;
    add_all<0>(r);
    add_all<1>(r);
    return r;
  }();
  return v;
}

std::atomic<int> g_forced{-1};
// Tile order and L2 hints (tuning knobs; -1 = the defaults below, chosen per problem in launch()):
// CY_RASTER 0 = groups of CY_GROUP_M m-blocks (A panels resident, B streams), 1 = groups of
// CY_GROUP_M n-blocks (B panels resident, A streams); CY_SERP=1 reverses the sweep of odd groups;
// CY_L2_POLICY = TMA L2 eviction hints for A/B (see Params::l2_policy).
// The knobs are read from the environment only in timing-experiment builds
// (scripts/build_experiment.py NAME CY_TUNING_KNOBS=1); the product library always runs the defaults.
int env_int(const char* name, int dflt) {
#ifdef CY_TUNING_KNOBS
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}
const int g_group_m = env_int("CY_GROUP_M", 0);
const int g_l2_policy = env_int("CY_L2_POLICY", -1);
const int g_serp = env_int("CY_SERP", -1);
const int g_raster = env_int("CY_RASTER", -1);
const int g_b4d = env_int("CY_B4D", 1);
const int g_d_policy = env_int("CY_D_POLICY", 0);  // L2 policy of the D stores (0 none, 1 first, 2 last)
const int g_c_pf = env_int("CY_C_PF", 0);  // epilogue C tiles prefetched into L2 during the main loop
const int g_pf_dist = env_int("CY_PF_DIST", 0);  // batched L2 prefetch distance in problems (0 = off)
// CY_SCHED: 0 = dynamic (cluster launch control) when there is more than one wave, 1 = static
const int g_sched = env_int("CY_SCHED", 0);
// CY_PDL=0 disables programmatic dependent launch (tuning / debugging knob)
const int g_pdl = env_int("CY_PDL", 1);
// CY_SLEEP_NS: epilogue wait backoff cap in ns (0 = spin); tuning knob
const int g_sleep_ns = env_int("CY_SLEEP_NS", 0);
// CY_A_REUSE=0 disables the A-operand collector reuse across the two accumulators (tuning knob)
const int g_a_reuse = env_int("CY_A_REUSE", 1);
std::atomic<int> g_last{-1};
std::atomic<int> g_last_splits{1};
std::atomic<int64_t> g_launches{0};

// ------------------------------------------------------------------------------------------
// per-device state
struct DevState {
  bool init = false;
  bool ok = false;
  int sms = 0;
  std::vector<char> attr_set;  // per menu entry: max dynamic smem attribute applied
  std::vector<int> max_clusters;  // per (menu entry, cluster size 1..8): co-resident clusters (0 = not queried)
};
std::mutex g_mu;
DevState g_dev[64];
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

cy_status_t device_state(int& dev, DevState*& st) {
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CY_ERR_UNSUPPORTED_DEVICE;
  std::lock_guard<std::mutex> lk(g_mu);
  st = &g_dev[dev];
  if (!st->init) {
    st->init = true;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&st->sms, cudaDevAttrMultiProcessorCount, dev);
    st->ok = (major == 10 && minor == 0);
    st->attr_set.assign(menu().size(), 0);
    st->max_clusters.assign(menu().size() * 9, 0);
    if (!g_encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cudaGetLastError();
  }
  if (!st->ok) return CY_ERR_UNSUPPORTED_DEVICE;
  if (!g_encode) return CY_ERR_INTERNAL;
  return CY_OK;
}

// ------------------------------------------------------------------------------------------
// TMA descriptors (3-D: columns, rows, batch), cached
// CY_L2_PROMO: TMA L2 sector promotion (tuning knob): 0 none, 1 64B, 2 128B, 3 256B (default)
CUtensorMapL2promotion promo() {
  static const int v = env_int("CY_L2_PROMO", 3);
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

struct MapKey {
  const void* ptr;
  uint64_t cols, rows, batch, ld, stride;
  uint32_t box_c, box_r;
  int dt, atoms;  // atoms > 0: 4-D map {64, rows, cols / 64, batch} with boxes of `atoms` 64-column atoms
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    // FNV-1a over the key bytes
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&k);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MapKey); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return static_cast<size_t>(h);
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;  // bounded: cleared when it grows past 4096

bool encode_map(CUtensorMap* out, int dt, const void* ptr, uint64_t cols, uint64_t rows, uint64_t batch,
                uint64_t ld, uint64_t stride, uint32_t box_c, uint32_t box_r, uint32_t atoms = 0) {
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.ptr = ptr; key.cols = cols; key.rows = rows; key.batch = batch; key.ld = ld; key.stride = stride;
  key.box_c = box_c; key.box_r = box_r; key.dt = dt; key.atoms = static_cast<int>(atoms);
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return true;
    }
  }
  CUtensorMap m;
  CUresult r;
  if (atoms > 0) {  // {64 columns, rows, cols / 64 atoms, batch}; strides: row, 128 B per atom, batch
    cuuint64_t dims[4] = {64, rows, cols / 64, batch};
    cuuint64_t strides[3] = {ld * 2, 128, stride * 2};
    cuuint32_t box[4] = {64, box_r, atoms, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    r = g_encode(&m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                 const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {cols, rows, batch};
    cuuint64_t strides[2] = {ld * 2, stride * 2};
    cuuint32_t box[3] = {box_c, box_r, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    r = g_encode(&m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                 const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return false;
  *out = m;
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (g_maps.size() >= 4096) g_maps.clear();
  g_maps.emplace(key, m);
  return true;
}

// ------------------------------------------------------------------------------------------
// validation helpers
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct Range {
  uintptr_t lo, hi;  // [lo, hi)
};
Range span(const void* p, int64_t rows, int64_t cols, int64_t ld, int64_t batch, int64_t stride, int64_t esz) {
  if (!p || rows <= 0 || cols <= 0 || batch <= 0) return Range{0, 0};
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p);
  const int64_t last = (batch - 1) * stride + (rows - 1) * ld + cols;
  return Range{lo, lo + static_cast<uintptr_t>(last * esz)};
}
bool overlap(Range a, Range b) { return a.lo < a.hi && b.lo < b.hi && a.lo < b.hi && b.lo < a.hi; }

// ------------------------------------------------------------------------------------------
// config choice: minimise (waves x tile area / efficiency)
// Kernel attributes (dynamic shared memory) of menu entry `idx`, set once per device.
bool ensure_attr(DevState* st, int idx) {
  const KDesc& kd = menu()[idx];
  std::lock_guard<std::mutex> lk(g_mu);
  if (!st->attr_set[idx]) {
    if (cudaFuncSetAttribute(kd.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kd.smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (kd.cg == 2) cudaFuncSetAttribute(kd.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    st->attr_set[idx] = 1;
  }
  return true;
}

// Co-resident clusters of `csize` CTAs of menu entry `idx` (clusters of 4 or 8 do not tile every
// GPC: ask the occupancy calculator once and cache it).
int active_clusters(DevState* st, int idx, int csize) {
  if (csize <= 2) return std::max(1, st->sms / csize);
  int& maxc = st->max_clusters[idx * 9 + csize];
  if (maxc > 0) return maxc;
  const KDesc& kd = menu()[idx];
  int nc = 0;
  if (ensure_attr(st, idx)) {
    cudaLaunchConfig_t q;
    std::memset(&q, 0, sizeof(q));
    q.gridDim = dim3(csize * 256, 1, 1);
    q.blockDim = dim3(kd.threads, 1, 1);
    q.dynamicSmemBytes = kd.smem;
    cudaLaunchAttribute qa;
    qa.id = cudaLaunchAttributeClusterDimension;
    qa.val.clusterDim.x = csize;
    qa.val.clusterDim.y = 1;
    qa.val.clusterDim.z = 1;
    q.attrs = &qa;
    q.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&nc, kd.fn, &q) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = st->sms / csize;
    }
  } else {
    nc = st->sms / csize;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  maxc = nc;
  return nc;
}

// Predicted time of one launch: waves x (tile area per SM) x (K + exposed epilogue) / efficiency.
// `units` = tiles in flight (co-resident clusters; a split-K cluster works on one tile).
double cfg_cost(int cg, int bn, int single_buf, int64_t m, int64_t n, int64_t k, int64_t L, int64_t units,
                int splits = 1, int bk = 64) {
  const int64_t bm = 128 * cg;
  const int64_t tiles = L * ((m + bm - 1) / bm) * ((n + bn - 1) / bn);
  const int64_t waves = (tiles + units - 1) / units;
  // relative per-SM efficiency of each tile shape, measured on B200 at 8192^3 under the power cap
  // (shared-memory operand bytes per MMA and L2 bytes per FLOP fall as the tile grows)
  double eff = 1.0;
  if (cg == 2 && bn == 512) eff = 1.25;  // 25 % fewer L2 bytes per FLOP: more clock under the power cap
  if (cg == 2 && bn == 128) eff = (bk == 128) ? 0.84 : 0.70;
  if (cg == 1 && bn == 256) eff = 0.80;
  if (cg == 1 && bn == 128) eff = 0.60;
  if (cg == 1 && bn == 64) eff = (bk == 128) ? 0.49 : 0.40;
  const int64_t kb = (k + 63) / 64;
  const int64_t kb_split = (kb + splits - 1) / splits;
  double kk = static_cast<double>(std::max<int64_t>(kb_split * 64, 64)) + (single_buf ? 128.0 : 0.0) + 128.0;
  // split-K: every CTA writes its 128 x bn fp32 partial (~8 bn cycles at ~64 B/clk of L2
  // bandwidth) and reads back the same volume for its share of the reduction; one k-block costs
  // 2 bn cycles per SM, so the reduction weighs ~8 k-blocks = 512 K elements
  if (splits > 1) kk += 512.0;
  // the last wave's epilogue is exposed whatever the buffering: draining 128 rows x bn columns per
  // SM costs about bn / 2 k-equivalents (calibrated on batched 8 x 1024^3, where one wave of 256 x 512
  // tiles measured 19.4 us against 18.1 us for two waves of 256 x 256; negligible for many waves)
  const double tail = 0.5 * bn;
  return (static_cast<double>(waves) * kk + tail) * static_cast<double>(bm * bn) / cg / eff;
}

// Menu entry and split count: the smallest predicted time.  max_splits > 1 lets split-K (V_GEMM
// with one accumulator per tile) compete; ws_bytes bounds the workspace a split may use.
struct Choice {
  int idx = -1, splits = 1;
};
size_t splitk_ws_bytes(const KDesc& kd, int64_t m, int64_t n, int64_t L, int splits);

Choice pick(int var, int dt, int64_t m, int64_t n, int64_t k, int64_t L, DevState* st, int max_splits = 1,
            size_t ws_bytes = 0, int forced_splits = 0, bool use_forced = true) {
  const auto& mn = menu();
  Choice best;
  double best_cost = 0;
  int64_t kb = (k + 63) / 64;
  const int forced = use_forced ? g_forced.load() : -1;
  // splits that leave no split empty: S -> ceil(kb / ceil(kb / S))
  auto eff_splits = [&](int sp) {
    if (kb <= 1 || sp <= 1) return 1;
    const int64_t kbs = (kb + sp - 1) / sp;
    return static_cast<int>((kb + kbs - 1) / kbs);
  };
  for (size_t i = 0; i < mn.size(); ++i) {
    if (mn[i].var != var || mn[i].dt != dt) continue;
    kb = (k + mn[i].bk - 1) / mn[i].bk;  // k-blocks of this config
    if (forced >= 0 && forced < kNumGemmCfg) {
      if (!(mn[i].cg == kGemmMenu[forced].cg && mn[i].bn == kGemmMenu[forced].bn && mn[i].mc == kGemmMenu[forced].mc &&
            mn[i].bk == kGemmMenu[forced].bk && mn[i].mx == kGemmMenu[forced].mx))
        continue;
    } else if (mn[i].mc != 1 || mn[i].mx) {
      continue;  // multicast clusters: only when forced (being evaluated)
    }
    const int acc_cols = ((var == cy::V_DUAL_PAIR || var == cy::V_DUAL_GLU) ? 2 : 1) * mn[i].bn;
    const int single = acc_cols * 2 > 512;
    const bool can_split = var == cy::V_GEMM && mn[i].mc == 1 && mn[i].mx == 0 && mn[i].bn <= 256;  // one accumulator (NSUB 1)
    if (!can_split && forced_splits > 1) continue;  // a requested split needs a splittable kernel
    // split-K clusters: cta_group x splits <= 8 CTAs (portable cluster size)
    const int s_cap = 8 / mn[i].cg;
    const int s_hi = can_split ? static_cast<int>(std::min<int64_t>(std::min(max_splits, s_cap), std::max<int64_t>(kb, 1)))
                               : 1;
    for (int sp = 1; sp <= s_hi; ++sp) {
      if (eff_splits(sp) != sp) continue;  // same k-block ranges as a smaller count
      if (can_split && forced_splits > 0 && sp != eff_splits(std::min(forced_splits, s_hi))) continue;
      if (sp > 1 && splitk_ws_bytes(mn[i], m, n, L, sp) > ws_bytes) continue;
      const int cl = mn[i].csize() * sp;
      const double c =
          cfg_cost(mn[i].cg, mn[i].bn, single, m, n, k, L, active_clusters(st, static_cast<int>(i), cl), sp, mn[i].bk);
      if (best.idx < 0 || c < best_cost) {
        best.idx = static_cast<int>(i);
        best.splits = sp;
        best_cost = c;
      }
    }
  }
  if (best.idx < 0 && forced >= 0)  // the forced shape has no kernel of this variant: heuristic
    return pick(var, dt, m, n, k, L, st, max_splits, ws_bytes, forced_splits, false);
  return best;
}

// Split-K workspace: the fp32 partial slices, tiles x CTAs per tile x 128 rows x TILE_N x splits.
size_t splitk_ws_bytes(const KDesc& kd, int64_t m, int64_t n, int64_t L, int splits) {
  if (splits <= 1) return 0;
  const int64_t bm = 128 * kd.cg * kd.mc;
  const int64_t tiles = L * ((m + bm - 1) / bm) * ((n + kd.bn - 1) / kd.bn);
  return static_cast<size_t>(tiles * kd.cg * 128 * kd.bn * 4) * splits;
}

// ------------------------------------------------------------------------------------------
struct Operand {
  const void* ptr;
  int64_t ld, stride;
};

cy_status_t launch(int var, int dt, int64_t m, int64_t n, int64_t k, int64_t L, float alpha, Operand A,
                   Operand B0, Operand B1, float beta, Operand C0, Operand C1, Operand D0, Operand D1, float* y,
                   void* stream, int act = 0, const Operand* extra_dst = nullptr, int n_extra = 0, int max_splits = 1,
                   void* ws = nullptr, size_t ws_bytes = 0, int forced_splits = 0) {
  int dev;
  DevState* st;
  cy_status_t s = device_state(dev, st);
  if (s != CY_OK) return s;
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX || L > INT32_MAX) return CY_ERR_INVALID_VALUE;
  const Choice ch = pick(var, dt, m, n, k, L, st, max_splits, ws_bytes, forced_splits);
  const int idx = ch.idx;
  if (idx < 0) return CY_ERR_INTERNAL;
  const KDesc& kd = menu()[idx];
  const int bm = kd.ct_m();  // rows per cluster tile
  const int bn_cta = kd.bn / kd.cg;

  CUtensorMap tA, tB0, tB1, tC0, tC1, tD0, tD1;
  std::memset(&tA, 0, sizeof(CUtensorMap));
  tB0 = tB1 = tC0 = tC1 = tD0 = tD1 = tA;
  auto enc = [&](CUtensorMap* out, Operand o, int64_t rows, int64_t cols, uint32_t bc, uint32_t br, uint32_t atoms = 0) {
    const int64_t stride = (L > 1) ? o.stride : rows * o.ld;
    return encode_map(out, dt, o.ptr, (uint64_t)cols, (uint64_t)rows, (uint64_t)L, (uint64_t)o.ld,
                      (uint64_t)stride, bc, br, atoms);
  };
  // B as 4-D boxes of all the slot's atoms (one TMA op per slot) when every atom is whole
  // (n % 64 == 0, so no box reads past a row) -- measured per-SM TMA rate 56 vs 35 B/clk for one
  // 4-atom box vs four 2-D boxes (scripts/experiments/tma_stream.cu)
  // (single-atom slots keep the 2-D form: measured 7.3 vs 7.6 us at 1024^3 on 128 x 64 tiles; the
  // multi-atom slots gain 0.5-1.5 %: 2048^3 16.5 -> 16.2 us, 4096^3, batched)
  const bool b4d = g_b4d && kd.mc == 1 && !kd.mx && (n % 64) == 0 && kd.bn_cta >= 128;
  const uint32_t b_atoms = b4d ? static_cast<uint32_t>(kd.bn_cta / 64) : 0;
  // K = 128 stages: A's two K-atoms in one 4-D box when every K-atom is whole (k % 64 == 0: a
  // partial atom would read past K, and garbage times B's zero-filled rows could be NaN)
  // (MX: each CTA loads one K-atom of A and one 64-row half of the B stage -- 3-D maps, 64-row B boxes)
  const bool a4d = kd.bk > 64 && (k % 64) == 0 && !kd.mx;
  bool ok = true;
  if (k > 0) {
    ok = ok && enc(&tA, A, m, k, 64, 128, a4d ? static_cast<uint32_t>(kd.bk / 64) : 0);
    ok = ok && enc(&tB0, B0, k, n, 64, kd.mx ? 64 : kd.bk, b_atoms);
    if (B1.ptr) ok = ok && enc(&tB1, B1, k, n, 64, kd.bk, b_atoms);
  }
  const bool has_c = (beta != 0.0f);
  if (has_c) {
    ok = ok && enc(&tC0, C0, m, n, 64, 32);
    if (C1.ptr) ok = ok && enc(&tC1, C1, m, n, 64, 32);
  }
  ok = ok && enc(&tD0, D0, m, n, 64, 32);
  if (D1.ptr) ok = ok && enc(&tD1, D1, m, n, 64, 32);
  cy::DstMaps extra;
  std::memset(&extra, 0, sizeof(extra));
  for (int j = 0; j < n_extra; ++j) ok = ok && enc(&extra.m[j], extra_dst[j], m, n, 64, 32);
  if (!ok) return CY_ERR_LAUNCH;
  (void)bn_cta;

  Params p;
  p.M = (int)m; p.N = (int)n; p.K = (int)k; p.L = (int)L;
  p.alpha = alpha; p.beta = beta; p.has_c = has_c ? 1 : 0;
  p.m_blocks = (int)((m + bm - 1) / bm);
  p.n_blocks = (int)((n + kd.ct_n() - 1) / kd.ct_n());
  p.k_blocks = (int)((k + kd.bk - 1) / kd.bk);
  p.splits = ch.splits;
  p.kb_split = p.splits > 1 ? (p.k_blocks + p.splits - 1) / p.splits : p.k_blocks;
  p.ws = p.splits > 1 ? static_cast<float*>(ws) : nullptr;
  if (L * p.m_blocks * p.n_blocks > INT32_MAX) return CY_ERR_INVALID_VALUE;
  p.tiles = (int)(L * p.m_blocks * p.n_blocks);
  // Single problems: groups of 4 n-blocks with B resident (evict_last hint on B only), A streaming,
  // odd groups sweeping m backwards.  Measured with ncu at 8192^3 (DRAM read 865 -> 785 MB) and
  // 65536 x 8192 x 8192 (6.76 -> 5.76 GB), +1.3 % sustained TFLOP/s on the row-reduce bench (clock
  // 1230 -> 1252 MHz under the power cap); larger resident groups thrash (64 MB of B: 7.6 GB).
  // Batched problems keep m-grouping by 12 with no hints (a batch's operands are not reused).
  const bool single = (L == 1);
  p.raster = g_raster >= 0 ? g_raster : (single ? 1 : 0);
  p.group_m = g_group_m > 0 ? g_group_m : (single ? 4 : 12);
  p.l2_policy = g_l2_policy >= 0 ? g_l2_policy : (single ? 6 : 5);
  p.serp = g_serp >= 0 ? g_serp : (single ? 1 : 0);
  p.b4d = b4d ? 1 : 0;
  p.a4d = a4d ? 1 : 0;
  // Batched: prefetch the operands of the problem pf_dist ahead into L2 (each problem's A and B
  // spans, padding between rows included; off for single problems and K = 0)
  p.pf_dist = (L > 1 && k > 0) ? g_pf_dist : 0;
  p.pf_a = static_cast<const char*>(A.ptr);
  p.pf_b = static_cast<const char*>(B0.ptr);
  p.pf_a_stride = A.stride * 2;
  p.pf_b_stride = B0.stride * 2;
  p.pf_a_bytes = ((m - 1) * A.ld + k) * 2 / 16 * 16;
  p.pf_b_bytes = ((k - 1) * B0.ld + n) * 2 / 16 * 16;
  if (B1.ptr) p.pf_dist = 0;
  p.c_pf = g_c_pf;
  p.d_policy = g_d_policy;
  p.sleep_ns = g_sleep_ns;
  p.a_reuse = g_a_reuse;
  p.act = act;
  p.n_extra = n_extra;
  p.y = y;

  if (!ensure_attr(st, idx)) return CY_ERR_LAUNCH;
  const int csize = kd.csize() * p.splits;  // split-K: the splits of a tile form one cluster
  if (csize > 8) return CY_ERR_INTERNAL;
  const int units = active_clusters(st, idx, csize);
  // More tiles than co-resident clusters: launch one cluster per tile and let running clusters
  // steal pending ones (cluster launch control) so the tiles in flight stay adjacent in the
  // raster; otherwise every tile gets its own resident cluster.
  // CY_SCHED=2: one cluster per tile and no stealing (the non-persistent launch) -- tuning knob
  p.dyn = (p.tiles > units && g_sched != 1) ? (g_sched == 2 ? 2 : 1) : 0;
  const int clusters = p.dyn ? p.tiles : std::max(1, std::min(p.tiles, units));

  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(clusters * csize, 1, 1);
  cfg.blockDim = dim3(kd.threads, 1, 1);
  cfg.dynamicSmemBytes = kd.smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = csize;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  // Programmatic dependent launch: our prologue may overlap the previous kernel's tail; the
  // kernel waits (griddepcontrol.wait) before its first global-memory access.
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  void* args[] = {&tA, &tB0, &tB1, &tC0, &tC1, &tD0, &tD1, &p, &extra};
  cudaError_t e = cudaLaunchKernelExC(&cfg, kd.fn, args);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return CY_ERR_LAUNCH;
  }
  g_last.store(idx);
  g_last_splits.store(p.splits);
  g_launches.fetch_add(1);
  return CY_OK;
}

bool ld_ok(int64_t ld) { return ld > 0 && (ld % 8) == 0; }

// y(i) = sum_k A(i,k) alone, for cy_gemm_rowreduce with n == 0 (no output tiles, so no reducer
// warps run; P:1579 still defines y).  One thread per row adds in k order in fp32 -- the order and
// precision of the fused reducer warps (cy_kernel.cuh), so y is bit-identical to the n > 0 path.
template <int DT>
__global__ void __launch_bounds__(128) rowsum_kernel(const uint16_t* __restrict__ A, int64_t lda, int m, int k,
                                                     float* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  const uint16_t* a = A + static_cast<int64_t>(row) * lda;
  float acc = 0.f;
  int kk = 0;
  for (; kk + 8 <= k; kk += 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(a + kk);  // 16-B aligned: A and lda*2 are
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = cy::unpack2<DT>(w[e]);
      acc += f.x;
      acc += f.y;
    }
  }
  for (; kk < k; ++kk) acc += cy::unpack2<DT>(static_cast<uint32_t>(a[kk])).x;
  y[row] = acc;
}

cy_status_t launch_rowsum(int dt, const void* A, int64_t lda, int64_t m, int64_t k, float* y, void* stream) {
  int dev;
  DevState* st;
  cy_status_t s = device_state(dev, st);
  if (s != CY_OK) return s;
  if (m > INT32_MAX || k > INT32_MAX) return CY_ERR_INVALID_VALUE;
  const dim3 grid(static_cast<unsigned>((m + 127) / 128));
  auto* a = static_cast<const uint16_t*>(A);
  if (dt == 0) rowsum_kernel<0><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a, lda, (int)m, (int)k, y);
  else rowsum_kernel<1><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a, lda, (int)m, (int)k, y);
  if (cudaGetLastError() != cudaSuccess) return CY_ERR_LAUNCH;
  g_launches.fetch_add(1);
  return CY_OK;
}

}  // namespace

#ifdef CY_GEMM_TRACE
// trace build only (scripts/build_experiment.py gtrace CY_GEMM_TRACE=1): not in the product ABI
extern "C" int cy_gemm_trace_read(unsigned long long* out, int clear) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(g_gemm_trace));
  if (clear) {
    static unsigned long long zero[64 * 16] = {};
    cudaMemcpyToSymbol(g_gemm_trace, zero, sizeof(zero));
  }
  return static_cast<int>(e);
}
extern "C" int cy_gemm_mtrace_read(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_gemm_mtrace, sizeof(g_gemm_mtrace)));
}
extern "C" int cy_gemm_etrace_read(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_gemm_etrace, sizeof(g_gemm_etrace)));
}
extern "C" int cy_gemm_ktrace_read(unsigned long long* ev, unsigned long long* gtime, int clear) {
  cudaError_t e = cudaMemcpyFromSymbol(ev, g_gemm_ktrace, sizeof(g_gemm_ktrace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(gtime, g_gemm_gtime, sizeof(g_gemm_gtime));
  if (clear) {
    static unsigned long long zero[1024 * 8] = {};
    cudaMemcpyToSymbol(g_gemm_ktrace, zero, sizeof(g_gemm_ktrace));
    cudaMemcpyToSymbol(g_gemm_gtime, zero, sizeof(g_gemm_gtime));
  }
  return static_cast<int>(e);
}
#endif

// shared with the attention entry point (cy_attention.cu): every kernel this library launches
namespace cy_internal {
void note_launch() { g_launches.fetch_add(1); }
}  // namespace cy_internal

// ============================================================================================
extern "C" {

const char* cy_status_string(cy_status_t s) {
  switch (s) {
    case CY_OK: return "CY_OK";
    case CY_ERR_INVALID_VALUE: return "CY_ERR_INVALID_VALUE: invalid size, leading dimension, pointer or overlap";
    case CY_ERR_MISALIGNED: return "CY_ERR_MISALIGNED: pointer not 16-byte aligned or ld/stride not a multiple of 8";
    case CY_ERR_UNSUPPORTED_DEVICE: return "CY_ERR_UNSUPPORTED_DEVICE: needs compute capability 10.0 (sm_100a)";
    case CY_ERR_LAUNCH: return "CY_ERR_LAUNCH: kernel launch or TMA descriptor encode failed";
    case CY_ERR_INTERNAL: return "CY_ERR_INTERNAL";
  }
  return "unknown cy_status_t";
}

int cy_num_configs(void) { return kNumGemmCfg; }

cy_status_t cy_config_info(int id, int* cta_group, int* tile_m, int* tile_n, int* stages) {
  if (id < 0 || id >= kNumGemmCfg) return CY_ERR_INVALID_VALUE;
  const auto& mn = menu();
  for (const auto& k : mn)
    if (k.var == cy::V_GEMM && k.cg == kGemmMenu[id].cg && k.bn == kGemmMenu[id].bn && k.mc == kGemmMenu[id].mc &&
        k.bk == kGemmMenu[id].bk && k.mx == kGemmMenu[id].mx) {
      if (cta_group) *cta_group = k.cg;
      if (tile_m) *tile_m = k.ct_m();
      if (tile_n) *tile_n = k.ct_n();
      if (stages) *stages = k.stages;
      return CY_OK;
    }
  return CY_ERR_INTERNAL;
}

cy_status_t cy_force_config(int id) {
  if (id < -1 || id >= kNumGemmCfg) return CY_ERR_INVALID_VALUE;
  g_forced.store(id);
  return CY_OK;
}

int cy_last_config(void) {
  const int idx = g_last.load();
  if (idx < 0) return -1;
  const auto& k = menu()[idx];
  for (int i = 0; i < kNumGemmCfg; ++i)
    if (kGemmMenu[i].cg == k.cg && kGemmMenu[i].bn == k.bn && kGemmMenu[i].mc == k.mc && kGemmMenu[i].bk == k.bk &&
        kGemmMenu[i].mx == k.mx)
      return i;
  return -1;
}

int64_t cy_launch_count(void) { return g_launches.load(); }

cy_status_t cy_last_kernel_info(int* variant, int* cta_group, int* tile_m, int* tile_n, int* stages, int* threads,
                                int* smem_bytes, int* dtype) {
  const int idx = g_last.load();
  if (idx < 0) return CY_ERR_INVALID_VALUE;
  const KDesc& k = menu()[idx];
  if (variant) *variant = k.var;
  if (cta_group) *cta_group = k.cg;
  if (tile_m) *tile_m = k.ct_m();
  if (tile_n) *tile_n = k.ct_n();
  if (stages) *stages = k.stages;
  if (threads) *threads = k.threads;
  if (smem_bytes) *smem_bytes = k.smem;
  if (dtype) *dtype = k.dt;
  return CY_OK;
}

static cy_status_t check_common(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch) {
  if (dt != CY_F16 && dt != CY_BF16) return CY_ERR_INVALID_VALUE;
  if (m < 0 || n < 0 || k < 0 || batch < 0) return CY_ERR_INVALID_VALUE;
  return CY_OK;
}

static cy_status_t check_batched(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, float beta,
                                 const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                                 int64_t strideB, const void* C, int64_t ldc, int64_t strideC, void* D, int64_t ldd,
                                 int64_t strideD) {
  cy_status_t s = check_common(dt, m, n, k, batch);
  if (s != CY_OK) return s;
  if (m == 0 || n == 0 || batch == 0) return CY_OK;
  const bool has_c = beta != 0.0f;
  if (!D || (k > 0 && (!A || !B)) || (has_c && !C)) return CY_ERR_INVALID_VALUE;
  if (ldd < n || (k > 0 && (lda < k || ldb < n)) || (has_c && ldc < n)) return CY_ERR_INVALID_VALUE;
  // batch strides must be positive (TMA has no zero stride; a broadcast operand is not supported)
  if (batch > 1 && (strideA <= 0 || strideB <= 0 || (has_c && strideC <= 0) || strideD <= 0))
    return CY_ERR_INVALID_VALUE;
  if (batch > 1 && strideD < m * ldd) return CY_ERR_INVALID_VALUE;  // D batches must not overlap
  if (!aligned16(D) || !ld_ok(ldd)) return CY_ERR_MISALIGNED;
  if (k > 0 && (!aligned16(A) || !aligned16(B) || !ld_ok(lda) || !ld_ok(ldb))) return CY_ERR_MISALIGNED;
  if (has_c && (!aligned16(C) || !ld_ok(ldc))) return CY_ERR_MISALIGNED;
  if (batch > 1 && ((strideA % 8) || (strideB % 8) || (has_c && (strideC % 8)) || (strideD % 8)))
    return CY_ERR_MISALIGNED;
  const Range rD = span(D, m, n, ldd, batch, strideD, 2);
  if (k > 0 && (overlap(rD, span(A, m, k, lda, batch, strideA, 2)) || overlap(rD, span(B, k, n, ldb, batch, strideB, 2))))
    return CY_ERR_INVALID_VALUE;
  if (has_c && !(C == D && ldc == ldd && strideC == strideD) && overlap(rD, span(C, m, n, ldc, batch, strideC, 2)))
    return CY_ERR_INVALID_VALUE;
  return CY_OK;
}

cy_status_t cy_gemm_batched(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, float alpha,
                            const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                            int64_t strideB, float beta, const void* C, int64_t ldc, int64_t strideC, void* D,
                            int64_t ldd, int64_t strideD, void* stream) {
  cy_status_t s = check_batched(dt, m, n, k, batch, beta, A, lda, strideA, B, ldb, strideB, C, ldc, strideC, D, ldd,
                                strideD);
  if (s != CY_OK || m == 0 || n == 0 || batch == 0) return s;
  return launch(cy::V_GEMM, dt, m, n, k, batch, alpha, {A, lda, strideA}, {B, ldb, strideB}, {nullptr, 0, 0}, beta,
                {C, ldc, strideC}, {nullptr, 0, 0}, {D, ldd, strideD}, {nullptr, 0, 0}, nullptr, stream);
}

// split-K: the choice the library makes for (shape, splits) with an unbounded workspace
static constexpr int kMaxAutoSplits = 16;
static Choice splitk_choice(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, int splits, DevState* st) {
  return pick(cy::V_GEMM, dt, m, n, k, batch, st, splits == 0 ? kMaxAutoSplits : splits, SIZE_MAX, splits);
}

size_t cy_gemm_splitk_workspace_size(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, int splits) {
  if (check_common(dt, m, n, k, batch) != CY_OK || splits < 0 || splits > 64 || m == 0 || n == 0 || batch == 0)
    return 0;
  int dev;
  DevState* st;
  if (device_state(dev, st) != CY_OK) return 0;
  const Choice ch = splitk_choice(dt, m, n, k, batch, splits, st);
  if (ch.idx < 0) return 0;
  return splitk_ws_bytes(menu()[ch.idx], m, n, batch, ch.splits);
}

cy_status_t cy_gemm_splitk(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, float alpha,
                           const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB,
                           float beta, const void* C, int64_t ldc, int64_t strideC, void* D, int64_t ldd,
                           int64_t strideD, int splits, void* workspace, size_t workspace_bytes, void* stream) {
  if (splits < 0 || splits > 64) return CY_ERR_INVALID_VALUE;
  cy_status_t s = check_batched(dt, m, n, k, batch, beta, A, lda, strideA, B, ldb, strideB, C, ldc, strideC, D, ldd,
                                strideD);
  if (s != CY_OK || m == 0 || n == 0 || batch == 0) return s;
  if (workspace_bytes > 0 && !workspace) return CY_ERR_INVALID_VALUE;
  if (workspace && (reinterpret_cast<uintptr_t>(workspace) & 15u)) return CY_ERR_MISALIGNED;
  if (workspace && workspace_bytes > 0) {
    const Range rW{reinterpret_cast<uintptr_t>(workspace), reinterpret_cast<uintptr_t>(workspace) + workspace_bytes};
    const bool has_c = beta != 0.0f;
    if (overlap(rW, span(D, m, n, ldd, batch, strideD, 2)) ||
        (k > 0 && (overlap(rW, span(A, m, k, lda, batch, strideA, 2)) || overlap(rW, span(B, k, n, ldb, batch, strideB, 2)))) ||
        (has_c && overlap(rW, span(C, m, n, ldc, batch, strideC, 2))))
      return CY_ERR_INVALID_VALUE;
  }
  if (splits > 1) {  // a requested split count must fit the workspace it was given
    int dev;
    DevState* st;
    s = device_state(dev, st);
    if (s != CY_OK) return s;
    const Choice ch = splitk_choice(dt, m, n, k, batch, splits, st);
    if (ch.idx >= 0 && splitk_ws_bytes(menu()[ch.idx], m, n, batch, ch.splits) > workspace_bytes)
      return CY_ERR_INVALID_VALUE;
  }
  return launch(cy::V_GEMM, dt, m, n, k, batch, alpha, {A, lda, strideA}, {B, ldb, strideB}, {nullptr, 0, 0}, beta,
                {C, ldc, strideC}, {nullptr, 0, 0}, {D, ldd, strideD}, {nullptr, 0, 0}, nullptr, stream, 0, nullptr, 0,
                splits == 0 ? kMaxAutoSplits : splits, workspace, workspace_bytes, splits);
}

int cy_last_splits(void) { return g_last_splits.load(); }

cy_status_t cy_gemm(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha, const void* A, int64_t lda,
                    const void* B, int64_t ldb, float beta, const void* C, int64_t ldc, void* D, int64_t ldd,
                    void* stream) {
  return cy_gemm_batched(dt, m, n, k, 1, alpha, A, lda, 0, B, ldb, 0, beta, C, ldc, 0, D, ldd, 0, stream);
}

cy_status_t cy_dual_gemm(cy_dtype_t dt, cy_dual_mode_t mode, int64_t m, int64_t n, int64_t k, float alpha,
                         const void* A, int64_t lda, const void* B0, int64_t ldb0, const void* B1, int64_t ldb1,
                         float beta, const void* C0, int64_t ldc0, const void* C1, int64_t ldc1, void* D0,
                         int64_t ldd0, void* D1, int64_t ldd1, void* stream) {
  cy_status_t s = check_common(dt, m, n, k, 1);
  if (s != CY_OK) return s;
  if (mode != CY_DUAL_PAIR && mode != CY_DUAL_SUM) return CY_ERR_INVALID_VALUE;
  const bool pair = (mode == CY_DUAL_PAIR);
  if (!pair && (C1 || D1)) return CY_ERR_INVALID_VALUE;
  if (m == 0 || n == 0) return CY_OK;
  const bool has_c = beta != 0.0f;
  if (!D0 || (pair && !D1) || (k > 0 && (!A || !B0 || !B1)) || (has_c && (!C0 || (pair && !C1))))
    return CY_ERR_INVALID_VALUE;
  if (ldd0 < n || (pair && ldd1 < n) || (k > 0 && (lda < k || ldb0 < n || ldb1 < n)) ||
      (has_c && (ldc0 < n || (pair && ldc1 < n))))
    return CY_ERR_INVALID_VALUE;
  if (!aligned16(D0) || !ld_ok(ldd0) || (pair && (!aligned16(D1) || !ld_ok(ldd1)))) return CY_ERR_MISALIGNED;
  if (k > 0 && (!aligned16(A) || !aligned16(B0) || !aligned16(B1) || !ld_ok(lda) || !ld_ok(ldb0) || !ld_ok(ldb1)))
    return CY_ERR_MISALIGNED;
  if (has_c && (!aligned16(C0) || !ld_ok(ldc0) || (pair && (!aligned16(C1) || !ld_ok(ldc1)))))
    return CY_ERR_MISALIGNED;
  const Range rD0 = span(D0, m, n, ldd0, 1, 0, 2);
  const Range rD1 = pair ? span(D1, m, n, ldd1, 1, 0, 2) : Range{0, 0};
  for (Range rd : {rD0, rD1}) {
    if (k > 0 && (overlap(rd, span(A, m, k, lda, 1, 0, 2)) || overlap(rd, span(B0, k, n, ldb0, 1, 0, 2)) ||
                  overlap(rd, span(B1, k, n, ldb1, 1, 0, 2))))
      return CY_ERR_INVALID_VALUE;
  }
  if (overlap(rD0, rD1)) return CY_ERR_INVALID_VALUE;
  if (has_c) {
    if (!(C0 == D0 && ldc0 == ldd0) && overlap(rD0, span(C0, m, n, ldc0, 1, 0, 2))) return CY_ERR_INVALID_VALUE;
    if (pair) {
      if (!(C1 == D1 && ldc1 == ldd1) && overlap(rD1, span(C1, m, n, ldc1, 1, 0, 2))) return CY_ERR_INVALID_VALUE;
      if (overlap(rD0, span(C1, m, n, ldc1, 1, 0, 2)) || overlap(rD1, span(C0, m, n, ldc0, 1, 0, 2)))
        return CY_ERR_INVALID_VALUE;
    }
  }
  return launch(pair ? cy::V_DUAL_PAIR : cy::V_DUAL_SUM, dt, m, n, k, 1, alpha, {A, lda, 0}, {B0, ldb0, 0},
                {B1, ldb1, 0}, beta, {C0, ldc0, 0}, {pair ? C1 : nullptr, ldc1, 0}, {D0, ldd0, 0},
                {pair ? D1 : nullptr, ldd1, 0}, nullptr, stream);
}

cy_status_t cy_gemm_replicated(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha, const void* A,
                               int64_t lda, const void* B, int64_t ldb, float beta, const void* C, int64_t ldc,
                               void* const* D_dst, int ndst, int64_t ldd, int64_t row_offset, int64_t rows_total,
                               void* stream) {
  cy_status_t s = check_common(dt, m, n, k, 1);
  if (s != CY_OK) return s;
  if (!D_dst || ndst < 1 || ndst > 1 + cy::kMaxExtraDst) return CY_ERR_INVALID_VALUE;
  if (row_offset < 0 || rows_total < 0 || row_offset + m > rows_total) return CY_ERR_INVALID_VALUE;
  if (m == 0 || n == 0) return CY_OK;
  const bool has_c = beta != 0.0f;
  if ((k > 0 && (!A || !B)) || (has_c && !C)) return CY_ERR_INVALID_VALUE;
  if (ldd < n || (k > 0 && (lda < k || ldb < n)) || (has_c && ldc < n)) return CY_ERR_INVALID_VALUE;
  if (!ld_ok(ldd)) return CY_ERR_MISALIGNED;
  if (k > 0 && (!aligned16(A) || !aligned16(B) || !ld_ok(lda) || !ld_ok(ldb))) return CY_ERR_MISALIGNED;
  if (has_c && (!aligned16(C) || !ld_ok(ldc))) return CY_ERR_MISALIGNED;
  Operand dst[1 + cy::kMaxExtraDst];
  for (int j = 0; j < ndst; ++j) {
    if (!D_dst[j] || !aligned16(D_dst[j])) return D_dst[j] ? CY_ERR_MISALIGNED : CY_ERR_INVALID_VALUE;
    // this shard's row block of destination j (TMA clips every store at the block's edge)
    dst[j] = {static_cast<const char*>(D_dst[j]) + row_offset * ldd * 2, ldd, 0};
    const Range rD = span(dst[j].ptr, m, n, ldd, 1, 0, 2);
    if (k > 0 && (overlap(rD, span(A, m, k, lda, 1, 0, 2)) || overlap(rD, span(B, k, n, ldb, 1, 0, 2))))
      return CY_ERR_INVALID_VALUE;
    if (has_c && overlap(rD, span(C, m, n, ldc, 1, 0, 2))) return CY_ERR_INVALID_VALUE;
    for (int i = 0; i < j; ++i)
      if (overlap(rD, span(dst[i].ptr, m, n, ldd, 1, 0, 2))) return CY_ERR_INVALID_VALUE;
  }
  return launch(cy::V_GEMM, dt, m, n, k, 1, alpha, {A, lda, 0}, {B, ldb, 0}, {nullptr, 0, 0}, beta, {C, ldc, 0},
                {nullptr, 0, 0}, dst[0], {nullptr, 0, 0}, nullptr, stream, 0, dst + 1, ndst - 1);
}

cy_status_t cy_dual_gemm_glu(cy_dtype_t dt, cy_act_t act, int64_t m, int64_t n, int64_t k, float alpha,
                             const void* A, int64_t lda, const void* B0, int64_t ldb0, const void* B1, int64_t ldb1,
                             void* D, int64_t ldd, void* stream) {
  cy_status_t s = check_common(dt, m, n, k, 1);
  if (s != CY_OK) return s;
  if (act != CY_ACT_SILU && act != CY_ACT_GELU_TANH) return CY_ERR_INVALID_VALUE;
  if (m == 0 || n == 0) return CY_OK;
  if (!D || (k > 0 && (!A || !B0 || !B1))) return CY_ERR_INVALID_VALUE;
  if (ldd < n || (k > 0 && (lda < k || ldb0 < n || ldb1 < n))) return CY_ERR_INVALID_VALUE;
  if (!aligned16(D) || !ld_ok(ldd)) return CY_ERR_MISALIGNED;
  if (k > 0 && (!aligned16(A) || !aligned16(B0) || !aligned16(B1) || !ld_ok(lda) || !ld_ok(ldb0) || !ld_ok(ldb1)))
    return CY_ERR_MISALIGNED;
  const Range rD = span(D, m, n, ldd, 1, 0, 2);
  if (k > 0 && (overlap(rD, span(A, m, k, lda, 1, 0, 2)) || overlap(rD, span(B0, k, n, ldb0, 1, 0, 2)) ||
                overlap(rD, span(B1, k, n, ldb1, 1, 0, 2))))
    return CY_ERR_INVALID_VALUE;
  return launch(cy::V_DUAL_GLU, dt, m, n, k, 1, alpha, {A, lda, 0}, {B0, ldb0, 0}, {B1, ldb1, 0}, 0.0f,
                {nullptr, 0, 0}, {nullptr, 0, 0}, {D, ldd, 0}, {nullptr, 0, 0}, nullptr, stream, static_cast<int>(act));
}

cy_status_t cy_gemm_rowreduce(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha, const void* A,
                              int64_t lda, const void* B, int64_t ldb, float beta, const void* C, int64_t ldc,
                              void* D, int64_t ldd, float* y, void* stream) {
  cy_status_t s = check_common(dt, m, n, k, 1);
  if (s != CY_OK) return s;
  if (m == 0) return CY_OK;
  if (!y) return CY_ERR_INVALID_VALUE;
  if (n == 0) {  // no D tiles; y is still defined: the stand-alone row-sum kernel
    if (k > 0 && !A) return CY_ERR_INVALID_VALUE;
    if (k > 0 && lda < k) return CY_ERR_INVALID_VALUE;
    if ((reinterpret_cast<uintptr_t>(y) & 3u) || (k > 0 && (!aligned16(A) || !ld_ok(lda)))) return CY_ERR_MISALIGNED;
    if (k > 0 && overlap(span(y, 1, m, m, 1, 0, 4), span(A, m, k, lda, 1, 0, 2))) return CY_ERR_INVALID_VALUE;
    return launch_rowsum(dt, A, lda, m, k, y, stream);
  }
  const bool has_c = beta != 0.0f;
  if (!D || (k > 0 && (!A || !B)) || (has_c && !C)) return CY_ERR_INVALID_VALUE;
  if (ldd < n || (k > 0 && (lda < k || ldb < n)) || (has_c && ldc < n)) return CY_ERR_INVALID_VALUE;
  if (!aligned16(D) || !ld_ok(ldd) || (reinterpret_cast<uintptr_t>(y) & 3u)) return CY_ERR_MISALIGNED;
  if (k > 0 && (!aligned16(A) || !aligned16(B) || !ld_ok(lda) || !ld_ok(ldb))) return CY_ERR_MISALIGNED;
  if (has_c && (!aligned16(C) || !ld_ok(ldc))) return CY_ERR_MISALIGNED;
  const Range rD = span(D, m, n, ldd, 1, 0, 2);
  const Range rY = span(y, 1, m, m, 1, 0, 4);
  const Range rA = k > 0 ? span(A, m, k, lda, 1, 0, 2) : Range{0, 0};
  const Range rB = k > 0 ? span(B, k, n, ldb, 1, 0, 2) : Range{0, 0};
  const Range rC = has_c ? span(C, m, n, ldc, 1, 0, 2) : Range{0, 0};
  if (overlap(rD, rA) || overlap(rD, rB) || overlap(rY, rA) || overlap(rY, rB) || overlap(rY, rC) || overlap(rY, rD))
    return CY_ERR_INVALID_VALUE;
  if (has_c && !(C == D && ldc == ldd) && overlap(rD, rC)) return CY_ERR_INVALID_VALUE;
  return launch(cy::V_ROWREDUCE, dt, m, n, k, 1, alpha, {A, lda, 0}, {B, ldb, 0}, {nullptr, 0, 0}, beta,
                {C, ldc, 0}, {nullptr, 0, 0}, {D, ldd, 0}, {nullptr, 0, 0}, y, stream);
}

}  // extern "C"
