// C ABI of the ADMM-LP decoder: graph construction, kernel selection and
// launch.  See include/admm_b200.h for the contract.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/admm_b200.h"
#include "bp_launch.h"
#include "cluster_launch.h"
#include "cluster_layout.h"
#include "cluster.cuh"
#include "steps.h"
#include "kernels.cuh"
#include "layout.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(ADMM_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Makes `dev` current for the scope of an entry point and restores the
// caller's current device on every return path.
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    err_ = prev_ == dev ? cudaSuccess : cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev_ >= 0 && changed()) cudaSetDevice(prev_);
  }
  cudaError_t error() const { return err_; }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  bool changed() const {
    int cur = -1;
    return cudaGetDevice(&cur) == cudaSuccess && cur != prev_;
  }
  int prev_ = -1;
  cudaError_t err_ = cudaSuccess;
};

#define ADMM_CUDA(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

}  // namespace

struct admm_graph {
  int device = 0;
  int n_vars = 0, n_checks = 0, n_edges = 0;
  int dmax = 0, dvmax_actual = 0;
  int D = 0, DVMAX = 0, CPT = 0, NT = 0, m_pad = 0, VPT = 0;
  int kind = 0;  // 1 = generic resident, 2 = regular resident, 3 = streaming
  int C = 0;
  int l2_bytes = 0;
  admm::StreamLaunch slaunch[2];
  admm::ShardLaunch shlaunch[2];
  bool shard_ok[2] = {false, false};
  admm::WideLaunch wlaunch[2];
  bool wide_ok[2] = {false, false};
  // cluster engine (cluster.cuh): one cluster per frame; fp64 on 8-CTA clusters only
  bool cluster_ok = false, cluster64_ok = false;
  int cl_nt = 0, cl_smem = 0, cl_clusters = 0, cl_regs = 0;
  int cl64_smem = 0, cl64_clusters = 0, cl64_regs = 0;
  int cl_NPL = 0, cl_NXS = 0, cl_NMS = 0, cl_MC = 0, cl_NO = 0;
  int cl_n_xs[admm::kClusterMax] = {}, cl_n_ms[admm::kClusterMax] = {};
  uint32_t cl_rx_x[admm::kClusterMax] = {}, cl_rx_m[admm::kClusterMax] = {};  // ELEMENTS received per iteration
  bool cl_dense = false;  // every part ships x to every other part (mbarrier-variant safety)
  long long cl_exchange = 0;
  int* cl_chk_slot = nullptr;
  int* cl_chk_orig = nullptr;
  int* cl_own_var = nullptr;
  uint32_t* cl_xsend = nullptr;
  uint32_t* cl_msend = nullptr;
  int* wctbl = nullptr;  // wide engine index tables (wide.cuh)
  int* wvtbl = nullptr;
  int engine_req = 0;
  int shard_G = 0, shard_dv = 0;
  long long shard_EB = 0;
  int smem_optin = 0;
  int num_sms = 0;
  // device arrays
  int* chk_var = nullptr;
  uint16_t* var_pos = nullptr;
  uint8_t* var_deg = nullptr;
  int* edge_base = nullptr;
  int* check_ptr_d = nullptr;   // [n_checks + 1] (step API, steps.cu)
  int* var_edge = nullptr;
  int* var_orig = nullptr;      // relabeled regular layout (kind 2)
  int* edge_ref = nullptr;
  int* var_edge_int = nullptr;
  int* cchk_var = nullptr;       // colored layout (fp32 regular kernels with DV | D)
  int* cvar_orig = nullptr;
  int* cedge_ref = nullptr;
  int* ccheck_rot = nullptr;     // colored layout, D mod DV = 1: per-check rotation
  int* chk_var_ref = nullptr;    // original numbering when chk_var is relabeled (kind 2), else == chk_var
  // BP (bp.cuh): its own CTA shape on the same graph arrays
  admm::BpLaunch bp_launch[2];
  bool bp_ok[2] = {false, false};
  int bp_nt = 0;
  double layout_cost[2] = {0, 0};
  // per-dtype launch data
  admm::ResidentLaunch launch[2];
};

namespace {

const int kBuckets[] = {4, 6, 8, 13, 16, 32};

// cudaFuncAttributeMaxDynamicSharedMemorySize is per kernel and process-wide,
// while one kernel serves many graphs with different shared-memory sizes:
// only ever raise it, so a graph placed earlier with a larger size stays
// launchable after a smaller one was placed.
cudaError_t ensure_smem(const void* fn, int smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& cur = granted[{dev, fn}];
  if (smem <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

int pick_bucket(int d) {
  for (int b : kBuckets)
    if (d <= b) return b;
  return 0;
}

}  // namespace

extern "C" {

int admm_version(void) { return ADMM_B200_VERSION; }

int admm_checked_probe(int bad, float* out, void* stream) {
  if (!out) return fail(ADMM_E_ARG, "null pointer argument");
  const cudaError_t e = admm::launch_checked_probe(bad, out, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "checked probe launch");
  return ADMM_OK;
}

int admm_build_flags(void) {
#ifdef ADMM_CHECKED
  return ADMM_BUILD_CHECKED;
#else
  return 0;
#endif
}

const char* admm_last_error(void) { return g_last_error.c_str(); }

int admm_graph_create(int device, int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                      const int32_t* edge_var, admm_graph** out) {
  return admm_graph_create_ex(device, n_vars, n_checks, check_ptr, edge_var, ADMM_ENGINE_AUTO, out);
}

int admm_graph_create_ex(int device, int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                         const int32_t* edge_var, int engine, admm_graph** out) {
  if (!out || !check_ptr || !edge_var) return fail(ADMM_E_ARG, "null pointer argument");
  if (engine != ADMM_ENGINE_AUTO && engine != ADMM_ENGINE_RESIDENT && engine != ADMM_ENGINE_STREAMING &&
      engine != ADMM_ENGINE_CLUSTER && engine != ADMM_ENGINE_WIDE)
    return fail(ADMM_E_ARG, "unknown engine");
  *out = nullptr;
  if (n_vars <= 0 || n_checks <= 0) return fail(ADMM_E_ARG, "n_vars and n_checks must be positive");
  if (check_ptr[0] != 0) return fail(ADMM_E_ARG, "check_ptr[0] must be 0");
  const int E = check_ptr[n_checks];
  std::vector<std::vector<int>> rows(n_checks);
  std::vector<int> vdeg(n_vars, 0);
  int dmax = 0;
  for (int c = 0; c < n_checks; ++c) {
    const int a = check_ptr[c], b = check_ptr[c + 1];
    if (b <= a) return fail(ADMM_E_ARG, "check " + std::to_string(c) + " has no variables");
    for (int e = a; e < b; ++e) {
      const int v = edge_var[e];
      if (v < 0 || v >= n_vars)
        return fail(ADMM_E_ARG, "check " + std::to_string(c) + " has a variable index out of range");
      rows[c].push_back(v);
    }
    std::sort(rows[c].begin(), rows[c].end());
    for (size_t k = 1; k < rows[c].size(); ++k)
      if (rows[c][k] == rows[c][k - 1])
        return fail(ADMM_E_ARG, "check " + std::to_string(c) + " has a parallel edge");
    for (int v : rows[c]) vdeg[v]++;
    dmax = std::max<int>(dmax, rows[c].size());
  }
  const int dvmax = *std::max_element(vdeg.begin(), vdeg.end());

  auto* g = new admm_graph();
  g->device = device;
  g->engine_req = engine;
  g->n_vars = n_vars;
  g->n_checks = n_checks;
  g->n_edges = E;
  g->dmax = dmax;
  g->dvmax_actual = dvmax;
  g->D = pick_bucket(dmax);
  g->DVMAX = dvmax <= 4 ? 4 : (dvmax <= 8 ? 8 : 0);
  if (!g->D || !g->DVMAX) {
    delete g;
    return fail(ADMM_E_UNSUPPORTED, "check degree > 32 or variable degree > 8 is not supported");
  }
  DeviceGuard guard(device);
  if (guard.error() != cudaSuccess) {
    delete g;
    return cuda_fail(guard.error(), "cudaSetDevice");
  }
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  g->smem_optin = smem_optin;
  cudaDeviceGetAttribute(&g->l2_bytes, cudaDevAttrL2CacheSize, device);

  bool regular = true;
  for (int c = 0; c < n_checks && regular; ++c) regular = (int)rows[c].size() == dmax;
  for (int v = 0; v < n_vars && regular; ++v) regular = vdeg[v] == dvmax;

  // Validate one candidate launch shape for both dtypes and record it.
  const bool dbg = std::getenv("ADMM_B200_DEBUG") != nullptr;
  auto check_one = [&](admm::ResidentLaunch& L, int smem, int nt) -> bool {
    if (smem > smem_optin) return false;
    cudaFuncAttributes fa{};
    const cudaError_t ge = cudaFuncGetAttributes(&fa, L.fn);
    if (dbg)
      std::fprintf(stderr, "[admm] candidate fn=%p nt=%d smem=%d colored=%d np_fixed=%d: %s regs=%d maxthr=%d\n",
                   L.fn, nt, smem, (int)L.colored, L.np_fixed, cudaGetErrorString(ge), fa.numRegs,
                   fa.maxThreadsPerBlock);
    if (ge != cudaSuccess) return false;
    if (fa.numRegs * nt > 65536 || nt > fa.maxThreadsPerBlock) return false;
    if (ensure_smem(L.fn, smem) != cudaSuccess) return false;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L.fn, nt, smem);
    if (dbg) std::fprintf(stderr, "[admm]   occupancy %d\n", occ);
    if (occ < 1) return false;
    L.smem = smem;
    L.occupancy = occ;
    L.regs = fa.numRegs;
    return true;
  };
  auto try_shape = [&](bool reg, int cpt, int nt, int* vpt_out) -> bool {
    const int m_pad = nt * cpt;
    admm::ResidentLaunch Ls[2];
    int vpt = 0;
    for (int dt = 0; dt < 2; ++dt) {
      bool ok = false;
      if (reg) {
        const int need = (n_vars + nt - 1) / nt;
        // tuning override: first fp32 variant to try
        const char* venv = dt == 0 ? std::getenv("ADMM_B200_F32_VARIANT") : nullptr;
        for (int variant = venv ? std::atoi(venv) : 0; !ok; ++variant) {
          admm::ResidentLaunch L{};
          if (!admm::regular_lookup(dt, dmax, dvmax, cpt, need, nt, n_vars, variant, &vpt, &L)) break;
          const int smem = admm::regular_smem_bytes(dt ? 8 : 4, dmax, dvmax, n_vars, L.colored, L.gm_smem, nt, vpt,
                                                    L.np_fixed, L.zs_cpt);
          ok = check_one(L, smem, nt);
          if (ok) Ls[dt] = L;
        }
      } else {
        admm::ResidentLaunch L{};
        if ((long long)g->D * m_pad < 65535 && admm::resident_lookup(dt, g->D, cpt, g->DVMAX, &L))
          ok = check_one(L, admm::ResidentSmem(dt ? 8 : 4, n_vars, g->D * m_pad, g->DVMAX).total, nt);
        if (ok) Ls[dt] = L;
      }
      if (!ok) return false;
    }
    g->launch[0] = Ls[0];
    g->launch[1] = Ls[1];
    *vpt_out = vpt;
    return true;
  };

  bool placed = false;
  const bool try_resident = engine == ADMM_ENGINE_AUTO || engine == ADMM_ENGINE_RESIDENT;
  for (int pass = regular ? 0 : 1; pass < 2 && !placed && try_resident; ++pass) {
    const bool reg = pass == 0;
    const int cpt_env = std::getenv("ADMM_B200_CPT") ? std::atoi(std::getenv("ADMM_B200_CPT")) : 0;
    // Two checks per thread first on the regular path: the second check's
    // independent instruction stream hides the sorting networks' ALU-pipe
    // bursts (measured +9 % over one check per thread on config 2).
    // The regular path keeps the shape with the most resident fp32 warps per
    // SM (ties: the order below), e.g. config 3: three checks per thread with
    // the edge state in shared memory, 2 x 14 warps, over two checks per
    // thread in registers, 1 x 21 warps.
    const int order_reg[4] = {2, 1, 3, 4}, order_gen[4] = {1, 2, 3, 4};
    int best_cpt = 0, best_warps = 0;
    for (int cpt : (reg ? order_reg : order_gen)) {
      if (cpt_env && cpt != cpt_env) continue;  // tuning override
      const int nt = ((n_checks + cpt - 1) / cpt + 31) / 32 * 32;
      if (nt > (reg ? 1024 : 512)) continue;
      int vpt = 0;
      if (!try_shape(reg, cpt, nt, &vpt)) continue;
      const int warps = g->launch[0].occupancy * nt / 32;
      if (dbg) std::fprintf(stderr, "[admm] shape cpt=%d nt=%d: %d fp32 warps/SM\n", cpt, nt, warps);
      if (warps > best_warps) {
        best_warps = warps;
        best_cpt = cpt;
      }
      if (!reg) break;  // generic kernels: first fit
    }
    if (best_cpt) {
      const int nt = ((n_checks + best_cpt - 1) / best_cpt + 31) / 32 * 32;
      int vpt = 0;
      if (try_shape(reg, best_cpt, nt, &vpt)) {
        g->kind = reg ? 2 : 1;
        g->CPT = best_cpt;
        g->NT = nt;
        g->m_pad = nt * best_cpt;
        g->VPT = vpt;
        placed = true;
      }
    }
  }
  if (!placed && (engine == ADMM_ENGINE_AUTO || engine == ADMM_ENGINE_STREAMING || engine == ADMM_ENGINE_WIDE ||
                  engine == ADMM_ENGINE_CLUSTER)) {
    // Streaming engine: batch-interleaved state in global memory (L2-resident).
    bool ok = true;
    for (int dt = 0; dt < 2 && ok; ++dt) {
      admm::StreamLaunch L{};
      const bool reg_stream = regular && dmax == g->D;
      if (!admm::stream_lookup(dt, g->D, g->DVMAX, reg_stream, &L)) { ok = false; break; }
      cudaFuncAttributes fa{};
      if (cudaFuncGetAttributes(&fa, L.fn) != cudaSuccess) { ok = false; break; }
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L.fn, admm::kStreamThreads, 0);
      if (occ < 1) { ok = false; break; }
      L.occupancy = occ;
      L.regs = fa.numRegs;
      g->slaunch[dt] = L;
    }
    if (ok) {
      // Sharded variant: one 512-thread CTA per SM, static graph slice,
      // z/lambda in shared memory (sharded.cuh).  Used when 32 slots fit.
      const int G = g->num_sms;
      const int MB = (n_checks + G - 1) / G;
      long long EB = 0;
      for (int b0 = 0; b0 < n_checks; b0 += MB) {
        const int b1 = std::min(n_checks, b0 + MB);
        EB = std::max<long long>(EB, (long long)check_ptr[b1] - check_ptr[b0]);
      }
      g->shard_G = G;
      g->shard_EB = EB;
      for (int dt = 0; dt < 2; ++dt) {
        admm::ShardLaunch SL{};
        const bool reg_stream = regular && dmax == g->D;
        const int dv_used = reg_stream && dvmax == 3 ? 3 : g->DVMAX;
        if (!admm::shard_lookup(dt, g->D, dv_used, reg_stream, &SL)) continue;
        g->shard_dv = dv_used;
        const admm::ShardGeom geo = admm::shard_geom(dt ? 8 : 4, g->D, dv_used, n_checks, n_vars, EB, G, 32);
        if (geo.total > smem_optin) continue;
        if (ensure_smem(SL.fn, smem_optin) != cudaSuccess) continue;
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, SL.fn) != cudaSuccess || fa.numRegs * (dt ? 512 : 1024) > 65536) continue;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, SL.fn, dt ? 512 : 1024, geo.total);
        if (occ < 1) continue;
        g->shlaunch[dt] = SL;
        g->shard_ok[dt] = std::getenv("ADMM_B200_NO_SHARD") == nullptr;
      }
      cudaGetLastError();
      // Wide HBM-streaming kernel (wide.cuh) for large batches.
      for (int dt = 0; dt < 2; ++dt) {
        admm::WideLaunch WL{};
        const bool reg_stream = regular && dmax == g->D;
        if (!admm::wide_lookup(dt, g->D, reg_stream && dvmax == 3 ? 3 : g->DVMAX, reg_stream, &WL)) continue;
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, WL.fn) != cudaSuccess) continue;
        if (WL.smem > smem_optin || ensure_smem(WL.fn, WL.smem) != cudaSuccess) continue;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, WL.fn, admm::kWideThreads, WL.smem);
        if (occ < 1) continue;
        WL.occupancy = occ;
        WL.regs = fa.numRegs;
        g->wlaunch[dt] = WL;
        g->wide_ok[dt] = std::getenv("ADMM_B200_NO_WIDE") == nullptr;
      }
      if (engine == ADMM_ENGINE_WIDE && !g->wide_ok[0] && !g->wide_ok[1]) {
        delete g;
        return fail(ADMM_E_UNSUPPORTED, "no wide streaming kernel for this graph");
      }
      // Cluster engine (fp32): one cluster per frame, state on chip.  C = 8
      // CTAs of 512 threads, two CTAs (of different clusters: the hardware
      // spreads a cluster over distinct SMs) per SM, measured 409 G
      // edge-updates/s on config 5 against 398 G for C = 4 CTAs of 1024
      // threads, which remains the fallback (ADMM_B200_CLUSTER forces a size).
      int cl_sizes[2] = {8, 4}, n_cl_sizes = 2;
      if (const char* e = std::getenv("ADMM_B200_CLUSTER")) {
        cl_sizes[0] = std::atoi(e);
        n_cl_sizes = 1;
      }
      for (int ci = 0; ci < n_cl_sizes && !g->cluster_ok; ++ci)
      if ((engine == ADMM_ENGINE_AUTO || engine == ADMM_ENGINE_CLUSTER) && regular && dmax == 6 && dvmax == 3 &&
          std::getenv("ADMM_B200_NO_CLUSTER") == nullptr) {
        const int C = cl_sizes[ci];
        const int CPT = 2, VPT = 4;
        const int NT = 4096 / std::max(C, 1);  // compiled CTA size (cluster.cu)
        const int nt_need = ((n_checks + C - 1) / C + CPT - 1) / CPT;
        if (admm::cluster_supported(0, 6, 3, C, CPT, VPT) && nt_need <= NT && n_vars <= C * NT * VPT) {
          long long pm = 20000000, bm = 20000000;
          if (const char* e = std::getenv("ADMM_B200_CLUSTER_MOVES")) pm = bm = std::atoll(e);
          const admm::ClusterLayout CL =
              admm::build_cluster_layout(rows, n_vars, 6, 3, C, NT, CPT, VPT, pm, bm, 4242);
          if (dbg)
            std::fprintf(stderr, "[admm] cluster layout ok=%d %s NPL=%d ghosts=%lld messages=%lld runs=%d bank %.0f->%.0f\n",
                         (int)CL.ok, CL.error.c_str(), CL.NPL, CL.ghost_total, CL.msg_total, CL.msg_runs,
                         CL.bank_cost_before, CL.bank_cost_after);
          if (CL.ok) {
            int npl = CL.NPL, smem = admm::cluster_smem_bytes(0, npl, 3, CL.NXS, CL.NMS);
            int clusters = 0, regs = 0;
            const bool fits = smem <= smem_optin && CL.NO <= 4096 && CL.NPL <= 8192;  // table fields
            const bool cl_placed = fits && admm::cluster_query(0, C, NT, smem, &clusters, &regs) == cudaSuccess && clusters > 0;
            // pad the slot space to a count with a compile-time kernel variant
            // (message rows at immediate offsets: +3 %) when that keeps the occupancy
            if (const int fixed = cl_placed ? admm::cluster_fixed_npl(C, npl) : 0) {
              const int smem_f = admm::cluster_smem_bytes(0, fixed, 3, CL.NXS, CL.NMS);
              int cl_f = 0, regs_f = 0;
              if (smem_f <= smem_optin && std::getenv("ADMM_B200_NO_FIXED_NPL") == nullptr &&
                  admm::cluster_query(0, C, NT, smem_f, &cl_f, &regs_f) == cudaSuccess && cl_f >= clusters) {
                npl = fixed;
                smem = smem_f;
              }
            }
            if (cl_placed) {
              // packed x-send table: own slot | ghost slot << 13 | rank << 29
              std::vector<uint32_t> xs((size_t)C * CL.NXS, 0);
              for (int p = 0; p < C; ++p) {
                for (int r = 0; r < C; ++r)
                  for (int i = CL.xs_start[p * (C + 1) + r]; i < CL.xs_start[p * (C + 1) + r + 1]; ++i) {
                    const uint32_t dst = CL.gbase[r * C + p] + (i - CL.xs_start[p * (C + 1) + r]);
                    xs[(size_t)p * CL.NXS + i] = admm::xs_pack(CL.xsend[(size_t)p * CL.NXS + i], dst, (uint32_t)r);
                  }
                g->cl_n_xs[p] = CL.xs_start[p * (C + 1) + C];
                g->cl_n_ms[p] = CL.n_ms[p];
              }
              // elements each CTA receives per iteration (mbarrier variant): ghost x;
              // messages (+ one 20-byte stop-rule header from every CTA, added at launch)
              bool dense = true;
              for (int p = 0; p < C; ++p) {
                uint32_t gx = 0, gm = 0;
                for (int o = 0; o < C; ++o) {
                  const int n = CL.xs_start[o * (C + 1) + p + 1] - CL.xs_start[o * (C + 1) + p];
                  gx += n;
                  dense = dense && (o == p || n > 0);
                }
                for (int q = 0; q < C; ++q)
                  for (int i = 0; i < CL.n_ms[q]; ++i) gm += (CL.msend[(size_t)q * CL.NMS + i] >> 27) == (uint32_t)p;
                g->cl_rx_x[p] = gx;
                g->cl_rx_m[p] = gm;
              }
              g->cl_dense = dense;
              auto upc = [&](void** dst, const void* src, size_t bytes) -> bool {
                if (*dst) cudaFree(*dst);  // a failed attempt at another cluster size
                *dst = nullptr;
                if (cudaMalloc(dst, bytes) != cudaSuccess) return false;
                return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
              };
              const bool up_ok =
                  upc((void**)&g->cl_chk_slot, CL.chk_slot.data(), CL.chk_slot.size() * sizeof(int)) &&
                  upc((void**)&g->cl_chk_orig, CL.chk_orig.data(), CL.chk_orig.size() * sizeof(int)) &&
                  upc((void**)&g->cl_own_var, CL.own_var.data(), CL.own_var.size() * sizeof(int)) &&
                  upc((void**)&g->cl_xsend, xs.data(), xs.size() * sizeof(uint32_t)) &&
                  upc((void**)&g->cl_msend, CL.msend.data(), CL.msend.size() * sizeof(uint32_t));
              if (up_ok) {
                g->cluster_ok = true;
                g->C = C;
                g->cl_nt = NT;
                g->cl_smem = smem;
                g->cl_clusters = clusters;
                g->cl_regs = regs;
                g->cl_NPL = npl;
                g->cl_NXS = CL.NXS;
                g->cl_NMS = CL.NMS;
                g->cl_MC = CL.MC;
                g->cl_NO = CL.NO;
                g->cl_exchange = CL.ghost_total + CL.msg_total;
                // fp64 (parity mode) on the same layout: twice the shared memory,
                // 128 registers, one 512-thread CTA per SM -- 8-CTA clusters only
                const int smem64 = admm::cluster_smem_bytes(1, npl, 3, CL.NXS, CL.NMS);
                int clusters64 = 0, regs64 = 0;
                if (admm::cluster_supported(1, 6, 3, C, CPT, VPT) && smem64 <= smem_optin &&
                    std::getenv("ADMM_B200_NO_CLUSTER64") == nullptr &&
                    admm::cluster_query(1, C, NT, smem64, &clusters64, &regs64) == cudaSuccess && clusters64 > 0) {
                  g->cluster64_ok = true;
                  g->cl64_smem = smem64;
                  g->cl64_clusters = clusters64;
                  g->cl64_regs = regs64;
                }
                if (dbg)
                  std::fprintf(stderr, "[admm] cluster fp32: C=%d smem=%d clusters=%d regs=%d; fp64: ok=%d smem=%d clusters=%d regs=%d\n",
                               C, smem, clusters, regs, (int)g->cluster64_ok, smem64, clusters64, regs64);
              }
            }
          }
          cudaGetLastError();
        }
      }
      if (engine == ADMM_ENGINE_CLUSTER && !g->cluster_ok) {
        admm_graph_destroy(g);
        return fail(ADMM_E_UNSUPPORTED, "no cluster engine for this graph ((3,6)-regular codes beyond one SM)");
      }
      g->kind = 3;
      g->CPT = 1;
      g->NT = admm::kStreamThreads;
      g->m_pad = (n_checks + admm::kStreamCK - 1) / admm::kStreamCK * admm::kStreamCK;
      placed = true;
    }
  }
  cudaGetLastError();
  if (!placed) {
    delete g;
    return fail(ADMM_E_UNSUPPORTED, "no engine fits this graph");
  }

  // Device layout.
  const int D = g->D, MP = g->m_pad;
  std::vector<int> chk_var((size_t)D * MP, -1);
  std::vector<int> edge_base(n_checks);
  std::vector<std::vector<int>> var_slots(n_vars);
  for (int c = 0; c < n_checks; ++c) {
    edge_base[c] = check_ptr[c];
    for (size_t k = 0; k < rows[c].size(); ++k) {
      chk_var[k * MP + c] = rows[c][k];
      var_slots[rows[c][k]].push_back((int)k * MP + c);  // appended in increasing check order
    }
  }
  std::vector<int> var_edge((size_t)n_vars * dvmax, -1);
  {
    std::vector<int> fill(n_vars, 0);
    for (int c = 0; c < n_checks; ++c)
      for (size_t k = 0; k < rows[c].size(); ++k) {
        const int v = rows[c][k];
        var_edge[(size_t)v * dvmax + fill[v]++] = check_ptr[c] + (int)k;  // increasing edge id
      }
  }
  // Index tables of the wide kernel's work items (wide.cuh ItemFeed).
  std::vector<int> wct, wvt;
  if (g->kind == 3 && (g->wide_ok[0] || g->wide_ok[1])) {
    const int dt = g->wide_ok[0] ? 0 : 1;
    const int WD = g->wlaunch[dt].D, WDV = g->wlaunch[dt].DV;
    if (g->wide_ok[1 - dt] && (g->wlaunch[1 - dt].D != WD || g->wlaunch[1 - dt].DV != WDV)) g->wide_ok[1 - dt] = false;
    const int CT = admm::wide_ct(WD), VT = admm::wide_vt(WDV), CB = admm::kWideCB, VB = admm::kWideVB;
    const int ncb = (n_checks + CB - 1) / CB, nvb = (n_vars + VB - 1) / VB;
    wct.assign((size_t)ncb * CT, -1);
    wvt.assign((size_t)nvb * VT, -1);
    for (int cb = 0; cb < ncb; ++cb)
      for (int q = 0; q < CB; ++q) wct[(size_t)cb * CT + WD * CB + q] = 0;
    for (int c = 0; c < n_checks; ++c) {
      const size_t base = (size_t)(c / CB) * CT;
      for (size_t k = 0; k < rows[c].size(); ++k) wct[base + k * CB + c % CB] = rows[c][k];
      wct[base + WD * CB + c % CB] = check_ptr[c];
    }
    for (int v = 0; v < n_vars; ++v)
      for (int j = 0; j < std::min(dvmax, WDV); ++j)
        wvt[(size_t)(v / VB) * VT + (v % VB) * WDV + j] = var_edge[(size_t)v * dvmax + j];
  }
  std::vector<uint16_t> var_pos((size_t)n_vars * g->DVMAX, 0);
  std::vector<uint8_t> var_deg(n_vars);
  for (int v = 0; v < n_vars; ++v) {
    var_deg[v] = (uint8_t)var_slots[v].size();
    for (size_t j = 0; j < var_slots[v].size(); ++j) var_pos[(size_t)v * g->DVMAX + j] = (uint16_t)var_slots[v][j];
  }
  auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  cudaError_t e1 = up((void**)&g->chk_var, chk_var.data(), chk_var.size() * sizeof(int));
  cudaError_t e2 = up((void**)&g->var_pos, var_pos.data(), var_pos.size() * sizeof(uint16_t));
  cudaError_t e3 = up((void**)&g->var_deg, var_deg.data(), var_deg.size());
  cudaError_t e4 = up((void**)&g->edge_base, edge_base.data(), edge_base.size() * sizeof(int));
  if (e4 == cudaSuccess) e4 = up((void**)&g->check_ptr_d, check_ptr, (size_t)(n_checks + 1) * sizeof(int));
  cudaError_t e5 = up((void**)&g->var_edge, var_edge.data(), var_edge.size() * sizeof(int));
  if (e5 == cudaSuccess && !wct.empty()) e5 = up((void**)&g->wctbl, wct.data(), wct.size() * sizeof(int));
  if (e5 == cudaSuccess && !wvt.empty()) e5 = up((void**)&g->wvtbl, wvt.data(), wvt.size() * sizeof(int));
  cudaError_t e6 = cudaSuccess, e7 = cudaSuccess, e8 = cudaSuccess;
  g->chk_var_ref = g->chk_var;
  if (g->kind == 2 && e1 == cudaSuccess)
    e1 = up((void**)&g->chk_var_ref, chk_var.data(), chk_var.size() * sizeof(int));
  // BP placement: generic check-degree bucket, one or two checks per thread.
  for (int dt = 0; dt < 2; ++dt) {
    for (int cpt : {1, 2}) {
      const int nt = ((n_checks + cpt - 1) / cpt + 31) / 32 * 32;
      if (nt > 512) continue;
      if (g->bp_nt && nt != g->bp_nt) continue;  // one CTA shape for both dtypes
      admm::BpLaunch L{};
      if (!admm::bp_lookup(dt, D, cpt, g->DVMAX, &L)) continue;
      const int smem = admm::bp_smem_bytes(dt ? 8 : 4, n_vars, D * MP, g->DVMAX);
      if (smem > smem_optin) continue;
      cudaFuncAttributes fa{};
      if (cudaFuncGetAttributes(&fa, L.fn) != cudaSuccess || fa.numRegs * nt > 65536) continue;
      if (ensure_smem(L.fn, smem) != cudaSuccess) continue;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L.fn, nt, smem);
      if (occ < 1) continue;
      L.smem = smem;
      L.occupancy = occ;
      L.regs = fa.numRegs;
      g->bp_launch[dt] = L;
      g->bp_ok[dt] = true;
      g->bp_nt = nt;
      break;
    }
  }
  cudaGetLastError();
  if (g->kind == 2) {
    // Bank-conflict-free layout (layout.h): internal variable numbering and
    // the slot of every edge inside its check, with the message of edge
    // (c, v) stored at msg[slot][pi(v)].  chk_var is rewritten in internal
    // variables; the kernel maps back through var_orig / edge_ref.
    long long moves = std::min<long long>(20000000, 4000ll * E);
    if (const char* env = std::getenv("ADMM_B200_LAYOUT_MOVES")) moves = std::atoll(env);
    admm::Layout lay = admm::optimize_layout(rows, n_vars, dmax, moves, 12345);
    for (int retry = 1; retry < 4 && lay.clashes > 0; ++retry)
      lay = admm::optimize_layout(rows, n_vars, dmax, moves * (retry + 1), 12345 + retry);
    if (lay.clashes > 0) {
      admm_graph_destroy(g);
      return fail(ADMM_E_UNSUPPORTED, "no clash-free message layout found");
    }
    g->layout_cost[0] = lay.cost_before;
    g->layout_cost[1] = lay.cost_after;
    std::vector<int> chk2((size_t)D * MP, -1), eref((size_t)MP * dmax, 0), vorig(n_vars), vint((size_t)n_vars * dvmax);
    for (int c = 0; c < n_checks; ++c)
      for (int r = 0; r < dmax; ++r) {
        const int e = c * dmax + r, k = lay.edge_slot[e];
        chk2[(size_t)k * MP + c] = lay.slot_of_var[rows[c][r]];
        eref[(size_t)c * dmax + k] = check_ptr[c] + r;
      }
    std::vector<int> fill(n_vars, 0);
    for (int c = 0; c < n_checks; ++c)  // increasing check order per variable
      for (int r = 0; r < dmax; ++r) {
        const int v = rows[c][r], i = lay.slot_of_var[v];
        vint[(size_t)i * dvmax + fill[v]++] = c * dmax + lay.edge_slot[c * dmax + r];
      }
    for (int i = 0; i < n_vars; ++i) vorig[i] = lay.var_of_slot[i];
    cudaMemcpy(g->chk_var, chk2.data(), chk2.size() * sizeof(int), cudaMemcpyHostToDevice);
    e6 = up((void**)&g->var_orig, vorig.data(), vorig.size() * sizeof(int));
    e7 = up((void**)&g->edge_ref, eref.data(), eref.size() * sizeof(int));
    e8 = up((void**)&g->var_edge_int, vint.data(), vint.size() * sizeof(int));
  }
  if (g->kind == 2 && (g->launch[0].colored || g->launch[1].colored)) {
    // Colored layout (layout.h): message of edge (c, v) at msgc[color][pi(v)].
    long long moves = std::min<long long>(20000000, 4000ll * E);
    if (const char* env = std::getenv("ADMM_B200_LAYOUT_MOVES")) moves = std::atoll(env);
    const admm::Layout lay = admm::optimize_colored_layout(rows, n_vars, dmax, dvmax, moves, 777);
    if (lay.clashes > 0) {
      admm_graph_destroy(g);
      return fail(ADMM_E_UNSUPPORTED, "no equitable edge coloring found");
    }
    g->layout_cost[0] = lay.cost_before;
    g->layout_cost[1] = lay.cost_after;
    std::vector<int> chk2((size_t)D * MP, -1), eref((size_t)MP * dmax, 0), vorig(n_vars);
    for (int c = 0; c < n_checks; ++c)
      for (int r = 0; r < dmax; ++r) {
        const int k = lay.edge_slot[c * dmax + r];
        chk2[(size_t)k * MP + c] = lay.slot_of_var[rows[c][r]];
        eref[(size_t)c * dmax + k] = check_ptr[c] + r;
      }
    for (int i = 0; i < n_vars; ++i) vorig[i] = lay.var_of_slot[i];
    cudaError_t c1 = up((void**)&g->cchk_var, chk2.data(), chk2.size() * sizeof(int));
    cudaError_t c2 = up((void**)&g->cvar_orig, vorig.data(), vorig.size() * sizeof(int));
    cudaError_t c3 = up((void**)&g->cedge_ref, eref.data(), eref.size() * sizeof(int));
    if (c3 == cudaSuccess && dmax % dvmax != 0) {
      std::vector<int> rot((size_t)MP, 0);
      for (int c = 0; c < n_checks; ++c) rot[c] = lay.check_rot[c];
      c3 = up((void**)&g->ccheck_rot, rot.data(), rot.size() * sizeof(int));
    }
    if (e6 == cudaSuccess) e6 = c1;
    if (e7 == cudaSuccess) e7 = c2;
    if (e8 == cudaSuccess) e8 = c3;
  }
  for (cudaError_t e : {e1, e2, e3, e4, e5, e6, e7, e8}) {
    if (e != cudaSuccess) {
      admm_graph_destroy(g);
      return cuda_fail(e, "graph upload");
    }
  }
  *out = g;
  return ADMM_OK;
}

int admm_graph_destroy(admm_graph* g) {
  if (!g) return ADMM_OK;
  DeviceGuard guard(g->device);
  cudaFree(g->chk_var);
  cudaFree(g->var_pos);
  cudaFree(g->var_deg);
  cudaFree(g->edge_base);
  cudaFree(g->check_ptr_d);
  cudaFree(g->var_edge);
  cudaFree(g->wctbl);
  cudaFree(g->cl_chk_slot);
  cudaFree(g->cl_chk_orig);
  cudaFree(g->cl_own_var);
  cudaFree(g->cl_xsend);
  cudaFree(g->cl_msend);
  cudaFree(g->wvtbl);
  cudaFree(g->var_orig);
  cudaFree(g->edge_ref);
  cudaFree(g->var_edge_int);
  cudaFree(g->cchk_var);
  cudaFree(g->cvar_orig);
  cudaFree(g->cedge_ref);
  cudaFree(g->ccheck_rot);
  if (g->chk_var_ref != g->chk_var) cudaFree(g->chk_var_ref);
  delete g;
  return ADMM_OK;
}

int admm_graph_get_info(const admm_graph* g, admm_graph_info* info) {
  if (!g || !info) return fail(ADMM_E_ARG, "null pointer argument");
  std::memset(info, 0, sizeof(*info));
  info->n_vars = g->n_vars;
  info->n_checks = g->n_checks;
  info->n_edges = g->n_edges;
  info->max_check_degree = g->dmax;
  info->max_var_degree = g->dvmax_actual;
  info->engine = g->kind;
  info->degree_bucket = g->D;
  info->checks_per_thread = g->CPT;
  info->threads_per_cta = g->NT;
  const bool st = g->kind == 3;
  info->ctas_per_sm_f32 = st ? g->slaunch[0].occupancy : g->launch[0].occupancy;
  info->ctas_per_sm_f64 = st ? g->slaunch[1].occupancy : g->launch[1].occupancy;
  info->smem_bytes_f32 = st ? 0 : g->launch[0].smem;
  info->smem_bytes_f64 = st ? 0 : g->launch[1].smem;
  info->regs_f32 = st ? g->slaunch[0].regs : g->launch[0].regs;
  info->regs_f64 = st ? g->slaunch[1].regs : g->launch[1].regs;
  info->cluster_size = g->cluster_ok ? g->C : 0;
  info->cluster_active = g->cl_clusters;
  info->cluster_threads = g->cl_nt;
  info->cluster_smem = g->cl_smem;
  info->cluster_regs = g->cl_regs;
  info->cluster_exchange = g->cl_exchange;
  info->layout_cost_before = g->layout_cost[0];
  info->layout_cost_after = g->layout_cost[1];
  info->num_sms = g->num_sms;
  return ADMM_OK;
}

namespace {

// Frame slots of the streaming engine: as many as keep the whole state in
// ~55 % of L2, a multiple of 32, and no more than the batch needs.
int shard_slots(const admm_graph* g, int dtype, int64_t batch) {
  int best = 0;
  for (int S = 32; S <= 512; S *= 2) {
    const admm::ShardGeom geo = admm::shard_geom(dtype ? 8 : 4, g->D, g->shard_dv, g->n_checks, g->n_vars,
                                                 g->shard_EB, g->shard_G, S);
    if (geo.total <= g->smem_optin) best = S;
  }
  if (const char* env = std::getenv("ADMM_B200_STREAM_SLOTS")) {
    const int v = std::atoi(env) / 32 * 32;
    if (v >= 32 && v <= best) best = v;
  }
  const long long need = std::max<long long>(32, (batch + 31) / 32 * 32);
  while (best > 32 && best / 2 >= need) best /= 2;
  return best;
}

// Wide kernel for this call?  Large batches of codes beyond one SM: the
// sharded kernel holds ~64 slots and is latency-bound, the wide kernel
// streams thousands of slots through HBM (wide.cuh).
bool use_wide(const admm_graph* g, int dtype, int64_t batch) {
  if (g->kind != 3 || !g->wide_ok[dtype]) return false;
  if (g->engine_req == ADMM_ENGINE_WIDE) return true;
  long long min_batch = 1024;  // measured crossover (cfg5 fp32): 512 frames sharded 111 G vs wide 82 G, 1024: 81 G vs 127 G
  if (const char* env = std::getenv("ADMM_B200_WIDE_MIN")) min_batch = std::atoll(env);
  return batch >= min_batch;
}

// Cluster engine for this call?  fp32 on graphs that placed it, unless the
// caller forced the streaming kernels.
bool use_cluster(const admm_graph* g, int dtype, int64_t /*batch*/) {
  if (g->kind != 3 || !(dtype == ADMM_F32 ? g->cluster_ok : g->cluster64_ok)) return false;
  return g->engine_req == ADMM_ENGINE_AUTO || g->engine_req == ADMM_ENGINE_CLUSTER;
}

// Slots of the wide kernel: a multiple of the stripe width, up to 8192
// (ADMM_B200_WIDE_SLOTS overrides), no more than the batch needs.
int wide_slots(const admm_graph* g, int dtype, int64_t batch) {
  const long long W = 32ll * g->wlaunch[dtype].vs;
  long long s = 8192;  // measured: 2048 slots 188 G, 4096 201 G, 8192 203 G edge-updates/s (cfg5 fp32)
  if (const char* env = std::getenv("ADMM_B200_WIDE_SLOTS")) s = std::max<long long>(W, std::atoll(env));
  s = s / W * W;
  const long long need = std::max<long long>(W, (batch + W - 1) / W * W);
  return (int)std::min(s, need);
}

int stream_slots(const admm_graph* g, int dtype, int64_t batch) {
  if (g->shard_ok[dtype]) return shard_slots(g, dtype, batch);
  const size_t elem = dtype ? 8 : 4;
  const long long ncblk = (g->n_checks + admm::kStreamCK - 1) / admm::kStreamCK;
  const size_t per = admm::StreamLayout(elem, g->n_edges, g->n_vars, ncblk, 32).total / 32 + 1;
  long long s = (long long)(0.55 * (double)g->l2_bytes) / (long long)per;
  s = std::max<long long>(32, s / 32 * 32);
  s = std::min<long long>(s, 4096);
  if (const char* env = std::getenv("ADMM_B200_STREAM_SLOTS")) {  // tuning override
    const long long v = std::atoll(env);
    if (v >= 32) s = v / 32 * 32;
  }
  const long long need = std::max<long long>(32, (batch + 31) / 32 * 32);
  return (int)std::min(s, need);
}

}  // namespace

int admm_decode_kernel(const admm_graph* g, int dtype, int64_t batch) {
  if (!g) return fail(ADMM_E_ARG, "null graph");
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (g->kind == 3 && use_cluster(g, dtype, batch)) return ADMM_KERNEL_CLUSTER;
  if (g->kind == 3 && use_wide(g, dtype, batch)) return ADMM_KERNEL_WIDE;
  return g->kind;
}

size_t admm_workspace_bytes(const admm_graph* g, int dtype, int64_t batch) {
  if (!g) return 0;
  if (g->kind == 3) {
    if (dtype < 0 || dtype > 1) return 0;
    if (use_cluster(g, dtype, batch)) return 256;  // the frame queue counter (padded)
    if (use_wide(g, dtype, batch)) {
      const int S = wide_slots(g, dtype, batch);
      // upper bound: the synthesis buffer is only laid out for admm_decode_synth
      return admm::WideLayout(dtype ? 8 : 4, g->n_edges, g->n_vars, admm::wide_ncb(g->n_checks), S, true).total;
    }
    const int S = stream_slots(g, dtype, batch);
    if (g->shard_ok[dtype]) return admm::StreamLayout(dtype ? 8 : 4, g->n_edges, g->n_vars, g->shard_G, S, true).total;
    const long long ncblk = (g->n_checks + admm::kStreamCK - 1) / admm::kStreamCK;
    return admm::StreamLayout(dtype ? 8 : 4, g->n_edges, g->n_vars, ncblk, S).total;
  }
  return 256;  // the frame queue counter (padded)
}

}  // extern "C"

namespace {

int make_synth(const admm_channel* ch, uint64_t seed, uint32_t point, int64_t trial0, admm::SynthParams* s) {
  *s = admm::SynthParams{};
  if (!ch) return fail(ADMM_E_ARG, "null channel");
  s->seed_lo = static_cast<uint32_t>(seed);
  s->seed_hi = static_cast<uint32_t>(seed >> 32);
  s->point = point;
  s->trial0 = trial0;
  if (trial0 < 0) return fail(ADMM_E_ARG, "trial0 must be non-negative");
  if (ch->kind == ADMM_CHANNEL_BSC) {
    if (!(ch->p > 0.0 && ch->p <= 0.5)) return fail(ADMM_E_ARG, "BSC crossover probability must be in (0, 0.5]");
    s->kind = 1;
    s->bsc_p = ch->p;
    s->bsc_llr = std::log((1.0 - ch->p) / ch->p);
    return ADMM_OK;
  }
  if (ch->kind == ADMM_CHANNEL_AWGN) {
    if (!(ch->rate > 0.0 && ch->rate <= 1.0)) return fail(ADMM_E_ARG, "code rate must be in (0, 1]");
    if (!std::isfinite(ch->snr_db)) return fail(ADMM_E_ARG, "snr_db must be finite");
    const double var = 1.0 / (2.0 * ch->rate * std::pow(10.0, ch->snr_db / 10.0));  // channels.py:59-61
    s->kind = 2;
    s->sigma = std::sqrt(var);
    s->two_over_var = 2.0 / var;
    return ADMM_OK;
  }
  return fail(ADMM_E_ARG, "unknown channel kind");
}

int decode_impl(const admm_graph* g, int dtype, int64_t batch, const void* gamma, int64_t ld_gamma,
                const admm::SynthParams& synth, double mu, double epsilon, int32_t t_max, double rho,
                void* x_out, int64_t ld_x, uint8_t* hard_out, int64_t ld_hard, int32_t* iters_out,
                uint8_t* flags_out, int32_t* weight_out, const void* z_in, const void* lam_in, void* z_out,
                void* lam_out, int64_t ld_edge, void* workspace, size_t workspace_bytes, void* stream) {
  if (!g) return fail(ADMM_E_ARG, "null graph");
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (batch < 0) return fail(ADMM_E_ARG, "batch must be non-negative");
  if (batch == 0) return ADMM_OK;
  if (synth.kind == 0) {
    if (!gamma) return fail(ADMM_E_ARG, "gamma is null");
    if (ld_gamma < g->n_vars) return fail(ADMM_E_ARG, "ld_gamma < n_vars");
  }
  if (x_out && ld_x < g->n_vars) return fail(ADMM_E_ARG, "ld_x < n_vars");
  if (hard_out && ld_hard < g->n_vars) return fail(ADMM_E_ARG, "ld_hard < n_vars");
  if (!(mu > 0)) return fail(ADMM_E_ARG, "mu must be positive");
  if (!(epsilon > 0)) return fail(ADMM_E_ARG, "epsilon must be positive");
  if (t_max < 1) return fail(ADMM_E_ARG, "t_max must be at least 1");
  if (!(rho >= 1.0 && rho < 2.0)) return fail(ADMM_E_ARG, "rho must be in [1, 2)");
  if ((z_in == nullptr) != (lam_in == nullptr)) return fail(ADMM_E_ARG, "z_in and lam_in go together");
  if ((z_out == nullptr) != (lam_out == nullptr)) return fail(ADMM_E_ARG, "z_out and lam_out go together");
  if ((z_in || z_out) && ld_edge < g->n_edges) return fail(ADMM_E_ARG, "ld_edge < n_edges");
  if (!workspace || workspace_bytes < admm_workspace_bytes(g, dtype, batch))
    return fail(ADMM_E_WORKSPACE, "workspace too small");
  if (batch > (1ll << 31) - 1024) return fail(ADMM_E_ARG, "batch too large for one call");

  DeviceGuard guard(g->device);
  ADMM_CUDA(guard.error());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g->kind == 3 && g->engine_req == ADMM_ENGINE_CLUSTER && dtype == ADMM_F64 && !g->cluster64_ok)
    return fail(ADMM_E_UNSUPPORTED, "the fp64 cluster engine needs 8-CTA clusters with room for the fp64 state "
                                    "(fp64 runs on the streaming engine for this graph)");
  if (g->kind == 3 && use_cluster(g, dtype, batch)) {
    if (z_in || z_out) return fail(ADMM_E_UNSUPPORTED, "state input/output is not supported by the cluster engine");
    ADMM_CUDA(cudaMemsetAsync(workspace, 0, sizeof(int), st));
    const double thr = epsilon * epsilon * (double)g->n_edges;  // admm_decoder.py:169
    auto launch = [&](auto tag) -> cudaError_t {
      using T = decltype(tag);
      constexpr int ES = sizeof(T);
      admm::ClusterParamsT<T> cp{};
      cp.chk_slot = g->cl_chk_slot;
      cp.chk_orig = g->cl_chk_orig;
      cp.own_var = g->cl_own_var;
      cp.xsend = g->cl_xsend;
      cp.msend = g->cl_msend;
      cp.NPL = g->cl_NPL;
      cp.NXS = g->cl_NXS;
      cp.NMS = g->cl_NMS;
      cp.MC = g->cl_MC;
      cp.NO = g->cl_NO;
      const admm::ClusterSmem L(ES, cp.NPL, 3, cp.NXS, cp.NMS);
      cp.sm_xs = L.xs;
      cp.sm_ms = L.ms;
      cp.sm_hdr = L.hdr;
      cp.sm_mbar = L.mbar;
      cp.sm_misc = L.misc;
      for (int r = 0; r < admm::kClusterMax; ++r) {
        cp.n_xs[r] = g->cl_n_xs[r];
        cp.n_ms[r] = g->cl_n_ms[r];
        // bytes received per iteration: ghost x; messages + one 20-byte header from every CTA
        cp.rx_x[r] = ES * g->cl_rx_x[r];
        cp.rx_m[r] = ES * g->cl_rx_m[r] + 20 * g->C;
      }
      cp.dense = g->cl_dense ? 1 : 0;
      cp.n_vars = g->n_vars;
      cp.n_checks = g->n_checks;
      cp.batch = batch;
      cp.gamma = static_cast<const T*>(gamma);
      cp.ld_gamma = ld_gamma;
      cp.mu = static_cast<T>(mu);
      cp.rho = static_cast<T>(rho);
      cp.one_minus_rho = static_cast<T>(1.0 - rho);
      cp.thr = admm::thr_round_up<T>(thr);
      cp.thr_d = thr;
      cp.fx_scale = admm::fx_scale_of(thr);
      cp.fx_thr = admm::fx_thr_of(thr);
      cp.t_max = t_max;
      cp.x_out = static_cast<T*>(x_out);
      cp.ld_x = ld_x;
      cp.hard_out = hard_out;
      cp.ld_hard = ld_hard;
      cp.iters_out = iters_out;
      cp.flags_out = flags_out;
      cp.weight_out = weight_out;
      cp.queue = reinterpret_cast<int*>(workspace);
      cp.synth = synth;
      const bool f64 = ES == 8;
      const int clusters = (int)std::min<long long>(batch, f64 ? g->cl64_clusters : g->cl_clusters);
      return admm::cluster_launch(g->C, cp, clusters, g->cl_nt, f64 ? g->cl64_smem : g->cl_smem, st);
    };
    const cudaError_t le = dtype == ADMM_F64 ? launch(double()) : launch(float());
    if (le != cudaSuccess) return cuda_fail(le, "cluster kernel launch");
    return ADMM_OK;
  }
  if (g->kind == 3) {
    if (z_in || z_out) return fail(ADMM_E_UNSUPPORTED, "state input/output is not supported by the streaming engine");
    const double thr = epsilon * epsilon * (double)g->n_edges;  // admm_decoder.py:169
    admm::StreamGraphArgs sg{g->n_vars, g->n_checks, g->n_edges, g->m_pad, g->dvmax_actual,
                             g->chk_var, g->edge_base, g->var_edge};
    if (use_wide(g, dtype, batch)) {
      const admm::WideLaunch& WL = g->wlaunch[dtype];
      sg.ctbl = g->wctbl;
      sg.vtbl = g->wvtbl;
      admm::ResidentFrameArgs fa{batch, gamma, ld_gamma, mu, rho, thr, t_max, nullptr, nullptr, 0,
                                 x_out, ld_x, hard_out, ld_hard, iters_out, flags_out, weight_out,
                                 nullptr, nullptr, nullptr, synth};
      const int rc = WL.launch(sg, fa, wide_slots(g, dtype, batch), workspace, WL.occupancy * g->num_sms, st);
      if (rc != 0) return cuda_fail((cudaError_t)rc, "cudaLaunchCooperativeKernel(wide)");
      ADMM_CUDA(cudaGetLastError());
      return ADMM_OK;
    }
    const int S = stream_slots(g, dtype, batch);
    const admm::StreamLaunch& L = g->slaunch[dtype];
    const int grid = L.occupancy * g->num_sms;
    admm::ResidentFrameArgs fa{batch, gamma, ld_gamma, mu, rho, thr, t_max, nullptr, nullptr, 0,
                               x_out, ld_x, hard_out, ld_hard, iters_out, flags_out, weight_out,
                               nullptr, nullptr, nullptr, synth};
    int rc;
    if (g->shard_ok[dtype]) {
      const admm::ShardGeom geo = admm::shard_geom(dtype ? 8 : 4, g->D, g->shard_dv, g->n_checks, g->n_vars,
                                                   g->shard_EB, g->shard_G, S);
      rc = g->shlaunch[dtype].launch(sg, fa, S, workspace, g->shard_G, geo, st);
    } else {
      rc = L.launch(sg, fa, S, workspace, grid, st);
    }
    if (rc != 0) return cuda_fail((cudaError_t)rc, "cudaLaunchCooperativeKernel");
    ADMM_CUDA(cudaGetLastError());
    return ADMM_OK;
  }
  ADMM_CUDA(cudaMemsetAsync(workspace, 0, sizeof(int), st));
  const admm::ResidentLaunch& L = g->launch[dtype];
  const long long grid = std::min<long long>(batch, (long long)L.occupancy * g->num_sms);
  const double thr = epsilon * epsilon * (double)g->n_edges;  // admm_decoder.py:169

  admm::ResidentGraphArgs ga{g->n_vars, g->n_checks, g->m_pad, g->chk_var, g->var_pos, g->var_deg,
                             g->edge_base, g->var_edge, g->var_orig, g->edge_ref, g->var_edge_int};
  if (L.colored) {
    ga.chk_var = g->cchk_var;
    ga.var_orig = g->cvar_orig;
    ga.edge_ref = g->cedge_ref;
    ga.var_edge_int = nullptr;
    ga.check_rot = g->ccheck_rot;
  }
  admm::ResidentFrameArgs fa{batch, gamma, ld_gamma, mu, rho, thr, t_max, z_in, lam_in, ld_edge,
                             x_out, ld_x, hard_out, ld_hard, iters_out, flags_out, weight_out,
                             z_out, lam_out, reinterpret_cast<int*>(workspace), synth};
  const cudaError_t le = L.launch(ga, fa, (int)grid, g->NT, L.smem, st);
  if (le != cudaSuccess) return cuda_fail(le, "resident kernel launch");
  return ADMM_OK;
}

}  // namespace

extern "C" {

int admm_decode_batch(const admm_graph* g, int dtype, int64_t batch, const void* gamma,
                      int64_t ld_gamma, double mu, double epsilon, int32_t t_max, double rho,
                      void* x_out, int64_t ld_x, uint8_t* hard_out, int64_t ld_hard,
                      int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out,
                      const void* z_in, const void* lam_in, void* z_out, void* lam_out,
                      int64_t ld_edge, void* workspace, size_t workspace_bytes, void* stream) {
  return decode_impl(g, dtype, batch, gamma, ld_gamma, admm::SynthParams{}, mu, epsilon, t_max, rho, x_out,
                     ld_x, hard_out, ld_hard, iters_out, flags_out, weight_out, z_in, lam_in, z_out, lam_out,
                     ld_edge, workspace, workspace_bytes, stream);
}

int admm_decode_synth(const admm_graph* g, int dtype, int64_t batch, const admm_channel* channel,
                      uint64_t seed, uint32_t point, int64_t trial0, double mu, double epsilon,
                      int32_t t_max, double rho, void* x_out, int64_t ld_x, uint8_t* hard_out,
                      int64_t ld_hard, int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out,
                      void* workspace, size_t workspace_bytes, void* stream) {
  admm::SynthParams sp;
  const int rc = make_synth(channel, seed, point, trial0, &sp);
  if (rc) return rc;
  return decode_impl(g, dtype, batch, nullptr, 0, sp, mu, epsilon, t_max, rho, x_out, ld_x, hard_out, ld_hard,
                     iters_out, flags_out, weight_out, nullptr, nullptr, nullptr, nullptr, 0, workspace,
                     workspace_bytes, stream);
}

int admm_synth_llr(int dtype, int64_t batch, int32_t n_vars, const admm_channel* channel, uint64_t seed,
                   uint32_t point, int64_t trial0, void* out, int64_t ld, void* stream) {
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (batch < 0 || n_vars <= 0) return fail(ADMM_E_ARG, "bad shape");
  if (ld < n_vars) return fail(ADMM_E_ARG, "ld < n_vars");
  admm::SynthParams sp;
  const int rc = make_synth(channel, seed, point, trial0, &sp);
  if (rc) return rc;
  if (batch == 0) return ADMM_OK;
  if (!out) return fail(ADMM_E_ARG, "null output");
  admm::launch_synth(dtype, batch, n_vars, sp, out, ld, reinterpret_cast<cudaStream_t>(stream));
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

int admm_bp_decode_batch(const admm_graph* g, int dtype, int64_t batch, const void* gamma, int64_t ld_gamma,
                         int32_t t_max, double llr_clip, int32_t early_stop, void* beliefs_out,
                         int64_t ld_beliefs, void* x_out, int64_t ld_x, uint8_t* hard_out, int64_t ld_hard,
                         int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (!g) return fail(ADMM_E_ARG, "null graph");
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (batch < 0) return fail(ADMM_E_ARG, "negative batch");
  if (t_max < 1) return fail(ADMM_E_ARG, "t_max must be at least 1");          // bp_decoder.py:31-32
  if (!(llr_clip > 0)) return fail(ADMM_E_ARG, "llr_clip must be positive");   // bp_decoder.py:33-34
  if (batch == 0) return ADMM_OK;
  if (!gamma) return fail(ADMM_E_ARG, "null gamma");
  if (ld_gamma < g->n_vars) return fail(ADMM_E_ARG, "ld_gamma < n_vars");
  if (beliefs_out && ld_beliefs < g->n_vars) return fail(ADMM_E_ARG, "ld_beliefs < n_vars");
  if (x_out && ld_x < g->n_vars) return fail(ADMM_E_ARG, "ld_x < n_vars");
  if (hard_out && ld_hard < g->n_vars) return fail(ADMM_E_ARG, "ld_hard < n_vars");
  if (!workspace || workspace_bytes < 16) return fail(ADMM_E_WORKSPACE, "workspace too small (16 bytes)");
  if (!g->bp_ok[dtype]) return fail(ADMM_E_UNSUPPORTED, "BP: the graph does not fit one SM");
  if (batch > (1ll << 31) - 1024) return fail(ADMM_E_ARG, "batch too large for one call");
  DeviceGuard guard(g->device);
  ADMM_CUDA(guard.error());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ADMM_CUDA(cudaMemsetAsync(workspace, 0, sizeof(int), st));
  const admm::BpLaunch& L = g->bp_launch[dtype];
  const long long grid = std::min<long long>(batch, (long long)L.occupancy * g->num_sms);
  admm::BpGraphArgs ga{g->n_vars, g->n_checks, g->m_pad, g->chk_var_ref, g->var_pos, g->var_deg};
  admm::BpFrameArgs fa{batch, gamma, ld_gamma, llr_clip, t_max, early_stop ? 1 : 0, beliefs_out, ld_beliefs,
                       x_out, ld_x, hard_out, ld_hard, iters_out, flags_out, weight_out,
                       reinterpret_cast<int*>(workspace), admm::SynthParams{}};
  const cudaError_t le = L.launch(ga, fa, (int)grid, g->bp_nt, L.smem, st);
  if (le != cudaSuccess) return cuda_fail(le, "BP kernel launch");
  return ADMM_OK;
}

int admm_phase_profile(int enable, uint64_t* cycles8) {
  if (!admm::phase_profile(enable, reinterpret_cast<unsigned long long*>(cycles8)))
    return fail(ADMM_E_CUDA, "phase profile: CUDA error");
  return ADMM_OK;
}

int admm_wide_phase_profile(int enable, uint64_t* cycles8) {
  if (!admm::wide_phase_profile(enable, reinterpret_cast<unsigned long long*>(cycles8)))
    return fail(ADMM_E_CUDA, "wide phase profile: CUDA error");
  return ADMM_OK;
}

int admm_cluster_phase_profile(int enable, uint64_t* cycles8) {
  if (!admm::cluster_phase_profile(enable, reinterpret_cast<unsigned long long*>(cycles8)))
    return fail(ADMM_E_CUDA, "cluster phase profile: CUDA error");
  return ADMM_OK;
}

int admm_project_batch(int dtype, int64_t m, int32_t d, const void* values, void* out, void* stream) {
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (m < 0 || d < 1) return fail(ADMM_E_ARG, "project_batch expects an (m, d) array with d >= 1");
  if (d > 32) return fail(ADMM_E_UNSUPPORTED, "project_batch supports d <= 32");
  if (m == 0) return ADMM_OK;
  if (!values || !out) return fail(ADMM_E_ARG, "null pointer argument");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!admm::launch_project(dtype, pick_bucket(d), m, d, values, out, st))
    return fail(ADMM_E_UNSUPPORTED, "no projection kernel for this degree");
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

// ---- step API (steps.cu): x_update / z_update / lambda_update, membership ----

namespace {

admm::StepGraph step_graph(const admm_graph* g) {
  return admm::StepGraph{g->n_vars, g->n_checks, g->m_pad, g->D, g->dvmax_actual, g->chk_var_ref, g->check_ptr_d,
                         g->var_edge, g->var_deg};
}

int step_args(const admm_graph* g, int dtype, int64_t batch, int64_t ld_edge) {
  if (!g) return fail(ADMM_E_ARG, "null graph");
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (batch < 0) return fail(ADMM_E_ARG, "batch must be non-negative");
  if (ld_edge < g->n_edges) return fail(ADMM_E_ARG, "ld_edge < n_edges");
  return ADMM_OK;
}

}  // namespace

int admm_x_update(const admm_graph* g, int dtype, int64_t batch, const void* z, const void* lam, int64_t ld_edge,
                  const void* gamma, int64_t ld_gamma, double mu, void* x_out, int64_t ld_x, void* stream) {
  if (const int rc = step_args(g, dtype, batch, ld_edge)) return rc;
  if (ld_gamma < g->n_vars || ld_x < g->n_vars) return fail(ADMM_E_ARG, "ld_gamma / ld_x < n_vars");
  if (!(mu > 0)) return fail(ADMM_E_ARG, "mu must be positive");
  if (batch == 0) return ADMM_OK;
  if (!z || !lam || !gamma || !x_out) return fail(ADMM_E_ARG, "null pointer argument");
  DeviceGuard guard(g->device);
  ADMM_CUDA(guard.error());
  cudaGetLastError();
  admm::launch_x_update(dtype, step_graph(g), batch, z, lam, ld_edge, gamma, ld_gamma, mu, x_out, ld_x,
                        reinterpret_cast<cudaStream_t>(stream));
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

int admm_z_update(const admm_graph* g, int dtype, int64_t batch, const void* x, int64_t ld_x, const void* z_old,
                  const void* lam, int64_t ld_edge, double mu, double rho, void* z_out, void* w_out, void* stream) {
  if (const int rc = step_args(g, dtype, batch, ld_edge)) return rc;
  if (ld_x < g->n_vars) return fail(ADMM_E_ARG, "ld_x < n_vars");
  if (!(mu > 0)) return fail(ADMM_E_ARG, "mu must be positive");
  if (!(rho >= 1.0 && rho < 2.0)) return fail(ADMM_E_ARG, "rho must be in [1, 2)");
  if (batch == 0) return ADMM_OK;
  if (!x || !z_old || !lam || !z_out) return fail(ADMM_E_ARG, "null pointer argument");
  DeviceGuard guard(g->device);
  ADMM_CUDA(guard.error());
  cudaGetLastError();
  if (!admm::launch_z_update(dtype, step_graph(g), batch, x, ld_x, z_old, lam, ld_edge, mu, rho, z_out, w_out,
                             reinterpret_cast<cudaStream_t>(stream)))
    return fail(ADMM_E_UNSUPPORTED, "no z-update kernel for this check-degree bucket");
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

int admm_lambda_update(const admm_graph* g, int dtype, int64_t batch, const void* lam, const void* w, const void* z,
                       int64_t ld_edge, double mu, void* lam_out, void* stream) {
  if (const int rc = step_args(g, dtype, batch, ld_edge)) return rc;
  if (batch == 0) return ADMM_OK;
  if (!lam || !w || !z || !lam_out) return fail(ADMM_E_ARG, "null pointer argument");
  DeviceGuard guard(g->device);
  ADMM_CUDA(guard.error());
  cudaGetLastError();
  admm::launch_lambda_update(dtype, batch, g->n_edges, lam, w, z, ld_edge, mu, lam_out,
                             reinterpret_cast<cudaStream_t>(stream));
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

int admm_membership_batch(int dtype, int64_t m, int32_t d, const void* values, double tol, uint8_t* out,
                          void* stream) {
  if (dtype != ADMM_F32 && dtype != ADMM_F64) return fail(ADMM_E_ARG, "dtype must be ADMM_F32 or ADMM_F64");
  if (m < 0 || d < 1) return fail(ADMM_E_ARG, "membership expects a non-empty 1-D vector per row");
  if (d > 32) return fail(ADMM_E_UNSUPPORTED, "membership supports d <= 32");
  if (!(tol >= 0)) return fail(ADMM_E_ARG, "tol must be non-negative");
  if (m == 0) return ADMM_OK;
  if (!values || !out) return fail(ADMM_E_ARG, "null pointer argument");
  cudaGetLastError();
  if (!admm::launch_membership(dtype, pick_bucket(d), m, d, values, tol, out, reinterpret_cast<cudaStream_t>(stream)))
    return fail(ADMM_E_UNSUPPORTED, "no membership kernel for this degree");
  ADMM_CUDA(cudaGetLastError());
  return ADMM_OK;
}

}  // extern "C"
