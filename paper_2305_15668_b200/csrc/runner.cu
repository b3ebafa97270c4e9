// Native single-GPU round loop: the host side of FederatedRunner's serving loop (engine.py:326-365 for
// sync FedAvg) in two GIL-free calls per round instead of ~40 Python / torch / ctypes operations.
//
//   fedhc_runner_plan   [planner thread]  selection (CPython random.sample on the selector's MT19937
//                       state, engine.py:327) -> native DES (engine.run_round, engine.py:53-230) -> per-client
//                       seeds, descriptors, FedAvg coefficients and the device batch-order block packed into
//                       the slot's pinned staging block (fedhc_round_pack) -> on the plan stream: one H2D
//                       copy + the PCG64 permutations kernel, recorded on the slot's plan event.
//   fedhc_runner_launch [launching thread] on the caller's stream: wait plan -> local_train (all
//                       participants, one launch) -> FedAvg (fp64, list order) -> on the accuracy stream: the
//                       accuracy of the new params (overlapping the next round's training) + an 8-byte D2H.
//   fedhc_runner_result waits for a slot's accuracy count.
//
// Stream / event protocol (per slot s, SLOTS rotating plan buffers):
//   plan stream : wait used[s] (the slot's previous round no longer reads its descriptors / coefficients /
//                 permutations) -> H2D stage -> permutations -> record planned[s]
//   main stream : wait planned[s] -> train -> [wait the previous round's accuracy: it reads the params] ->
//                 FedAvg -> record used[s], agg[s]
//   eval stream : wait agg[s] -> zero count -> accuracy -> D2H count -> record result[s]
// The host reuses a slot's pinned staging block only after planned[s] (its H2D) completed.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace fedhc {
int local_train_entry(const fedhc_client* clients, int n_clients, const double* params, int n_features, int n_classes,
                      int max_batch, bool split, int64_t split_off, void* stream);
}

struct fedhc_runner {
  fedhc_runner_config c;
  std::vector<cudaEvent_t> planned, used, agg, result;
  cudaEvent_t prev_result = nullptr;  // the previous launched round's accuracy (reads the params)
  std::vector<int32_t> order, wi32;
  std::vector<int64_t> wi64;
  std::vector<double> w, starts, ends;
  std::vector<int32_t> k_of;        // participants per slot (launch needs it)
  std::vector<int32_t> chunks_of;   // aggregation chunks per slot (1 for sync FedAvg)
  std::vector<int32_t> sorted;      // async: participants in (end time, id) order
  std::vector<std::vector<int32_t>> chunk_len;  // per slot: chunk sizes
};

namespace {
void destroy_events(fedhc_runner* r) {
  for (auto* v : {&r->planned, &r->used, &r->agg, &r->result})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
}
}  // namespace

using namespace fedhc;

extern "C" int fedhc_runner_create(const fedhc_runner_config* cfg, fedhc_runner** out) {
  if (!cfg || !out) return fail(FEDHC_ERR_VALUE, "runner: null argument");
  if (cfg->slots < 2 || cfg->n_fleet < 0 || cfg->participants < 0 || cfg->participants > cfg->n_fleet)
    return fail(FEDHC_ERR_VALUE, "runner: need slots >= 2 and 0 <= participants <= fleet size");
  auto* r = new fedhc_runner();
  r->c = *cfg;
  const int S = cfg->slots;
  for (auto* v : {&r->planned, &r->used, &r->agg, &r->result}) v->assign(S, nullptr);
  for (int s = 0; s < S; ++s)
    for (auto* v : {&r->planned, &r->used, &r->agg, &r->result}) {
      cudaError_t e = cudaEventCreateWithFlags(&(*v)[s], cudaEventDisableTiming);
      if (e != cudaSuccess) {
        destroy_events(r);
        delete r;
        return cuda_status(e, "runner: cudaEventCreate");
      }
    }
  const int kp = cfg->participants;
  r->order.resize(kp + 1);
  r->wi32.resize(kp + 1);
  r->wi64.resize(kp + 1);
  r->w.resize(kp + 1);
  r->starts.resize(kp + 1);
  r->ends.resize(kp + 1);
  r->k_of.assign(S, 0);
  r->chunks_of.assign(S, 1);
  r->sorted.resize(kp + 1);
  r->chunk_len.assign(S, std::vector<int32_t>(kp + 1, 0));
  if (cfg->async_buffer < 0 || (cfg->async_buffer > 0 && (!cfg->async_host || !cfg->async_dev || !cfg->snapshots))) {
    destroy_events(r);
    delete r;
    return fail(FEDHC_ERR_VALUE, "runner: async aggregation needs the async blocks and snapshots");
  }
  *out = r;
  return FEDHC_OK;
}

extern "C" void fedhc_runner_destroy(fedhc_runner* r) {
  if (!r) return;
  for (cudaEvent_t e : r->result) cudaEventSynchronize(e);
  destroy_events(r);
  delete r;
}

extern "C" int fedhc_runner_plan(fedhc_runner* r, int64_t round_index, double t0, int slot, fedhc_runner_plan_info* info) {
  if (!r || !info || slot < 0 || slot >= r->c.slots) return fail(FEDHC_ERR_VALUE, "runner_plan: bad argument");
  const fedhc_runner_config& c = r->c;
  const int kp = c.participants;
  info->n_launched = info->n_uploaded = info->n_par = info->over_theta = info->degenerate = info->max_rows = 0;
  info->n_chunks = 0;
  info->makespan = info->utilization = info->vacancy_area = info->throughput = info->total_weight = 0.0;
  info->perm_words = info->h2d_bytes = 0;
  // ---- selection (engine.py:327): CPython random.sample(range(n_fleet), kp) on the selector state ----
  int rc = fedhc_mt_sample(c.mt_state, c.n_fleet, kp, r->wi32.data());
  if (rc != FEDHC_OK) return rc;
  memcpy(info->selected, r->wi32.data(), sizeof(int32_t) * (size_t)kp);
  for (int i = 0; i < kp; ++i) {
    if (c.over_theta[r->wi32[i]]) {  // the caller re-runs this selection through the raising DES path
      info->over_theta = 1;
      return FEDHC_OK;
    }
  }
  // ---- the round's DES (engine.run_round) with its trace ----
  for (int i = 0; i < kp; ++i) r->order[i] = c.sim_index[r->wi32[i]];
  fedhc_des_report rep{};
  rc = fedhc_des_run_round(c.sim, c.des_clients, c.des_ids, r->order.data(), kp, &c.des_cfg, t0,
                           static_cast<int>(round_index), 1, r->starts.data(), r->ends.data(), &rep);
  if (rc != FEDHC_OK) return rc;
  info->makespan = rep.makespan;
  info->utilization = rep.utilization;
  info->vacancy_area = rep.vacancy_area;
  info->throughput = rep.throughput;
  info->degenerate = rep.degenerate;
  memcpy(info->starts, r->starts.data(), sizeof(double) * (size_t)kp);
  memcpy(info->ends, r->ends.data(), sizeof(double) * (size_t)kp);
  {
    const fedhc_des_event* ev = nullptr;
    const int32_t* ac = nullptr;
    const double* ash = nullptr;
    const double* pt = nullptr;
    const int32_t* pn = nullptr;
    int npar = 0;
    rc = fedhc_des_trace(c.sim, &ev, &ac, &ash, &pt, &pn, &npar);
    if (rc != FEDHC_OK) return rc;
    int nl = 0, nu = 0;
    for (int e = 0; e < rep.n_events; ++e) {
      if (ev[e].kind == FEDHC_EV_LAUNCHED && nl < kp) info->launch_order[nl++] = ev[e].client;
      if (ev[e].kind == FEDHC_EV_UPLOADED && nu < kp) info->upload_order[nu++] = ev[e].client;
    }
    info->n_launched = nl;
    info->n_uploaded = nu;
    info->n_par = npar <= info->par_cap ? npar : -npar;  // negative: the caller's timeline buffer is too small
    if (npar <= info->par_cap && npar > 0) {
      memcpy(info->par_t, pt, sizeof(double) * (size_t)npar);
      memcpy(info->par_n, pn, sizeof(int32_t) * (size_t)npar);
    }
  }
  // ---- FedAvg weights (fl_core.py:201-212 validation, raised before any device work) ----
  for (int i = 0; i < kp; ++i) r->w[i] = c.weight[r->wi32[i]];
  const double total = fedhc_py_float_sum(r->w.data(), kp);
  if (kp == 0) return fail(FEDHC_ERR_AGGREGATION, "no deltas to aggregate");
  if (total == 0.0) return fail(FEDHC_ERR_AGGREGATION, "weights must not all be zero");
  info->total_weight = total;
  // ---- pack seeds / descriptors / coefficients / batch-order block into the slot's pinned block ----
  cudaError_t e = cudaEventSynchronize(r->planned[slot]);  // the slot's previous H2D has read the block
  if (e != cudaSuccess) return cuda_status(e, "runner_plan: wait for the slot's previous copy");
  for (int i = 0; i < kp; ++i) r->wi64[i] = r->wi32[i];
  int64_t words = 0;
  int32_t mrows = 0;
  rc = fedhc_round_pack(c.seed, round_index, kp, r->wi64.data(), c.reprs, c.rows, c.n_perms, c.n_batches,
                        c.batch_size, c.xptr, c.yptr, c.weight, total, c.lr,
                        reinterpret_cast<uint64_t>(c.plan_dev[slot]), reinterpret_cast<uint64_t>(c.deltas),
                        c.delta_stride_bytes, c.stage_host[slot], &words, &mrows);
  if (rc != FEDHC_OK) return rc;
  if (words > c.plan_cap_words) return fail(FEDHC_ERR_VALUE, "runner_plan: permutation buffer too small");
  info->perm_words = words;
  info->max_rows = mrows;
  const int64_t tot = (int64_t)kp * (24 + (int64_t)sizeof(fedhc_client) + 8);
  info->h2d_bytes = tot;
  int n_chunks = 1;
  if (c.async_buffer > 0) {
    // engine.py:355-364: participants in (per_client_end, id) order, chunks of async_buffer, each chunk's FedAvg
    // normalised by its own weights (fl_core.fedavg on the chunk, CPython float sum)
    for (int i = 0; i < kp; ++i) r->sorted[i] = i;
    std::sort(r->sorted.begin(), r->sorted.begin() + kp, [&](int a, int b) {
      if (r->ends[a] != r->ends[b]) return r->ends[a] < r->ends[b];
      return strcmp(c.des_ids[r->order[a]], c.des_ids[r->order[b]]) < 0;
    });
    double* acoef = reinterpret_cast<double*>(c.async_host[slot]);
    uint64_t* arow = reinterpret_cast<uint64_t*>(c.async_host[slot] + 8 * (size_t)kp);
    n_chunks = 0;
    std::vector<double> cw(c.async_buffer);
    for (int at = 0; at < kp; at += c.async_buffer, ++n_chunks) {
      const int len = std::min(c.async_buffer, kp - at);
      for (int j = 0; j < len; ++j) cw[j] = c.weight[r->wi32[r->sorted[at + j]]];
      const double wc = fedhc_py_float_sum(cw.data(), len);
      if (wc == 0.0) return fail(FEDHC_ERR_AGGREGATION, "weights must not all be zero");
      for (int j = 0; j < len; ++j) {
        const int i = r->sorted[at + j];
        acoef[at + j] = cw[j] / wc;
        arow[at + j] = reinterpret_cast<uint64_t>(c.deltas) + (uint64_t)i * (uint64_t)c.delta_stride_bytes;
      }
      r->chunk_len[slot][n_chunks] = len;
      info->chunk_end[n_chunks] = r->ends[r->sorted[at + len - 1]];
    }
    info->h2d_bytes = tot + 16 * (int64_t)kp;
  }
  info->n_chunks = n_chunks;
  // ---- plan stream: H2D of the block, then the batch order on the device ----
  cudaStream_t ps = static_cast<cudaStream_t>(c.plan_stream);
  e = cudaStreamWaitEvent(ps, r->used[slot], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c.stage_dev[slot], c.stage_host[slot], tot, cudaMemcpyHostToDevice, ps);
  if (e == cudaSuccess && c.async_buffer > 0)
    e = cudaMemcpyAsync(c.async_dev[slot], c.async_host[slot], 16 * (size_t)kp, cudaMemcpyHostToDevice, ps);
  if (e != cudaSuccess) return cuda_status(e, "runner_plan: H2D");
  if (words > 0) {
    uint8_t* md = c.stage_dev[slot];
    rc = fedhc_batch_permutations_device(reinterpret_cast<const uint64_t*>(md),
                                         reinterpret_cast<const int32_t*>(md + 8 * (size_t)kp),
                                         reinterpret_cast<const int32_t*>(md + 12 * (size_t)kp),
                                         reinterpret_cast<const int64_t*>(md + 16 * (size_t)kp), kp, c.plan_dev[slot],
                                         c.rows_max, ps);
    if (rc != FEDHC_OK) return rc;
  }
  e = cudaEventRecord(r->planned[slot], ps);
  if (e != cudaSuccess) return cuda_status(e, "runner_plan: record");
  r->k_of[slot] = kp;
  r->chunks_of[slot] = n_chunks;
  return FEDHC_OK;
}

extern "C" int fedhc_runner_launch(fedhc_runner* r, int slot, void* stream) {
  if (!r || slot < 0 || slot >= r->c.slots) return fail(FEDHC_ERR_VALUE, "runner_launch: bad argument");
  const fedhc_runner_config& c = r->c;
  const int k = r->k_of[slot];
  cudaStream_t ms = static_cast<cudaStream_t>(stream), es = static_cast<cudaStream_t>(c.eval_stream);
  FEDHC_CUDA_TRY(cudaStreamWaitEvent(ms, r->planned[slot], 0));
  uint8_t* md = c.stage_dev[slot];
  const fedhc_client* desc = reinterpret_cast<const fedhc_client*>(md + 24 * (size_t)k);
  const double* coef = reinterpret_cast<const double*>(md + (24 + sizeof(fedhc_client)) * (size_t)k);
  int rc = local_train_entry(desc, k, c.params, c.n_features, c.n_classes, c.max_batch, c.split != 0, c.split_offset,
                             ms);
  if (rc != FEDHC_OK) return rc;
  const int64_t P = (int64_t)c.n_features * c.n_classes + c.n_classes;
  const int kp = c.participants > 0 ? c.participants : 1;
  unsigned long long* cnt = c.correct_dev + (size_t)slot * kp;
  if (c.async_buffer == 0) {
    if (r->prev_result) FEDHC_CUDA_TRY(cudaStreamWaitEvent(ms, r->prev_result, 0));  // it reads the params
    rc = fedhc_fedavg(nullptr, c.deltas, c.delta_stride_bytes / 4, FEDHC_F32, coef, k, c.params, c.params, P, ms);
    if (rc != FEDHC_OK) return rc;
    FEDHC_CUDA_TRY(cudaEventRecord(r->used[slot], ms));
    FEDHC_CUDA_TRY(cudaEventRecord(r->agg[slot], ms));
    FEDHC_CUDA_TRY(cudaStreamWaitEvent(es, r->agg[slot], 0));
    FEDHC_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), es));
    if (c.n_test > 0) {
      rc = fedhc_eval_ctas(c.x_test, c.y_test, c.n_test, c.n_features, c.n_classes, c.params, cnt, c.eval_ctas, es);
      if (rc != FEDHC_OK) return rc;
    }
    FEDHC_CUDA_TRY(cudaMemcpyAsync(c.correct_host + (size_t)slot * kp, cnt, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, es));
  } else {
    // chunked FedAvg in (end, id) order on the params; each chunk's result is snapshotted so its accuracy
    // (eval stream) overlaps the next chunks and the next round's training
    const uint8_t* ad = c.async_dev[slot];
    const double* acoef = reinterpret_cast<const double*>(ad);
    const void* const* arow = reinterpret_cast<const void* const*>(ad + 8 * (size_t)kp);
    double* snap = c.snapshots[slot];
    FEDHC_CUDA_TRY(cudaStreamWaitEvent(ms, r->result[slot], 0));  // the slot's previous accuracy read its snapshots
    int at = 0;
    for (int ch = 0; ch < r->chunks_of[slot]; ++ch) {
      const int len = r->chunk_len[slot][ch];
      rc = fedhc_fedavg(arow + at, nullptr, 0, FEDHC_F32, acoef + at, len, c.params, c.params, P, ms);
      if (rc != FEDHC_OK) return rc;
      FEDHC_CUDA_TRY(cudaMemcpyAsync(snap + (size_t)ch * P, c.params, sizeof(double) * P, cudaMemcpyDeviceToDevice, ms));
      at += len;
    }
    FEDHC_CUDA_TRY(cudaEventRecord(r->used[slot], ms));
    FEDHC_CUDA_TRY(cudaEventRecord(r->agg[slot], ms));
    FEDHC_CUDA_TRY(cudaStreamWaitEvent(es, r->agg[slot], 0));
    const int nc = r->chunks_of[slot];
    FEDHC_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * nc, es));
    if (c.n_test > 0)
      for (int ch = 0; ch < nc; ++ch) {
        rc = fedhc_eval_ctas(c.x_test, c.y_test, c.n_test, c.n_features, c.n_classes, snap + (size_t)ch * P, cnt + ch,
                             c.eval_ctas, es);
        if (rc != FEDHC_OK) return rc;
      }
    FEDHC_CUDA_TRY(cudaMemcpyAsync(c.correct_host + (size_t)slot * kp, cnt, sizeof(unsigned long long) * nc,
                                   cudaMemcpyDeviceToHost, es));
  }
  FEDHC_CUDA_TRY(cudaEventRecord(r->result[slot], es));
  r->prev_result = r->result[slot];
  return FEDHC_OK;
}

extern "C" int fedhc_runner_result(fedhc_runner* r, int slot, int64_t* correct) {
  if (!r || !correct || slot < 0 || slot >= r->c.slots) return fail(FEDHC_ERR_VALUE, "runner_result: bad argument");
  FEDHC_CUDA_TRY(cudaEventSynchronize(r->result[slot]));
  const int kp = r->c.participants > 0 ? r->c.participants : 1;
  for (int ch = 0; ch < r->chunks_of[slot]; ++ch)
    correct[ch] = static_cast<int64_t>(r->c.correct_host[(size_t)slot * kp + ch]);
  return FEDHC_OK;
}
