// Native serving runtime: the discrete-event loop of fragserve's _Sim (simulator.py:430-463) with
// its batching (_service / _enqueue / _stage_done, simulator.py:387-426) and admission control
// (_arrive, simulator.py:377-385), for one deployed plan (or a sequence of per-epoch plans) over
// one horizon.
//
// GX_CLOCK_VIRTUAL replays the reference exactly: the same event heap keyed (t, rank, seq), the same
// push order (so request seqs match _Request.seq), the same float arithmetic; a batch completes at
// dispatch time + the stage's latency table entry for k.  GX_CLOCK_WALL runs the same state machine
// against the wall clock: every dispatched batch executes on the GPU (gx_stage_run on a free
// instance, on a pooled stream of that instance's device) and completes when its CUDA event fires.
// GX_CLOCK_REPLAY keeps the virtual clock (so dispatch order and batch composition are the
// reference's, bit for bit) and also executes every dispatched batch on the GPU, synchronously,
// with the real per-request activations flowing align -> shared through the ragged gather: the
// numerics-parity mode.
//
// Placement (multi-GPU, placement.py:24-70): a stage's instances may live on different GPUs of
// the box.  Each stage keeps ONE global FIFO (simulator.py:91); a dispatched batch goes to a free
// instance, preferring the GPU that holds most of the batch's current activations.  A request's
// activation lives in a device slot on the GPU of the instance that produced it; a batch on another
// GPU gathers it over NVLink through peer access (no copy, no collective).  Per GPU: a stream pool,
// a slot pool, copy streams for DMA ingress and a recycled event pool.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "gx_internal.h"
#include "gx_runtime.h"

namespace {
constexpr int kDoneFlags = 1 << 16;  // completion words (indexed by batch record id)
typedef CUresult (*PFN_streamWriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_streamWriteValue32 stream_write_value32() {
  static const PFN_streamWriteValue32 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_streamWriteValue32>(p);
  }();
  return fn;
}
}  // namespace

using namespace gx;

namespace {

enum { R_REPLAN = 0, R_GEN = 1, R_ARRIVE = 2, R_TIMEOUT = 3, R_DONE = 4 };
constexpr double kEps = 1e-9;  // simulator.py:39

struct Ev {
  double t;
  int rank;
  int64_t seq;
  int64_t a, b;  // payload
  bool operator>(const Ev& o) const {
    if (t != o.t) return t > o.t;
    if (rank != o.rank) return rank > o.rank;
    return seq > o.seq;
  }
};

struct Req {
  int64_t seq;
  int client;
  double gen, slo, deadline, worst_rem;
  int route;
  int stage_idx = 0;
  double stage_enq = 0.0;
  int status = 2;  // 0 completed, 1 dropped, 2 inflight
  double done = NAN;
  int loc = -1;  // device-table index of the GPU holding the current activation (routing)
  // GPU clocks: where the request's current activation lives
  const void* cur = nullptr;
  int cur_dtype = GX_F32;
  int cur_channels = 0;
  int slot = -1, slot_dev = -1;  // device slot holding the activation (DMA ingress / stage outputs)
  int old_slot = -1, old_dev = -1;  // slot the running batch reads; freed when the batch completes
  int64_t result_seq = -1;  // completion slot number; its output lives in ring row result_seq % result_rows
  int h2d_ev = -1, h2d_dev = -1;  // GX_INGRESS_DMA: event of the arrival-time H2D copy into the slot
};

struct Batch {
  int stage;
  int inst = -1;
  int dev = -1;  // device-table index the batch runs on
  std::vector<int> reqs;
  int ev = -1;           // completion event (pool of `dev`; WALL: only with GX_SERVE_DEBUG timing)
  uint32_t flag = 0;     // WALL: value the batch's stream writes to done_flags[batch id] when it completes
  int ev0 = -1;          // GX_SERVE_DEBUG: event recorded ahead of the batch's first command
  double t_disp = 0.0;   // wall ms at dispatch (diagnostics)
  int lane = -1;         // stream-pool lane the batch runs on
  double t_start_est = 0.0;  // GX_LANE_EARLIEST: when the lane was expected to start it (wall ms)
};

struct Stage {
  int batch, instances, free;
  double budget;
  std::vector<double> lat;  // [batch + 1]
  std::deque<int> queue;
  int64_t armed_seq = -1;
  std::vector<gx_stage*> inst;
  std::vector<int> inst_dev;  // device-table index per instance
  std::vector<char> busy;
  int out_final = 0;
  int prio_class = 0;       // stream-priority class of its batches (0 = highest; see lane_class)
  double expected_us = 0.0;  // roofline time of one full batch on an instance's SM budget
  double est_ms = 0.0;       // GX_LANE_EARLIEST: running estimate of one batch's time on its lane
  // wall-clock diagnostics (GX_SERVE_DEBUG): observed dispatch->completion time per batch
  double obs_ms = 0.0, plan_ms = 0.0, exec_ms = 0.0;  // exec: GPU time from the batch's first command
  int64_t obs_n = 0, obs_k = 0;
};

struct Client {
  double rate, slo;
  int route;
  std::vector<double> gaps;  // pre-drawn inter-arrival gaps (Poisson); empty = deterministic
  size_t gap_idx = 0;
  std::vector<double> tr_t, tr_mbps;  // bandwidth trace (piecewise constant, workload.py:46-52)
  std::vector<int> epoch_route;       // per-epoch route (plan transitions); empty = `route` always
};

struct Route {
  int n_stages;
  int stage[2];
  double worst_rem;
  double mobile_ms;
  int64_t payload_bytes;
  const void* ingress;
  int64_t ingress_bytes;
  int ingress_dtype;
  int ingress_channels;
  int home = 0;  // device-table index of the first stage's instance 0 (DMA ingress slots live there)
};

// Per-GPU serving resources.  Stream pool: a batch runs on an idle pooled stream rather than on
// its instance's own stream.  A device has at most CUDA_DEVICE_MAX_CONNECTIONS (32) hardware
// queues; with one stream per instance, plans with > 32 instances alias streams onto shared queues
// and unrelated instances serialise.  Pooling keeps every in-flight batch on its own queue while
// <= pool size.
struct DevRes {
  int device = 0;
  std::vector<cudaStream_t> pool;
  std::vector<int> pool_cls;      // priority class of each lane
  std::vector<int> pool_n;        // batches in flight per lane
  std::vector<double> pool_last;  // wall ms of the lane's last dispatch
  std::vector<double> pool_free;  // GX_LANE_EARLIEST: expected wall ms the lane's queued work ends
  std::vector<cudaStream_t> copy_streams;
  int64_t n_copies = 0;
  void* slots = nullptr;
  std::vector<int> free_slots;
  std::vector<cudaEvent_t> events;  // recycled: batch completions and H2D copies on this device
  std::vector<int> free_events;
};

}  // namespace

struct gx_serve {
  gx_ctx* ctx = nullptr;
  gx_serve_cfg cfg;
  std::vector<Stage> stages;
  std::vector<Route> routes;
  std::vector<Client> clients;
  std::vector<Req> reqs;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap;
  int64_t seq = 0;
  int cur_epoch = 0;  // advanced by REPLAN events (simulator.py:457-458 -> _plan_epoch)
  // dispatch log
  std::vector<double> d_t;
  std::vector<int32_t> d_stage, d_k, d_inst, d_gpu;
  std::vector<int64_t> d_seqs;
  // devices: table index -> GPU ordinal (index 0 = the context's device)
  std::vector<int> gpus;
  std::vector<DevRes> devs;
  int cur_device = -1;
  // batches
  std::vector<Batch> batches;
  std::vector<int> free_batches;
  std::vector<int> inflight;  // batch ids in flight (WALL)
  std::vector<int> pending;   // GX_LANE_EDF: batches decided but held until a lane of their pool is idle
  void* results = nullptr;  // fp32 outputs ring (context device) or mapped pinned host
  int32_t* top1s = nullptr;  // GX_TOP1_*: int32 argmax ring, same rows and memory kind as `results`
  int64_t result_elems = 0;
  int64_t result_cursor = 0;
  double wall_ms = 0.0;
  int64_t n_batches = 0, n_kernels = 0;
  int64_t drops_no_slot = 0, remote_gathers = 0;
  double host_dispatch_ms = 0.0, host_copy_ms = 0.0;  // diagnostics (GX_SERVE_DEBUG)
  int64_t loop_iters = 0;
  double poll_ms = 0.0, busy_ms = 0.0;  // diagnostics: completion polling, iterations that did work
  // WALL completions: each batch's stream writes a sequence value into a pinned, mapped host word
  // (cuStreamWriteValue32) once its work is done, so the host loop polls plain memory instead of
  // one cudaEventQuery per batch in flight (~100 ns each: 90 in flight kept the loop busy ~90%)
  volatile uint32_t* done_flags = nullptr;
  uint32_t flag_seq = 0;
  size_t max_inflight_seen = 0;
  int n_classes = 1;  // stream-priority classes (GX_LANE_PRIO_*)
  int short_lanes = 4;  // GX_LANE_SPLIT / EDF: hardware queues of the first (shortest) pool
  std::vector<int> class_lanes;  // GX_LANE_SPLIT / EDF: hardware queues per stage group
  bool dbg_timing = false;  // GX_SERVE_DEBUG: timing events around each batch (diagnostics only)
  std::chrono::steady_clock::time_point t0;

  bool gpu() const { return cfg.clock != GX_CLOCK_VIRTUAL; }
  void push(double t, int rank, int64_t a, int64_t b = 0) {
    ++seq;
    heap.push(Ev{t, rank, seq, a, b});
  }
  double now_wall() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  double bandwidth_at(const Client& c, double t_s) const {
    // bisect_right(times, t_s) - 1, clamped at 0 (workload.py:46-52)
    auto it = std::upper_bound(c.tr_t.begin(), c.tr_t.end(), t_s);
    long idx = static_cast<long>(it - c.tr_t.begin()) - 1;
    if (idx < 0) idx = 0;
    return c.tr_mbps[idx];
  }
  double next_gen(Client& c, double now) {
    if (!c.gaps.empty()) {
      if (c.gap_idx >= c.gaps.size()) return INFINITY;
      return now + c.gaps[c.gap_idx++];
    }
    return now + 1000.0 / c.rate;
  }
  int dev_index(int gpu_ordinal) {
    for (size_t i = 0; i < gpus.size(); ++i)
      if (gpus[i] == gpu_ordinal) return static_cast<int>(i);
    gpus.push_back(gpu_ordinal);
    return static_cast<int>(gpus.size()) - 1;
  }
  int set_device(int d) {
    if (cur_device != gpus[d]) {
      GX_CUDA(cudaSetDevice(gpus[d]));
      cur_device = gpus[d];
    }
    return GX_OK;
  }
  uint8_t* slot_ptr(int d, int slot) const {
    return static_cast<uint8_t*>(devs[d].slots) + static_cast<size_t>(slot) * cfg.slot_bytes;
  }
  void free_slot(int d, int& slot) {
    if (slot >= 0) devs[d].free_slots.push_back(slot);
    slot = -1;
  }
  int take_event(int d, int* out) {
    DevRes& r = devs[d];
    if (r.free_events.empty()) {
      if (int rc = set_device(d)) return rc;
      cudaEvent_t ev = nullptr;
      GX_CUDA(cudaEventCreateWithFlags(&ev, dbg_timing ? cudaEventDefault : cudaEventDisableTiming));
      r.events.push_back(ev);
      r.free_events.push_back(static_cast<int>(r.events.size()) - 1);
    }
    *out = r.free_events.back();
    r.free_events.pop_back();
    return GX_OK;
  }

  int gen_request(int cid, double now);
  int arrive(int ri, double now);
  int enqueue(int si, int ri, double now);
  int service(int si, double now);
  int stage_done(int bi, double now);
  int complete(int ri, double now);
  int pick_instance(Stage& st, const Batch& b) const;
  int dispatch_gpu(int si, int bi);
  bool lane_idle(int dev, int cls) const {
    const DevRes& dr = devs[dev];
    for (size_t i = 0; i < dr.pool.size(); ++i)
      if (dr.pool_cls[i] == cls && dr.pool_n[i] == 0) return true;
    return false;
  }
  int launch_pending();
  int run();
};

int gx_serve::complete(int ri, double now) {
  Req& r = reqs[ri];
  r.status = 0;
  r.done = now;
  if (r.slot >= 0) free_slot(r.slot_dev, r.slot);
  if (r.old_slot >= 0) free_slot(r.old_dev, r.old_slot);
  return GX_OK;
}

int gx_serve::gen_request(int cid, double now) {
  Client& c = clients[cid];
  Req r;
  r.seq = seq;  // _Request(self.seq, ...) before the ARRIVE push (simulator.py:355)
  r.client = cid;
  r.gen = now;
  r.slo = c.slo;
  r.deadline = now + c.slo;
  r.worst_rem = 0.0;
  // self.routes.get(client_id) of the current epoch (simulator.py:360-365)
  r.route = c.epoch_route.empty() ? c.route
                                  : c.epoch_route[std::min<size_t>(static_cast<size_t>(cur_epoch), c.epoch_route.size() - 1)];
  reqs.push_back(r);
  const int ri = static_cast<int>(reqs.size()) - 1;
  if (reqs[ri].route < 0) {
    reqs[ri].status = 1;
    return GX_OK;
  }
  const Route& rt = routes[reqs[ri].route];
  const double bw = bandwidth_at(c, now / 1000.0);
  // transfer_ms (workload.py:141-142), same operation order
  const double xfer = static_cast<double>(rt.payload_bytes) * 8.0 / (bw * 1e6) * 1000.0;
  const double arrive_t = now + rt.mobile_ms + xfer;
  reqs[ri].worst_rem = rt.worst_rem;
  push(arrive_t, R_ARRIVE, ri);
  return GX_OK;
}

int gx_serve::arrive(int ri, double now) {
  Req& r = reqs[ri];
  const double elapsed = now - r.gen;
  if (elapsed + r.worst_rem > r.slo + kEps) {
    r.status = 1;
    return GX_OK;
  }
  const Route& rt = routes[r.route];
  if (rt.n_stages == 0) return complete(ri, now);
  r.loc = rt.home;
  if (gpu()) {
    r.cur = rt.ingress;
    r.cur_dtype = rt.ingress_dtype;
    r.cur_channels = rt.ingress_channels;
    // zero-copy ingress: r.cur stays the pinned host pointer (UVA) and the first stage's gather
    // reads it over PCIe; only DMA ingress and multi-stage routes need a device slot
    const bool needs_slot = cfg.ingress_from_host == GX_INGRESS_DMA || rt.n_stages > 1 ||
                            !stages[rt.stage[0]].out_final;
    if (needs_slot) {
      DevRes& home = devs[rt.home];
      if (home.free_slots.empty()) {  // out of device slots: counts as an admission drop
        r.status = 1;
        ++drops_no_slot;
        return GX_OK;
      }
      r.slot = home.free_slots.back();
      r.slot_dev = rt.home;
      home.free_slots.pop_back();
      if (cfg.ingress_from_host == GX_INGRESS_DMA) {
        // the copy engine moves the request's activation into its slot as soon as it arrives
        // (it waits in the stage queue anyway); the batch that takes it waits on this copy only
        const double t_c = now_wall();
        if (int rc = set_device(rt.home)) return rc;
        int ei = -1;
        if (int rc = take_event(rt.home, &ei)) return rc;
        cudaStream_t cs = home.copy_streams[home.n_copies++ % home.copy_streams.size()];
        void* dst = slot_ptr(rt.home, r.slot);
        GX_CUDA(cudaMemcpyAsync(dst, rt.ingress, rt.ingress_bytes, cudaMemcpyHostToDevice, cs));
        GX_CUDA(cudaEventRecord(home.events[ei], cs));
        r.h2d_ev = ei;
        r.h2d_dev = rt.home;
        r.cur = dst;
        host_copy_ms += now_wall() - t_c;
      }
    }
  }
  return enqueue(rt.stage[0], ri, now);
}

int gx_serve::enqueue(int si, int ri, double now) {
  reqs[ri].stage_enq = now;
  stages[si].queue.push_back(ri);
  return service(si, now);
}

// A free instance on the GPU that holds most of the batch's activations; ties -> lowest index.
int gx_serve::pick_instance(Stage& st, const Batch& b) const {
  int best = -1, best_score = -1;
  for (int i = 0; i < static_cast<int>(st.busy.size()); ++i) {
    if (st.busy[i]) continue;
    int score = 0;
    for (int ri : b.reqs) score += reqs[ri].loc == st.inst_dev[i];
    if (score > best_score) {
      best = i;
      best_score = score;
    }
  }
  return best;
}

int gx_serve::dispatch_gpu(int si, int bi) {
  Stage& st = stages[si];
  Batch& b = batches[bi];
  gx_stage* g = st.inst[b.inst];
  const int d = b.dev;
  DevRes& dr = devs[d];
  const int k = static_cast<int>(b.reqs.size());
  if (k < 1 || k > 64 || k > g->max_batch) return fail(GX_EINTERNAL, "dispatched batch larger than the instance");
  if (int rc = set_device(d)) return rc;
  const void* src[64];
  int32_t sdt[64];
  void* dst[64];
  int32_t* t1[64];
  int channels = 0;
  // an idle lane of the stage's priority class if there is one, else the class's lane with the
  // fewest / oldest batches in flight
  int lane = -1;
  if (cfg.lane_policy == GX_LANE_EDF) {
    for (int i = 0; i < static_cast<int>(dr.pool.size()) && lane < 0; ++i)
      if (dr.pool_cls[i] == st.prio_class && dr.pool_n[i] == 0) lane = i;
  } else if (cfg.lane_policy == GX_LANE_EARLIEST || cfg.lane_policy == GX_LANE_SPLIT) {
    // the lane (= hardware queue) of the stage's pool expected to free first; ties -> fewer in flight
    for (int i = 0; i < static_cast<int>(dr.pool.size()); ++i) {
      if (dr.pool_cls[i] != st.prio_class) continue;
      const double fi = std::max(b.t_disp, dr.pool_free[i]);
      const double fl = lane < 0 ? 0.0 : std::max(b.t_disp, dr.pool_free[lane]);
      if (lane < 0 || fi < fl - 1e-9 || (fi <= fl + 1e-9 && dr.pool_n[i] < dr.pool_n[lane])) lane = i;
    }
    b.t_start_est = std::max(b.t_disp, dr.pool_free[lane]);
    dr.pool_free[lane] = b.t_start_est + st.est_ms;
  } else {
    for (int i = 0; i < static_cast<int>(dr.pool.size()); ++i) {
      if (dr.pool_cls[i] != st.prio_class) continue;
      if (lane < 0 || dr.pool_n[i] < dr.pool_n[lane] ||
          (dr.pool_n[i] == dr.pool_n[lane] && dr.pool_last[i] < dr.pool_last[lane]))
        lane = i;
    }
  }
  if (lane < 0) return fail(GX_EINTERNAL, "no stream lane for the stage's priority class");
  cudaStream_t sm = dr.pool[lane];
  if (dbg_timing) {
    if (int e = take_event(d, &b.ev0)) return e;
    GX_CUDA(cudaEventRecord(dr.events[b.ev0], sm));
  }
  for (int i = 0; i < k; ++i) {
    Req& r = reqs[b.reqs[i]];
    if (r.h2d_ev >= 0) {  // (cross-device event waits are allowed)
      GX_CUDA(cudaStreamWaitEvent(sm, devs[r.h2d_dev].events[r.h2d_ev], 0));
      devs[r.h2d_dev].free_events.push_back(r.h2d_ev);
      r.h2d_ev = -1;
    }
    src[i] = r.cur;
    sdt[i] = r.cur_dtype;
    channels = std::max(channels, r.cur_channels);
    if (r.loc != d && r.slot >= 0) ++remote_gathers;
    if (st.out_final) {
      r.result_seq = result_cursor++;
      const int64_t row = r.result_seq % cfg.result_rows;
      dst[i] = results ? static_cast<uint8_t*>(results) + row * result_elems * 4 : nullptr;
      t1[i] = top1s ? top1s + row : nullptr;
    } else {
      // the output goes to a slot on this GPU: the request's own if it is here, else a fresh one
      // (the old one is read by this batch's gather and freed when the batch completes); with no
      // free slot here, the scatter writes the request's existing slot over NVLink
      if (r.slot_dev != d && !dr.free_slots.empty()) {
        r.old_slot = r.slot;
        r.old_dev = r.slot_dev;
        r.slot = dr.free_slots.back();
        r.slot_dev = d;
        dr.free_slots.pop_back();
      }
      if (r.slot < 0) return fail(GX_EINTERNAL, "request without an output slot");
      dst[i] = slot_ptr(r.slot_dev, r.slot);
    }
  }
  b.lane = lane;
  dr.pool_n[lane] += 1;
  dr.pool_last[lane] = b.t_disp;
  const int out_dt = st.out_final ? GX_F32 : g->m->tensors[g->out_tid].dtype;
  const bool with_top1 = st.out_final && top1s;
  int rc = gx::stage_run_on(g, sm, k, src, sdt, channels, (st.out_final && !results) ? nullptr : dst, out_dt,
                            with_top1 ? t1 : nullptr);
  if (rc != GX_OK) return rc;
  int kc = 0;
  gx_stage_kernel_count(g, k, &kc);
  n_kernels += kc;
  if (cfg.clock == GX_CLOCK_WALL && done_flags) {
    if (bi >= kDoneFlags) return fail(GX_EINTERNAL, "more batch records than completion words");
    if (dbg_timing) {
      if (int e = take_event(d, &b.ev)) return e;
      GX_CUDA(cudaEventRecord(dr.events[b.ev], sm));
    }
    b.flag = ++flag_seq;
    if (b.flag == 0) b.flag = ++flag_seq;  // 0 marks "no flag"
    const CUresult cr = stream_write_value32()(reinterpret_cast<CUstream>(sm),
                                               reinterpret_cast<CUdeviceptr>(done_flags + bi), b.flag, 0);
    if (cr != CUDA_SUCCESS) return fail(GX_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string(cr) + ")");
  } else {
    b.flag = 0;
    if (int e = take_event(d, &b.ev)) return e;
    GX_CUDA(cudaEventRecord(dr.events[b.ev], sm));
  }
  for (int i = 0; i < k; ++i) {
    Req& r = reqs[b.reqs[i]];
    if (!st.out_final) {
      r.cur = dst[i];
      r.cur_dtype = out_dt;
      r.cur_channels = 0;
    }
  }
  inflight.push_back(bi);
  return GX_OK;
}

// GX_LANE_EDF: every hardware queue runs at most one batch; batches that find no idle lane of their
// pool wait here and are launched earliest-deadline-first (the earliest deadline among their
// requests) as lanes free, instead of queueing FIFO behind whatever batch holds a hardware queue.
int gx_serve::launch_pending() {
  while (!pending.empty()) {
    int best = -1;
    double best_dl = 0.0;
    for (size_t i = 0; i < pending.size(); ++i) {
      const Batch& b = batches[pending[i]];
      if (!lane_idle(b.dev, stages[b.stage].prio_class)) continue;
      double dl = 1e300;
      for (int ri : b.reqs) dl = std::min(dl, reqs[ri].deadline);
      if (best < 0 || dl < best_dl) {
        best = static_cast<int>(i);
        best_dl = dl;
      }
    }
    if (best < 0) return GX_OK;
    const int bi = pending[best];
    pending.erase(pending.begin() + best);
    const double t_a = now_wall();
    int rc = dispatch_gpu(batches[bi].stage, bi);
    host_dispatch_ms += now_wall() - t_a;
    if (rc != GX_OK) return rc;
  }
  return GX_OK;
}

int gx_serve::service(int si, double now) {
  Stage& st = stages[si];
  auto& q = st.queue;
  while (st.free > 0 && !q.empty()) {
    int k;
    if (static_cast<int>(q.size()) >= st.batch) {
      k = st.batch;
    } else if (now - reqs[q.front()].stage_enq >= st.budget - kEps) {
      k = static_cast<int>(q.size());
    } else {
      break;
    }
    int bi;
    if (!free_batches.empty()) {
      bi = free_batches.back();
      free_batches.pop_back();
    } else {
      batches.emplace_back();
      bi = static_cast<int>(batches.size()) - 1;
    }
    Batch& b = batches[bi];
    b.stage = si;
    b.reqs.clear();
    for (int i = 0; i < k; ++i) {
      b.reqs.push_back(q.front());
      q.pop_front();
    }
    st.free -= 1;
    ++n_batches;
    b.inst = pick_instance(st, b);
    if (b.inst < 0) return fail(GX_EINTERNAL, "no free instance although free > 0");
    st.busy[b.inst] = 1;
    b.dev = st.inst_dev[b.inst];
    if (cfg.record_dispatch) {
      d_t.push_back(now);
      d_stage.push_back(si);
      d_k.push_back(k);
      d_inst.push_back(b.inst);
      d_gpu.push_back(gpus[b.dev]);
      for (int ri : b.reqs) d_seqs.push_back(reqs[ri].seq);
    }
    if (cfg.clock == GX_CLOCK_VIRTUAL) {
      push(now + st.lat[k], R_DONE, bi);
    } else if (cfg.clock == GX_CLOCK_REPLAY) {
      // execute now and finish before anything else is dispatched (the next stage's gather reads
      // this batch's outputs); completion stays on the virtual clock
      int rc = dispatch_gpu(si, bi);
      if (rc != GX_OK) return rc;
      GX_CUDA(cudaStreamSynchronize(devs[b.dev].pool[b.lane]));
      inflight.pop_back();
      devs[b.dev].pool_n[b.lane] -= 1;
      devs[b.dev].free_events.push_back(b.ev);
      b.ev = -1;
      push(now + st.lat[k], R_DONE, bi);
    } else {
      const double t_a = now_wall();
      b.t_disp = t_a;
      if (cfg.lane_policy == GX_LANE_EDF && !lane_idle(b.dev, st.prio_class)) {
        pending.push_back(bi);  // launched by launch_pending when a lane of its pool frees
        continue;
      }
      int rc = dispatch_gpu(si, bi);
      host_dispatch_ms += now_wall() - t_a;
      if (rc != GX_OK) return rc;
    }
  }
  if (!q.empty()) {
    // arm the partial-batch timer only when the head is not yet overdue (simulator.py:409-416)
    const Req& head = reqs[q.front()];
    const double tfire = head.stage_enq + st.budget;
    if (tfire > now + kEps && st.armed_seq != head.seq) {
      st.armed_seq = head.seq;
      push(tfire, R_TIMEOUT, si, head.seq);
    }
  }
  return GX_OK;
}

int gx_serve::stage_done(int bi, double now) {
  Batch& b = batches[bi];
  Stage& st = stages[b.stage];
  st.free += 1;
  st.busy[b.inst] = 0;
  if (cfg.clock == GX_CLOCK_WALL) {
    st.obs_ms += now - b.t_disp;
    if (b.reqs.size() < st.lat.size()) st.plan_ms += st.lat[b.reqs.size()];
    st.obs_n += 1;
    st.obs_k += static_cast<int64_t>(b.reqs.size());
  }
  std::vector<int> reqs_copy = b.reqs;
  const int si = b.stage;
  const int dev = b.dev;
  free_batches.push_back(bi);
  for (int ri : reqs_copy) {
    Req& r = reqs[ri];
    if (!st.out_final) r.loc = dev;  // its output now lives on the GPU that ran the batch
    if (r.old_slot >= 0) free_slot(r.old_dev, r.old_slot);
    r.stage_idx += 1;
    const Route& rt = routes[r.route];
    if (r.stage_idx < rt.n_stages) {
      int rc = enqueue(rt.stage[r.stage_idx], ri, now);
      if (rc != GX_OK) return rc;
    } else {
      complete(ri, now);
    }
  }
  return service(si, now);
}

int gx_serve::run() {
  const double horizon = cfg.horizon_ms;
  // _plan_epoch(0) then one REPLAN per later epoch (simulator.py:432-437): they consume seqs
  if (cfg.epoch_ms > 0) {
    long k = 1;
    while (k * cfg.epoch_ms < horizon) {
      push(k * cfg.epoch_ms, R_REPLAN, k);
      ++k;
    }
  }
  for (int cid = 0; cid < static_cast<int>(clients.size()); ++cid) {  // clients pre-sorted by id
    Client& c = clients[cid];
    const double first = c.gaps.empty() ? 0.0 : next_gen(c, 0.0);
    if (first < horizon) push(first, R_GEN, cid);
  }
  t0 = std::chrono::steady_clock::now();
  int rc = GX_OK;
  if (cfg.clock != GX_CLOCK_WALL) {
    while (!heap.empty() && heap.top().t <= horizon + kEps && rc == GX_OK) {
      Ev e = heap.top();
      heap.pop();
      switch (e.rank) {
        case R_REPLAN:
          cur_epoch = static_cast<int>(e.a);
          break;
        case R_GEN: {
          rc = gen_request(static_cast<int>(e.a), e.t);
          const double nxt = next_gen(clients[e.a], e.t);
          if (nxt < horizon) push(nxt, R_GEN, e.a);
          break;
        }
        case R_ARRIVE:
          rc = arrive(static_cast<int>(e.a), e.t);
          break;
        case R_TIMEOUT: {
          Stage& st = stages[e.a];
          if (st.armed_seq == e.b) {
            st.armed_seq = -1;
            rc = service(static_cast<int>(e.a), e.t);
          }
          break;
        }
        default:
          rc = stage_done(static_cast<int>(e.a), e.t);
      }
    }
  } else {
    // Wall clock: scheduled events fire when the clock passes them; completions fire when the
    // batch's CUDA event has completed (polled).  Generation stops at the horizon; requests
    // already generated keep being served (arrivals, partial-batch timeouts, completions) for up
    // to drain_ms more, so the last windows' tails are measured; anything still unfinished then
    // stays "inflight" (status 2), as at the reference's horizon (simulator.py:460-463).
    const double limit = horizon + std::max(0.0, cfg.drain_ms);
    for (;;) {
      const double now = now_wall();
      ++loop_iters;
      max_inflight_seen = std::max(max_inflight_seen, inflight.size());
      const size_t n_before = inflight.size(), heap_before = heap.size();
      for (size_t i = 0; i < inflight.size();) {
        const int bi = inflight[i];
        Batch& b = batches[bi];
        DevRes& dr = devs[b.dev];
        cudaError_t q = cudaSuccess;
        if (b.flag)
          q = done_flags[bi] == b.flag ? cudaSuccess : cudaErrorNotReady;
        else
          q = cudaEventQuery(dr.events[b.ev]);
        if (q == cudaSuccess) {
          inflight[i] = inflight.back();
          inflight.pop_back();
          dr.pool_n[b.lane] -= 1;
          if (cfg.lane_policy == GX_LANE_EARLIEST || cfg.lane_policy == GX_LANE_SPLIT ||
              cfg.lane_policy == GX_LANE_EDF) {
            // the batch ran from about max(dispatch, expected start) to now: refine the stage's estimate
            Stage& xs = stages[b.stage];
            const double took = now - b.t_start_est;
            if (took > 0.0) xs.est_ms += 0.1 * (took - xs.est_ms);
            if (dr.pool_n[b.lane] == 0) dr.pool_free[b.lane] = now;
          }
          if (b.ev0 >= 0) {
            float ms = 0.0f;
            if (b.ev >= 0 && cudaEventElapsedTime(&ms, dr.events[b.ev0], dr.events[b.ev]) == cudaSuccess)
              stages[b.stage].exec_ms += ms;
            cudaGetLastError();
            dr.free_events.push_back(b.ev0);
            b.ev0 = -1;
          }
          if (b.ev >= 0) dr.free_events.push_back(b.ev);
          b.ev = -1;
          if (now <= limit) {
            rc = stage_done(bi, now);
          } else {
            Stage& st = stages[b.stage];
            st.free += 1;
            st.busy[b.inst] = 0;
          }
          if (rc != GX_OK) break;
        } else if (q == cudaErrorNotReady) {
          ++i;
        } else {
          return cuda_fail(q, "batch completion");
        }
      }
      const double t_polled = dbg_timing ? now_wall() : 0.0;
      if (dbg_timing) poll_ms += t_polled - now;
      bool worked = inflight.size() != n_before;
      if (rc == GX_OK && !pending.empty()) rc = launch_pending();
      if (rc != GX_OK) break;
      while (!heap.empty() && heap.top().t <= now && heap.top().t <= limit + kEps && rc == GX_OK) {
        Ev e = heap.top();
        heap.pop();
        worked = true;
        // events fire at their scheduled time (the clock has passed it); state uses that time
        switch (e.rank) {
          case R_REPLAN:
            cur_epoch = static_cast<int>(e.a);
            break;
          case R_GEN: {
            rc = gen_request(static_cast<int>(e.a), e.t);
            const double nxt = next_gen(clients[e.a], e.t);
            if (nxt < horizon) push(nxt, R_GEN, e.a);
            break;
          }
          case R_ARRIVE:
            rc = arrive(static_cast<int>(e.a), e.t);
            break;
          case R_TIMEOUT: {
            Stage& st = stages[e.a];
            if (st.armed_seq == e.b) {
              st.armed_seq = -1;
              rc = service(static_cast<int>(e.a), now);
            }
            break;
          }
          default:
            break;
        }
      }
      if (rc != GX_OK) break;
      if (dbg_timing && worked) busy_ms += now_wall() - now;
      (void)heap_before;
      if (now > horizon && inflight.empty() && pending.empty() && (now > limit || heap.empty() || heap.top().t > limit + kEps)) break;
      if (now > limit + 60000.0) return fail(GX_EINTERNAL, "wall-clock serving did not drain");
    }
  }
  wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (cfg.clock == GX_CLOCK_WALL && getenv("GX_SERVE_DEBUG")) {  // diagnostics only: prints, changes nothing
    std::string groups;
    for (int q : class_lanes) groups += (groups.empty() ? "" : "/") + std::to_string(q);
    fprintf(stderr,
            "[serve] lane_groups=%s wall=%.0fms batches=%lld host_copy=%.0fms host_dispatch=%.0fms (%.1fus/batch) host_busy=%.0fms "
            "event_poll=%.0fms loop_iters=%lld max_inflight=%zu gpus=%zu remote_gathers=%lld\n",
            groups.empty() ? "-" : groups.c_str(), wall_ms, static_cast<long long>(n_batches), host_copy_ms, host_dispatch_ms,
            n_batches ? 1000.0 * host_dispatch_ms / n_batches : 0.0, busy_ms, poll_ms, static_cast<long long>(loop_iters),
            max_inflight_seen, gpus.size(), static_cast<long long>(remote_gathers));
    for (size_t i = 0; i < stages.size(); ++i) {
      const Stage& st = stages[i];
      if (!st.obs_n) continue;
      fprintf(stderr, "[serve] stage %zu: cls=%d exp=%.0fus batches=%lld mean_k=%.2f obs=%.3fms gpu=%.3fms plan=%.3fms ratio=%.2f busy=%.0f%%\n", i,
              st.prio_class, st.expected_us,
              static_cast<long long>(st.obs_n), double(st.obs_k) / st.obs_n, st.obs_ms / st.obs_n, st.exec_ms / st.obs_n,
              st.plan_ms / st.obs_n, st.obs_ms / std::max(1e-9, st.plan_ms),
              100.0 * st.obs_ms / std::max(1e-9, wall_ms * st.instances));
    }
  }
  return rc;
}

namespace {
constexpr double kSplitShortUs = 150.0;    // GX_LANE_SPLIT: group bounds on a stage's expected batch time
// a middle group (bound 1.5 ms) measured worse: the long stages carry most of the GPU time and need
// most of the queues (profiles/r02_lanes_oversubscribe.log), so medium batches share the long group
constexpr double kSplitMediumUs = 1e30;

// GPU-clock resources: per device a stream pool, copy streams, a slot pool; peer access between
// every pair of devices the plan spans (batches gather activations produced on another GPU).
int create_gpu_resources(gx_serve* s) {
  const gx_serve_cfg& cfg = s->cfg;
  for (size_t a = 0; a < s->gpus.size(); ++a)
    for (size_t b = 0; b < s->gpus.size(); ++b) {
      if (a == b) continue;
      int can = 0;
      GX_CUDA(cudaDeviceCanAccessPeer(&can, s->gpus[a], s->gpus[b]));
      if (!can)
        return fail(GX_EINFEASIBLE, "GPU " + std::to_string(s->gpus[a]) + " cannot access GPU " +
                                        std::to_string(s->gpus[b]) + " (peer access needed across the placement)");
      GX_CUDA(cudaSetDevice(s->gpus[a]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(s->gpus[b], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
  s->devs.resize(s->gpus.size());
  for (size_t d = 0; d < s->gpus.size(); ++d) {
    DevRes& r = s->devs[d];
    r.device = s->gpus[d];
    GX_CUDA(cudaSetDevice(r.device));
    if (cfg.slot_bytes > 0) GX_CUDA(cudaMalloc(&r.slots, static_cast<size_t>(cfg.slot_bytes) * cfg.max_inflight));
    for (int i = cfg.max_inflight - 1; i >= 0; --i) r.free_slots.push_back(i);
    // more lanes than the 32 hardware queues: the least-loaded-lane choice then spreads in-flight
    // batches over every queue (measured: 30 lanes -> p99 205 ms, 64 -> 101 ms at 1536 clients)
    // lanes split over the priority classes in use; class c streams get priority greatest + c
    // (lower value = scheduled first when CTAs wait for SMs)
    // GX_LANE_EARLIEST: one lane per hardware queue (the DMA copy stream takes one of the 32)
    const bool per_queue = cfg.lane_policy == GX_LANE_EARLIEST || cfg.lane_policy == GX_LANE_SPLIT ||
                           cfg.lane_policy == GX_LANE_EDF;
    const int lanes = per_queue ? (cfg.ingress_from_host == GX_INGRESS_DMA ? 31 : 32) : std::max(1, dev().serve_streams);
    int least = 0, greatest = 0;
    GX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (int c = 0; c < s->n_classes; ++c) {
      int n = std::max(1, lanes / s->n_classes + (c < lanes % s->n_classes ? 1 : 0));
      int prio = std::min(least, greatest + c);
      if ((cfg.lane_policy == GX_LANE_SPLIT || cfg.lane_policy == GX_LANE_EDF) &&
          static_cast<int>(s->class_lanes.size()) == s->n_classes) {  // queues per stage group
        n = s->class_lanes[c];
        prio = 0;
      }
      for (int i = 0; i < n; ++i) {
        cudaStream_t q = nullptr;
        GX_CUDA(cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, prio));
        r.pool.push_back(q);
        r.pool_cls.push_back(c);
      }
    }
    r.pool_n.assign(r.pool.size(), 0);
    r.pool_last.assign(r.pool.size(), 0.0);
    r.pool_free.assign(r.pool.size(), 0.0);
    if (d == 0 && cfg.clock == GX_CLOCK_WALL && stream_write_value32()) {
      // completion words: written by each batch's stream, read by the host loop (portable: every GPU
      // of a placed plan writes them); a failed probe write keeps the event path
      void* p = nullptr;
      GX_CUDA(cudaHostAlloc(&p, kDoneFlags * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
      std::memset(p, 0, kDoneFlags * sizeof(uint32_t));
      s->done_flags = static_cast<volatile uint32_t*>(p);
      const CUresult cr = stream_write_value32()(reinterpret_cast<CUstream>(r.pool[0]),
                                                 reinterpret_cast<CUdeviceptr>(p), 0u, 0);
      if (cr != CUDA_SUCCESS || cudaStreamSynchronize(r.pool[0]) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeHost(p);
        s->done_flags = nullptr;
      }
    }
    // one FIFO copy stream: arrival order is deadline order, and concurrent copies only share
    // the PCIe link (measured at 1152 clients: p99 88 ms with 1 stream, 205-220 ms with 4 or 16)
    const int ncopy = cfg.ingress_from_host == GX_INGRESS_DMA ? std::max(1, dev().copy_streams) : 0;
    for (int i = 0; i < ncopy; ++i) {
      cudaStream_t q = nullptr;
      GX_CUDA(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
      r.copy_streams.push_back(q);
    }
  }
  int64_t relems = 0;
  for (auto& x : s->stages)
    if (x.out_final && !x.inst.empty()) {
      const gx_stage* g = x.inst[0];
      relems = std::max<int64_t>(relems, tensor_elems(g->m->tensors[g->out_tid]));
    }
  s->result_elems = relems;
  GX_CUDA(cudaSetDevice(s->gpus[0]));
  s->cur_device = s->gpus[0];
  if (relems > 0 && cfg.top1 != GX_TOP1_ONLY) {
    const size_t bytes = static_cast<size_t>(relems) * 4 * cfg.result_rows;
    if (cfg.egress_to_host)
      GX_CUDA(cudaHostAlloc(&s->results, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    else
      GX_CUDA(cudaMalloc(&s->results, bytes));
  }
  if (relems > 0 && cfg.top1 != GX_TOP1_NONE) {
    void* p = nullptr;
    const size_t bytes = static_cast<size_t>(cfg.result_rows) * 4;
    if (cfg.egress_to_host)
      GX_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    else
      GX_CUDA(cudaMalloc(&p, bytes));
    s->top1s = static_cast<int32_t*>(p);
  }
  return GX_OK;
}

// Stream priorities by expected batch time (GX_LANE_PRIO_BY_TIME): the roofline time of one full
// batch on the instance's SM budget (tensor peak or the per-SM L2 feed per op, plus a launch
// allowance).  Short stages (the tail spans planned at batch 1-2) go to the highest-priority lanes:
// when the GPU's SMs are all held by persistent grids, their CTAs are placed first as SMs free up,
// instead of queueing behind long batches (shortest-job-first at the block scheduler).
double expected_batch_us(const gx_stage* g, int k) {
  double us = 0.0;
  const double sm = std::max(1, g->sm_budget);
  for (int oi : g->ops) {
    double f = 0.0, b = 0.0;
    gx::op_work(g->m->ops[oi], g->m->tensors.data(), k, &f, &b);
    us += std::max(f / (sm * 11.2e6), b / (sm * 1.7e5)) + 3.0;  // 11.2 TFLOP/s and ~170 GB/s per SM
  }
  return us;
}

void classify_stages(gx_serve* s) {
  s->n_classes = 1;
  for (Stage& x : s->stages) {
    x.prio_class = 0;
    x.expected_us = x.inst.empty() ? 0.0 : expected_batch_us(x.inst[0], x.batch);
  }
  for (Stage& x : s->stages) x.est_ms = 1.5e-3 * x.expected_us;  // refined by measured batch times
  if (s->cfg.lane_policy == GX_LANE_SPLIT || s->cfg.lane_policy == GX_LANE_EDF) {
    // stages grouped by expected batch time (< 150 us: the tail spans at batch 1-2; < 1.5 ms; longer),
    // each group with hardware queues of its own, so a batch never waits in a queue behind a batch
    // of a much longer kind; queues per group follow the group's expected occupancy: per stage its
    // request rate (the clients routed through it, any epoch) / batch x ~3x its roofline batch time
    std::vector<double> rate(s->stages.size(), 0.0);
    for (const Client& c : s->clients) {
      std::vector<int> rs = c.epoch_route;
      if (rs.empty()) rs.push_back(c.route);
      std::vector<char> seen(s->stages.size(), 0);
      for (int ri : rs) {
        if (ri < 0) continue;
        const Route& rt = s->routes[ri];
        for (int j = 0; j < rt.n_stages; ++j)
          if (!seen[rt.stage[j]]) {
            seen[rt.stage[j]] = 1;
            rate[rt.stage[j]] += c.rate;
          }
      }
    }
    double occ[3] = {0.0, 0.0, 0.0};
    for (size_t i = 0; i < s->stages.size(); ++i) {
      Stage& x = s->stages[i];
      x.prio_class = x.expected_us < kSplitShortUs ? 0 : x.expected_us < kSplitMediumUs ? 1 : 2;
      occ[x.prio_class] += rate[i] / x.batch * std::max(50.0, 3.0 * x.expected_us) * 1e-6;
    }
    // compact the classes in use to 0..n-1
    int remap[3] = {-1, -1, -1}, n = 0;
    std::vector<int> used;
    for (const Stage& x : s->stages) used.push_back(x.prio_class);
    for (int c = 0; c < 3; ++c)
      if (std::find(used.begin(), used.end(), c) != used.end()) remap[c] = n++;
    for (Stage& x : s->stages) x.prio_class = remap[x.prio_class];
    s->n_classes = n;
    s->class_lanes.assign(n, 0);
    const int lanes = s->cfg.ingress_from_host == GX_INGRESS_DMA ? 31 : 32;
    // the shorter groups get twice their expected occupancy plus one queue (headroom: their
    // batches are many and latency-critical), the longest group the rest (at least 8)
    int given = 0, last = -1;
    for (int c = 0; c < 3; ++c)
      if (remap[c] >= 0) last = c;
    for (int c = 0; c < 3; ++c) {
      if (remap[c] < 0 || c == last) continue;
      const int q = std::min(16, std::max(2, static_cast<int>(std::ceil(2.0 * occ[c])) + 1));
      s->class_lanes[remap[c]] = q;
      given += q;
    }
    s->class_lanes[remap[last]] = lanes - given;
    while (s->class_lanes[remap[last]] < 8) {  // keep >= 8 for the longest group: trim the others
      int big = -1;
      for (int c = 0; c < n; ++c)
        if (c != remap[last] && (big < 0 || s->class_lanes[c] > s->class_lanes[big])) big = c;
      if (big < 0 || s->class_lanes[big] <= 2) break;
      --s->class_lanes[big];
      ++s->class_lanes[remap[last]];
    }
    s->short_lanes = s->class_lanes[0];
    return;
  }
  if (s->cfg.lane_policy != GX_LANE_PRIO_BY_TIME) return;
  // three classes: < 300 us, < 2 ms, longer
  for (Stage& x : s->stages) x.prio_class = x.expected_us < 300.0 ? 0 : x.expected_us < 2000.0 ? 1 : 2;
  s->n_classes = 3;
}

int device_of_pointer(const void* p, int fallback) {
  cudaPointerAttributes at;
  if (p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice) return at.device;
  cudaGetLastError();
  return fallback;
}
}  // namespace

extern "C" {

int gx_serve_create(gx_ctx* ctx, int n_stages, const gx_serve_stage* st, int n_routes, const gx_serve_route* rt,
                    int n_clients, const gx_serve_client* cl, const gx_serve_cfg* cfg, gx_serve** out) {
  if (!ctx || !out || !cfg || (n_stages && !st) || (n_routes && !rt) || (n_clients && !cl))
    return fail(GX_EINVAL, "null arg");
  gx_serve* s = new gx_serve();
  s->ctx = ctx;
  s->cfg = *cfg;
  const bool gpu_clock = cfg->clock != GX_CLOCK_VIRTUAL;
  s->dbg_timing = cfg->clock == GX_CLOCK_WALL && getenv("GX_SERVE_DEBUG") != nullptr;  // diagnostics only
  s->gpus.push_back(gpu_clock ? ctx->device : 0);
  for (int i = 0; i < n_stages; ++i) {
    Stage x;
    x.batch = st[i].batch;
    x.instances = st[i].instances;
    x.free = st[i].instances;
    x.budget = st[i].budget_ms;
    x.out_final = st[i].out_final;
    if (x.batch < 1 || x.batch > 64 || x.instances < 1) {
      delete s;
      return fail(GX_EINVAL, "stage needs 1 <= batch <= 64 and instances >= 1");
    }
    if (st[i].lat_ms) x.lat.assign(st[i].lat_ms, st[i].lat_ms + x.batch + 1);
    if (cfg->clock == GX_CLOCK_REPLAY && x.lat.empty()) {
      delete s;
      return fail(GX_EINVAL, "replay clock needs a latency table per stage");
    }
    x.busy.assign(x.instances, 0);
    if (gpu_clock) {
      if (!st[i].inst) {
        delete s;
        return fail(GX_EINVAL, "wall clock needs executor instances per stage");
      }
      for (int j = 0; j < x.instances; ++j) {
        gx_stage* g = static_cast<gx_stage*>(st[i].inst[j]);
        if (!g || g->max_batch < x.batch) {
          delete s;
          return fail(GX_EINVAL, "stage " + std::to_string(i) + ": executor instance " + std::to_string(j) +
                                     (g ? " has max_batch " + std::to_string(g->max_batch) + " < stage batch " +
                                              std::to_string(x.batch)
                                        : " is null"));
        }
        x.inst.push_back(g);
        x.inst_dev.push_back(s->dev_index(g->m->ctx->device));
      }
    } else {
      if (x.lat.empty()) {
        delete s;
        return fail(GX_EINVAL, "virtual clock needs a latency table per stage");
      }
      for (int j = 0; j < x.instances; ++j) x.inst_dev.push_back(s->dev_index(st[i].inst_gpu ? st[i].inst_gpu[j] : 0));
    }
    s->stages.push_back(std::move(x));
  }
  for (int i = 0; i < n_routes; ++i) {
    Route r;
    r.n_stages = rt[i].n_stages;
    r.stage[0] = rt[i].stage[0];
    r.stage[1] = rt[i].stage[1];
    r.worst_rem = rt[i].worst_rem_ms;
    r.mobile_ms = rt[i].mobile_ms;
    r.payload_bytes = rt[i].payload_bytes;
    r.ingress = rt[i].ingress;
    r.ingress_bytes = rt[i].ingress_bytes;
    r.ingress_dtype = rt[i].ingress_dtype;
    r.ingress_channels = rt[i].ingress_channels;
    for (int j = 0; j < r.n_stages; ++j)
      if (r.stage[j] < 0 || r.stage[j] >= n_stages) {
        delete s;
        return fail(GX_EINVAL, "route references a bad stage");
      }
    if (r.ingress && (reinterpret_cast<uintptr_t>(r.ingress) & 15u)) {
      // the gather and the DMA copy move 16-byte vectors: every ingress row starts 16-byte aligned
      delete s;
      return fail(GX_EINVAL, "route ingress pointer is not 16-byte aligned");
    }
    if (r.n_stages > 0) {
      // where the request's activation is when it arrives: DMA ingress lands on the first stage's
      // instance-0 GPU; device-resident ingress lives where it was allocated
      r.home = s->stages[r.stage[0]].inst_dev[0];
      if (gpu_clock && cfg->ingress_from_host != GX_INGRESS_DMA && r.ingress)
        r.home = s->dev_index(device_of_pointer(r.ingress, s->gpus[r.home]));
    }
    s->routes.push_back(r);
  }
  for (int i = 0; i < n_clients; ++i) {
    Client c;
    c.rate = cl[i].rate_rps;
    c.slo = cl[i].slo_ms;
    c.route = cl[i].route;
    if (cl[i].gen_gaps_ms && cl[i].n_gaps > 0) c.gaps.assign(cl[i].gen_gaps_ms, cl[i].gen_gaps_ms + cl[i].n_gaps);
    if (cl[i].n_trace < 1 || !cl[i].trace_t_s || !cl[i].trace_mbps) {
      delete s;
      return fail(GX_EINVAL, "client needs a bandwidth trace");
    }
    c.tr_t.assign(cl[i].trace_t_s, cl[i].trace_t_s + cl[i].n_trace);
    if (cl[i].epoch_route && cl[i].n_epoch_route > 0) {
      c.epoch_route.assign(cl[i].epoch_route, cl[i].epoch_route + cl[i].n_epoch_route);
      for (int rix : c.epoch_route)
        if (rix >= n_routes) {
          delete s;
          return fail(GX_EINVAL, "client references a bad epoch route");
        }
    }
    c.tr_mbps.assign(cl[i].trace_mbps, cl[i].trace_mbps + cl[i].n_trace);
    if (c.route >= n_routes) {
      delete s;
      return fail(GX_EINVAL, "client references a bad route");
    }
    s->clients.push_back(std::move(c));
  }
  if (gpu_clock) {
    if (cfg->max_inflight < 1) {
      delete s;
      return fail(GX_EINVAL, "max_inflight must be >= 1 when batches execute");
    }
    // Every route's ingress must exist, and a request that needs a device slot (DMA ingress, or a
    // stage whose output feeds another stage) must fit it: the slot holds the DMA-copied ingress
    // and then each intermediate boundary the route writes (stage output elems x element size).
    int64_t need = 0;
    for (size_t i = 0; i < s->routes.size(); ++i) {
      const Route& r = s->routes[i];
      if (r.n_stages == 0) continue;
      if (!r.ingress || r.ingress_bytes <= 0) {
        delete s;
        return fail(GX_EINVAL, "route " + std::to_string(i) + " has no ingress buffer");
      }
      if (cfg->ingress_from_host == GX_INGRESS_DMA) need = std::max(need, r.ingress_bytes);
      for (int j = 0; j < r.n_stages; ++j) {
        const Stage& x = s->stages[r.stage[j]];
        if (x.out_final) continue;
        const gx_stage* g = x.inst[0];
        const gx_tensor& to = g->m->tensors[g->out_tid];
        need = std::max<int64_t>(need, tensor_elems(to) * elem_size(to.dtype));
      }
    }
    if (s->cfg.slot_bytes == 0) s->cfg.slot_bytes = (need + 255) / 256 * 256;
    if (s->cfg.slot_bytes < need) {
      const int64_t have = s->cfg.slot_bytes;
      delete s;
      return fail(GX_EINVAL, "slot_bytes " + std::to_string(have) + " < " + std::to_string(need) +
                                 " bytes a route needs (ingress copy or intermediate boundary)");
    }
    if (s->cfg.result_rows <= 0) s->cfg.result_rows = cfg->max_inflight;
    classify_stages(s);
    if (cfg->top1 < GX_TOP1_NONE || cfg->top1 > GX_TOP1_ONLY) {
      delete s;
      return fail(GX_EINVAL, "top1 must be GX_TOP1_NONE, GX_TOP1_WITH_LOGITS or GX_TOP1_ONLY");
    }
    if (cfg->top1 != GX_TOP1_NONE)
      for (const Stage& x : s->stages)
        if (x.out_final && !x.inst.empty() && x.inst[0]->m->tensors[x.inst[0]->out_tid].dtype != GX_F32) {
          delete s;
          return fail(GX_EINVAL, "top-1 needs a classifier chain (fp32 logits as the chain output)");
        }
    if (int rc = create_gpu_resources(s)) {
      gx_serve_destroy(s);
      return rc;
    }
  }
  *out = s;
  return GX_OK;
}

int gx_serve_run(gx_serve* s) {
  if (!s) return fail(GX_EINVAL, "null arg");
  if (s->gpu()) {
    GX_CUDA(cudaSetDevice(s->gpus[0]));
    s->cur_device = s->gpus[0];
  }
  return s->run();
}

int gx_serve_count_requests(gx_serve* s, int64_t* n) {
  if (!s || !n) return fail(GX_EINVAL, "null arg");
  *n = static_cast<int64_t>(s->reqs.size());
  return GX_OK;
}

int gx_serve_requests(gx_serve* s, int32_t* client, double* gen_ms, double* done_ms, double* deadline_ms,
                      int32_t* status) {
  if (!s) return fail(GX_EINVAL, "null arg");
  for (size_t i = 0; i < s->reqs.size(); ++i) {
    const Req& r = s->reqs[i];
    if (client) client[i] = r.client;
    if (gen_ms) gen_ms[i] = r.gen;
    if (done_ms) done_ms[i] = r.done;
    if (deadline_ms) deadline_ms[i] = r.deadline;
    if (status) status[i] = r.status;
  }
  return GX_OK;
}

int gx_serve_count_dispatch(gx_serve* s, int64_t* n_batches, int64_t* n_items) {
  if (!s) return fail(GX_EINVAL, "null arg");
  if (n_batches) *n_batches = static_cast<int64_t>(s->d_t.size());
  if (n_items) *n_items = static_cast<int64_t>(s->d_seqs.size());
  return GX_OK;
}

int gx_serve_dispatch(gx_serve* s, double* t_ms, int32_t* stage, int32_t* k, int64_t* seqs) {
  if (!s) return fail(GX_EINVAL, "null arg");
  if (t_ms) std::copy(s->d_t.begin(), s->d_t.end(), t_ms);
  if (stage) std::copy(s->d_stage.begin(), s->d_stage.end(), stage);
  if (k) std::copy(s->d_k.begin(), s->d_k.end(), k);
  if (seqs) std::copy(s->d_seqs.begin(), s->d_seqs.end(), seqs);
  return GX_OK;
}

int gx_serve_dispatch_placement(gx_serve* s, int32_t* inst, int32_t* gpu) {
  if (!s) return fail(GX_EINVAL, "null arg");
  if (inst) std::copy(s->d_inst.begin(), s->d_inst.end(), inst);
  if (gpu) std::copy(s->d_gpu.begin(), s->d_gpu.end(), gpu);
  return GX_OK;
}

int gx_serve_stats(gx_serve* s, double* wall_ms, int64_t* batches, int64_t* kernels) {
  if (!s) return fail(GX_EINVAL, "null arg");
  if (wall_ms) *wall_ms = s->wall_ms;
  if (batches) *batches = s->n_batches;
  if (kernels) *kernels = s->n_kernels;
  return GX_OK;
}

int gx_serve_outputs(gx_serve* s, float* out, int64_t n_requests, int64_t elems) {
  if (!s || !out) return fail(GX_EINVAL, "null arg");
  if (n_requests < static_cast<int64_t>(s->reqs.size())) return fail(GX_EINVAL, "output array too small");
  if (s->gpu() && s->result_cursor > s->cfg.result_rows)
    return fail(GX_EINVAL, "outputs were overwritten (more completions than result_rows)");
  std::vector<int64_t> all(s->reqs.size());
  for (size_t i = 0; i < all.size(); ++i) all[i] = static_cast<int64_t>(i);
  int64_t held = 0;
  return gx_serve_outputs_for(s, static_cast<int64_t>(all.size()), all.data(), out, elems, &held);
}

int gx_serve_top1_for(gx_serve* s, int64_t n, const int64_t* req, int32_t* out, int64_t* held) {
  if (!s || (n > 0 && (!req || !out))) return fail(GX_EINVAL, "null arg");
  if (!s->gpu()) return fail(GX_EINVAL, "outputs exist only when batches execute on the GPU");
  if (!s->top1s) return fail(GX_EINVAL, "serving ran without top-1 (gx_serve_cfg.top1 = GX_TOP1_NONE)");
  for (int g : s->gpus) {
    GX_CUDA(cudaSetDevice(g));
    GX_CUDA(cudaDeviceSynchronize());
  }
  GX_CUDA(cudaSetDevice(s->gpus[0]));
  s->cur_device = s->gpus[0];
  std::vector<int32_t> ring(static_cast<size_t>(s->cfg.result_rows));
  GX_CUDA(cudaMemcpy(ring.data(), s->top1s, ring.size() * 4, cudaMemcpyDefault));
  int64_t got = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ri = req[i];
    const bool ok = ri >= 0 && ri < static_cast<int64_t>(s->reqs.size()) && s->reqs[ri].status == 0 &&
                    s->reqs[ri].result_seq >= 0 && s->reqs[ri].result_seq >= s->result_cursor - s->cfg.result_rows;
    out[i] = ok ? ring[s->reqs[ri].result_seq % s->cfg.result_rows] : -1;
    got += ok;
  }
  if (held) *held = got;
  return GX_OK;
}

int gx_serve_outputs_for(gx_serve* s, int64_t n, const int64_t* req, float* out, int64_t elems, int64_t* held) {
  if (!s || (n > 0 && (!req || !out))) return fail(GX_EINVAL, "null arg");
  if (!s->gpu()) return fail(GX_EINVAL, "outputs exist only when batches execute on the GPU");
  if (!s->results) return fail(GX_EINVAL, "serving kept no logits (gx_serve_cfg.top1 = GX_TOP1_ONLY)");
  if (elems != s->result_elems) return fail(GX_EINVAL, "output row size mismatch");
  for (int g : s->gpus) {
    GX_CUDA(cudaSetDevice(g));
    GX_CUDA(cudaDeviceSynchronize());
  }
  GX_CUDA(cudaSetDevice(s->gpus[0]));
  s->cur_device = s->gpus[0];
  int64_t got = 0;
  for (int64_t i = 0; i < n; ++i) {
    float* dst = out + i * elems;
    const int64_t ri = req[i];
    const bool ok = ri >= 0 && ri < static_cast<int64_t>(s->reqs.size()) && s->reqs[ri].status == 0 &&
                    s->reqs[ri].result_seq >= 0 && s->reqs[ri].result_seq >= s->result_cursor - s->cfg.result_rows;
    if (!ok) {  // not completed, or its ring row was reused by a later completion
      for (int64_t j = 0; j < elems; ++j) dst[j] = NAN;
      continue;
    }
    const uint8_t* src =
        static_cast<const uint8_t*>(s->results) + (s->reqs[ri].result_seq % s->cfg.result_rows) * elems * 4;
    GX_CUDA(cudaMemcpy(dst, src, elems * 4, cudaMemcpyDefault));
    ++got;
  }
  if (held) *held = got;
  return GX_OK;
}

int gx_serve_destroy(gx_serve* s) {
  if (!s) return GX_OK;
  if (s->gpu()) {
    for (DevRes& r : s->devs) {
      cudaSetDevice(r.device);
      cudaDeviceSynchronize();
      for (cudaEvent_t ev : r.events) cudaEventDestroy(ev);
      for (cudaStream_t q : r.copy_streams) cudaStreamDestroy(q);
      for (cudaStream_t q : r.pool) cudaStreamDestroy(q);
      if (r.slots) cudaFree(r.slots);
    }
    if (s->done_flags) cudaFreeHost(const_cast<uint32_t*>(s->done_flags));
    if (!s->gpus.empty()) cudaSetDevice(s->gpus[0]);
    for (void* p : {s->results, static_cast<void*>(s->top1s)}) {
      if (!p) continue;
      if (s->cfg.egress_to_host)
        cudaFreeHost(p);
      else
        cudaFree(p);
    }
  }
  delete s;
  return GX_OK;
}

}  // extern "C"
