// Thin PyTorch C++ extension over the step-loop entry points of libneurocomm_b200
// (BASELINE.json north_star: "Python host code calls CUDA through a thin PyTorch C++
// extension"; SURVEY 8(b) "Proposed C ABI (torch ops, TORCH_LIBRARY(neurocomm_b200, m))").
//
// Every per-step launch of the simulators (sim.py, distributed.py) goes through these
// ops: torch.ops.neurocomm_b200.<name>(...).  The descriptors -- nc_shard_t,
// nc_lif_params_t, nc_xchg_t -- travel as uint8 CPU tensors that view the host structs
// (torch.frombuffer over the ctypes objects, no copy), device buffers as tensors, and
// the CUDA stream as an int (the launch stream the caller chose: the current stream, a
// capture stream, or one stream per virtual rank).  Each op checks sizes, calls the
// C-ABI function and turns an error code into an exception carrying nc_last_error()
// (ValueError for NC_E_ARG, as _native.check does; RuntimeError otherwise).
// The planner / builder / I/O entry points stay on the plain C ABI (_native.py).

#include <torch/library.h>

#include <cstdint>
#include <string>

#include "../../include/neurocomm_b200.h"

namespace {

template <typename T>
const T* desc(const at::Tensor& t, const char* what) {
  TORCH_CHECK(t.device().is_cpu() && t.scalar_type() == at::kByte && t.is_contiguous(), what,
              ": expected a contiguous uint8 CPU tensor viewing the C struct");
  TORCH_CHECK((size_t)t.numel() == sizeof(T), what, ": ", t.numel(), " bytes, the struct has ", sizeof(T));
  return reinterpret_cast<const T*>(t.data_ptr());
}

// NC_E_ARG -> ValueError (as _native.check), anything else -> RuntimeError
void check(int rc, const char* what) {
  if (rc == NC_OK) return;
  TORCH_CHECK_VALUE(rc != NC_E_ARG, what, ": ", nc_last_error());
  TORCH_CHECK(false, what, " failed (", rc, "): ", nc_last_error());
}

void* stream_of(int64_t s) { return reinterpret_cast<void*>(static_cast<intptr_t>(s)); }

void* dptr(const c10::optional<at::Tensor>& t) { return t.has_value() ? t->data_ptr() : nullptr; }

void sim_init(const at::Tensor& shard, const at::Tensor& lif, int64_t stream) {
  check(nc_sim_init(desc<nc_shard_t>(shard, "shard"), desc<nc_lif_params_t>(lif, "lif"), stream_of(stream)),
        "nc_sim_init");
}

void sim_step_fused(const at::Tensor& shard, const at::Tensor& lif, int64_t stream) {
  check(nc_sim_step_fused(desc<nc_shard_t>(shard, "shard"), desc<nc_lif_params_t>(lif, "lif"), stream_of(stream)),
        "nc_sim_step_fused");
}

void sim_step_binned(const at::Tensor& shard, const at::Tensor& lif, int64_t stream) {
  check(nc_sim_step_binned(desc<nc_shard_t>(shard, "shard"), desc<nc_lif_params_t>(lif, "lif"), stream_of(stream)),
        "nc_sim_step_binned");
}

void sim_deliver_push(const at::Tensor& shard, int64_t g_inh, int64_t stream) {
  check(nc_sim_deliver_push(desc<nc_shard_t>(shard, "shard"), (int32_t)g_inh, stream_of(stream)),
        "nc_sim_deliver_push");
}

void sim_deliver_pull(const at::Tensor& shard, int64_t g_inh, int64_t stream) {
  check(nc_sim_deliver_pull(desc<nc_shard_t>(shard, "shard"), (int32_t)g_inh, stream_of(stream)),
        "nc_sim_deliver_pull");
}

void sim_lif_update(const at::Tensor& shard, const at::Tensor& lif, int64_t stream) {
  check(nc_sim_lif_update(desc<nc_shard_t>(shard, "shard"), desc<nc_lif_params_t>(lif, "lif"), stream_of(stream)),
        "nc_sim_lif_update");
}

void sim_end_step(const at::Tensor& shard, int64_t stream) {
  check(nc_sim_end_step(desc<nc_shard_t>(shard, "shard"), stream_of(stream)), "nc_sim_end_step");
}

// shards: n_shards nc_shard_t structs back to back (the ctypes array)
void exchange_local(const at::Tensor& shards, int64_t n_shards, const at::Tensor& dest_mask,
                    const at::Tensor& fwd_table, const at::Tensor& fwd_ids, const at::Tensor& fwd_count,
                    int64_t fwd_cap, const at::Tensor& hop_ids, const at::Tensor& deliv_ids, int64_t per_step,
                    int64_t stream) {
  TORCH_CHECK(shards.device().is_cpu() && shards.scalar_type() == at::kByte &&
                  (size_t)shards.numel() == sizeof(nc_shard_t) * (size_t)n_shards,
              "shards: expected n_shards nc_shard_t structs as uint8");
  TORCH_CHECK(fwd_table.device().is_cpu() && fwd_table.numel() >= n_shards * n_shards,
              "fwd_table: expected a CPU tensor of n*n uint16");
  check(nc_exchange_local(reinterpret_cast<const nc_shard_t*>(shards.data_ptr()), (int32_t)n_shards,
                          static_cast<const uint16_t*>(dest_mask.data_ptr()),
                          static_cast<const uint16_t*>(fwd_table.data_ptr()),
                          static_cast<uint32_t*>(fwd_ids.data_ptr()), static_cast<int32_t*>(fwd_count.data_ptr()),
                          fwd_cap, static_cast<long long*>(hop_ids.data_ptr()),
                          static_cast<long long*>(deliv_ids.data_ptr()), (int32_t)per_step, stream_of(stream)),
        "nc_exchange_local");
}

void xchg_p2p(const at::Tensor& x, int64_t stream) {
  check(nc_xchg_p2p(desc<nc_xchg_t>(x, "xchg"), stream_of(stream)), "nc_xchg_p2p");
}

void xchg_seal(const at::Tensor& x, int64_t phase, int64_t stream) {
  check(nc_xchg_seal(desc<nc_xchg_t>(x, "xchg"), (int32_t)phase, stream_of(stream)), "nc_xchg_seal");
}

void xchg_scatter(const at::Tensor& x, int64_t phase, int64_t stream) {
  check(nc_xchg_scatter(desc<nc_xchg_t>(x, "xchg"), (int32_t)phase, stream_of(stream)), "nc_xchg_scatter");
}

void nccl_exchange(int64_t comm, const at::Tensor& x, int64_t phase, int64_t stream) {
  check(nc_nccl_exchange(reinterpret_cast<void*>(static_cast<intptr_t>(comm)), desc<nc_xchg_t>(x, "xchg"),
                         (int32_t)phase, stream_of(stream)),
        "nc_nccl_exchange");
}

void stamp(const at::Tensor& dst, const at::Tensor& step, int64_t max_steps, int64_t stream) {
  check(nc_stamp(static_cast<unsigned long long*>(dst.data_ptr()), static_cast<const int32_t*>(step.data_ptr()),
                 (int32_t)max_steps, stream_of(stream)),
        "nc_stamp");
}

void run_persistent(const at::Tensor& shard, const at::Tensor& lif, const c10::optional<at::Tensor>& x,
                    int64_t n_steps, int64_t blocks_per_peer, const at::Tensor& gbar,
                    const c10::optional<at::Tensor>& stamp_ready, const c10::optional<at::Tensor>& stamp_done,
                    int64_t stamp_cap, int64_t stream) {
  check(nc_run_persistent(desc<nc_shard_t>(shard, "shard"), desc<nc_lif_params_t>(lif, "lif"),
                          x.has_value() ? desc<nc_xchg_t>(*x, "xchg") : nullptr, (int32_t)n_steps,
                          (int32_t)blocks_per_peer, static_cast<unsigned int*>(gbar.data_ptr()),
                          static_cast<unsigned long long*>(dptr(stamp_ready)),
                          static_cast<unsigned long long*>(dptr(stamp_done)), (int32_t)stamp_cap, stream_of(stream)),
        "nc_run_persistent");
}

int64_t abi_version() { return nc_abi_version(); }

}  // namespace

TORCH_LIBRARY(neurocomm_b200, m) {
  m.def("abi_version() -> int", abi_version);
  m.def("sim_init(Tensor shard, Tensor lif, int stream) -> ()", sim_init);
  m.def("sim_step_fused(Tensor shard, Tensor lif, int stream) -> ()", sim_step_fused);
  m.def("sim_step_binned(Tensor shard, Tensor lif, int stream) -> ()", sim_step_binned);
  m.def("sim_deliver_push(Tensor shard, int g_inh, int stream) -> ()", sim_deliver_push);
  m.def("sim_deliver_pull(Tensor shard, int g_inh, int stream) -> ()", sim_deliver_pull);
  m.def("sim_lif_update(Tensor shard, Tensor lif, int stream) -> ()", sim_lif_update);
  m.def("sim_end_step(Tensor shard, int stream) -> ()", sim_end_step);
  m.def("exchange_local(Tensor shards, int n_shards, Tensor dest_mask, Tensor fwd_table, Tensor fwd_ids, "
        "Tensor fwd_count, int fwd_cap, Tensor hop_ids, Tensor deliv_ids, int per_step, int stream) -> ()",
        exchange_local);
  m.def("xchg_p2p(Tensor x, int stream) -> ()", xchg_p2p);
  m.def("xchg_seal(Tensor x, int phase, int stream) -> ()", xchg_seal);
  m.def("xchg_scatter(Tensor x, int phase, int stream) -> ()", xchg_scatter);
  m.def("nccl_exchange(int comm, Tensor x, int phase, int stream) -> ()", nccl_exchange);
  m.def("stamp(Tensor dst, Tensor step, int max_steps, int stream) -> ()", stamp);
  m.def("run_persistent(Tensor shard, Tensor lif, Tensor? x, int n_steps, int blocks_per_peer, Tensor gbar, "
        "Tensor? stamp_ready, Tensor? stamp_done, int stamp_cap, int stream) -> ()",
        run_persistent);
}
