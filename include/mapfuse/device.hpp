// mapfuse/device.hpp -- device parameters.
//
// DeviceConfig keeps the reference's keys and text format
// (/root/reference/proj/include/mapfuse/device.hpp, data/device.cfg) so
// existing configs still parse; B200Device adds what the B200 cost model and
// kernel configuration actually use (SM count, HBM bandwidth, shared memory
// per block, L2, launch overhead), filled from the CUDA device properties and
// the measured peaks when a GPU is present.
#pragma once

#include <cstdint>
#include <string>

namespace mapfuse::vm {

struct DeviceConfig {
  int warp_size = 32;
  int max_threads_per_block = 1024;
  int shared_bytes_per_block = 48 * 1024;
  int sm_count = 16;
  int max_blocks_per_sm = 8;
  int cycles_per_global_word = 8;
  int cycles_per_shared_word = 1;
  int cycles_per_arith_op = 1;
  int cycles_per_barrier = 32;
  int cycles_per_atomic = 4;
  int latency_hiding_divisor = 4;

  bool operator==(const DeviceConfig&) const = default;

  int occupancy(int shared_bytes, int threads) const;
  double latency_factor(int occ) const;
  void validate() const;
};

DeviceConfig parse_device_config(const std::string& text);
std::string print_device_config(const DeviceConfig& c);
uint64_t device_config_hash(const DeviceConfig& c);

// B200 additions ----------------------------------------------------------
struct B200Device {
  std::string name = "NVIDIA B200";
  int sm_count = 148;
  int64_t shared_bytes_per_block = 232448;  // opt-in maximum
  int64_t l2_bytes = 132644864;
  double hbm_gbs = 6545.6;      // measured copy bandwidth (MEASURED_PEAKS.json)
  double fp32_tflops = 75.0;    // non-tensor FFMA peak (2 * 148 * 128 * 1.965 GHz)
  double launch_us = 2.5;       // per-kernel launch + ramp overhead
  bool live = false;            // filled from a real device
};

// Queries device 0 when the CUDA runtime sees one, else the B200 defaults.
B200Device b200_device();

}  // namespace mapfuse::vm
