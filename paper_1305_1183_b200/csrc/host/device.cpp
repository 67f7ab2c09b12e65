// host/device.cpp -- DeviceConfig text format (keys of the reference's
// data/device.cfg, proj/src/device.cpp:40-70) and the B200 device query.
#include "mapfuse/device.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <sstream>
#include <stdexcept>

namespace mapfuse::vm {

namespace {
struct Key {
  const char* name;
  int DeviceConfig::*field;
};
const Key kKeys[] = {
    {"warp_size", &DeviceConfig::warp_size},
    {"max_threads_per_block", &DeviceConfig::max_threads_per_block},
    {"shared_bytes_per_block", &DeviceConfig::shared_bytes_per_block},
    {"sm_count", &DeviceConfig::sm_count},
    {"max_blocks_per_sm", &DeviceConfig::max_blocks_per_sm},
    {"cycles_per_global_word", &DeviceConfig::cycles_per_global_word},
    {"cycles_per_shared_word", &DeviceConfig::cycles_per_shared_word},
    {"cycles_per_arith_op", &DeviceConfig::cycles_per_arith_op},
    {"cycles_per_barrier", &DeviceConfig::cycles_per_barrier},
    {"cycles_per_atomic", &DeviceConfig::cycles_per_atomic},
    {"latency_hiding_divisor", &DeviceConfig::latency_hiding_divisor},
};
}  // namespace

int DeviceConfig::occupancy(int shared_bytes, int threads) const {
  int occ = max_blocks_per_sm;
  if (shared_bytes > 0) occ = std::min(occ, shared_bytes_per_block / shared_bytes);
  if (threads > 0) occ = std::min(occ, max_threads_per_block / threads);
  return std::max(occ, 0);
}

double DeviceConfig::latency_factor(int occ) const {
  return occ <= 0 ? 0.0 : std::min(1.0, double(occ) / latency_hiding_divisor);
}

void DeviceConfig::validate() const {
  for (const auto& k : kKeys)
    if (this->*k.field <= 0)
      throw std::runtime_error(std::string("device config: ") + k.name + " must be positive");
  if (max_threads_per_block % warp_size)
    throw std::runtime_error("device config: warp_size must divide max_threads_per_block");
}

DeviceConfig parse_device_config(const std::string& text) {
  DeviceConfig c;
  std::istringstream in(text);
  int no = 0;
  for (std::string line; std::getline(in, line);) {
    ++no;
    if (auto p = line.find("//"); p != std::string::npos) line.erase(p);
    std::istringstream ls(line);
    std::string key;
    if (!(ls >> key)) continue;
    int v = 0;
    if (!(ls >> v))
      throw std::runtime_error("device config line " + std::to_string(no) + ": missing value");
    auto it = std::find_if(std::begin(kKeys), std::end(kKeys),
                           [&](const Key& k) { return key == k.name; });
    if (it == std::end(kKeys))
      throw std::runtime_error("device config line " + std::to_string(no) + ": unknown key '" +
                               key + "'");
    c.*(it->field) = v;
  }
  c.validate();
  return c;
}

std::string print_device_config(const DeviceConfig& c) {
  std::string o;
  for (const auto& k : kKeys) o += std::string(k.name) + " " + std::to_string(c.*k.field) + "\n";
  return o;
}

uint64_t device_config_hash(const DeviceConfig& c) {
  uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a over the canonical text
  for (unsigned char ch : print_device_config(c)) h = (h ^ ch) * 0x100000001b3ull;
  return h;
}

B200Device b200_device() {
  B200Device d;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return d;
  }
  cudaDeviceProp p{};
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return d;
  d.name = p.name;
  d.sm_count = p.multiProcessorCount;
  d.shared_bytes_per_block = static_cast<int64_t>(p.sharedMemPerBlockOptin);
  d.l2_bytes = p.l2CacheSize;
  d.live = true;
  return d;
}

}  // namespace mapfuse::vm
