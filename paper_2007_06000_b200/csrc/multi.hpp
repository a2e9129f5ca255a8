// Several GPUs of one node in one process: the batch-sharded successor of
// simulate_graph (reference fused_exec.cpp:313-349) for 1..8 B200s.
// Inference is embarrassingly parallel over images: every device
// holds the weights and its own Engine, device k owns a contiguous image range
// of the batch, and nothing is exchanged on the data path.  One persistent
// host worker thread per device (CUDA context bound once, its own stream)
// enqueues that device's work, so the devices run concurrently.
#pragma once

#include <condition_variable>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace xlf {

// Images [first, first + count) of device slot k when `batch` images are split
// over n devices: contiguous, sizes differ by at most one (the first
// batch % n slots take one more).  n * B images with n slots give slot k
// exactly [k*B, (k+1)*B) -- the weak-scaling shard of bench.py.
void shard_range(int batch, int n, int k, int* first, int* count);

class DeviceWorker {
public:
    explicit DeviceWorker(int device);
    ~DeviceWorker();
    DeviceWorker(const DeviceWorker&) = delete;
    DeviceWorker& operator=(const DeviceWorker&) = delete;
    // Runs `job` on the worker thread (device current, `stream()` valid).
    std::future<void> submit(std::function<void()> job);
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }

private:
    void loop();
    int device_;
    cudaStream_t stream_ = nullptr;
    std::mutex mu_;
    std::condition_variable cv_;
    std::queue<std::packaged_task<void()>> jobs_;
    bool stop_ = false;
    std::thread thread_;
};

class MultiEngine {
public:
    MultiEngine(const Graph& g, const std::vector<int>& devices, Partition part, Precision prec, const float* weights, size_t nweights,
                int max_batch_per_device, const Knobs& knobs = Knobs{});
    ~MultiEngine();
    int devices() const { return int(engines_.size()); }
    Engine& engine(int k) { return *engines_[size_t(k)]; }
    // Every device tunes its own engine at `batch_per_device` (concurrently).
    void autotune(int batch_per_device, int reps, int topk);
    // End to end from host memory: device k copies in its image range of h_in,
    // runs it and copies its slice of `out_name` back into h_out (the gather).
    // Synchronous; returns the per-device wall times (ms).
    std::vector<double> run_host(const float* h_in, int batch, const std::string& out_name, float* h_out);
    // Device-resident throughput: device k generates images [k*B, (k+1)*B) of
    // SeededStream(seed) (B = batch_per_device), runs `warmup` untimed and
    // `steps` timed forwards (CUDA events on its stream); returns the per-device
    // ms per forward (the job's step time is their max).
    std::vector<double> time_seeded(uint64_t seed, int batch_per_device, int steps, int warmup);

private:
    void all(const std::function<void(int)>& job);  // job(k) on every worker, waits, rethrows the first error
    std::vector<std::unique_ptr<DeviceWorker>> workers_;
    std::vector<std::unique_ptr<Engine>> engines_;
    int max_batch_;
};

}  // namespace xlf
