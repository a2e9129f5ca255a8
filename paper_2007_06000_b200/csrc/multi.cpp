#include "multi.hpp"

#include <algorithm>
#include <chrono>

#include "common.hpp"

namespace xlf {

void shard_range(int batch, int n, int k, int* first, int* count) {
    if (batch < 0 || n < 1 || k < 0 || k >= n) fail(ErrorKind::validation, "shard: bad batch / device count / slot");
    const int base = batch / n, extra = batch % n;
    *first = k * base + std::min(k, extra);
    *count = base + (k < extra ? 1 : 0);
}

DeviceWorker::DeviceWorker(int device) : device_(device) {
    std::promise<void> ready;
    std::future<void> f = ready.get_future();
    thread_ = std::thread([this, &ready] {
        try {
            cuda_check(cudaSetDevice(device_), "cudaSetDevice(worker)");
            cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate(worker)");
            ready.set_value();
        } catch (...) {
            ready.set_exception(std::current_exception());
            return;
        }
        loop();
    });
    try {
        f.get();
    } catch (...) {
        thread_.join();
        throw;
    }
}

DeviceWorker::~DeviceWorker() {
    {
        std::lock_guard<std::mutex> l(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    if (thread_.joinable()) thread_.join();
}

void DeviceWorker::loop() {
    for (;;) {
        std::packaged_task<void()> job;
        {
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait(l, [&] { return stop_ || !jobs_.empty(); });
            if (jobs_.empty()) break;  // stop_ and drained
            job = std::move(jobs_.front());
            jobs_.pop();
        }
        job();
    }
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
}

std::future<void> DeviceWorker::submit(std::function<void()> job) {
    std::packaged_task<void()> t(std::move(job));
    std::future<void> f = t.get_future();
    {
        std::lock_guard<std::mutex> l(mu_);
        jobs_.push(std::move(t));
    }
    cv_.notify_one();
    return f;
}

MultiEngine::MultiEngine(const Graph& g, const std::vector<int>& devices, Partition part, Precision prec, const float* weights,
                         size_t nweights, int max_batch_per_device, const Knobs& knobs)
    : max_batch_(max_batch_per_device) {
    if (devices.empty() || devices.size() > 64) fail(ErrorKind::validation, "multi-GPU engine: 1..64 devices");
    for (int d : devices) workers_.push_back(std::make_unique<DeviceWorker>(d));
    engines_.resize(devices.size());
    // weights replicated: each worker builds its engine on its own device, concurrently
    all([&](int k) {
        engines_[size_t(k)] = std::make_unique<Engine>(g, workers_[size_t(k)]->device(), part, prec, weights, nweights, max_batch_per_device, knobs);
    });
}

MultiEngine::~MultiEngine() {
    // engines die on their own device's thread (their CUDA resources)
    try {
        all([&](int k) { engines_[size_t(k)].reset(); });
    } catch (...) {
    }
}

void MultiEngine::all(const std::function<void(int)>& job) {
    std::vector<std::future<void>> fs;
    for (size_t k = 0; k < workers_.size(); ++k) fs.push_back(workers_[k]->submit([&job, k] { job(int(k)); }));
    std::exception_ptr first;
    for (auto& f : fs) {
        try {
            f.get();
        } catch (...) {
            if (!first) first = std::current_exception();
        }
    }
    if (first) std::rethrow_exception(first);
}

void MultiEngine::autotune(int batch_per_device, int reps, int topk) {
    all([&](int k) {
        Engine& e = *engines_[size_t(k)];
        const int b = batch_per_device > 0 ? std::min(batch_per_device, max_batch_) : max_batch_;
        e.set_input_seeded(e.graph().inputs[0].name, 42, uint64_t(k) * b, b, workers_[size_t(k)]->stream());
        e.forward(b, workers_[size_t(k)]->stream(), false);
        cuda_check(cudaStreamSynchronize(workers_[size_t(k)]->stream()), "sync");
        e.autotune(b, reps, topk);
    });
}

std::vector<double> MultiEngine::run_host(const float* h_in, int batch, const std::string& out_name, float* h_out) {
    const int n = devices();
    if (batch < 1 || batch > n * max_batch_) fail(ErrorKind::validation, "batch out of range for the devices' max_batch");
    std::vector<double> ms(size_t(n), 0.0);
    const size_t img_in = engines_[0]->user_input_elements();
    all([&](int k) {
        int first = 0, count = 0;
        shard_range(batch, n, k, &first, &count);
        if (!count) return;
        Engine& e = *engines_[size_t(k)];
        const size_t img_out = e.tensor_elements(out_name);
        const auto t0 = std::chrono::steady_clock::now();
        e.run_host(h_in + size_t(first) * img_in, count, out_name, h_out + size_t(first) * img_out, workers_[size_t(k)]->stream());
        ms[size_t(k)] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    return ms;
}

std::vector<double> MultiEngine::time_seeded(uint64_t seed, int batch_per_device, int steps, int warmup) {
    if (batch_per_device < 1 || batch_per_device > max_batch_) fail(ErrorKind::validation, "batch out of range");
    std::vector<double> ms(size_t(devices()), 0.0);
    all([&](int k) {
        Engine& e = *engines_[size_t(k)];
        const cudaStream_t st = workers_[size_t(k)]->stream();
        e.set_input_seeded(e.graph().inputs[0].name, seed, uint64_t(k) * batch_per_device, batch_per_device, st);
        for (int i = 0; i < warmup; ++i) e.forward(batch_per_device, st, true);
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "cudaEventCreate"), cuda_check(cudaEventCreate(&b), "cudaEventCreate");
        cuda_check(cudaEventRecord(a, st), "cudaEventRecord");
        for (int i = 0; i < steps; ++i) e.forward(batch_per_device, st, true);
        cuda_check(cudaEventRecord(b, st), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
        float t = 0;
        cuda_check(cudaEventElapsedTime(&t, a, b), "cudaEventElapsedTime");
        cudaEventDestroy(a), cudaEventDestroy(b);
        ms[size_t(k)] = double(t) / std::max(1, steps);
    });
    return ms;
}

}  // namespace xlf
