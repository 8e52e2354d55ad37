// pd_stage.cu — pinned staging rings for pageable host buffers (see pd_stage.h). Host code only.
#include "pd_stage.h"

#include <algorithm>
#include <atomic>
#include <cstring>

namespace pdb {

bool host_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// ---------------- worker pool ----------------

struct StagePool::Batch {
    const std::function<void(unsigned)>* fn;
    unsigned left;  // guarded by mu
    std::mutex mu;
    std::condition_variable cv;
};

StagePool::StagePool(unsigned workers) {
    for (unsigned k = 0; k < workers; ++k) threads_.emplace_back([this] { loop(); });
}

StagePool::~StagePool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
}

void StagePool::loop() {
    for (;;) {
        std::pair<Batch*, unsigned> job;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
            if (queue_.empty()) return;
            job = queue_.front();
            queue_.pop_front();
        }
        Batch* b = job.first;
        (*b->fn)(job.second);
        // decrement under the batch mutex: the caller returns (and destroys the batch) only
        // after it has seen the count reach 0 under that mutex, i.e. after this block is done
        std::lock_guard<std::mutex> lk(b->mu);
        if (--b->left == 0) b->cv.notify_all();
    }
}

void StagePool::parallel(unsigned parts, const std::function<void(unsigned)>& fn) {
    if (parts <= 1 || threads_.empty()) {
        for (unsigned k = 0; k < parts; ++k) fn(k);
        return;
    }
    Batch b;
    b.fn = &fn;
    b.left = parts - 1;
    {
        std::lock_guard<std::mutex> lk(mu_);
        for (unsigned k = 1; k < parts; ++k) queue_.emplace_back(&b, k);
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(b.mu);
    b.cv.wait(lk, [&] { return b.left == 0; });
}

// ---------------- stager ----------------

namespace {
constexpr size_t kPieceMin = size_t{1} << 20;  // smallest share of a band per thread
}

Stager::Stager(int device, size_t slot_bytes, unsigned up_slots, unsigned down_slots, unsigned workers)
    : device_(device), slot_bytes_(slot_bytes), pool_(workers), up_(up_slots), down_(down_slots) {
    for (auto* ring : {&up_, &down_})
        for (Slot& s : *ring) {
            if (cudaHostAlloc(reinterpret_cast<void**>(&s.host), slot_bytes, cudaHostAllocDefault) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
        }
    drainer_ = std::thread([this] { drain_loop(); });
    ok_ = true;
}

Stager::~Stager() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    if (drainer_.joinable()) drainer_.join();
    for (auto* ring : {&up_, &down_})
        for (Slot& s : *ring) {
            if (s.done) {
                cudaEventSynchronize(s.done);
                cudaEventDestroy(s.done);
            }
            if (s.host) cudaFreeHost(s.host);
        }
}

cudaError_t Stager::upload_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                              size_t height, cudaStream_t stream) {
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    // rows wider than a slot go up as 1-row pieces
    const size_t piece_w = std::min(width, slot_bytes_);
    const size_t band_rows = width <= slot_bytes_ ? std::max<size_t>(1, slot_bytes_ / width) : 1;
    for (size_t r0 = 0; r0 < height; r0 += band_rows) {
        const size_t rows = std::min(band_rows, height - r0);
        for (size_t c0 = 0; c0 < width; c0 += piece_w) {
            const size_t w = std::min(piece_w, width - c0);
            Slot& slot = up_[up_next_];
            up_next_ = (up_next_ + 1) % up_.size();
            if (slot.used) {
                if (cudaError_t e = cudaEventSynchronize(slot.done)) return e;
            }
            // the band as rows x w bytes, packed in the slot; split into equal linear shares
            const size_t total = rows * w;
            const unsigned parts = static_cast<unsigned>(
                std::max<size_t>(1, std::min<size_t>(pool_.workers() + 1, total / kPieceMin)));
            pool_.parallel(parts, [&](unsigned k) {
                size_t a = total * k / parts;
                const size_t b = total * (k + 1) / parts;
                while (a < b) {
                    const size_t r = a / w, c = a % w;
                    const size_t n = std::min(b - a, w - c);
                    std::memcpy(slot.host + a, s + (r0 + r) * spitch + c0 + c, n);
                    a += n;
                }
            });
            cudaError_t e = cudaMemcpy2DAsync(d + r0 * dpitch + c0, dpitch, slot.host, w, w, rows,
                                              cudaMemcpyHostToDevice, stream);
            if (e == cudaSuccess) e = cudaEventRecord(slot.done, stream);
            if (e != cudaSuccess) return e;
            slot.used = true;
        }
    }
    return cudaSuccess;
}

cudaError_t Stager::take_down_slot(unsigned* out) {
    std::unique_lock<std::mutex> lk(mu_);
    Slot& s = down_[down_next_];
    cv_.wait(lk, [&] { return !s.busy || drain_error_ != cudaSuccess; });
    if (drain_error_ != cudaSuccess) return drain_error_;
    *out = down_next_;
    down_next_ = (down_next_ + 1) % down_.size();
    return cudaSuccess;
}

cudaError_t Stager::download(const Piece* pieces, size_t count, cudaEvent_t after,
                             cudaStream_t stream) {
    if (after) {
        if (cudaError_t e = cudaStreamWaitEvent(stream, after, 0)) return e;
    }
    unsigned k = 0;
    size_t fill = 0;   // bytes of the open slot in use
    bool open = false;
    std::vector<Seg> segs;
    auto close = [&]() -> cudaError_t {
        if (!open) return cudaSuccess;
        cudaError_t e = cudaEventRecord(down_[k].done, stream);
        if (e != cudaSuccess) return e;
        {
            std::lock_guard<std::mutex> lk(mu_);
            down_[k].busy = true;
            drains_.push_back({k, std::move(segs)});
        }
        cv_.notify_all();
        segs.clear();
        open = false;
        return cudaSuccess;
    };
    for (size_t i = 0; i < count; ++i) {
        const char* s = static_cast<const char*>(pieces[i].src);
        char* d = static_cast<char*>(pieces[i].dst);
        for (size_t off = 0; off < pieces[i].bytes;) {
            if (open && fill == slot_bytes_) {
                if (cudaError_t e = close()) return e;
            }
            if (!open) {
                if (cudaError_t e = take_down_slot(&k)) return e;
                open = true;
                fill = 0;
            }
            const size_t n = std::min(slot_bytes_ - fill, pieces[i].bytes - off);
            if (cudaError_t e = cudaMemcpyAsync(down_[k].host + fill, s + off, n, cudaMemcpyDeviceToHost,
                                                stream))
                return e;
            segs.push_back({d + off, fill, n});
            fill += n;
            off += n;
        }
    }
    return close();
}

void Stager::scatter(const std::vector<Seg>& segs, const char* slot) {
    size_t total = 0;
    for (const Seg& g : segs) total += g.bytes;
    const unsigned parts = static_cast<unsigned>(
        std::max<size_t>(1, std::min<size_t>(pool_.workers() + 1, total / kPieceMin)));
    pool_.parallel(parts, [&](unsigned k) {
        // linear share [a, b) of the slot's bytes, i.e. of the segments laid end to end
        size_t a = total * k / parts;
        const size_t b = total * (k + 1) / parts;
        size_t base = 0;
        for (const Seg& g : segs) {
            if (a >= b) break;
            if (a < base + g.bytes) {
                const size_t in = a - base, n = std::min(b, base + g.bytes) - a;
                std::memcpy(g.dst + in, slot + g.off + in, n);
                a += n;
            }
            base += g.bytes;
        }
    });
}

void Stager::drain_loop() {
    cudaSetDevice(device_);
    for (;;) {
        Drain job;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || !drains_.empty(); });
            if (drains_.empty()) return;
            job = std::move(drains_.front());
        }
        Slot& slot = down_[job.slot];
        const cudaError_t e = cudaEventSynchronize(slot.done);
        if (e == cudaSuccess) scatter(job.segs, slot.host);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (e != cudaSuccess && drain_error_ == cudaSuccess) drain_error_ = e;
            drains_.pop_front();
            slot.busy = false;
        }
        cv_.notify_all();
    }
}

cudaError_t Stager::finish() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return drains_.empty(); });
    const cudaError_t e = drain_error_;
    drain_error_ = cudaSuccess;
    return e;
}

}  // namespace pdb
