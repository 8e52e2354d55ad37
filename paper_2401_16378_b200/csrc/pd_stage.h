// pd_stage.h — host-buffer transfers for pageable (ordinary malloc / numpy) caller memory.
//
// A cudaMemcpy*Async on pageable memory is staged by the driver through its own pinned buffer
// on the calling thread, one copy at a time (measured on the box at N=14: 11.3 GB/s H2D,
// 16.2 GB/s D2H, and decompose() of a numpy array 1,071 ms against 354 ms with pinned buffers).
// Registering the caller's 4 GiB for the call costs 414 ms + 105 ms to unregister, more than
// the whole decomposition. So pageable buffers go through rings of pinned slots instead:
//   * uploads: the calling thread fills a slot with the host rows of the next band (split over
//     the worker threads), enqueues the slot's H2D and moves on to the next slot while the
//     copy engine drains it; a slot is refilled once its previous H2D has completed;
//   * downloads: the calling thread enqueues each piece's D2H into a free slot after the
//     event that publishes the piece; a drain thread waits for the copy in order and scatters
//     the slot into the caller's buffer over the worker threads (which also takes the first-touch
//     page faults of a fresh output array off the calling thread).
// Pinned callers (cudaHostAlloc / cudaHostRegister / torch pin_memory) keep the direct copies.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pdb {

// true when p is ordinary pageable host memory (not device, managed or page-locked)
bool host_pageable(const void* p);

class StagePool {  // worker threads running memcpy pieces
public:
    explicit StagePool(unsigned workers);
    ~StagePool();
    // run fn(k) for k in [0, parts) over the workers and the calling thread; returns when done
    void parallel(unsigned parts, const std::function<void(unsigned)>& fn);
    unsigned workers() const { return static_cast<unsigned>(threads_.size()); }

private:
    struct Batch;
    void loop();
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::pair<Batch*, unsigned>> queue_;
    std::vector<std::thread> threads_;
    bool stop_ = false;
};

class Stager {
public:
    Stager(int device, size_t slot_bytes, unsigned up_slots, unsigned down_slots, unsigned workers);
    ~Stager();
    bool ok() const { return ok_; }
    size_t slot_bytes() const { return slot_bytes_; }

    // H2D of a height x width-byte rectangle (row pitches spitch on the host, dpitch on the
    // device) from pageable host memory, enqueued on `stream` in row bands
    cudaError_t upload_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                          size_t height, cudaStream_t stream);
    cudaError_t upload(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
        return upload_2d(dst, bytes, src, bytes, bytes, 1, stream);
    }
    // D2H of `bytes` from device src to pageable host dst once `after` (may be null) has fired;
    // the D2H is enqueued on `stream`, the host scatter happens on the drain thread
    struct Piece {
        void* dst;
        const void* src;
        size_t bytes;
    };
    cudaError_t download(void* dst, const void* src, size_t bytes, cudaEvent_t after,
                         cudaStream_t stream) {
        const Piece p{dst, src, bytes};
        return download(&p, 1, after, stream);
    }
    // several pieces packed into the slots back to back (a slot's pieces drain as one job)
    cudaError_t download(const Piece* pieces, size_t count, cudaEvent_t after, cudaStream_t stream);
    // wait until every download has landed in host memory; the first error seen, if any
    cudaError_t finish();

private:
    struct Slot {
        char* host = nullptr;
        cudaEvent_t done = nullptr;  // the slot's last transfer
        bool used = false;
        bool busy = false;           // download slot: waiting for its drain
    };
    struct Seg {
        char* dst;
        size_t off;  // in the slot
        size_t bytes;
    };
    struct Drain {
        unsigned slot;
        std::vector<Seg> segs;
    };
    cudaError_t take_down_slot(unsigned* slot);
    void drain_loop();
    void scatter(const std::vector<Seg>& segs, const char* slot);

    int device_;
    size_t slot_bytes_;
    StagePool pool_;
    std::vector<Slot> up_, down_;
    unsigned up_next_ = 0, down_next_ = 0;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Drain> drains_;
    cudaError_t drain_error_ = cudaSuccess;
    bool stop_ = false;
    bool ok_ = false;
    std::thread drainer_;
};

}  // namespace pdb
