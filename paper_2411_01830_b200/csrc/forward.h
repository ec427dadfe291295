// K2 — the staged host->gFunc forward (internal to libfaastube; used by the pacer).
//
// A staged route lands its bytes on a staging GPU's chunk ring by copy engine and
// forwards them into the target over NVLink. Per chunk the copy-engine stream
// writes the slot's `landed` word (cuStreamWriteValue32, ordered after the DMA);
// ONE forward kernel per batch of chunks polls those words on the device, pulls
// each chunk as it lands, and counts the slot free in `freed` (each CTA adds 1
// after its share was read); the CE stream waits on `freed` (cuStreamWaitValue32
// GEQ) before it reuses a slot. No host round trip, no per-chunk launch or
// event. Every wait points at work enqueued earlier (a batch holds at most one
// chunk per slot), so a context-wide synchronisation (lazy module loading) can
// always drain — no stream ever waits on host progress.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ft {

constexpr int kFwdMaxChunks = 32;  // chunks per forward launch (<= ring slots)
constexpr int kFwdCtas = 32;       // CTAs of every forward launch (the `freed` unit)

struct FwdChunk {
  uint64_t dst_off;   // offset in the destination
  uint32_t slot;      // ring slot
  uint32_t gen;       // the slot's use number this chunk is (landed value to wait for)
  uint64_t len;       // bytes
};
struct FwdBatch {
  FwdChunk c[kFwdMaxChunks];
  int n;
};

// ring words (device memory of the staging GPU, 2 x slots uint32) + error word (mapped host)
int fwd_ring_words(int device, int slots, uint32_t** landed, uint32_t** freed, uint32_t** err_host);
void fwd_ring_words_free(int device, uint32_t* landed, uint32_t* err_host);
// load the forward kernel's module now (a lazy load later could synchronise the
// context while a CE stream waits on a kernel that is not launched yet)
int fwd_preload(int device);
// stream memory ops (driver API through the runtime's entry points)
int mem_write32(cudaStream_t st, uint32_t* addr, uint32_t value);
int mem_wait_geq32(cudaStream_t st, uint32_t* addr, uint32_t value);
// one forward launch on `st` (device `device`): chunks of `ring` (slot_bytes each) -> dst
int fwd_launch(int device, cudaStream_t st, uint8_t* dst, const uint8_t* ring, uint64_t slot_bytes,
               const uint32_t* landed, uint32_t* freed, uint32_t* err, const FwdBatch& b);

}  // namespace ft
