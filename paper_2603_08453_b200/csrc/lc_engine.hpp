// Internal engine definition shared by the ABI translation units.
#pragma once

#include "../../include/lychee_b200.h"
#include "lc_common.cuh"

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace lc {
size_t select3_pick_smem(const Arena& a);
cudaError_t launch_select3(const Arena& a, const float* q, uint32_t unit_topk, uint32_t mode, uint32_t cluster_topk,
                           unsigned long long budget, uint32_t sink, uint32_t flags, const uint32_t* buf_off,
                           const uint32_t* buf_ids, unsigned char* scratch, uint32_t qcap, uint32_t max_union,
                           uint32_t pmax, uint32_t n_slots, uint32_t* fine_ctr, uint32_t* pick_ord,
                           cudaStream_t stream, const float* q_in = nullptr);  // q_in: k_coarse reads q here and copies it to q
extern thread_local char g_select3_where[96];  // failing stage of the last launch_select3
cudaError_t launch_fused(const Arena& a, const float* q, const float* q_in, uint32_t unit_topk, uint32_t mode,
                         uint32_t cluster_topk, unsigned long long budget, uint32_t sink, uint32_t flags,
                         const uint32_t* buf_off, const uint32_t* buf_ids, unsigned char* scratch, uint32_t kc,
                         uint32_t uc, uint32_t pmax, uint32_t max_fanout, uint32_t n_slots, cudaStream_t stream,
                         const AttQueueDev* aq = nullptr);
uint32_t attend_grid(uint32_t d);
uint32_t attend_queue_cap(uint32_t d, uint32_t G, uint32_t n_slots);
size_t attend_partials_floats(uint32_t d, uint32_t G, uint32_t n_slots);
cudaError_t launch_attend(const Arena& a, const float* q, float* out, float* part, uint32_t n_slots,
                          cudaStream_t stream, const PeerGather* pg = nullptr, const AttQueueDev* aq = nullptr,
                          cudaEvent_t* att_ev = nullptr);
cudaError_t launch_gather_wait(unsigned int* flag, unsigned int* done, unsigned int expect, uint32_t* err,
                               cudaStream_t stream);
cudaError_t launch_append(const Arena& a, const void* keys, const void* values, cudaStream_t stream);
size_t compact_smem(const Arena& a);
cudaError_t launch_compact(const Arena& a, uint32_t min_grafted, cudaStream_t stream);
cudaError_t launch_chunk_rep(const Arena& a, uint32_t slot, uint32_t start, uint32_t take, uint32_t pooling,
                             float* rep_dev, cudaStream_t stream);
cudaError_t launch_graft(const Arena& a, const uint32_t* take_dev, uint32_t pooling, void* reports,
                         const float* reps_dev, cudaStream_t stream, const uint32_t* kind_dev = nullptr,
                         const uint32_t* level_dev = nullptr);
}  // namespace lc

namespace lcx {

inline thread_local std::string g_err;

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Status(code, msg); }

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(LC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return LC_OK;
    } catch (const Status& s) {
        g_err = s.what();
        return s.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return LC_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LC_ERUNTIME;
    }
}

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(LC_ENOMEM, std::string("cudaMalloc ") + std::to_string(n * sizeof(T)) + " B: " +
                            cudaGetErrorString(e));
    }
    owned.push_back(p);
    return static_cast<T*>(p);
}

}  // namespace lcx

using namespace lc;
using namespace lcx;

struct HostSlot {
    uint32_t n_tokens = 0, chunked_end = 0, n_chunks = 0, L = 0, P = 0;
    bool loaded = false;
    std::vector<uint32_t> kind, level;   // per chunk (host-only fields of ChunkSpan)
    std::vector<float> rep;              // prefill reps when the device keeps none
    std::vector<uint32_t> fanout;        // n_u per unit (fixed after build)
    std::vector<uint32_t> internal_of;   // reference cluster id -> internal id (lazy; fixed after upload)
    lc_index_config cfg{2.0, 64, 10, 0, 2, 0};  // IndexConfig defaults (index.hpp:13-22)
};

struct lc_index_s {
    lc_index_desc desc{};
    Arena a{};
    std::vector<void*> owned;
    std::vector<HostSlot> hs;
    float* q_stage = nullptr;    // device staging for lc_retrieve_host
    float* out_stage = nullptr;
    uint32_t* take_dev = nullptr;
    lc_graft_report* rep_scratch = nullptr;
    float* reps_dev = nullptr;     // caller-supplied representatives (lc_graft_rep)
    uint32_t kv_elem = 2;          // bytes per K/V element (2 bf16, 4 fp32)
    void* kv_ptr(int which, uint32_t slot) const {
        const size_t off = kv_off(a, slot);
        if (a.kv_f32) return (which ? a.Vf : a.Kf) + off;
        return (which ? a.V : a.K) + off;
    }
    uint32_t last_flags = 0;
    uint32_t last_valid = 0;
    uint32_t last_launches = 0;                // kernels of the last selection + attention
    std::vector<cudaEvent_t> att_ev;           // lc_attend_timing: event pairs around k_attend launches
    unsigned char* sel_stage = nullptr;        // lc_selection_stage: page-locked copy of one head's selection
    size_t sel_stage_bytes = 0;
    uint32_t stage_slot = 0, stage_g = 0;
    bool stage_valid = false;
    size_t att_ev_used = 0;
    std::map<uint32_t, uint32_t> cand_cache;  // unit_topk -> max candidates over slots
    unsigned char* sel_scratch = nullptr;      // per-head candidate keys + weights (k_fine -> k_pickq)
    size_t sel_scratch_bytes = 0;
    float* att_part = nullptr;                 // k_attend per-(warp, slot) segment partials + counters
    uint32_t* fine_ctr = nullptr;              // k_fine / k_pickq counters, 32 per slot group (zeroed)
    uint32_t* pick_ord = nullptr;              // k_pickq's size-class lists, 16 x G per slot
    std::vector<cudaStream_t> group_streams;   // one per slot group
    uint64_t version = 0;                      // bumped by every upload / append / graft
    cudaStream_t host_stream = nullptr;        // lc_retrieve_host's graph replay stream
    cudaEvent_t host_event = nullptr;
    cudaGraphExec_t host_exec = nullptr;
    uint64_t host_version = 0;
    uint32_t host_flags = 0;
    lc_budgets host_budgets{};
    const float* host_q = nullptr;  // the graph's q source (mapped host buffer) or nullptr (staged)
    float* host_out = nullptr;      // the graph's output buffer (mapped host buffer or out_stage)
    unsigned char* host_scratch = nullptr;  // sel_scratch the graph was captured with
    std::vector<cudaEvent_t> group_events;     // fork + one join per group
    // lc_decode_step_async advances the per-slot stream cursors on the device
    // only; the host copies in `hs` are re-read (sync_host) before any call that
    // needs them
    bool dev_ahead = false;
    uint32_t steps_since_compact = 0;  // decode steps since the last chunk-table compaction
    // streamed attention (selection publishes tasks, attention claims them)
    void* aq_mem = nullptr;
    AttQueueDev aq{};
    // fused all-gather epilogue (lc_set_gather)
    PeerGather pg{nullptr, nullptr, nullptr, 0u};
    void* pg_mem = nullptr;            // device: peer out pointers, flag pointers, rows, wait count
    unsigned int* pg_done = nullptr;
    unsigned int* pg_myflag = nullptr;
    uint32_t pg_expect = 0;

    ~lc_index_s() {
        for (void* p : owned) cudaFree(p);
        if (sel_scratch) cudaFree(sel_scratch);
        for (auto s : group_streams) cudaStreamDestroy(s);
        if (host_exec) cudaGraphExecDestroy(host_exec);
        if (host_stream) cudaStreamDestroy(host_stream);
        if (host_event) cudaEventDestroy(host_event);
        for (auto e : group_events) cudaEventDestroy(e);
        for (auto e : att_ev) cudaEventDestroy(e);
        if (sel_stage) cudaFreeHost(sel_stage);
        if (pg_mem) cudaFree(pg_mem);
        if (aq_mem) cudaFree(aq_mem);
    }
    void set_device() { ck(cudaSetDevice(desc.device), "cudaSetDevice"); }
};


// host mirror <- device after lc_decode_step_async steps: per-slot cursors
// (n_tokens, chunked_end, n_chunks) and the grafted chunks' kind / level
void sync_host(lc_index_t h);

// chunk_representative of every chunk of a slot, recomputed on the device from
// the bf16 store (lc_build.cu); chunk_bounds = chunk_start[0..M]
void recompute_slot_reps(lc_index_t h, uint32_t slot, const uint32_t* chunk_bounds, uint32_t M, float* out);
