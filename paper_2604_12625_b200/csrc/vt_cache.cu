// vt_cache.cu -- the residency side of the page cache:
// page table + strict-LRU slot manager with time buckets, host C++ (no device
// code; compiled with the library so the C-ABI stays one .so).
//
// P:229  "on each frame we fetch the parameters of the required tiles on
//        demand ... write the results to the physical texture ... For tiles
//        already resident ... we can reuse the cached content for a period"
// P:521  page table = "indirection texture that maps each virtual tile to its
//        location in the physical texture"
// P:524  "identifies missing tiles ... the page table is updated ... Tiles
//        that have not been referenced within a interval may be evicted"
// Readings (R24): an entry is (slot, time bucket); with nb buckets
// per unit of t, bucket(t) = floor(t * nb) (t = 1 in the last bucket; exact in
// fp64 for fp32 t); a tile decoded for bucket b is decoded at the bucket
// centre (b + 1/2) / nb; eviction is strict LRU over slots; never-used slots
// are handed out first, in increasing order.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/ndgi.h"

struct ndgi_vt {
    uint32_t num_tiles = 0, capacity = 0;
    int32_t nbuckets = 0;
    std::vector<int32_t> pt;          // [num_tiles][2] = (slot, bucket); slot -1 = absent
    std::vector<uint32_t> slot_tile;  // tile held by a slot, UINT32_MAX = free
    std::vector<uint32_t> prev, next; // LRU list over used slots (head = least recent)
    uint32_t head = UINT32_MAX, tail = UINT32_MAX;
    uint32_t fresh = 0;               // slots [fresh, capacity) never used
    std::vector<uint64_t> seen;       // per tile: id of the last request that touched it
    uint64_t req_id = 0;
    uint64_t stats[4] = {0, 0, 0, 0}; // tile requests, hits, decode jobs, evictions
    uint64_t version = 1;             // bumped by every page-table change
    const void* uploaded_ptr = nullptr;
    uint64_t uploaded_version = 0;    // what uploaded_ptr holds
    std::string err;
};

namespace ndgi {
ndgi_status set_error(ndgi_status s, const char* msg);   // host.cu
}

namespace {

constexpr uint32_t kNone = UINT32_MAX;

void lru_unlink(ndgi_vt* v, uint32_t s) {
    const uint32_t p = v->prev[s], n = v->next[s];
    if (p != kNone) v->next[p] = n; else v->head = n;
    if (n != kNone) v->prev[n] = p; else v->tail = p;
    v->prev[s] = v->next[s] = kNone;
}

void lru_push_back(ndgi_vt* v, uint32_t s) {
    v->prev[s] = v->tail;
    v->next[s] = kNone;
    if (v->tail != kNone) v->next[v->tail] = s; else v->head = s;
    v->tail = s;
}

int32_t bucket_of(const ndgi_vt* v, double t) {
    int32_t b = (int32_t)std::floor(t * (double)v->nbuckets);
    if (b >= v->nbuckets) b = v->nbuckets - 1;
    if (b < 0) b = 0;
    return b;
}

}  // namespace

extern "C" {

ndgi_status ndgi_vt_create(uint32_t num_tiles, uint32_t capacity, uint32_t num_buckets, ndgi_vt** out) {
    if (!out || num_tiles == 0 || capacity == 0 || num_buckets == 0 || num_buckets > (1u << 20))
        return ndgi::set_error(NDGI_ERR_ARG, "ndgi_vt_create: NULL out, or 0 tiles / slots / buckets, or > 2^20 buckets");
    ndgi_vt* v = new (std::nothrow) ndgi_vt();
    if (!v) return ndgi::set_error(NDGI_ERR_NOMEM, "host allocation");
    try {
        v->num_tiles = num_tiles;
        v->capacity = capacity;
        v->nbuckets = (int32_t)num_buckets;
        v->pt.assign((size_t)num_tiles * 2, -1);
        v->slot_tile.assign(capacity, kNone);
        v->prev.assign(capacity, kNone);
        v->next.assign(capacity, kNone);
        v->seen.assign(num_tiles, 0);
    } catch (...) {
        delete v;
        return ndgi::set_error(NDGI_ERR_NOMEM, "host allocation");
    }
    *out = v;
    return NDGI_OK;
}

ndgi_status ndgi_vt_free(ndgi_vt* v) {
    if (!v) return NDGI_ERR_ARG;
    delete v;
    return NDGI_OK;
}

ndgi_status ndgi_vt_request(ndgi_vt* v, const uint32_t* ids, uint32_t n, float t, uint32_t* job_ids,
                            uint32_t* job_slots, uint32_t* n_jobs, float* t_decode, int32_t* bucket) {
    if (!v || (!ids && n) || !job_ids || !job_slots || !n_jobs) return ndgi::set_error(NDGI_ERR_ARG, "NULL argument");
    if (!std::isfinite(t) || t < 0.0f || t > 1.0f) return ndgi::set_error(NDGI_ERR_RANGE, "t outside [0,1]");
    // validate the whole request before touching any state
    const uint64_t rid = ++v->req_id;
    uint32_t distinct = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (ids[i] >= v->num_tiles) return ndgi::set_error(NDGI_ERR_ARG, "tile id >= num_tiles");
        if (v->seen[ids[i]] != rid) {
            v->seen[ids[i]] = rid;
            ++distinct;
        }
    }
    if (distinct > v->capacity)   // the request cannot be resident at once
        return ndgi::set_error(NDGI_ERR_RANGE, "more distinct tiles requested than cache slots");
    const int32_t b = bucket_of(v, (double)t);
    const double td = ((double)b + 0.5) / (double)v->nbuckets;
    const uint64_t rid2 = ++v->req_id;   // second pass: dedupe marker
    uint32_t nj = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t id = ids[i];
        if (v->seen[id] == rid2) continue;   // duplicate within this request
        v->seen[id] = rid2;
        ++v->stats[0];
        int32_t slot = v->pt[2 * (size_t)id];
        if (slot >= 0) {
            lru_unlink(v, (uint32_t)slot);
            lru_push_back(v, (uint32_t)slot);
            if (v->pt[2 * (size_t)id + 1] == b) {
                ++v->stats[1];
                continue;
            }
        } else {
            uint32_t s;
            if (v->fresh < v->capacity) {
                s = v->fresh++;
            } else {
                s = v->head;   // least recently used; never one touched by this request (distinct <= capacity)
                lru_unlink(v, s);
                const uint32_t old = v->slot_tile[s];
                if (old != kNone) {
                    v->pt[2 * (size_t)old] = -1;
                    v->pt[2 * (size_t)old + 1] = -1;
                    ++v->stats[3];
                }
            }
            lru_push_back(v, s);
            v->slot_tile[s] = id;
            slot = (int32_t)s;
            v->pt[2 * (size_t)id] = slot;
        }
        v->pt[2 * (size_t)id + 1] = b;
        job_ids[nj] = id;
        job_slots[nj] = (uint32_t)slot;
        ++nj;
        ++v->stats[2];
    }
    if (nj) ++v->version;   // jobs (and any evictions, which come with a job) changed the table
    *n_jobs = nj;
    if (t_decode) *t_decode = (float)td;
    if (bucket) *bucket = b;
    return NDGI_OK;
}

ndgi_status ndgi_vt_bucket(const ndgi_vt* v, float t, int32_t* bucket, float* t_decode) {
    if (!v || !bucket) return ndgi::set_error(NDGI_ERR_ARG, "NULL argument");
    if (!std::isfinite(t) || t < 0.0f || t > 1.0f) return ndgi::set_error(NDGI_ERR_RANGE, "t outside [0,1]");
    const int32_t b = bucket_of(v, (double)t);
    *bucket = b;
    if (t_decode) *t_decode = (float)(((double)b + 0.5) / (double)v->nbuckets);
    return NDGI_OK;
}

ndgi_status ndgi_vt_page_table(const ndgi_vt* v, int32_t* out_host) {
    if (!v || !out_host) return NDGI_ERR_ARG;
    std::memcpy(out_host, v->pt.data(), v->pt.size() * sizeof(int32_t));
    return NDGI_OK;
}

ndgi_status ndgi_vt_upload(ndgi_vt* v, int32_t* page_table_dev, void* stream) {
    if (!v || !page_table_dev) return ndgi::set_error(NDGI_ERR_ARG, "NULL argument");
    // unchanged since the last upload to this buffer: nothing to copy (an
    // all-hit frame costs no transfer)
    if (v->uploaded_ptr == page_table_dev && v->uploaded_version == v->version) return NDGI_OK;
    // pageable source: the call returns once the table is staged, so the next
    // request may modify it while the copy is in flight
    const cudaError_t e = cudaMemcpyAsync(page_table_dev, v->pt.data(), v->pt.size() * sizeof(int32_t),
                                          cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return ndgi::set_error(NDGI_ERR_CUDA, cudaGetErrorString(e));
    v->uploaded_ptr = page_table_dev;
    v->uploaded_version = v->version;
    return NDGI_OK;
}

ndgi_status ndgi_vt_stats(const ndgi_vt* v, uint64_t out[4]) {
    if (!v || !out) return NDGI_ERR_ARG;
    for (int i = 0; i < 4; ++i) out[i] = v->stats[i];
    return NDGI_OK;
}

}  // extern "C"
