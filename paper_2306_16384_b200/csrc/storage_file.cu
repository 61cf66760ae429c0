// storage_file.cu -- file-backed storage tier with a page-granular access
// accumulator (north-star subsystems 2 and 5).
//
// The backing store is the reference's .gfea file (graph.py:304-327): a
// header of `offset` bytes (24) followed by fp32 rows, read in pages of
// `page_bytes` (the paper's GIDS init parameters: offset, cache-line size,
// number of elements).  Per served batch:
//
//   control stream  the storage-tier rows of the batch (the gather's host
//                   work list, backing entries only) mark the pages their
//                   bytes span in a page bitmap; the bitmap is compacted to
//                   an ascending, de-duplicated page list (the accumulator's
//                   request batch: every page once, adjacent pages adjacent),
//                   each listed page gets its staging slot, and the list is
//                   copied to pinned host memory.
//   host            the list is coalesced into runs of consecutive pages and
//                   read with pread() by `io_threads` threads into pinned
//                   staging, slot-contiguous (a run is one read).
//   gather stream   one DMA copy of the staged pages to HBM, then the row
//                   kernel: storage rows from the HBM staging (a row that
//                   straddles two pages reads on into the next slot, which is
//                   the next page), constant-buffer rows zero-copy from
//                   pinned host, cache insertion as in the pinned tier.
//
// Rows are the file's bytes, so results are bit-identical to the pinned tier.
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gids_internal.cuh"

struct FileTier {
    int fd = -1;
    bool direct = false;
    int64_t offset = 0, page = 0, npages = 0, row_bytes = 0, cap = 0;
    int io_threads = 1;
    uint32_t* page_bits = nullptr;  // device [ceil(npages/32)]
    int32_t* page_list = nullptr;   // device [cap]
    // device [npages] per decision set: batch b+1's plan (control stream) must
    // not overwrite the slots batch b's gather (gather stream) is reading
    int32_t* page_slot[2] = {nullptr, nullptr};
    int64_t* page_cnt = nullptr;    // device [2]: count, overflow
    int32_t* hlist[2] = {nullptr, nullptr};  // pinned [cap]
    int64_t* hcnt[2] = {nullptr, nullptr};   // pinned [2]
    char* hstage[2] = {nullptr, nullptr};    // pinned, page aligned [cap * page]
    char* dstage = nullptr;                  // HBM [cap * page]
    cudaEvent_t listed[2] = {nullptr, nullptr};
    // statistics (since the tier was attached)
    int64_t pages_read = 0, bytes_read = 0, runs = 0;
    double io_ms = 0.0;
};

namespace {

constexpr int BLOCK = 256;

// pages spanned by the bytes of each storage-tier row of the host work list
__global__ void k_page_mark(const int2* __restrict__ host_list, const int64_t* __restrict__ list_cnt,
                            int64_t offset, int64_t row_bytes, int64_t page, uint32_t* bits) {
    const int64_t n = list_cnt[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int2 it = host_list[i];
        if (it.y >= 0) continue;  // constant-buffer row: not a storage access
        const int64_t x = -(int64_t)(it.y + 1);
        const int64_t b0 = offset + x * row_bytes;
        const int64_t p0 = b0 / page, p1 = (b0 + row_bytes - 1) / page;
        for (int64_t p = p0; p <= p1; p++) atomicOr(bits + (p >> 5), 1u << (p & 31));
    }
}

__global__ void k_page_slot(const int32_t* __restrict__ list, const int64_t* __restrict__ cnt,
                            int32_t* slot) {
    const int64_t n = cnt[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        slot[list[i]] = (int32_t)i;
}

// storage rows from the HBM page staging, buffer rows zero-copy from pinned
// host; T = 8-byte words (offset, row and page sizes are multiples of 8) or
// fp32 words otherwise
template <typename T, int U>
__global__ void __launch_bounds__(BLOCK)
k_gather_file(const int2* __restrict__ host_list, const int64_t* __restrict__ list_cnt,
              const int32_t* __restrict__ ins, const T* __restrict__ buffer_rows,
              const char* __restrict__ dstage, const int32_t* __restrict__ page_slot,
              int64_t offset, int64_t page, T* __restrict__ cache_rows, T* __restrict__ out,
              uint32_t cpr) {
    const uint64_t total = (uint64_t)list_cnt[1] * cpr;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)BLOCK + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * BLOCK) >> 5;
    const int64_t rb = (int64_t)cpr * sizeof(T);
    for (uint64_t base = warp * U * 32; base < total; base += nwarps * U * 32) {
        T v[U];
        int64_t d[U], d2[U];
#pragma unroll
        for (int k = 0; k < U; k++) {
            const uint64_t i = base + k * 32 + lane;
            d[k] = -1;
            if (i < total) {
                const uint64_t r = i / cpr, c = i - r * cpr;
                const int2 it = host_list[r];
                const T* src;
                if (it.y >= 0) {
                    src = buffer_rows + (int64_t)it.y * cpr;
                } else {
                    const int64_t x = -(int64_t)(it.y + 1);
                    const int64_t b0 = offset + x * rb;
                    src = reinterpret_cast<const T*>(dstage + (int64_t)page_slot[b0 / page] * page +
                                                     b0 % page);
                }
                v[k] = src[c];
                d[k] = (int64_t)it.x * cpr + (int64_t)c;
                const int32_t t = ins[it.x];
                d2[k] = t >= 0 ? (int64_t)t * cpr + (int64_t)c : (int64_t)-1;
            }
        }
#pragma unroll
        for (int k = 0; k < U; k++)
            if (d[k] >= 0) {
                out[d[k]] = v[k];
                if (d2[k] >= 0) cache_rows[d2[k]] = v[k];
            }
    }
}

// read one run of consecutive pages into staging (handles short reads)
bool read_run(int fd, char* dst, int64_t file_off, int64_t len, std::string* err) {
    int64_t done = 0;
    while (done < len) {
        ssize_t r = pread(fd, dst + done, (size_t)(len - done), (off_t)(file_off + done));
        if (r < 0) {
            if (errno == EINTR) continue;
            *err = std::string("pread: ") + strerror(errno);
            return false;
        }
        if (r == 0) {  // past the end of the file: the tail page is partial
            memset(dst + done, 0, (size_t)(len - done));
            return true;
        }
        done += r;
    }
    return true;
}

}  // namespace

int gids_file_plan(gids_handle* h, int par, cudaStream_t st) {
    FileTier* f = h->ft;
    const int g = gids_grid(h->serve_cap, BLOCK, 8 * GIDS_SMS);
    k_page_mark<<<g, BLOCK, 0, st>>>(h->host_list, h->list_cnt, f->offset, f->row_bytes, f->page,
                                     f->page_bits);
    GIDS_LAUNCH_CHECK(h);
    GIDS_CUDA_TRY(cudaMemsetAsync(f->page_cnt, 0, 2 * sizeof(int64_t), st));
    int rc = gids_bitmap_compact_n(h, f->page_bits, f->npages, f->page_list, f->page_cnt, f->cap,
                                   true, f->page_cnt + 1, h->serve_word_parts, st);
    if (rc) return rc;
    k_page_slot<<<gids_grid(f->cap, BLOCK, 8 * GIDS_SMS), BLOCK, 0, st>>>(
        f->page_list, f->page_cnt, f->page_slot[par]);
    GIDS_LAUNCH_CHECK(h);
    GIDS_CUDA_TRY(cudaMemcpyAsync(f->hcnt[par], f->page_cnt, 2 * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaMemcpyAsync(f->hlist[par], f->page_list, sizeof(int32_t) * f->cap,
                                  cudaMemcpyDeviceToHost, st));
    GIDS_CUDA_TRY(cudaEventRecord(f->listed[par], st));
    return GIDS_OK;
}

int gids_file_fetch_and_gather(gids_handle* h, int par, float* out, cudaStream_t gst) {
    FileTier* f = h->ft;
    GIDS_CUDA_TRY(cudaEventSynchronize(f->listed[par]));
    const int64_t cnt = f->hcnt[par][0];
    if (f->hcnt[par][1] || cnt > f->cap) {
        gids_set_error("file tier: a batch spans more pages than the staging holds "
                       "(raise max_pages)");
        return GIDS_E_CAPACITY;
    }
    auto t0 = std::chrono::steady_clock::now();
    // coalesce the ascending page list into runs of consecutive pages
    const int32_t* pl = f->hlist[par];
    std::vector<int64_t> run_start, run_len, run_slot;
    for (int64_t i = 0; i < cnt;) {
        int64_t j = i + 1;
        while (j < cnt && pl[j] == pl[j - 1] + 1) j++;
        run_start.push_back(pl[i]);
        run_len.push_back(j - i);
        run_slot.push_back(i);
        i = j;
    }
    const int64_t nruns = (int64_t)run_start.size();
    // split the runs over the I/O threads by page count
    int nt = f->io_threads;
    if (nt > nruns) nt = (int)std::max<int64_t>(1, nruns);
    std::vector<int64_t> cut(nt + 1, nruns);
    cut[0] = 0;
    {
        int64_t per = (cnt + nt - 1) / std::max(1, nt), acc = 0;
        int t = 1;
        for (int64_t r = 0; r < nruns && t < nt; r++) {
            acc += run_len[r];
            if (acc >= per * t) cut[t++] = r + 1;
        }
    }
    std::vector<std::string> errs(nt);
    auto work = [&](int t) {
        for (int64_t r = cut[t]; r < cut[t + 1]; r++)
            if (!read_run(f->fd, f->hstage[par] + run_slot[r] * f->page, run_start[r] * f->page,
                          run_len[r] * f->page, &errs[t]))
                return;
    };
    if (nt <= 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; t++) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }
    for (auto& e : errs)
        if (!e.empty()) {
            gids_set_error("file tier: " + e);
            return GIDS_E_CUDA;
        }
    f->io_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count();
    f->pages_read += cnt;
    f->bytes_read += cnt * f->page;
    f->runs += nruns;
    if (cnt > 0)
        GIDS_CUDA_TRY(cudaMemcpyAsync(f->dstage, f->hstage[par], (size_t)(cnt * f->page),
                                      cudaMemcpyHostToDevice, gst));
    const int64_t dim = h->row_floats;
    const bool w8 = (f->offset % 8 == 0) && (f->row_bytes % 8 == 0) && (f->page % 8 == 0);
    const int grid = gids_grid(h->serve_cap, BLOCK / 32, 4 * GIDS_SMS);
    if (w8) {
        k_gather_file<int2, 4><<<grid, BLOCK, 0, gst>>>(
            h->host_list, h->list_cnt, h->ins, reinterpret_cast<const int2*>(h->buffer_rows),
            f->dstage, f->page_slot[par], f->offset, f->page,
            reinterpret_cast<int2*>(h->cache_rows),
            reinterpret_cast<int2*>(out), (uint32_t)(dim / 2));
    } else {
        k_gather_file<float, 4><<<grid, BLOCK, 0, gst>>>(
            h->host_list, h->list_cnt, h->ins, h->buffer_rows, f->dstage, f->page_slot[par],
            f->offset,
            f->page, h->cache_rows, out, (uint32_t)dim);
    }
    GIDS_LAUNCH_CHECK(h);
    return GIDS_OK;
}

void gids_file_free(gids_handle* h) {
    FileTier* f = h->ft;
    if (!f) return;
    if (f->fd >= 0) close(f->fd);
    void* dev[] = {f->page_bits, f->page_list, f->page_slot[0], f->page_slot[1], f->page_cnt,
                   f->dstage};
    for (void* p : dev)
        if (p) cudaFree(p);
    for (int b = 0; b < 2; b++) {
        if (f->hlist[b]) cudaFreeHost(f->hlist[b]);
        if (f->hcnt[b]) cudaFreeHost(f->hcnt[b]);
        if (f->hstage[b]) cudaFreeHost(f->hstage[b]);
        if (f->listed[b]) cudaEventDestroy(f->listed[b]);
    }
    delete f;
    h->ft = nullptr;
}

extern "C" {

int gids_set_storage_file(gids_handle* h, const char* path, int64_t offset, int32_t page_bytes,
                          int64_t max_pages, int32_t io_threads, int32_t direct) {
    if (h) gids_drop_serve_graphs(h);
    if (!h || !path || offset < 0 || page_bytes < 16 || io_threads < 1) {
        gids_set_error("set_storage_file: need a path, offset >= 0, page_bytes >= 16, threads >= 1");
        return GIDS_E_INVALID;
    }
    GIDS_CUDA_TRY(cudaSetDevice(h->device));
    const int64_t rb = h->row_floats * 4;
    if (rb > page_bytes) {
        gids_set_error("set_storage_file: a feature row is larger than one page");
        return GIDS_E_INVALID;
    }
    int fd = -1;
    bool is_direct = false;
    if (direct && page_bytes % 4096 == 0) {
        fd = open(path, O_RDONLY | O_DIRECT);
        is_direct = fd >= 0;
    }
    if (fd < 0) fd = open(path, O_RDONLY);
    if (fd < 0) {
        gids_set_error(std::string("set_storage_file: open ") + path + ": " + strerror(errno));
        return GIDS_E_INVALID;
    }
    struct stat sb;
    if (fstat(fd, &sb) != 0 || sb.st_size < offset + h->N * rb) {
        close(fd);
        gids_set_error("set_storage_file: file shorter than offset + num_nodes * row_bytes");
        return GIDS_E_INVALID;
    }
    if (h->ft) gids_file_free(h);
    FileTier* f = new FileTier();
    h->ft = f;
    f->fd = fd;
    f->direct = is_direct;
    f->offset = offset;
    f->page = page_bytes;
    f->row_bytes = rb;
    f->io_threads = io_threads;
    f->npages = (offset + h->N * rb + page_bytes - 1) / page_bytes;
    int64_t cap = 2 * h->serve_cap;  // a row spans at most two pages
    if (cap > f->npages) cap = f->npages;
    if (max_pages > 0 && max_pages < cap) cap = max_pages;
    f->cap = cap > 0 ? cap : 1;
    cudaError_t e = cudaSuccess;
    auto ck = [&](cudaError_t x) {
        if (x != cudaSuccess && e == cudaSuccess) e = x;
    };
    ck(cudaMalloc((void**)&f->page_bits, sizeof(uint32_t) * ceil_div(f->npages, 32)));
    ck(cudaMalloc((void**)&f->page_list, sizeof(int32_t) * f->cap));
    ck(cudaMalloc((void**)&f->page_slot[0], sizeof(int32_t) * f->npages));
    ck(cudaMalloc((void**)&f->page_slot[1], sizeof(int32_t) * f->npages));
    ck(cudaMalloc((void**)&f->page_cnt, 2 * sizeof(int64_t)));
    ck(cudaMalloc((void**)&f->dstage, (size_t)(f->cap * f->page)));
    for (int b = 0; b < 2; b++) {
        ck(cudaMallocHost((void**)&f->hlist[b], sizeof(int32_t) * f->cap));
        ck(cudaMallocHost((void**)&f->hcnt[b], 2 * sizeof(int64_t)));
        ck(cudaMallocHost((void**)&f->hstage[b], (size_t)(f->cap * f->page)));
        ck(cudaEventCreateWithFlags(&f->listed[b], cudaEventDisableTiming));
    }
    if (e == cudaSuccess) e = cudaMemset(f->page_bits, 0, sizeof(uint32_t) * ceil_div(f->npages, 32));
    if (e != cudaSuccess) {
        gids_file_free(h);
        gids_set_error(std::string("set_storage_file: ") + cudaGetErrorString(e));
        return GIDS_E_CUDA;
    }
    return GIDS_OK;
}

int gids_storage_file_stats(gids_handle* h, int64_t* pages, int64_t* bytes, int64_t* runs,
                            double* io_ms, int32_t* direct) {
    if (!h || !h->ft) {
        gids_set_error("no file-backed storage tier attached");
        return GIDS_E_STATE;
    }
    *pages = h->ft->pages_read;
    *bytes = h->ft->bytes_read;
    *runs = h->ft->runs;
    *io_ms = h->ft->io_ms;
    *direct = h->ft->direct ? 1 : 0;
    return GIDS_OK;
}

}  // extern "C"
