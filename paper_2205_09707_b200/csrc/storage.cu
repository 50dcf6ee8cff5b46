// storage.cu — on-disk index format (SPEC.md "storage" module, SPEC.md:425-472;
// SURVEY.md §8f rank 1): save, and load = mmap -> HBM upload -> checksums
// verified ON THE GPU over the uploaded arrays -> validate_index.
//
// The reference ships no loader: its SPEC fixes the layout —
// manifest.json + little-endian centroids.f32 (K x d), codes.u32 (T),
// residuals.bin (T x b*d/8), doclens.u32 (N), ivf_offsets.u64 (K + 1),
// ivf_postings.u32 — and leaves the checksum open.  Ours (FORMAT.md):
//   fnv(h, w) = (h ^ w) * 0x100000001b3, h0 = 0xcbf29ce484222325, on 64-bit
//   little-endian words (a file's tail zero-padded to 8 bytes);
//   a 64 KiB block's 8192 words are dealt to 32 lanes (word i -> lane i % 32),
//   lane digest = fnv-fold of its words in order, block digest = fnv-fold of
//   the 32 lane digests; file digest = fnv-fold of the block digests followed
//   by the byte length.
// The lane split makes a warp hash a block with coalesced loads (one warp per
// block on the GPU); the host computes the same digest with threads.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "storage.hpp"

namespace plaid {
namespace {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr uint64_t kBlockBytes = 64 * 1024;
constexpr uint64_t kBlockWords = kBlockBytes / 8;

__host__ __device__ __forceinline__ uint64_t fnv(uint64_t h, uint64_t w) { return (h ^ w) * kFnvPrime; }

__host__ __device__ __forceinline__ uint64_t load_word(const uint8_t* p, uint64_t bytes, uint64_t i) {
    const uint64_t off = i * 8;
    if (off + 8 <= bytes) {
        uint64_t w;
        memcpy(&w, p + off, 8);
        return w;
    }
    uint64_t w = 0;
    for (uint64_t b = 0; off + b < bytes; ++b) w |= uint64_t(p[off + b]) << (8 * b);
    return w;
}

// one warp per 64 KiB block: lane l folds words l, l + 32, ...
__global__ void block_hash_kernel(const uint8_t* __restrict__ data, uint64_t bytes, uint64_t nblocks,
                                  uint64_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t b = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nblocks; b += warps) {
        const uint8_t* base = data + b * kBlockBytes;
        const uint64_t len = bytes - b * kBlockBytes < kBlockBytes ? bytes - b * kBlockBytes : kBlockBytes;
        const uint64_t nw = (len + 7) / 8;
        uint64_t h = kFnvBasis;
        const bool full = len == kBlockBytes && (reinterpret_cast<uintptr_t>(base) & 7) == 0;
        for (uint64_t i = lane; i < nw; i += 32)
            h = fnv(h, full ? __ldg(reinterpret_cast<const unsigned long long*>(base) + i) : load_word(base, len, i));
        uint64_t d = kFnvBasis;
        for (int l = 0; l < 32; ++l) d = fnv(d, __shfl_sync(0xffffffffu, h, l));
        if (lane == 0) out[b] = d;
    }
}

uint64_t host_block_hash(const uint8_t* base, uint64_t len) {
    uint64_t lanes[32];
    for (auto& h : lanes) h = kFnvBasis;
    const uint64_t nw = (len + 7) / 8;
    for (uint64_t i = 0; i < nw; ++i) lanes[i % 32] = fnv(lanes[i % 32], load_word(base, len, i));
    uint64_t d = kFnvBasis;
    for (uint64_t h : lanes) d = fnv(d, h);
    return d;
}

uint64_t fold_blocks(const std::vector<uint64_t>& blocks, uint64_t bytes) {
    uint64_t h = kFnvBasis;
    for (uint64_t b : blocks) h = fnv(h, b);
    return fnv(h, bytes);
}

// ---- files ------------------------------------------------------------------------
struct Mapped {
    void* p = nullptr;
    uint64_t bytes = 0;
    ~Mapped() {
        if (p && bytes) munmap(p, bytes);
    }
};

std::string join(const std::string& dir, const char* name) { return dir + "/" + name; }

void map_file(const std::string& path, Mapped& m) {
    const int fd = open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(PLAID_IO_ERROR, "cannot open " + path + ": " + strerror(errno));
    struct stat st {};
    if (fstat(fd, &st) != 0) {
        close(fd);
        fail(PLAID_IO_ERROR, "cannot stat " + path);
    }
    m.bytes = uint64_t(st.st_size);
    if (m.bytes) {
        m.p = mmap(nullptr, m.bytes, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
        if (m.p == MAP_FAILED) {
            m.p = nullptr;
            close(fd);
            fail(PLAID_IO_ERROR, "cannot mmap " + path);
        }
    }
    close(fd);
}

void write_file(const std::string& path, const void* data, uint64_t bytes) {
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) fail(PLAID_IO_ERROR, "cannot create " + path + ": " + strerror(errno));
    const uint8_t* p = static_cast<const uint8_t*>(data);
    uint64_t done = 0;
    while (done < bytes) {
        const size_t chunk = size_t(std::min<uint64_t>(bytes - done, 1ull << 28));
        const size_t w = fwrite(p + done, 1, chunk, f);
        if (w != chunk) {
            fclose(f);
            remove(path.c_str());
            fail(PLAID_IO_ERROR, "short write to " + path + " (disk full?)");
        }
        done += w;
    }
    if (fclose(f) != 0) {
        remove(path.c_str());
        fail(PLAID_IO_ERROR, "cannot close " + path);
    }
}

// ---- manifest (our own writer's JSON; a small reader for exactly that shape) -------------
struct Manifest {
    std::map<std::string, std::string> scalars;          // key -> raw token
    std::map<std::string, std::vector<std::string>> arrays;
    std::map<std::string, std::string> checksums;        // file -> hex digest
};

class JsonReader {
public:
    explicit JsonReader(const std::string& s) : s_(s) {}
    Manifest parse() {
        Manifest m;
        expect('{');
        if (peek() == '}') return ++i_, m;
        for (;;) {
            const std::string key = string();
            expect(':');
            const char c = peek();
            if (c == '[') {
                m.arrays[key] = array();
            } else if (c == '{') {
                ++i_;
                if (peek() != '}') {
                    for (;;) {
                        const std::string k = string();
                        expect(':');
                        m.checksums[k] = string();
                        if (peek() == ',') { ++i_; continue; }
                        break;
                    }
                }
                expect('}');
            } else {
                m.scalars[key] = c == '"' ? string() : token();
            }
            if (peek() == ',') { ++i_; continue; }
            break;
        }
        expect('}');
        return m;
    }

private:
    char peek() {
        while (i_ < s_.size() && isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
        if (i_ >= s_.size()) bad();
        return s_[i_];
    }
    void expect(char c) {
        if (peek() != c) bad();
        ++i_;
    }
    std::string string() {
        expect('"');
        const size_t e = s_.find('"', i_);
        if (e == std::string::npos) bad();
        std::string out = s_.substr(i_, e - i_);
        i_ = e + 1;
        return out;
    }
    std::string token() {
        peek();
        const size_t b = i_;
        while (i_ < s_.size() && (isalnum(static_cast<unsigned char>(s_[i_])) || strchr("+-.eE", s_[i_]))) ++i_;
        if (i_ == b) bad();
        return s_.substr(b, i_ - b);
    }
    std::vector<std::string> array() {
        std::vector<std::string> out;
        expect('[');
        if (peek() == ']') return ++i_, out;
        for (;;) {
            out.push_back(token());
            if (peek() == ',') { ++i_; continue; }
            break;
        }
        expect(']');
        return out;
    }
    [[noreturn]] void bad() { fail(PLAID_HEADER_MISMATCH, "manifest.json is not valid JSON of the expected shape"); }
    const std::string& s_;
    size_t i_ = 0;
};

uint64_t get_u64(const Manifest& m, const char* key) {
    auto it = m.scalars.find(key);
    if (it == m.scalars.end()) fail(PLAID_HEADER_MISMATCH, std::string("manifest.json lacks ") + key);
    char* end = nullptr;
    const unsigned long long v = strtoull(it->second.c_str(), &end, 10);
    if (!end || *end) fail(PLAID_HEADER_MISMATCH, std::string("manifest.json: bad integer for ") + key);
    return v;
}

std::vector<uint32_t> get_bits(const Manifest& m, const char* key, size_t n) {
    auto it = m.arrays.find(key);
    if (it == m.arrays.end() || it->second.size() != n)
        fail(PLAID_HEADER_MISMATCH, std::string("manifest.json: ") + key + " missing or of the wrong length");
    std::vector<uint32_t> out;
    for (const auto& t : it->second) out.push_back(uint32_t(strtoul(t.c_str(), nullptr, 10)));
    return out;
}

const char* kFiles[6] = {"centroids.f32", "codes.u32", "residuals.bin", "doclens.u32", "ivf_offsets.u64",
                         "ivf_postings.u32"};

std::string hex64(uint64_t v) {
    char b[17];
    snprintf(b, sizeof b, "%016" PRIx64, v);
    return b;
}

}  // namespace

uint64_t checksum_host(const void* data, uint64_t bytes) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    const uint64_t nb = (bytes + kBlockBytes - 1) / kBlockBytes;
    std::vector<uint64_t> blocks(nb);
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const uint64_t nt = std::min<uint64_t>(hw, std::max<uint64_t>(1, nb / 64));
    std::vector<std::thread> pool;
    for (uint64_t t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (uint64_t b = t; b < nb; b += nt)
                blocks[b] = host_block_hash(p + b * kBlockBytes, std::min(kBlockBytes, bytes - b * kBlockBytes));
        });
    for (auto& th : pool) th.join();
    return fold_blocks(blocks, bytes);
}

uint64_t checksum_device(const void* d_data, uint64_t bytes, cudaStream_t st) {
    const uint64_t nb = (bytes + kBlockBytes - 1) / kBlockBytes;
    if (nb == 0) return fold_blocks({}, 0);
    uint64_t* d_out = nullptr;
    PLAID_CUDA(cudaMalloc(&d_out, nb * sizeof(uint64_t)));
    const uint64_t grid = std::min<uint64_t>((nb + 7) / 8, 148ull * 16);
    block_hash_kernel<<<uint32_t(grid), 256, 0, st>>>(static_cast<const uint8_t*>(d_data), bytes, nb, d_out);
    std::vector<uint64_t> blocks(nb);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(blocks.data(), d_out, nb * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_out);
    PLAID_CUDA(e);
    return fold_blocks(blocks, bytes);
}

void save_index(const plaid_index_desc& d, const std::string& dir, uint64_t rng_seed) {
    validate_index_host(d);
    struct stat st {};
    if (stat(dir.c_str(), &st) != 0 || !S_ISDIR(st.st_mode)) fail(PLAID_IO_ERROR, "not a directory: " + dir);
    const uint64_t K = d.num_centroids, T = d.num_embeddings, N = d.num_passages;
    const uint64_t P = d.ivf_offsets[K];
    const void* data[6] = {d.centroids, d.codes, d.residuals, d.doclens, d.ivf_offsets, d.ivf_postings};
    const uint64_t bytes[6] = {K * d.dim * 4, T * 4, T * (uint64_t(d.nbits) * d.dim / 8), N * 4, (K + 1) * 8, P * 4};
    std::string sums;
    try {
        for (int f = 0; f < 6; ++f) {
            write_file(join(dir, kFiles[f]), data[f], bytes[f]);
            sums += std::string(f ? ", " : "") + "\"" + kFiles[f] + "\": \"" + hex64(checksum_host(data[f], bytes[f])) + "\"";
        }
        const uint64_t nb = uint64_t(1) << d.nbits;
        std::string cut, wts, cutb, wtsb;
        char buf[64];
        for (uint64_t i = 0; i < nb; ++i) {
            uint32_t u;
            if (i + 1 < nb) {
                memcpy(&u, d.bucket_cutoffs + i, 4);
                snprintf(buf, sizeof buf, "%s%.9g", i ? ", " : "", d.bucket_cutoffs[i]);
                cut += buf;
                snprintf(buf, sizeof buf, "%s%u", i ? ", " : "", u);
                cutb += buf;
            }
            memcpy(&u, d.bucket_weights + i, 4);
            snprintf(buf, sizeof buf, "%s%.9g", i ? ", " : "", d.bucket_weights[i]);
            wts += buf;
            snprintf(buf, sizeof buf, "%s%u", i ? ", " : "", u);
            wtsb += buf;
        }
        char head[512];
        snprintf(head, sizeof head,
                 "{\n  \"format_version\": %d,\n  \"dim\": %u,\n  \"nbits\": %u,\n  \"num_passages\": %" PRIu64
                 ",\n  \"num_embeddings\": %" PRIu64 ",\n  \"num_centroids\": %" PRIu64 ",\n  \"num_postings\": %" PRIu64
                 ",\n  \"rng_seed\": %" PRIu64 ",\n",
                 kFormatVersion, d.dim, d.nbits, N, T, K, P, rng_seed);
        std::string js = head;
        js += "  \"bucket_cutoffs\": [" + cut + "],\n  \"bucket_weights\": [" + wts + "],\n";
        js += "  \"bucket_cutoffs_bits\": [" + cutb + "],\n  \"bucket_weights_bits\": [" + wtsb + "],\n";
        js += "  \"checksum\": \"fnv1a64-lane32-block64k\",\n  \"checksums\": {" + sums + "}\n}\n";
        write_file(join(dir, "manifest.json"), js.data(), js.size());
    } catch (...) {
        for (const char* f : kFiles) remove(join(dir, f).c_str());  // no partial index left behind
        remove(join(dir, "manifest.json").c_str());
        throw;
    }
}

DeviceIndex* open_index(const std::string& dir, int device, uint32_t flags) {
    Mapped man;
    map_file(join(dir, "manifest.json"), man);
    const std::string text(static_cast<const char*>(man.p), man.bytes);
    const Manifest m = JsonReader(text).parse();
    const uint64_t version = get_u64(m, "format_version");
    if (version != uint64_t(kFormatVersion))
        fail(PLAID_UNSUPPORTED_VERSION, "index format_version " + std::to_string(version) + " (this build reads " +
                                            std::to_string(kFormatVersion) + ")");
    plaid_index_desc d{};
    d.dim = uint32_t(get_u64(m, "dim"));
    d.nbits = uint32_t(get_u64(m, "nbits"));
    d.num_passages = get_u64(m, "num_passages");
    d.num_embeddings = get_u64(m, "num_embeddings");
    d.num_centroids = get_u64(m, "num_centroids");
    if (d.nbits != 1 && d.nbits != 2 && d.nbits != 4) fail(PLAID_PACKING_UNSUPPORTED, "manifest nbits must be 1, 2 or 4");
    const uint64_t nb = uint64_t(1) << d.nbits;
    const std::vector<uint32_t> cb = get_bits(m, "bucket_cutoffs_bits", nb - 1);
    const std::vector<uint32_t> wb = get_bits(m, "bucket_weights_bits", nb);
    std::vector<float> cut(nb - 1), wts(nb);
    memcpy(cut.data(), cb.data(), cut.size() * 4);
    memcpy(wts.data(), wb.data(), wts.size() * 4);
    Mapped files[6];
    for (int f = 0; f < 6; ++f) map_file(join(dir, kFiles[f]), files[f]);
    // dimensional bookkeeping (SPEC.md storage invariants) before touching the data
    const uint64_t K = d.num_centroids, T = d.num_embeddings, N = d.num_passages;
    const uint64_t want[5] = {K * d.dim * 4, T * 4, T * (uint64_t(d.nbits) * d.dim / 8), N * 4, (K + 1) * 8};
    for (int f = 0; f < 5; ++f)
        if (files[f].bytes != want[f])
            fail(PLAID_LENGTH_MISMATCH, std::string(kFiles[f]) + " has " + std::to_string(files[f].bytes) +
                                            " bytes, manifest implies " + std::to_string(want[f]));
    const uint64_t* ivo = static_cast<const uint64_t*>(files[4].p);
    if (files[5].bytes != ivo[K] * 4) fail(PLAID_LENGTH_MISMATCH, "ivf_postings.u32 length != ivf_offsets[K]");
    d.centroids = static_cast<const float*>(files[0].p);
    d.codes = static_cast<const uint32_t*>(files[1].p);
    d.residuals = static_cast<const uint8_t*>(files[2].p);
    d.doclens = static_cast<const uint32_t*>(files[3].p);
    d.ivf_offsets = ivo;
    d.ivf_postings = static_cast<const uint32_t*>(files[5].p);
    d.bucket_cutoffs = cut.data();
    d.bucket_weights = wts.data();
    if (flags & PLAID_OPEN_VALIDATE) validate_index_host(d);
    auto* ix = new DeviceIndex(d, device, 0);
    try {
        if (!(flags & PLAID_OPEN_NO_CHECKSUMS)) {
            // checksums over the arrays as they sit in HBM: the upload is verified too
            DeviceGuard g(device);
            const IndexView& v = ix->view();
            const void* dev[6] = {v.centroids, v.codes, v.residuals, v.doclens, v.ivf_offsets, v.ivf_postings};
            const uint64_t sizes[6] = {files[0].bytes, files[1].bytes, files[2].bytes,
                                       files[3].bytes, files[4].bytes, files[5].bytes};
            for (int f = 0; f < 6; ++f) {
                auto it = m.checksums.find(kFiles[f]);
                if (it == m.checksums.end()) fail(PLAID_HEADER_MISMATCH, std::string("no checksum for ") + kFiles[f]);
                const uint64_t got = checksum_device(dev[f], sizes[f], nullptr);
                if (hex64(got) != it->second)
                    fail(PLAID_CHECKSUM_MISMATCH, std::string(kFiles[f]) + ": checksum " + hex64(got) +
                                                      " != manifest " + it->second);
            }
        }
    } catch (...) {
        delete ix;
        throw;
    }
    return ix;
}

}  // namespace plaid

// ---- measured read floor (bench.py's roofline context) ---------------------------------
namespace plaid {
namespace {
__global__ void read_stream_kernel(const uint4* __restrict__ src, uint64_t n16, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(src + i);
        acc += v.x ^ v.w;
    }
    if (acc == 0x9e3779b97f4a7c15ull) *sink = acc;  // keeps the loads alive
}
}  // namespace
}  // namespace plaid

// Best-of-`iters` GB/s of a plain coalesced read of `bytes` from HBM (L2
// flushed by a 256 MiB write before each pass): the achievable streaming rate
// of a one-pass kernel of that size, next to the copy peak of MEASURED_PEAKS.
extern "C" int plaid_measure_read_gbs(int device, uint64_t bytes, int iters, double* out_gbs) {
    using namespace plaid;
    *out_gbs = 0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    uint8_t *src = nullptr, *flush = nullptr;
    unsigned long long* sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    int rc = int(cudaMalloc(&src, bytes));
    if (!rc) rc = int(cudaMalloc(&flush, 256ull << 20));
    if (!rc) rc = int(cudaMalloc(&sink, 8));
    if (!rc) rc = int(cudaMemset(src, 1, bytes));
    if (!rc) rc = int(cudaEventCreate(&a));
    if (!rc) rc = int(cudaEventCreate(&b));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float best = 1e30f;
    for (int it = 0; !rc && it < iters + 1; ++it) {
        cudaMemset(flush, it, 256ull << 20);
        cudaEventRecord(a);
        read_stream_kernel<<<sms * 32, 256>>>(reinterpret_cast<const uint4*>(src), bytes / 16, sink);
        cudaEventRecord(b);
        rc = int(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
    }
    if (!rc) *out_gbs = double(bytes) / (double(best) * 1e-3) / 1e9;
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFree(src);
    cudaFree(flush);
    cudaFree(sink);
    cudaSetDevice(prev);
    return rc;
}
