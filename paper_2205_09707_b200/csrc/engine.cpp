// engine.cpp — DeviceIndex / Searcher: the host orchestration of lir::search
// (pipeline.cpp:232-283) over the sm_100a kernels in kernels.cuh.
#include "engine.hpp"

#include "device.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>

namespace plaid {

// ---------------------------------------------------------------- launch counter
namespace launch {
namespace {
thread_local uint64_t g_launches = 0;
thread_local int64_t g_pdl_issued = 0;
std::atomic<int64_t> g_launch_cap{-1};
}
uint64_t launches() { return g_launches; }
void reset_launches() { g_launches = 0; g_pdl_issued = 0; }
bool pdl_skip() {
    const int64_t cap = g_launch_cap.load(std::memory_order_relaxed);
    return cap >= 0 && g_pdl_issued++ >= cap;
}
int64_t set_launch_cap(int64_t cap) { return g_launch_cap.exchange(cap); }
// Every launcher calls this right after its <<<>>>: a failed launch (bad
// config, missing smem opt-in) surfaces here instead of as stale results.
void count_launch() {
    ++g_launches;
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(PLAID_CUDA_ERROR, std::string("kernel launch failed: ") + cudaGetErrorString(e));
    }
}
void fail_cuda_driver(int code, const char* what) {
    fail(PLAID_CUDA_ERROR, std::string(what) + " failed with CUresult " + std::to_string(code));
}
}  // namespace launch

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        fail(PLAID_OUT_OF_MEMORY, std::string("CUDA out of memory in ") + what);
    }
    fail(PLAID_CUDA_ERROR, std::string(cudaGetErrorString(e)) + " in " + what);
}

namespace {

bool nbits_supported(uint32_t b) { return b == 1 || b == 2 || b == 4; }

uint32_t np_bucket(uint64_t nprobe) {
    uint32_t b = 1;
    while (b < nprobe) b <<= 1;
    return b;
}


// Counter slots in Searcher::counters_.
enum : int {
    kN1 = 0,        // stage1_candidates
    kN2 = 1,        // stage2_out
    kN3 = 2,        // stage3_out
    kNOut = 3,      // final_out
    kRows2 = 4,     // stage2_rows_gathered
    kRows3 = 5,     // stage3_rows_gathered
    kNFin = 6,      // decompressed_passages
    kKConst = 7,    // K (for generic selects)
    kTmpN = 8,      // scratch count
    kEntryN = 9,    // entry-point input count
    kT4 = 13,       // stage-4 stream tokens (trace.decompressed_tokens)
    kUsedN = 14,    // range_stage2: keys of candidates owning a kept token (ukeys_)
    kFinTicket = 15,  // finalize_rank: CTAs done reading `run`
    kKeptN = 10,    // stage 2: kept centroids, their postings, queued owners (3 slots)
    kGthr = 16,     // 32 u32 per-token top-nprobe bounds (tensor S_cq kernel)
    kNumCounters = 32
};

}  // namespace

// ---------------------------------------------------------------- validation
// types.cpp:61-72 (check_unit_rows types.cpp:10-19, tolerance types.hpp:16)
void validate_query_host(const float* q, uint64_t rows, uint64_t dim, uint64_t index_dim) {
    if (rows == 0) fail(PLAID_INVALID_PARAMS, "query must contain at least one token");
    if (dim != index_dim)
        fail(PLAID_DIMENSION_MISMATCH, "query dim " + std::to_string(dim) +
                                           " does not match index dim " + std::to_string(index_dim));
    const double tol = double(1e-3f);
    // each row's sum in dim order, eight rows' chains interleaved (the
    // search path's host cost; same per-row rounding as one row at a time)
    constexpr uint64_t kR = 8;
    for (uint64_t r0 = 0; r0 < rows; r0 += kR) {
        const uint64_t nr = rows - r0 < kR ? rows - r0 : kR;
        double acc[kR] = {};
        for (uint64_t d = 0; d < dim; ++d)
            for (uint64_t j = 0; j < kR; ++j)
                if (j < nr) {
                    const double x = double(q[(r0 + j) * dim + d]);
                    acc[j] += x * x;
                }
        for (uint64_t j = 0; j < nr; ++j) {
            const double norm = std::sqrt(acc[j]);
            if (std::fabs(norm - 1.0) > tol)
                fail(PLAID_NOT_NORMALIZED,
                     "query row " + std::to_string(r0 + j) + " has L2 norm " + std::to_string(norm));
        }
    }
}

// types.cpp:88-99
void validate_params_host(const plaid_params& p, uint64_t num_centroids) {
    if (p.k < 1) fail(PLAID_INVALID_PARAMS, "k must be >= 1");
    if (p.nprobe < 1 || p.nprobe > num_centroids)
        fail(PLAID_INVALID_PARAMS, "nprobe " + std::to_string(p.nprobe) + " outside [1, " +
                                       std::to_string(num_centroids) + "]");
    if (p.ndocs < p.k) fail(PLAID_INVALID_PARAMS, "ndocs must be >= k");
    if (!(p.t_cs >= -1.0f && p.t_cs <= 1.0f)) fail(PLAID_INVALID_PARAMS, "t_cs must lie in [-1, 1]");
}

// types.cpp:74-86
void default_params_for_k(uint64_t k, plaid_params* out) {
    out->k = k;
    out->disable_filter = 0;
    if (k <= 10) {
        out->nprobe = 1; out->t_cs = 0.5f; out->ndocs = 256;
    } else if (k <= 100) {
        out->nprobe = 2; out->t_cs = 0.45f; out->ndocs = 1024;
    } else {
        out->nprobe = 4; out->t_cs = 0.4f; out->ndocs = 4096;
    }
    if (out->ndocs < k) out->ndocs = k;
}

// pipeline.cpp:227-230
uint64_t stage3_width(const plaid_params& p) { return std::max<uint64_t>((p.ndocs + 3) / 4, p.k); }

// index.cpp:12-84 (+ validate_centroids types.cpp:50-59, validate_quantizer
// residual_codec.cpp:15-40), on the host arrays before upload.
void validate_index_host(const plaid_index_desc& d) {
    auto bad = [](const std::string& m) { fail(PLAID_INVARIANT_VIOLATION, m); };
    if (!nbits_supported(d.nbits)) bad("nbits must be one of {1,2,4}");
    if (d.dim == 0 || d.dim % (8 / d.nbits) != 0) bad("dim must be positive and divisible by 8/nbits");
    const uint64_t K = d.num_centroids;
    if (K == 0) bad("index must contain at least one centroid");
    const double tol = double(1e-3f);
    for (uint64_t c = 0; c < K; ++c) {
        double acc = 0;
        for (uint32_t j = 0; j < d.dim; ++j) acc += double(d.centroids[c * d.dim + j]) * double(d.centroids[c * d.dim + j]);
        if (std::fabs(std::sqrt(acc) - 1.0) > tol) fail(PLAID_NOT_NORMALIZED, "centroid row " + std::to_string(c) + " not unit norm");
    }
    if (d.num_passages == 0) bad("index must contain at least one passage");
    uint64_t total = 0;
    for (uint64_t p = 0; p < d.num_passages; ++p) total += d.doclens[p];
    if (d.num_embeddings != total) bad("codes length must equal the doclens total");
    for (uint64_t t = 0; t < total; ++t)
        if (d.codes[t] >= K) bad("token code " + std::to_string(t) + " out of centroid range");
    const uint64_t nb = uint64_t(1) << d.nbits;
    for (uint64_t i = 1; i + 1 < nb; ++i)
        if (d.bucket_cutoffs[i] < d.bucket_cutoffs[i - 1]) bad("quantizer cutoffs not ascending");
    for (uint64_t i = 0; i < nb; ++i) {
        const float lo = i == 0 ? -INFINITY : d.bucket_cutoffs[i - 1];
        const float hi = i + 1 == nb ? INFINITY : d.bucket_cutoffs[i];
        const float w = d.bucket_weights[i];
        if (!(w >= lo && w <= hi)) bad("quantizer weight " + std::to_string(i) + " outside its bucket interval");
    }
    if (d.ivf_offsets[0] != 0) bad("inverted list offsets must start at 0");
    for (uint64_t c = 0; c < K; ++c) {
        if (d.ivf_offsets[c + 1] < d.ivf_offsets[c]) bad("inverted list offsets must be monotone");
        for (uint64_t j = d.ivf_offsets[c]; j < d.ivf_offsets[c + 1]; ++j) {
            if (d.ivf_postings[j] >= d.num_passages) bad("posting references unknown passage");
            if (j > d.ivf_offsets[c] && d.ivf_postings[j] <= d.ivf_postings[j - 1])
                bad("postings must be strictly increasing within a centroid");
        }
    }
    // content check: passage p listed under centroid c iff some token of p has code c
    std::vector<uint64_t> cursor(d.ivf_offsets, d.ivf_offsets + K);
    std::vector<uint32_t> seen(K, UINT32_MAX);
    uint64_t t = 0;
    for (uint64_t p = 0; p < d.num_passages; ++p)
        for (uint32_t j = 0; j < d.doclens[p]; ++j, ++t) {
            const uint32_t c = d.codes[t];
            if (seen[c] == p) continue;
            seen[c] = uint32_t(p);
            if (cursor[c] >= d.ivf_offsets[c + 1] || d.ivf_postings[cursor[c]] != p)
                bad("inverted list does not match token codes");
            ++cursor[c];
        }
    for (uint64_t c = 0; c < K; ++c)
        if (cursor[c] != d.ivf_offsets[c + 1]) bad("inverted list contains postings with no matching token code");
}

// ---------------------------------------------------------------- DevBuf
std::atomic<uint64_t> g_alloc_generation{0};  // bumped by every reallocation (captured graphs go stale)

template <typename T>
void DevBuf<T>::ensure(uint64_t count) {
    if (count <= n && p) return;
    g_alloc_generation.fetch_add(1);
    release();
    const uint64_t c = count ? count : 1;
    PLAID_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), c * sizeof(T)));
    n = c;
}
template <typename T>
void DevBuf<T>::release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
}
template struct DevBuf<float>;
template struct DevBuf<uint32_t>;
template struct DevBuf<uint64_t>;
template struct DevBuf<unsigned char>;
template struct DevBuf<SelectState>;
template struct DevBuf<SelectHist>;
template struct DevBuf<int>;

// ---------------------------------------------------------------- DeviceIndex
void DeviceIndex::build_range_table(cudaStream_t st) {
    // per (centroid, pid range): where the list's run in the range starts —
    // index-side, once (binary searches on the GPU).  Ranges of about N / SMs
    // ids: range_stage2 runs one CTA per range, one wave
    const uint64_t N = view_.N, K = view_.K;
    if (!N || !K || N > 0xFFFFFFFFull) return;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_);
    const uint32_t W = launch::range_width_for(N, uint32_t(sms)), R = uint32_t((N + W - 1) / W);
    uint32_t* tab = upload<uint32_t>(nullptr, K * (uint64_t(R) + 1));
    launch::wave_range_table(view_, W, R, tab, st);
    PLAID_CUDA(cudaStreamSynchronize(st));
    PLAID_CUDA(cudaGetLastError());
    view_.range_tab = tab, view_.range_w = W, view_.range_n = R;
}

template <typename T>
T* DeviceIndex::upload(const T* src, uint64_t count) {
    void* p = nullptr;
    const uint64_t bytes = std::max<uint64_t>(count, 1) * sizeof(T);
    PLAID_CUDA(cudaMalloc(&p, bytes));
    allocs_.push_back(p);
    bytes_ += bytes;
    if (count && src) PLAID_CUDA(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return static_cast<T*>(p);
}

// mult[j] for posting j = (centroid c, passage p): how many tokens of p have
// code c, saturated at 255 (kernels recount a saturated entry from the codes).
// Stage 2 scores candidates from the kept centroids' posting lists and needs
// it for the reference's gathered-row counter (pipeline.cpp:108, :133).  One
// pass over the codes per passage range; ranges run on all host threads.
static std::vector<uint8_t> posting_multiplicity(const plaid_index_desc& d, const std::vector<uint64_t>& offsets) {
    const uint64_t K = d.num_centroids, N = d.num_passages;
    const uint64_t P = d.ivf_offsets[K];
    std::vector<uint8_t> mult(P, 0);
    if (P == 0 || N == 0) return mult;
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    if (nt > 32) nt = 32;
    if (uint64_t(nt) * 4096 > N) nt = unsigned(std::max<uint64_t>(1, N / 4096));
    auto work = [&](uint64_t pb, uint64_t pe) {
        std::vector<uint64_t> cursor(K);
        std::vector<uint32_t> seen(K, UINT32_MAX);
        std::vector<uint64_t> at(K, UINT64_MAX);
        for (uint64_t c = 0; c < K; ++c) {
            const uint32_t* b = d.ivf_postings + d.ivf_offsets[c];
            const uint32_t* e = d.ivf_postings + d.ivf_offsets[c + 1];
            cursor[c] = uint64_t(std::lower_bound(b, e, uint32_t(pb)) - d.ivf_postings);
        }
        for (uint64_t p = pb; p < pe; ++p)
            for (uint64_t t = offsets[p]; t < offsets[p + 1]; ++t) {
                const uint32_t c = d.codes[t];
                if (c >= K) continue;
                if (seen[c] != uint32_t(p)) {
                    seen[c] = uint32_t(p);
                    const uint64_t j = cursor[c];
                    if (j < d.ivf_offsets[c + 1] && d.ivf_postings[j] == p) {
                        at[c] = j;
                        ++cursor[c];
                    } else {
                        at[c] = UINT64_MAX;  // inconsistent IVF (validate_index reports it)
                    }
                }
                if (at[c] != UINT64_MAX && mult[at[c]] < 255) ++mult[at[c]];
            }
    };
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i) th.emplace_back(work, N * i / nt, N * (i + 1) / nt);
    for (auto& x : th) x.join();
    return mult;
}

DeviceIndex::DeviceIndex(const plaid_index_desc& d, int device, uint64_t pid_base)
    : device_(device), pid_base_(pid_base) {
    if (!nbits_supported(d.nbits)) fail(PLAID_PACKING_UNSUPPORTED, "nbits must be one of {1,2,4}");
    if (d.dim == 0 || d.dim % 4 != 0 || d.dim > 256)
        fail(PLAID_UNSUPPORTED, "engine supports dim in {4, 8, ..., 256}");
    if (d.num_centroids == 0 || d.num_centroids > 0xFFFFFFFFull)
        fail(PLAID_INVALID_PARAMS, "centroid count must be in [1, 2^32)");
    if (d.num_passages > 0xFFFFFFFFull) fail(PLAID_INVALID_PARAMS, "corpora above 2^32 passages are not supported");
    DeviceGuard g(device);
    view_.dim = d.dim;
    view_.nbits = d.nbits;
    view_.K = d.num_centroids;
    view_.N = d.num_passages;
    view_.T = d.num_embeddings;
    view_.P = d.ivf_offsets[d.num_centroids];
    h_doclens_.assign(d.doclens, d.doclens + d.num_passages);
    std::vector<uint64_t> offsets(d.num_passages + 1, 0);
    for (uint64_t p = 0; p < d.num_passages; ++p) {
        offsets[p + 1] = offsets[p] + d.doclens[p];
        max_doclen_ = std::max(max_doclen_, d.doclens[p]);
    }
    if (offsets.back() != d.num_embeddings) fail(PLAID_LENGTH_MISMATCH, "doclens total does not match codes length");
    view_.max_doclen = max_doclen_;
    set_list_bounds(d.ivf_offsets);
    const uint64_t nb = uint64_t(1) << d.nbits;
    for (uint64_t i = 0; i < nb; ++i) view_.weights[i] = d.bucket_weights[i];
    for (uint64_t i = 0; i + 1 < nb; ++i) cutoffs_[i] = d.bucket_cutoffs[i];
    try {
        view_.centroids = upload(d.centroids, d.num_centroids * d.dim);
        view_.codes = upload(d.codes, d.num_embeddings);
        view_.residuals = upload(d.residuals, d.num_embeddings * (uint64_t(d.nbits) * d.dim / 8));
        view_.doclens = upload(d.doclens, d.num_passages);
        view_.offsets = upload(offsets.data(), offsets.size());
        view_.ivf_offsets = upload(d.ivf_offsets, d.num_centroids + 1);
        view_.ivf_postings = upload(d.ivf_postings, view_.P);
        const std::vector<uint8_t> mult = posting_multiplicity(d, offsets);
        view_.ivf_mult = upload(mult.data(), mult.size());
        if (d.dim == 128 && d.num_embeddings) {
            // per-token 1/||v|| for the tensor-core stage 4 (TENSOR mode)
            float* inv = upload<float>(nullptr, d.num_embeddings);
            launch::token_inv_norms(view_, inv, 0);
            PLAID_CUDA(cudaStreamSynchronize(0));
            PLAID_CUDA(cudaGetLastError());
            view_.tok_inv = inv;
        }
        build_range_table(0);
    } catch (...) {
        for (void* p : allocs_) cudaFree(p);
        allocs_.clear();
        throw;
    }
}

void DeviceIndex::set_list_bounds(const uint64_t* ivo) {
    const uint64_t K = view_.K;
    std::vector<uint64_t> len(K);
    for (uint64_t c = 0; c < K; ++c) len[c] = ivo[c + 1] - ivo[c];
    std::sort(len.begin(), len.end(), std::greater<uint64_t>());
    longest_prefix_.assign(K + 1, 0);
    for (uint64_t j = 0; j < K; ++j) longest_prefix_[j + 1] = longest_prefix_[j] + len[j];
}

uint64_t DeviceIndex::candidate_bound(uint64_t nprobe) const {
    const uint64_t N = view_.N, K = view_.K;
    if (longest_prefix_.size() != K + 1) return N;
    const uint64_t lists = nprobe >= K / 32 ? K : 32 * nprobe;
    return std::min<uint64_t>(N, longest_prefix_[std::min<uint64_t>(lists, K)]);
}

void DeviceIndex::validate_device() {
    DeviceGuard g(device_);
    const IndexView& v = view_;
    std::vector<float> C(v.K * v.dim);
    std::vector<uint32_t> codes(v.T), post(v.P);
    std::vector<uint8_t> res(v.T * (uint64_t(v.nbits) * v.dim / 8));
    std::vector<uint64_t> ivo(v.K + 1);
    PLAID_CUDA(cudaMemcpy(C.data(), v.centroids, C.size() * 4, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(codes.data(), v.codes, codes.size() * 4, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(post.data(), v.ivf_postings, post.size() * 4, cudaMemcpyDeviceToHost));
    PLAID_CUDA(cudaMemcpy(ivo.data(), v.ivf_offsets, ivo.size() * 8, cudaMemcpyDeviceToHost));
    plaid_index_desc d{};
    d.dim = v.dim;
    d.nbits = v.nbits;
    d.num_centroids = v.K;
    d.num_passages = v.N;
    d.num_embeddings = v.T;
    d.centroids = C.data();
    d.codes = codes.data();
    d.residuals = res.data();
    d.doclens = h_doclens_.data();
    d.ivf_offsets = ivo.data();
    d.ivf_postings = post.data();
    d.bucket_cutoffs = cutoffs_;
    d.bucket_weights = v.weights;
    validate_index_host(d);
}

DeviceIndex::~DeviceIndex() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    for (void* p : allocs_) cudaFree(p);
    cudaSetDevice(prev);
}

// ---------------------------------------------------------------- Searcher
Searcher::Searcher(DeviceIndex* index, int device, const plaid_searcher_config& cfg)
    : index_(index), device_(index ? index->device() : device), cfg_(cfg) {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    for (auto& e : ev_) PLAID_CUDA(cudaEventCreate(&e));
    const uint64_t words = index_ ? (index_->view().N + 31) / 32 : 0;
    // [candidate bitmap | used bitmap | per-chunk compaction status (u64) +
    // the compaction's ticket counter], whole 16-byte units, cleared per
    // query by the prologue kernel
    const uint64_t chunks = index_ ? launch::bitmap_chunks(index_->view().N) : 1;
    const uint64_t bm_words = (2 * words + 3) / 4 * 4;
    zero_.ensure(bm_words + (2 * (chunks + 1) + 3) / 4 * 4);
    PLAID_CUDA(cudaMemset(zero_.p, 0, zero_.n * sizeof(uint32_t)));
    bitmap_.p = zero_.p;
    compact_status_ = reinterpret_cast<unsigned long long*>(zero_.p + bm_words);
    ensure_result_block(1);
    kconst_.ensure(1);
    status_.ensure(1);
    PLAID_CUDA(cudaMemset(status_.p, 0, sizeof(int)));
    sel_state_.ensure(1);
    PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_q_), 32 * 256 * sizeof(float)));
    PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_flag_), 64));
    *h_flag_ = 0;
    pub_seq_.ensure(1);
    PLAID_CUDA(cudaMemset(pub_seq_.p, 0, sizeof(uint32_t)));
    q_.ensure(32 * 256);
    if (index_) {
        const IndexView& ix = index_->view();
        scores_.ensure(ix.K * kScoresPitch);
        rowmax_.ensure(ix.K);
        keep_.ensure((ix.K + 31) / 32);
        npartial_warps_ = std::max(launch::scores_max_warps(), launch::scores_tensor_max_warps());
        partial_.ensure(npartial_warps_ * 32 * 32);
        chunk_counts_.ensure(launch::bitmap_chunks(ix.N));
        c1_.ensure(ix.N);
        slot_of_.ensure(ix.N);
        bkeys_.ensure(ix.N);
        sel_hist_.ensure(1);
        PLAID_CUDA(cudaMemset(sel_hist_.p, 0, sizeof(SelectHist)));  // re-zeroed by every select after
        kept_list_.ensure(ix.K);
        keys2_.ensure(ix.N);
        ukeys_.ensure(ix.N);
        keys4_.ensure(ix.N);
        const uint64_t K = ix.K;
        PLAID_CUDA(cudaMemcpy(kconst_.p, &K, sizeof K, cudaMemcpyHostToDevice));
        tensor_ = cfg_.score_mode == PLAID_SCORES_TENSOR && launch::tensor_scores_supported(ix);
        if (tensor_) launch::make_centroid_tensor_map(ix, tmap_);
        if (tensor_ && ix.tok_inv) qimg_.ensure((launch::kQImgBytes + launch::kQFragImgBytes) / 4);
    }
    // the zero fills above run on the legacy default stream, which does not
    // order the searcher's non-blocking streams: finish them before any search
    PLAID_CUDA(cudaDeviceSynchronize());
}

uint32_t Searcher::launch_scores(const float* d_q, uint32_t rows, float t_cs, uint32_t npb, cudaStream_t st) {
    const IndexView& ix = index_->view();
    if (tensor_)
        return launch::scores_tensor(tmap_, ix, d_q, rows, t_cs, scores_.p, keep_.p, partial_.p, npb,
                                     reinterpret_cast<uint32_t*>(counters_.p + kGthr), st);
    return launch::scores_exact(ix, d_q, rows, t_cs, scores_.p, rowmax_.p, keep_.p, partial_.p, npb, st);
}

Searcher::~Searcher() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& e : graphs_) cudaGraphExecDestroy(e.exec);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (h_q_) cudaFreeHost(h_q_);
    if (h_res_) cudaFreeHost(h_res_);
    if (h_flag_) cudaFreeHost(h_flag_);
    if (stream_) cudaStreamDestroy(stream_);
    cudaSetDevice(prev);
}

void Searcher::require_index() const {
    if (!index_) fail(PLAID_INVALID_PARAMS, "searcher has no index");
}

void Searcher::ensure_param_buffers(const plaid_params& p) {
    // buffers that grow here are zero-filled on the legacy default stream
    // (cudaMemset), which does NOT order the non-blocking stream the search
    // runs on: wait for the fills before enqueueing (growth is rare)
    const uint64_t gen0 = g_alloc_generation.load();
    ensure_param_buffers_impl(p);
    if (g_alloc_generation.load() != gen0) PLAID_CUDA(cudaDeviceSynchronize());
}

void Searcher::ensure_param_buffers_impl(const plaid_params& p) {
    // first: the result block holds the counters, and pointers into it are
    // cached below (rank_scratch_.tokens) — growing it later would leave them
    // pointing at the freed block
    ensure_result_block(p.k);
    const IndexView& ix = index_->view();
    const uint64_t K = ix.K, N = ix.N;
    const uint64_t nsel = p.nprobe == K ? K : 32 * std::max<uint64_t>(p.nprobe, 32);
    sel_.ensure(nsel);
    if (p.nprobe > 32 && p.nprobe < K) tok_keys_.ensure(K);
    const uint64_t nd = std::min<uint64_t>(p.ndocs, N);
    const uint64_t n3 = std::min<uint64_t>(stage3_width(p), N);
    // stage-2 accumulators: [slot of a candidate][query token], slots < |C1|;
    // every consumer re-zeroes the slots it read, so only growth is filled
    const uint64_t n1cap = index_->candidate_bound(p.nprobe);
    if (acc2_.n < n1cap * 32) {
        acc2_.ensure(n1cap * 32);
        PLAID_CUDA(cudaMemset(acc2_.p, 0, acc2_.n * sizeof(uint32_t)));
    }
    sel2_.ensure(nd);
    keys3_.ensure(nd);
    if (nd <= launch::kSmallSortMax) cand_len_.ensure(nd), cand_off_.ensure(nd);
    sel3_.ensure(n3);
    if (ix.dim == 128 && n3 <= launch::kStreamMaxPassages) {
        pref_.ensure(n3 + 1);
        if (run_.n < n3 * 32) {
            run_.ensure(n3 * 32);
            PLAID_CUDA(cudaMemset(run_.p, 0, run_.n * sizeof(uint32_t)));
        }
        fin_base_.ensure(n3);
        rank_scratch_.pref = pref_.p;
        rank_scratch_.run = run_.p;
        rank_scratch_.tensor_S = tensor_ && ix.tok_inv ? scores_.p : nullptr;
        rank_scratch_.fin_base = fin_base_.p;
        rank_scratch_.tokens = counters_.p + kT4;
        rank_scratch_.pass_cap =
            std::min<uint64_t>({pref_.n - 1, run_.n / 32, fin_base_.n, launch::kStreamMaxPassages});
        if (rank_scratch_.tensor_S) {
            run_p0_.ensure((rank_scratch_.pass_cap * ix.max_doclen + 31) / 32 + 1);
            rank_scratch_.run_p0 = run_p0_.p;
            rank_scratch_.qimg = qimg_.p;
        }
    }
    tmp_keys_.ensure(std::max<uint64_t>(std::min<uint64_t>(p.k, N), std::min<uint64_t>(p.nprobe, K)));
    uint64_t tmp = 0;
    tmp = std::max(tmp, launch::sort_tmp_capacity(nd));
    tmp = std::max(tmp, launch::sort_tmp_capacity(std::min<uint64_t>(p.k, N)));
    tmp = std::max(tmp, launch::sort_tmp_capacity(n3));
    if (tmp) sort_tmp_.ensure(tmp);
}

// res_ = [32 u64 counters | k u32 pids | k f32 scores] (16-byte aligned
// parts): the host path reads counters and results back with ONE copy.
void Searcher::ensure_result_block(uint64_t k) {
    const uint64_t kk = (std::max<uint64_t>(k, 1) + 3) / 4 * 4;
    if (res_.p && res_k_ >= kk) return;
    res_.ensure(2 * kNumCounters + 2 * kk);
    PLAID_CUDA(cudaMemset(res_.p, 0, res_.n * sizeof(uint32_t)));
    res_k_ = kk;
    counters_.p = reinterpret_cast<uint64_t*>(res_.p);
    out_pids_p_ = res_.p + 2 * kNumCounters;
    out_scores_p_ = reinterpret_cast<float*>(res_.p + 2 * kNumCounters + kk);
    if (h_res_) cudaFreeHost(h_res_);
    h_res_ = nullptr;
    PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_res_), (res_.n + 3) / 4 * 4 * sizeof(uint32_t)));
}

void Searcher::record(int slot, cudaStream_t st, bool times) {
    if (times) PLAID_CUDA(cudaEventRecord(ev_[slot], st));
}

// The four stages of lir::search (pipeline.cpp:232-283) as one launch sequence.
void Searcher::enqueue(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t* d_pids,
                       float* d_scores, uint64_t* d_n, cudaStream_t st, bool times, bool validate) {
    pending_rows_ = rows;
    enqueue_front(d_q, rows, p, st, times, validate);
    enqueue_stage3(p, st, times, true);
    enqueue_back(d_q, rows, p, d_pids, d_scores, d_n, st, times);
}

// Stage 1 (S_cq, candidates) and stage 2 (pruned interaction + top-ndocs
// select): survivors in sel2_ (keys, count counters[kN2]).
void Searcher::enqueue_front(const float* d_q, uint32_t rows, const plaid_params& p, cudaStream_t st,
                             bool times, bool validate) {
    const IndexView& ix = index_->view();
    const uint64_t K = ix.K, N = ix.N;
    uint64_t* c = counters_.p;
    uint32_t* bitmap = bitmap_.p;
    uint32_t* owners = bitmap_.p + (N + 31) / 32;
    // one PDL-chained prologue kernel validates the query rows on the device
    // (device-resident queries) and clears the per-query counters, the
    // candidate bitmap and the stage-2 used bitmap (contiguous in zero_); the
    // "scores" phase then brackets the S_cq kernel alone
    // host path: the prologue also copies Q from the pinned staging buffer
    const float* qsrc = host_q_ ? host_q_ : d_q;
    // the range path reads neither bitmap: only the counters are cleared
    launch::query_prologue(validate ? d_q : nullptr, rows, ix.dim, status_.p, zero_.p,
                           range_path(rows, p) ? 0 : zero_.n, res_.p,
                           2 * kNumCounters, st, qsrc, rank_scratch_.qimg ? qimg_.p : nullptr,
                           host_q_ ? const_cast<float*>(d_q) : nullptr);
    record(0, st, times);

    // Stage 1: S_cq (+ row max, keep bits, per-warp top-nprobe), candidates.
    const uint32_t npb = p.nprobe <= 32 ? np_bucket(p.nprobe) : 1;
    const uint32_t warps = launch_scores(d_q, rows, p.t_cs, npb, st);
    record(1, st, times);
    front_after_scores(rows, p, warps, st, times);
}

bool Searcher::final_fused_ok(uint32_t rows, const plaid_params& p) const {
    const IndexView& ix = index_->view();
    if (p.disable_filter || !rank_scratch_.run || ix.dim != 128 || rows > 32) return false;
    const uint64_t fin_max = std::min<uint64_t>(stage3_width(p), ix.N);
    return fin_max >= launch::kFinalRankMin && fin_max <= launch::kSmallSortMax &&
           launch::rank_stream128_ok(ix, rows, fin_max, rank_scratch_);
}

bool Searcher::range_path(uint32_t rows, const plaid_params& p) const {
    static const bool off = getenv("PLAID_NO_RANGE_STAGE2") != nullptr;
    const IndexView& ix = index_->view();
    return !off && p.nprobe != ix.K && p.nprobe <= 8 && !p.disable_filter &&
           launch::range_stage2_ok(ix, rows, uint64_t(rows) * p.nprobe);
}

// Stage 1 after S_cq (top-nprobe merge, candidate generation) and stage 2.
void Searcher::front_after_scores(uint32_t rows, const plaid_params& p, uint32_t warps, cudaStream_t st,
                                  bool times) {
    const IndexView& ix = index_->view();
    const uint64_t K = ix.K, N = ix.N;
    uint64_t* c = counters_.p;
    uint32_t* bitmap = bitmap_.p;
    uint32_t* owners = bitmap_.p + (N + 31) / 32;
    const uint32_t npb = p.nprobe <= 32 ? np_bucket(p.nprobe) : 1;
    uint64_t nsel;
    bool bitmap_done = false, kept_ready = false;
    if (p.nprobe == K) {
        launch::iota(sel_.p, K, st);
        nsel = K;
    } else if (range_path(rows, p)) {
        // candidates + stage 2 in one launch, a CTA per pid range
        // (range_stage2.cu): topn_postings only merges the top-nprobe lists
        // and builds the kept list; no bitmap, no compaction, no slot map
        launch::KeepListArgs kl{keep_.p, kept_list_.p, reinterpret_cast<unsigned long long*>(c + kKeptN)};
        launch::topn_postings(partial_.p, warps, npb, rows, uint32_t(p.nprobe), ix, sel_.p, nullptr, &kl, st);
        record(2, st, times);
        launch::range_stage2(ix, scores_.p, rows, sel_.p, rows * uint32_t(p.nprobe), keep_.p, kept_list_.p,
                             reinterpret_cast<unsigned long long*>(c + kKeptN), keys2_.p, c + kN1,
                             reinterpret_cast<unsigned long long*>(c + kRows2), sel_hist_.p, ukeys_.p, c + kUsedN,
                             st);
        record(3, st, times);
        launch::select_top_hist(keys2_.p, c + kN1, N, p.ndocs, sel_hist_.p, bkeys_.p, sel2_.p, c + kN2, st,
                                ukeys_.p, c + kUsedN);
        record(4, st, times);
        return;
    } else if (p.nprobe <= 32) {
        // the kept-centroid list rides in the same launch unless stage 2 is skipped
        launch::KeepListArgs kl{keep_.p, kept_list_.p, reinterpret_cast<unsigned long long*>(c + kKeptN)};
        kept_ready = !p.disable_filter;
        launch::topn_postings(partial_.p, warps, npb, rows, uint32_t(p.nprobe), ix, sel_.p, bitmap,
                              kept_ready ? &kl : nullptr, st);
        nsel = uint64_t(rows) * p.nprobe;
        bitmap_done = true;
    } else {
        for (uint32_t i = 0; i < rows; ++i) {
            launch::token_keys(scores_.p, K, i, tok_keys_.p, st);
            launch::select_top_large(tok_keys_.p, kconst_.p, K, p.nprobe, sel_state_.p,
                                     tmp_keys_.p, c + kTmpN, st);
            launch::keys_to_ids(tmp_keys_.p, c + kTmpN, p.nprobe, sel_.p + uint64_t(i) * p.nprobe, st);
        }
        nsel = uint64_t(rows) * p.nprobe;
    }
    if (!bitmap_done) launch::postings_to_bitmap(ix, sel_.p, uint32_t(nsel), bitmap, st);
    launch::bitmap_compact_1pass(bitmap, N, compact_status_, c1_.p, c + kN1, slot_of_.p, st);
    record(2, st, times);
    if (p.disable_filter) {
        record(3, st, times);
        record(4, st, times);
        return;
    }
    // Stage 2: pruned centroid interaction over C1, keep ndocs.  Only the
    // candidates owning a kept token are read (see kept_owners).
    launch::stage2_masked(ix, scores_.p, rows, c1_.p, c + kN1, N, keep_.p, bitmap, owners, kept_list_.p,
                          slot_of_.p, acc2_.p, reinterpret_cast<unsigned long long*>(c + kKeptN), keys2_.p,
                          reinterpret_cast<unsigned long long*>(c + kRows2), sel_hist_.p, kept_ready, st);
    record(3, st, times);
    launch::select_top_hist(keys2_.p, c + kN1, N, p.ndocs, sel_hist_.p, bkeys_.p, sel2_.p, c + kN2, st);
    record(4, st, times);
}

// Stage 3: full centroid interaction over sel2_, keep max(ceil(ndocs/4), k)
// into sel3_ (sorted, count counters[kN3]).
void Searcher::enqueue_stage3(const plaid_params& p, cudaStream_t st, bool times, bool fuse_scan) {
    scan_fused_ = false;
    if (p.disable_filter) {
        record(5, st, times);
        return;
    }
    const IndexView& ix = index_->view();
    uint64_t* c = counters_.p;
    const uint64_t nd = std::min<uint64_t>(p.ndocs, ix.N);
    // stage 4 needs only the top-stage3_width SET (the final select orders it)
    // unsharded, stage 4's finalist scan runs in the select's own CTA, on the
    // (doclen, offset) pairs the stage-3 scorer carries over
    const uint64_t fin_max = std::min<uint64_t>(stage3_width(p), ix.N);
    scan_fused_ = fuse_scan && nd <= launch::kSmallSortMax && rank_scratch_.pref &&
                  launch::rank_stream128_ok(ix, pending_rows_, fin_max, rank_scratch_);
    const bool carry = scan_fused_ && cand_len_.n >= nd && cand_off_.n >= nd;
    launch::centroid_interaction(ix, scores_.p, pending_rows_, nullptr, sel2_.p, c + kN2, nd, nullptr, nullptr,
                                 keys3_.p, nullptr, reinterpret_cast<unsigned long long*>(c + kRows3), st,
                                 carry ? cand_len_.p : nullptr, carry ? cand_off_.p : nullptr);
    launch::FinalistScanArgs fs{ix.doclens, ix.offsets, rank_scratch_.pref, rank_scratch_.fin_base,
                                rank_scratch_.tokens, rank_scratch_.run_p0,
                                carry ? cand_len_.p : nullptr, carry ? cand_off_.p : nullptr};
    if (nd <= launch::kSmallSortMax)
        launch::select_set(keys3_.p, c + kN2, nd, stage3_width(p), sel3_.p, c + kN3, scan_fused_ ? &fs : nullptr, st);
    else
        launch::sort_top(keys3_.p, c + kN2, nd, stage3_width(p), sel3_.p, nullptr, nullptr, c + kN3, 0,
                         sort_tmp_.p, st);
    record(5, st, times);
}

// Stage 4: decompress + exact MaxSim of the finalists, top-k (global ids).
void Searcher::enqueue_back(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t* d_pids,
                            float* d_scores, uint64_t* d_n, cudaStream_t st, bool times) {
    const IndexView& ix = index_->view();
    uint64_t* c = counters_.p;
    const uint64_t want_final = p.k;
    const uint64_t* fin_keys = nullptr;
    const uint32_t* fin_ids = nullptr;
    const uint64_t* fin_n = nullptr;
    uint64_t fin_max = 0;
    if (p.disable_filter) {
        // pipeline.cpp:255-258: every stage-1 candidate goes to stage 4
        fin_ids = c1_.p;
        fin_n = c + kN1;
        fin_max = ix.N;
    } else {
        fin_keys = sel3_.p;
        fin_n = c + kN3;
        fin_max = std::min<uint64_t>(stage3_width(p), ix.N);
    }
    rank_scratch_.prescanned = scan_fused_ && !p.disable_filter;
    const uint32_t base = uint32_t(index_->pid_base());
    // finalize + top-k in one launch (the ticket slot was cleared by this query's prologue)
    const launch::RankScratch::Final fin{want_final, d_pids, d_scores, d_n, base,
                                         reinterpret_cast<unsigned int*>(c + kFinTicket)};
    static const bool s4_tiles = getenv("PLAID_S4_TILES") != nullptr;  // stage4_tensor_kernel instead
    rank_scratch_.warp_s4 = !s4_tiles && rank_scratch_.tensor_S != nullptr;
    const bool fused_final = !rank_scratch_.warp_s4 && final_fused_ok(rows, p);
    rank_scratch_.final_out = fused_final ? &fin : nullptr;
    launch::rank_exact(ix, d_q, rows, fin_ids, fin_keys, fin_n, fin_max, keys4_.p, &rank_scratch_, st);
    rank_scratch_.prescanned = scan_fused_ = false;
    rank_scratch_.final_out = nullptr;
    rank_scratch_.warp_s4 = false;
    record(6, st, times);
    if (fused_final) {
        record(7, st, times);
        return;
    }
    if (fin_max <= launch::kSmallSortMax) {
        launch::sort_top(keys4_.p, fin_n, fin_max, want_final, nullptr, d_pids, d_scores, d_n, base,
                         sort_tmp_.p, st);
    } else {
        launch::select_top_large(keys4_.p, fin_n, fin_max, want_final, sel_state_.p, tmp_keys_.p,
                                 c + kTmpN, st);
        const uint64_t m = std::min<uint64_t>(want_final, fin_max);
        launch::sort_top(tmp_keys_.p, c + kTmpN, m, want_final, nullptr, d_pids, d_scores, d_n, base,
                         sort_tmp_.p, st);
    }
    record(7, st, times);
}

// ---- global-exact passage sharding -------------------------------------
// Three device phases; between them the caller all-gathers the exported key
// rows of every shard (zero-padded to a common stride).  The survivors of
// each threshold filter are exactly this shard's members of the reference's
// single-index stage-2 / stage-3 selections, so the merged top-k — and the
// summed trace counters — equal lir::search over the unsharded index.
void Searcher::shard_phase1(const float* d_q, uint64_t rows, uint64_t dim, const plaid_params& p, uint64_t* d_x2,
                            uint64_t stride2, cudaStream_t st) {
    require_index();
    const IndexView& ix = index_->view();
    if (dim != ix.dim) fail(PLAID_DIMENSION_MISMATCH, "query dim does not match index dim");
    if (rows == 0) fail(PLAID_INVALID_PARAMS, "query must contain at least one token");
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    validate_params_host(p, ix.K);
    if (!p.disable_filter && stride2 < std::min<uint64_t>(p.ndocs, ix.N))
        fail(PLAID_INVALID_PARAMS, "exchange stride below this shard's stage-2 width");
    DeviceGuard g(device_);
    ensure_param_buffers(p);
    if (!st) st = stream_;
    launch::reset_launches();
    const uint64_t l0 = launch::launches();
    pending_ = p;
    pending_q_ = d_q;
    pending_rows_ = uint32_t(rows);
    pending_stride2_ = stride2;
    pending_stride3_ = 0;
    phase_ = 1;
    const bool times = cfg_.record_times != 0;
    enqueue_front(d_q, uint32_t(rows), p, st, times, true);
    if (!p.disable_filter)
        launch::export_keys(sel2_.p, counters_.p + kN2, stride2, uint32_t(index_->pid_base()), d_x2, st);
    PLAID_CUDA(cudaGetLastError());
    phase_launches_ = launch::launches() - l0;
}

void Searcher::shard_phase2(const uint64_t* d_g2, uint64_t shards, uint64_t* d_x3, uint64_t stride3,
                            cudaStream_t st) {
    if (phase_ != 1) fail(PLAID_INVALID_PARAMS, "shard_phase2 without a preceding shard_phase1");
    const plaid_params& p = pending_;
    if (!p.disable_filter && stride3 < std::min<uint64_t>(stage3_width(p), index_->view().N))
        fail(PLAID_INVALID_PARAMS, "exchange stride below this shard's stage-3 width");
    DeviceGuard g(device_);
    if (!st) st = stream_;
    const bool times = cfg_.record_times != 0;
    const uint32_t base = uint32_t(index_->pid_base());
    const uint64_t l0 = launch::launches();
    if (!p.disable_filter) {
        launch::threshold_filter(d_g2, shards * pending_stride2_, p.ndocs, sel2_.p, counters_.p + kN2, base, st);
        enqueue_stage3(p, st, times, false);
        launch::export_keys(sel3_.p, counters_.p + kN3, stride3, base, d_x3, st);
    }
    pending_stride3_ = stride3;
    phase_ = 2;
    PLAID_CUDA(cudaGetLastError());
    phase_launches_ += launch::launches() - l0;
}

void Searcher::shard_phase3(const uint64_t* d_g3, uint64_t shards, uint32_t* d_pids, float* d_scores,
                            uint64_t* d_n, cudaStream_t st) {
    if (phase_ != 2) fail(PLAID_INVALID_PARAMS, "shard_phase3 without a preceding shard_phase2");
    const plaid_params& p = pending_;
    DeviceGuard g(device_);
    if (!st) st = stream_;
    const bool times = cfg_.record_times != 0;
    const uint64_t l0 = launch::launches();
    if (!p.disable_filter)
        launch::threshold_filter(d_g3, shards * pending_stride3_, stage3_width(p), sel3_.p, counters_.p + kN3,
                                 uint32_t(index_->pid_base()), st);
    enqueue_back(pending_q_, pending_rows_, p, d_pids, d_scores, d_n, st, times);
    phase_ = 0;
    PLAID_CUDA(cudaGetLastError());
    last_launches_ = phase_launches_ + (launch::launches() - l0);
}

// ---- batched S_cq (BatchSearcher): the query's prologue on this lane's
// stream, then the shared S_cq launch writes this lane's S / keep bits /
// partial lists / bounds, then the rest of the pipeline.
bool Searcher::batch_scores_ok(const plaid_params& p, uint64_t rows, uint64_t dim) const {
    const IndexView& ix = index_->view();
    return tensor_ && dim == ix.dim && rows <= 32 && p.nprobe < ix.K && p.nprobe <= 8;
}

void Searcher::batch_prepare(const float* d_q, uint64_t rows, uint64_t dim, const plaid_params& p,
                             cudaStream_t st) {
    require_index();
    const IndexView& ix = index_->view();
    if (dim != ix.dim) fail(PLAID_DIMENSION_MISMATCH, "query dim does not match index dim");
    if (rows == 0) fail(PLAID_INVALID_PARAMS, "query must contain at least one token");
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    validate_params_host(p, ix.K);
    DeviceGuard g(device_);
    ensure_param_buffers(p);
    launch::reset_launches();
    launch::query_prologue(d_q, uint32_t(rows), uint32_t(dim), status_.p, zero_.p, zero_.n, res_.p, 2 * kNumCounters,
                           st, d_q, rank_scratch_.qimg ? qimg_.p : nullptr);
}

void Searcher::batch_targets(TfOut& out, uint32_t qi, const float* d_q) {
    out.Q[qi] = d_q;
    out.S[qi] = scores_.p;
    out.keep[qi] = keep_.p;
    out.partial[qi] = partial_.p;
    out.gthr[qi] = reinterpret_cast<uint32_t*>(counters_.p + kGthr);
}

void Searcher::batch_finish(const float* d_q, uint32_t rows, const plaid_params& p, uint32_t warps, uint32_t* d_pids,
                            float* d_scores, uint64_t* d_n, cudaStream_t st) {
    DeviceGuard g(device_);
    pending_rows_ = rows;
    front_after_scores(rows, p, warps, st, false);
    enqueue_stage3(p, st, false, true);
    enqueue_back(d_q, rows, p, d_pids, d_scores, d_n, st, false);
    PLAID_CUDA(cudaGetLastError());
    last_launches_ = launch::launches();
}

// Trace counters of the last enqueued query, on the device: [stage1_candidates,
// stage2_out, stage3_out, final_out (host path only), stage2_rows_gathered,
// stage3_rows_gathered].
void Searcher::trace_counters_device(uint64_t* d_out, cudaStream_t st) {
    DeviceGuard g(device_);
    if (!st) st = stream_;
    PLAID_CUDA(cudaMemcpyAsync(d_out, counters_.p, 6 * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
}

// Phase durations of the last enqueued query (record_times): K1, candidate
// generation, stage-2 interaction, stage-2 select, stage 3, stage-4 kernel,
// final select.
void Searcher::phase_ms(double* out) {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaEventSynchronize(ev_[7]));
    for (int i = 0; i < 7; ++i) {
        float ms = 0;
        PLAID_CUDA(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
        out[i] = ms;
    }
}

// Spin on the publish kernel's flag (every search publishes exactly once, so
// the host's count is the value to expect); poll the stream now and then so a
// fault surfaces instead of a hang.
void Searcher::wait_published() {
    const unsigned int expect = ++pub_seq_host_;
    volatile unsigned int* flag = h_flag_;
    for (uint64_t spins = 1; *flag != expect; ++spins) {
        if ((spins & 4095) == 0) {
            const cudaError_t e = cudaStreamQuery(stream_);
            if (e == cudaSuccess && *flag != expect) {
                pub_seq_host_ = *flag;  // resynchronise before failing
                fail(PLAID_CUDA_ERROR, "search finished without publishing its results");
            }
            if (e != cudaSuccess && e != cudaErrorNotReady) PLAID_CUDA(e);
        }
    }
}

void Searcher::search(const float* q, uint64_t rows, uint64_t dim, const plaid_params& p,
                      uint32_t* out_pids, float* out_scores, uint64_t* out_n, plaid_trace* trace) {
    require_index();
    *out_n = 0;
    if (trace) std::memset(trace, 0, sizeof *trace);
    const IndexView& ix = index_->view();
    validate_query_host(q, rows, dim, ix.dim);
    validate_params_host(p, ix.K);
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    DeviceGuard g(device_);
    ensure_param_buffers(p);
    launch::reset_launches();
    std::memcpy(h_q_, q, rows * dim * sizeof(float));
    const bool times = trace && cfg_.record_times;
    const uint64_t kk = res_k_;
    const uint64_t words = 2 * kNumCounters + kk + p.k;
    // the launch sequence with Q read from the pinned staging buffer by the
    // prologue and [counters | pids | scores] written to pinned memory by a
    // final publish kernel, which then raises a flag the host spins on: no
    // copy-engine round trips and no stream-synchronize wake-up on the path
    const uint64_t pub_words = (words + 3) / 4 * 4;
    auto body = [&] {
        host_q_ = h_q_;
        try {
            enqueue(q_.p, uint32_t(rows), p, out_pids_p_, out_scores_p_, counters_.p + kNOut, stream_, times, false);
        } catch (...) {
            host_q_ = nullptr;
            throw;
        }
        host_q_ = nullptr;
        launch::publish(res_.p, h_res_, pub_words, pub_seq_.p, h_flag_, stream_);
    };
    if (cfg_.use_graphs && !times) {
        // one CUDA graph per (rows, params): captured on first use, replayed
        // after; every buffer it touches is owned by this searcher, and any
        // reallocation (g_alloc_generation) makes the cached graphs stale
        GraphKey key{rows, p.k, p.nprobe, p.ndocs, p.disable_filter, 0};
        std::memcpy(&key.t_cs_bits, &p.t_cs, 4);
        const uint64_t gen = g_alloc_generation.load();
        GraphEntry* hit = nullptr;
        for (auto& e : graphs_)
            if (e.key == key) hit = &e;
        if (hit && hit->gen != gen) {
            cudaGraphExecDestroy(hit->exec);
            *hit = graphs_.back();
            graphs_.pop_back();
            hit = nullptr;
        }
        if (!hit) {
            cudaGraph_t graph = nullptr;
            PLAID_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            try {
                body();
            } catch (...) {
                cudaStreamEndCapture(stream_, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            PLAID_CUDA(cudaStreamEndCapture(stream_, &graph));
            GraphEntry e{key, gen, nullptr, launch::launches()};
            const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
            cudaGraphDestroy(graph);
            PLAID_CUDA(ie);
            graphs_.push_back(e);
            hit = &graphs_.back();
        }
        PLAID_CUDA(cudaGraphLaunch(hit->exec, stream_));
        last_launches_ = hit->launches;
    } else {
        body();
        last_launches_ = launch::launches();
    }
    wait_published();
    PLAID_CUDA(cudaGetLastError());
    const uint64_t* h_counters_ = reinterpret_cast<const uint64_t*>(h_res_);
    const uint64_t n = h_counters_[kNOut];
    *out_n = n;
    std::memcpy(out_pids, h_res_ + 2 * kNumCounters, n * sizeof(uint32_t));
    std::memcpy(out_scores, h_res_ + 2 * kNumCounters + kk, n * sizeof(float));
    if (trace) {
        trace->stage1_candidates = h_counters_[kN1];
        trace->centroid_matmul_count = 1;
        if (h_counters_[kN1] > 0) {  // pipeline.cpp:249-252: empty C1 returns early
            const bool df = p.disable_filter != 0;  // pipeline.cpp:255-258
            trace->stage2_out = df ? h_counters_[kN1] : h_counters_[kN2];
            trace->stage3_out = df ? h_counters_[kN1] : h_counters_[kN3];
            trace->final_out = n;
            trace->stage2_rows_gathered = h_counters_[kRows2];
            trace->stage3_rows_gathered = h_counters_[kRows3];
            trace->decompressed_passages = trace->stage3_out;
            trace->decompressed_tokens = h_counters_[kT4];
        }
        if (times) {
            double ms[7];
            phase_ms(ms);
            trace->candidate_generation_ms = ms[0] + ms[1];
            trace->stage2_ms = ms[2] + ms[3];
            trace->stage3_ms = ms[4];
            trace->lookup_ms = 0.0;  // fused into the stage-4 kernel
            trace->decompression_ms = ms[5];  // fused decompress + MaxSim kernel
            trace->scoring_ms = ms[6];        // final top-k select
            trace->total_ms = ms[0] + ms[1] + ms[2] + ms[3] + ms[4] + ms[5] + ms[6];
        }
    }
}

void Searcher::search_device(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim,
                             const plaid_params& p, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                             cudaStream_t st) {
    require_index();
    const IndexView& ix = index_->view();
    if (dim != ix.dim) fail(PLAID_DIMENSION_MISMATCH, "query dim does not match index dim");
    if (rows == 0) fail(PLAID_INVALID_PARAMS, "query must contain at least one token");
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    validate_params_host(p, ix.K);
    DeviceGuard g(device_);
    ensure_param_buffers(p);
    if (!st) st = stream_;
    launch::reset_launches();
    for (uint64_t j = 0; j < nq; ++j) {
        const float* q = d_q + j * rows * dim;
        enqueue(q, uint32_t(rows), p, d_pids + j * p.k, d_scores + j * p.k, d_n + j, st,
                cfg_.record_times != 0, true);
    }
    PLAID_CUDA(cudaGetLastError());
    last_launches_ = launch::launches();
}

void Searcher::sync() {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    PLAID_CUDA(cudaDeviceSynchronize());
    int status = 0;
    PLAID_CUDA(cudaMemcpy(&status, status_.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (status) {
        PLAID_CUDA(cudaMemset(status_.p, 0, sizeof(int)));
        PLAID_CUDA(cudaDeviceSynchronize());
        fail(status, "device-side query validation failed (row not unit norm)");
    }
}

// ---------------------------------------------------------------- entry points
namespace {
template <typename T>
void h2d(T* dst, const T* src, uint64_t n, cudaStream_t st) {
    if (n) PLAID_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}
template <typename T>
void d2h(T* dst, const T* src, uint64_t n, cudaStream_t st) {
    if (n) PLAID_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}
}  // namespace

void Searcher::compute_centroid_scores(const float* q, uint64_t rows, uint64_t dim, float* scores,
                                       float* row_max) {
    require_index();
    const IndexView& ix = index_->view();
    if (dim != ix.dim) fail(PLAID_DIMENSION_MISMATCH, "query dim does not match centroid dim");
    if (rows == 0 || rows > 32) fail(PLAID_UNSUPPORTED, "engine supports 1 <= |Q| <= 32");
    DeviceGuard g(device_);
    h2d(q_.p, q, rows * dim, stream_);
    PLAID_CUDA(cudaMemsetAsync(counters_.p + kGthr, 0, 16 * sizeof(uint64_t), stream_));
    launch_scores(q_.p, uint32_t(rows), INFINITY, 1, stream_);
    std::vector<float> S(ix.K * kScoresPitch);
    d2h(S.data(), scores_.p, S.size(), stream_);
    if (!tensor_) d2h(row_max, rowmax_.p, ix.K, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    for (uint64_t c = 0; c < ix.K; ++c) {
        std::memcpy(scores + c * rows, S.data() + c * kScoresPitch, rows * sizeof(float));
        if (tensor_) {  // the tensor kernel emits keep bits, not row maxima (pipeline.cpp:40-46)
            float m = -INFINITY;
            for (uint64_t i = 0; i < rows; ++i)
                if (S[c * kScoresPitch + i] > m) m = S[c * kScoresPitch + i];
            row_max[c] = m;
        }
    }
}

void Searcher::generate_candidates(const float* scores, uint64_t rows, uint64_t nprobe,
                                   uint32_t* out_ids, uint64_t* out_n) {
    require_index();
    const IndexView& ix = index_->view();
    *out_n = 0;
    if (nprobe < 1 || nprobe > ix.K) fail(PLAID_INVALID_PARAMS, "nprobe outside [1, K]");
    if (rows == 0 || rows > 32) fail(PLAID_UNSUPPORTED, "engine supports 1 <= |Q| <= 32");
    DeviceGuard g(device_);
    plaid_params p{};
    p.k = 1;
    p.nprobe = nprobe;
    p.ndocs = 1;
    ensure_param_buffers(p);
    std::vector<float> S(ix.K * kScoresPitch, 0.0f);
    for (uint64_t c = 0; c < ix.K; ++c) std::memcpy(S.data() + c * kScoresPitch, scores + c * rows, rows * 4);
    h2d(scores_.p, S.data(), S.size(), stream_);
    uint64_t* c = counters_.p;
    PLAID_CUDA(cudaMemsetAsync(bitmap_.p, 0, ((ix.N + 31) / 32) * sizeof(uint32_t), stream_));
    uint64_t nsel;
    if (nprobe == ix.K) {
        launch::iota(sel_.p, ix.K, stream_);
        nsel = ix.K;
    } else if (nprobe <= 32) {
        const uint32_t npb = np_bucket(nprobe);
        PLAID_CUDA(cudaMemsetAsync(counters_.p + kGthr, 0, 16 * sizeof(uint64_t), stream_));
        const uint32_t w = launch::topn_from_scores(scores_.p, ix.K, uint32_t(rows), partial_.p, npb,
                                                    reinterpret_cast<uint32_t*>(counters_.p + kGthr), stream_);
        launch::topn_merge(partial_.p, w, npb, uint32_t(rows), uint32_t(nprobe), sel_.p, stream_);
        nsel = rows * nprobe;
    } else {
        for (uint32_t i = 0; i < rows; ++i) {
            launch::token_keys(scores_.p, ix.K, i, tok_keys_.p, stream_);
            launch::select_top_large(tok_keys_.p, kconst_.p, ix.K, nprobe, sel_state_.p, tmp_keys_.p,
                                     c + kTmpN, stream_);
            launch::keys_to_ids(tmp_keys_.p, c + kTmpN, nprobe, sel_.p + uint64_t(i) * nprobe, stream_);
        }
        nsel = rows * nprobe;
    }
    launch::postings_to_bitmap(ix, sel_.p, uint32_t(nsel), bitmap_.p, stream_);
    launch::bitmap_compact(bitmap_.p, ix.N, chunk_counts_.p, c1_.p, c + kN1, nullptr, stream_);
    uint64_t n = 0;
    d2h(&n, c + kN1, 1, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    d2h(out_ids, c1_.p, n, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    *out_n = n;
}

void Searcher::centroid_interaction(const float* scores, uint64_t rows, const uint32_t* cand, uint64_t n,
                                    const uint8_t* mask, float* out_scores, uint64_t* rows_gathered) {
    require_index();
    const IndexView& ix = index_->view();
    if (n == 0) fail(PLAID_INVALID_PARAMS, "centroid interaction requires candidates");
    if (rows == 0 || rows > 32) fail(PLAID_UNSUPPORTED, "engine supports 1 <= |Q| <= 32");
    for (uint64_t i = 0; i < n; ++i)
        if (cand[i] >= ix.N) fail(PLAID_INDEX_OUT_OF_RANGE, "candidate id out of range");
    DeviceGuard g(device_);
    std::vector<float> S(ix.K * kScoresPitch, 0.0f);
    for (uint64_t c = 0; c < ix.K; ++c) std::memcpy(S.data() + c * kScoresPitch, scores + c * rows, rows * 4);
    h2d(scores_.p, S.data(), S.size(), stream_);
    ids_tmp_.ensure(n);
    h2d(ids_tmp_.p, cand, n, stream_);
    if (mask) {
        std::vector<uint32_t> bits((ix.K + 31) / 32, 0);
        for (uint64_t c = 0; c < ix.K; ++c)
            if (mask[c]) bits[c / 32] |= 1u << (c % 32);
        h2d(keep_.p, bits.data(), bits.size(), stream_);
    }
    uint64_t* c = counters_.p;
    PLAID_CUDA(cudaMemcpyAsync(c + kEntryN, &n, sizeof n, cudaMemcpyHostToDevice, stream_));
    PLAID_CUDA(cudaMemsetAsync(c + kRows2, 0, sizeof(uint64_t), stream_));
    DevBuf<uint64_t> keys;
    keys.ensure(n);
    DevBuf<float> sc;
    sc.ensure(n);
    uint32_t* owners = nullptr;
    if (mask) {  // same owner filter as the pipeline's stage 2
        owners = bitmap_.p + (ix.N + 31) / 32;
        PLAID_CUDA(cudaMemsetAsync(owners, 0, ((ix.N + 31) / 32) * sizeof(uint32_t), stream_));
        launch::kept_owners(ix, keep_.p, owners, stream_);
    }
    launch::centroid_interaction(ix, scores_.p, uint32_t(rows), ids_tmp_.p, nullptr, c + kEntryN, n,
                                 mask ? keep_.p : nullptr, owners, keys.p, sc.p,
                                 reinterpret_cast<unsigned long long*>(c + kRows2), stream_);
    d2h(out_scores, sc.p, n, stream_);
    uint64_t rg = 0;
    d2h(&rg, c + kRows2, 1, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    if (rows_gathered) *rows_gathered = rg;
}

void Searcher::select_top(const uint32_t* ids, const float* scores, uint64_t n, uint64_t keep,
                          uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    if (keep < 1) fail(PLAID_INVALID_PARAMS, "selection width must be >= 1");
    *out_n = 0;
    DeviceGuard g(device_);
    DevBuf<uint32_t> dids;
    DevBuf<float> dsc;
    DevBuf<uint64_t> keys, sel, tmp, out_nb;
    dids.ensure(n);
    dsc.ensure(n);
    keys.ensure(n);
    out_nb.ensure(2);
    h2d(dids.p, ids, n, stream_);
    h2d(dsc.p, scores, n, stream_);
    uint64_t* c = counters_.p;
    PLAID_CUDA(cudaMemcpyAsync(c + kEntryN, &n, sizeof n, cudaMemcpyHostToDevice, stream_));
    launch::make_keys(dids.p, dsc.p, n, keys.p, stream_);
    const uint64_t m = std::min(n, keep);
    DevBuf<uint32_t> oid;
    DevBuf<float> osc;
    oid.ensure(m);
    osc.ensure(m);
    if (n <= launch::kSmallSortMax) {
        launch::sort_top(keys.p, c + kEntryN, n, keep, nullptr, oid.p, osc.p, out_nb.p, 0, nullptr, stream_);
    } else {
        sel.ensure(m);
        launch::select_top_large(keys.p, c + kEntryN, n, keep, sel_state_.p, sel.p, out_nb.p + 1, stream_);
        const uint64_t cap = launch::sort_tmp_capacity(m);
        if (cap) tmp.ensure(cap);
        launch::sort_top(sel.p, out_nb.p + 1, m, keep, nullptr, oid.p, osc.p, out_nb.p, 0, tmp.p, stream_);
    }
    uint64_t got = 0;
    d2h(&got, out_nb.p, 1, stream_);
    d2h(out_ids, oid.p, m, stream_);
    d2h(out_scores, osc.p, m, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    *out_n = got;
}

void Searcher::rank_final(const float* q, uint64_t rows, const uint32_t* cand, uint64_t n, uint64_t k,
                          uint32_t* out_ids, float* out_scores, uint64_t* out_n) {
    require_index();
    const IndexView& ix = index_->view();
    *out_n = 0;
    if (n == 0) fail(PLAID_INVALID_PARAMS, "final ranking requires candidates");
    if (rows == 0 || rows > 32) fail(PLAID_UNSUPPORTED, "engine supports 1 <= |Q| <= 32");
    for (uint64_t i = 0; i < n; ++i) {  // maxsim.cpp:18-22 via rank_final's packed offsets
        if (cand[i] >= ix.N) fail(PLAID_INDEX_OUT_OF_RANGE, "candidate id out of range");
        if (index_->host_doclens()[cand[i]] == 0)
            fail(PLAID_EMPTY_PASSAGE_RANGE, "passage " + std::to_string(i) + " has no token rows");
    }
    DeviceGuard g(device_);
    ids_tmp_.ensure(n);
    h2d(q_.p, q, rows * ix.dim, stream_);
    h2d(ids_tmp_.p, cand, n, stream_);
    uint64_t* c = counters_.p;
    PLAID_CUDA(cudaMemcpyAsync(c + kEntryN, &n, sizeof n, cudaMemcpyHostToDevice, stream_));
    DevBuf<uint64_t> keys;
    keys.ensure(n);
    launch::rank_exact(ix, q_.p, uint32_t(rows), ids_tmp_.p, nullptr, c + kEntryN, n, keys.p, nullptr, stream_);
    std::vector<uint64_t> hk(n);
    d2h(hk.data(), keys.p, n, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    PLAID_CUDA(cudaGetLastError());
    std::vector<float> sc(n);
    for (uint64_t i = 0; i < n; ++i) sc[i] = dev::key_score(hk[i]);
    select_top(cand, sc.data(), n, k, out_ids, out_scores, out_n);
}

void Searcher::reconstruct(const uint32_t* codes, uint64_t n, const uint8_t* residuals, float* out) {
    require_index();
    const IndexView& ix = index_->view();
    DeviceGuard g(device_);
    for (uint64_t t = 0; t < n; ++t)
        if (codes[t] >= ix.K) fail(PLAID_INDEX_OUT_OF_RANGE, "code exceeds centroid count");
    const uint64_t bpt = uint64_t(ix.nbits) * ix.dim / 8;
    DevBuf<uint32_t> dc;
    DevBuf<unsigned char> dr;
    DevBuf<float> dout;
    dc.ensure(n);
    dr.ensure(n * bpt);
    dout.ensure(n * ix.dim);
    h2d(dc.p, codes, n, stream_);
    h2d(dr.p, residuals, n * bpt, stream_);
    launch::reconstruct(ix, dc.p, n, dr.p, dout.p, stream_);
    d2h(out, dout.p, n * ix.dim, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
}

void Searcher::unpack(const uint8_t* packed, uint64_t n, uint32_t nbits, uint8_t* out) {
    if (!nbits_supported(nbits)) fail(PLAID_PACKING_UNSUPPORTED, "nbits not in {1,2,4}");
    DeviceGuard g(device_);
    DevBuf<unsigned char> dp, dout;
    dp.ensure(n);
    dout.ensure(n * (8 / nbits));
    h2d(dp.p, packed, n, stream_);
    launch::unpack_via_lut(dp.p, n, nbits, dout.p, stream_);
    d2h(out, dout.p, n * (8 / nbits), stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
}

namespace {
// maxsim.cpp:11-27
void check_offsets_host(const uint64_t* offsets, uint64_t np, uint64_t total_rows) {
    if (offsets[0] != 0) fail(PLAID_INVALID_PARAMS, "offsets must start at 0");
    for (uint64_t p = 0; p < np; ++p) {
        if (offsets[p + 1] < offsets[p]) fail(PLAID_INVALID_PARAMS, "offsets must be monotone");
        if (offsets[p + 1] == offsets[p])
            fail(PLAID_EMPTY_PASSAGE_RANGE, "passage " + std::to_string(p) + " has no token rows");
    }
    if (offsets[np] != total_rows) fail(PLAID_LENGTH_MISMATCH, "last offset does not match row count");
}
}  // namespace

void Searcher::maxsim_packed(const float* scores, uint64_t nq, const uint64_t* offsets, uint64_t np,
                             float* out) {
    if (nq == 0) fail(PLAID_INVALID_PARAMS, "need at least one query token");
    if (nq > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32");
    check_offsets_host(offsets, np, offsets[np]);
    DeviceGuard g(device_);
    const uint64_t T = offsets[np];
    DevBuf<float> ds, dout;
    DevBuf<uint64_t> doff;
    ds.ensure(T * nq);
    doff.ensure(np + 1);
    dout.ensure(np);
    h2d(ds.p, scores, T * nq, stream_);
    h2d(doff.p, offsets, np + 1, stream_);
    launch::maxsim_packed(ds.p, uint32_t(nq), doff.p, np, dout.p, stream_);
    d2h(out, dout.p, np, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
}

void Searcher::maxsim_embeddings(const float* q, uint64_t rows, uint64_t dim, const float* emb,
                                 const uint64_t* offsets, uint64_t np, float* out) {
    if (rows == 0 || dim == 0) fail(PLAID_INVALID_PARAMS, "empty query matrix");
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32");
    check_offsets_host(offsets, np, offsets[np]);
    DeviceGuard g(device_);
    const uint64_t T = offsets[np];
    DevBuf<float> dq, de, dout;
    DevBuf<uint64_t> doff;
    dq.ensure(rows * dim);
    de.ensure(T * dim);
    doff.ensure(np + 1);
    dout.ensure(np);
    h2d(dq.p, q, rows * dim, stream_);
    h2d(de.p, emb, T * dim, stream_);
    h2d(doff.p, offsets, np + 1, stream_);
    launch::maxsim_embeddings(dq.p, uint32_t(rows), uint32_t(dim), de.p, doff.p, np, dout.p, stream_);
    d2h(out, dout.p, np, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
}

void Searcher::merge_topk_device(const uint32_t* d_pids, const float* d_scores, const uint64_t* d_counts,
                                 uint64_t shards, uint64_t stride, uint64_t k, uint32_t* d_out_pids,
                                 float* d_out_scores, uint64_t* d_out_n, cudaStream_t st) {
    if (k < 1) fail(PLAID_INVALID_PARAMS, "k must be >= 1");
    DeviceGuard g(device_);
    if (!st) st = stream_;
    const uint64_t total = shards * stride;
    tmp_keys_.ensure(std::max<uint64_t>(total, 1));
    const uint64_t cap = launch::sort_tmp_capacity(total);
    if (cap) sort_tmp_.ensure(cap);
    launch::merge_topk(d_pids, d_scores, d_counts, shards, stride, 1, stride, k, tmp_keys_.p, counters_.p + kTmpN,
                       d_out_pids, d_out_scores, d_out_n, sort_tmp_.p, st);
}

// Packed rows (one all-gather per query): row g = [k u32 pids | k f32 scores |
// u64 count] at d_rows + g * (2k + 2) words.
void Searcher::merge_topk_rows_device(const uint32_t* d_rows, uint64_t shards, uint64_t k, uint32_t* d_out_pids,
                                      float* d_out_scores, uint64_t* d_out_n, cudaStream_t st) {
    if (k < 1) fail(PLAID_INVALID_PARAMS, "k must be >= 1");
    DeviceGuard g(device_);
    if (!st) st = stream_;
    const uint64_t total = shards * k;
    tmp_keys_.ensure(std::max<uint64_t>(total, 1));
    const uint64_t cap = launch::sort_tmp_capacity(total);
    if (cap) sort_tmp_.ensure(cap);
    const uint64_t row = 2 * k + 2;
    const uint64_t l0 = launch::launches();
    launch::merge_topk(d_rows, reinterpret_cast<const float*>(d_rows + k),
                       reinterpret_cast<const uint64_t*>(d_rows + 2 * k), shards, row, row / 2, k, k, tmp_keys_.p,
                       counters_.p + kTmpN, d_out_pids, d_out_scores, d_out_n, sort_tmp_.p, st);
    last_launches_ = launch::launches() - l0;
}

void Searcher::merge_topk(const uint32_t* pids, const float* scores, const uint64_t* counts, uint64_t shards,
                          uint64_t stride, uint64_t k, uint32_t* out_pids, float* out_scores,
                          uint64_t* out_n) {
    DeviceGuard g(device_);
    const uint64_t total = shards * stride;
    DevBuf<uint32_t> dp, op;
    DevBuf<float> ds, os;
    DevBuf<uint64_t> dc, on;
    dp.ensure(total);
    ds.ensure(total);
    dc.ensure(shards);
    op.ensure(k);
    os.ensure(k);
    on.ensure(1);
    h2d(dp.p, pids, total, stream_);
    h2d(ds.p, scores, total, stream_);
    h2d(dc.p, counts, shards, stream_);
    merge_topk_device(dp.p, ds.p, dc.p, shards, stride, k, op.p, os.p, on.p, stream_);
    uint64_t n = 0;
    d2h(&n, on.p, 1, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    d2h(out_pids, op.p, n, stream_);
    d2h(out_scores, os.p, n, stream_);
    PLAID_CUDA(cudaStreamSynchronize(stream_));
    *out_n = n;
}

// ---------------------------------------------------------------- throughput mode
// ---------------------------------------------------------------- throughput: waves
WavePipeline::WavePipeline(DeviceIndex* index, int device, bool tensor)
    : index_(index), device_(device), tensor_(tensor) {
    DeviceGuard g(device_);
    const IndexView& ix = index_->view();
    if (tensor_ && launch::tensor_scores_supported(ix)) launch::make_wave_tensor_map(ix, tmap_);
    else tensor_ = false;
    status_.ensure(1);
    PLAID_CUDA(cudaMemset(status_.p, 0, sizeof(int)));
    PLAID_CUDA(cudaDeviceSynchronize());
    const char* tr = getenv("PLAID_WAVE_TRACE");
    tracing_ = tr && *tr && *tr != '0';
}

WavePipeline::~WavePipeline() {
    DeviceGuard g(device_);
    cudaDeviceSynchronize();
}

bool WavePipeline::supports(const plaid_params& p, uint64_t rows, uint64_t dim) const {
    const IndexView& ix = index_->view();
    return ix.dim == 128 && dim == 128 && rows >= 1 && rows <= 32 && ix.tok_inv && !p.disable_filter &&
           p.nprobe >= 1 && p.nprobe <= 8 && p.nprobe <= ix.K && ix.N < (1ull << 31) &&
           std::min<uint64_t>(stage3_width(p), ix.N) <= launch::kWaveSortCap && p.ndocs <= (1ull << 24) &&
           index_->candidate_bound(p.nprobe) < (1ull << 31);
}

// Scratch per slot: S (K x 32 f32), keep bits, partial lists, candidate
// bitmap + word prefix (N bits each, padded to whole compaction rounds), C1
// ids / keys / two side buffers / stage-2 accumulators (c1cap = the sum of
// the 32 nprobe longest posting lists), stage-2/3 selections.  The number of
// slots is the wave size: at most 512 (4 resident worker CTAs per SM hold a
// whole wave) and at most half of the free device memory.
void WavePipeline::ensure(uint64_t nq, const plaid_params& p) {
    const IndexView& ix = index_->view();
    const uint64_t K = ix.K, N = ix.N;
    const uint64_t c1cap = std::max<uint64_t>(index_->candidate_bound(p.nprobe), 1);
    const uint64_t nd = std::min<uint64_t>(p.ndocs, N), n3 = std::min<uint64_t>(stage3_width(p), N);
    const uint64_t sel_stride = (nd + n3 + 1) / 2 * 2;
    const uint64_t lists = std::max<uint64_t>(launch::wave_scores_lists(ix), launch::scores_max_warps());
    const uint64_t partial_stride = lists * 32 * 8;
    const uint64_t keep_stride = ((K + 31) / 32 + 3) / 4 * 4;
    const uint64_t s_stride = K * kScoresPitch;
    const uint64_t per_slot = s_stride * 4 + keep_stride * 4 + partial_stride * 8 + c1cap * (4 + 8 + 24) +
                              nd * 128 + sel_stride * 8 + 32;
    // a wave = the worker CTAs resident at once (one round of the worker)
    static const uint64_t resident = [&] {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return uint64_t(sms) * launch::wave_worker_ctas_per_sm(ix.nbits);
    }();
    uint64_t want = std::min<uint64_t>(std::max<uint64_t>(nq, 1), std::min<uint64_t>(resident, 1024));
    if (tensor_) want = (want + 3) / 4 * 4;
    if (ix.range_w == launch::kWaveRangeIds) {
        range_tab_p_ = ix.range_tab;  // the index's own table has the worker's range width
    } else if (!range_tab_.p) {
        const uint32_t W = launch::kWaveRangeIds, R = uint32_t((N + W - 1) / W);
        range_tab_.ensure(K * (uint64_t(R) + 1));
        launch::wave_range_table(ix, W, R, range_tab_.p, 0);
        PLAID_CUDA(cudaDeviceSynchronize());
        PLAID_CUDA(cudaGetLastError());
        range_tab_p_ = range_tab_.p;
    }
    const bool fits = slots_ >= want && c1cap_ >= c1cap && sel_stride_ >= sel_stride && nd_cap_ >= nd;
    if (fits) return;
    // grow: release first so the free-memory estimate sees the old buffers
    S_.release(), rowmax_.release(), keep_.release(), c1_.release(), acc_.release();
    partial_.release(), keys_.release(), side_.release(), sel_.release(), counters_.release();
    size_t free_b = 0, total_b = 0;
    PLAID_CUDA(cudaMemGetInfo(&free_b, &total_b));
    uint64_t cap = std::max<uint64_t>(uint64_t(free_b / 2) / per_slot, 1);
    uint64_t slots = std::max<uint64_t>(want, slots_);
    slots = std::min<uint64_t>(slots, cap);
    if (tensor_ && slots >= 4) slots = slots / 4 * 4;
    if (slots == 0) fail(PLAID_OUT_OF_MEMORY, "not enough device memory for one throughput-mode slot");
    c1cap_ = std::max(c1cap_, c1cap);
    sel_stride_ = std::max(sel_stride_, sel_stride);
    partial_stride_ = partial_stride, keep_stride_ = keep_stride, s_stride_ = s_stride;
    nd_cap_ = std::max(nd_cap_, nd);
    slots_ = uint32_t(slots);
    S_.ensure(slots * s_stride_);
    rowmax_.ensure(K);
    keep_.ensure(slots * keep_stride_);
    partial_.ensure(slots * partial_stride_);
    c1_.ensure(slots * c1cap_);
    acc_.ensure(slots * nd_cap_ * 32);
    keys_.ensure(slots * c1cap_);
    side_.ensure(slots * c1cap_ * 3);
    sel_.ensure(slots * sel_stride_);
    counters_.ensure(std::max<uint64_t>(nq, slots) * 4);
    if (tracing_) trace_.ensure(std::max<uint64_t>(nq, slots) * 16);
    PLAID_CUDA(cudaMemset(acc_.p, 0, acc_.n * sizeof(uint32_t)));
    PLAID_CUDA(cudaDeviceSynchronize());
}

void WavePipeline::run(const float* d_q, uint64_t nq, uint32_t rows, const plaid_params& p, uint32_t* d_pids,
                       float* d_scores, uint64_t* d_n, bool validate, cudaStream_t st) {
    DeviceGuard g(device_);
    const IndexView& ix = index_->view();
    ensure(nq, p);
    if (counters_.n < nq * 4 || (tracing_ && trace_.n < nq * 16)) {
        counters_.ensure(nq * 4);
        if (tracing_) trace_.ensure(nq * 16);
        PLAID_CUDA(cudaDeviceSynchronize());
    }
    launch::reset_launches();
    const uint32_t npb = np_bucket(p.nprobe);
    const uint64_t nd = std::min<uint64_t>(p.ndocs, ix.N), n3 = std::min<uint64_t>(stage3_width(p), ix.N);
    for (uint64_t j0 = 0; j0 < nq; j0 += slots_) {
        const uint32_t w = uint32_t(std::min<uint64_t>(slots_, nq - j0));
        const float* q = d_q + j0 * rows * 128;
        uint32_t lists = 0;
        if (tensor_) {
            lists = launch::wave_scores(tmap_, ix, q, w, rows, p.t_cs, npb, S_.p, s_stride_, keep_.p, keep_stride_,
                                        partial_.p, partial_stride_, st);
        } else {
            for (uint32_t i = 0; i < w; ++i)
                lists = launch::scores_exact(ix, q + uint64_t(i) * rows * 128, rows, p.t_cs, S_.p + i * s_stride_,
                                             rowmax_.p, keep_.p + i * keep_stride_, partial_.p + i * partial_stride_,
                                             npb, st);
        }
        launch::WaveArgs a;
        a.Q = q;
        a.rows = rows, a.nprobe = uint32_t(p.nprobe), a.ndocs = uint32_t(nd), a.n3 = uint32_t(n3);
        a.k = uint32_t(p.k), a.nlists = lists, a.pid_base = uint32_t(index_->pid_base()), a.validate = validate ? 1 : 0;
        static const bool s4_exact = getenv("PLAID_WAVE_S4_EXACT") != nullptr;
        a.s4_tensor = tensor_ && ix.tok_inv && !s4_exact ? 1u : 0u;
        a.S = S_.p, a.s_stride = s_stride_, a.keep = keep_.p, a.keep_stride = keep_stride_;
        a.partial = partial_.p, a.partial_stride = partial_stride_;
        a.range_tab = range_tab_p_, a.range_w = launch::kWaveRangeIds;
        a.range_n = uint32_t((ix.N + launch::kWaveRangeIds - 1) / launch::kWaveRangeIds);
        a.c1 = c1_.p, a.acc = acc_.p, a.keys = keys_.p, a.side = side_.p, a.c1cap = c1cap_;
        a.sel = sel_.p, a.sel_stride = sel_stride_;
        a.out_pids = d_pids + j0 * p.k, a.out_scores = d_scores + j0 * p.k, a.out_n = d_n + j0;
        a.counters = counters_.p + j0 * 4, a.status = status_.p;
        a.trace = tracing_ ? reinterpret_cast<unsigned long long*>(trace_.p + j0 * 16) : nullptr;
        launch::wave_worker(ix, a, w, npb, st);
    }
    PLAID_CUDA(cudaGetLastError());
    last_launches_ = launch::launches();
}

void WavePipeline::counters(uint64_t* out_host, uint64_t nq) {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaDeviceSynchronize());
    if (nq * 4 > counters_.n) fail(PLAID_INVALID_PARAMS, "counter request exceeds the last batch");
    PLAID_CUDA(cudaMemcpy(out_host, counters_.p, nq * 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
}

void WavePipeline::copy_scores(uint64_t j, float* out_host) {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaDeviceSynchronize());
    if (j >= slots_ || !S_.p) fail(PLAID_INVALID_PARAMS, "no such slot in the last wave");
    PLAID_CUDA(cudaMemcpy(out_host, S_.p + j * s_stride_, s_stride_ * sizeof(float), cudaMemcpyDeviceToHost));
}

void WavePipeline::trace(uint64_t* out_host, uint64_t nq) {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaDeviceSynchronize());
    if (!tracing_ || nq * 16 > trace_.n) fail(PLAID_INVALID_PARAMS, "no wave trace (set PLAID_WAVE_TRACE=1)");
    PLAID_CUDA(cudaMemcpy(out_host, trace_.p, nq * 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
}

void WavePipeline::check_status() {
    DeviceGuard g(device_);
    PLAID_CUDA(cudaDeviceSynchronize());
    int status = 0;
    PLAID_CUDA(cudaMemcpy(&status, status_.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (status) {
        PLAID_CUDA(cudaMemset(status_.p, 0, sizeof(int)));
        PLAID_CUDA(cudaDeviceSynchronize());
        fail(status, "device-side query validation failed (row not unit norm)");
    }
}

BatchSearcher::BatchSearcher(DeviceIndex* index, int device, const plaid_searcher_config& cfg, uint32_t lanes)
    : index_(index), device_(device) {
    if (!index) fail(PLAID_INVALID_PARAMS, "batch searcher needs an index");
    if (lanes == 0 || lanes > 64) fail(PLAID_INVALID_PARAMS, "lanes must be in [1, 64]");
    DeviceGuard g(device_);
    plaid_searcher_config c = cfg;
    c.record_times = 0;
    for (uint32_t l = 0; l < lanes; ++l) {
        lanes_.push_back(std::make_unique<Searcher>(index, device, c));
        streams_.push_back(lanes_.back()->stream());
        cudaEvent_t e;
        PLAID_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        joins_.push_back(e);
    }
    PLAID_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    for (uint32_t l = 0; l < lanes; ++l) {
        cudaEvent_t e;
        PLAID_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ready_.push_back(e);
        PLAID_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        sdone_.push_back(e);
    }
    // the S_cq pass needs whole SMs (215 KB of shared memory, the full register
    // file): give its stream the highest priority so freed SMs go to it before
    // the lanes' small kernels refill them
    int lo = 0, hi = 0;
    PLAID_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PLAID_CUDA(cudaStreamCreateWithPriority(&sstream_, cudaStreamNonBlocking, hi));
    if (cfg.batch_engine != PLAID_BATCH_LANES)
        wave_ = std::make_unique<WavePipeline>(index, device, cfg.score_mode == PLAID_SCORES_TENSOR);
}

BatchSearcher::~BatchSearcher() {
    DeviceGuard g(device_);
    cudaDeviceSynchronize();
    for (auto e : joins_) cudaEventDestroy(e);
    for (auto e : ready_) cudaEventDestroy(e);
    for (auto e : sdone_) cudaEventDestroy(e);
    if (sstream_) cudaStreamDestroy(sstream_);
    if (fork_) cudaEventDestroy(fork_);
    if (h_q_) cudaFreeHost(h_q_);
    if (h_pids_) cudaFreeHost(h_pids_);
    if (h_scores_) cudaFreeHost(h_scores_);
    if (h_n_) cudaFreeHost(h_n_);
}

void BatchSearcher::search_device(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim, const plaid_params& p,
                                  uint32_t* d_pids, float* d_scores, uint64_t* d_n, cudaStream_t st) {
    search_device_impl(d_q, nq, rows, dim, p, d_pids, d_scores, d_n, st, true);
}

void BatchSearcher::wave_counters(uint64_t* out_host, uint64_t nq) {
    if (!wave_ || !last_wave_) fail(PLAID_INVALID_PARAMS, "the last batch did not run on the wave engine");
    wave_->counters(out_host, nq);
}

void BatchSearcher::wave_scores(uint64_t j, float* out_host) {
    if (!wave_ || !last_wave_) fail(PLAID_INVALID_PARAMS, "the last batch did not run on the wave engine");
    wave_->copy_scores(j, out_host);
}

void BatchSearcher::wave_trace(uint64_t* out_host, uint64_t nq) {
    if (!wave_ || !last_wave_) fail(PLAID_INVALID_PARAMS, "the last batch did not run on the wave engine");
    wave_->trace(out_host, nq);
}

void BatchSearcher::search_device_impl(const float* d_q, uint64_t nq, uint64_t rows, uint64_t dim,
                                       const plaid_params& p, uint32_t* d_pids, float* d_scores, uint64_t* d_n,
                                       cudaStream_t st, bool validate) {
    DeviceGuard g(device_);
    if (!st) st = streams_[0];
    last_wave_ = false;
    if (wave_ && wave_->supports(p, rows, dim)) {
        validate_params_host(p, index_->view().K);
        if (nq == 0) return;
        wave_->run(d_q, nq, uint32_t(rows), p, d_pids, d_scores, d_n, validate, st);
        last_launches_ = wave_->last_launches();
        last_wave_ = true;
        return;
    }
    const uint64_t L = lanes_.size();
    PLAID_CUDA(cudaEventRecord(fork_, st));
    for (uint64_t l = 0; l < L && l < nq; ++l)
        if (streams_[l] != st) PLAID_CUDA(cudaStreamWaitEvent(streams_[l], fork_, 0));
    uint64_t launches = 0;
    const bool batched = L >= 2 && lanes_[0]->batch_scores_ok(p, rows, dim);
    if (batched) {
        // pairs of queries share one S_cq pass over C (scores_tensor_batch) on
        // the scores stream; each lane waits for it, then runs the rest
        PLAID_CUDA(cudaStreamWaitEvent(sstream_, fork_, 0));
        const uint32_t npb = np_bucket(p.nprobe);
        const uint64_t step = kMaxScoreBatch;
        for (uint64_t j0 = 0; j0 < nq; j0 += step) {
            const uint32_t qb = uint32_t(std::min<uint64_t>(step, nq - j0));
            TfOut out{};
            for (uint32_t qi = 0; qi < qb; ++qi) {
                const uint64_t j = j0 + qi, l = j % L;
                const float* q = d_q + j * rows * dim;
                lanes_[l]->batch_prepare(q, rows, dim, p, streams_[l]);
                lanes_[l]->batch_targets(out, qi, q);
                PLAID_CUDA(cudaEventRecord(ready_[l], streams_[l]));
                PLAID_CUDA(cudaStreamWaitEvent(sstream_, ready_[l], 0));
            }
            const uint32_t warps = launch::scores_tensor_batch(lanes_[0]->tensor_map(), index_->view(), out, qb,
                                                               uint32_t(rows), p.t_cs, npb, sstream_);
            PLAID_CUDA(cudaEventRecord(sdone_[(j0 / step) % sdone_.size()], sstream_));
            for (uint32_t qi = 0; qi < qb; ++qi) {
                const uint64_t j = j0 + qi, l = j % L;
                PLAID_CUDA(cudaStreamWaitEvent(streams_[l], sdone_[(j0 / step) % sdone_.size()], 0));
                lanes_[l]->batch_finish(d_q + j * rows * dim, uint32_t(rows), p, warps, d_pids + j * p.k,
                                        d_scores + j * p.k, d_n + j, streams_[l]);
                launches += lanes_[l]->last_launches() + (qi == 0);
            }
        }
    } else {
        for (uint64_t j = 0; j < nq; ++j) {
            Searcher& s = *lanes_[j % L];
            s.search_device(d_q + j * rows * dim, 1, rows, dim, p, d_pids + j * p.k, d_scores + j * p.k, d_n + j,
                            streams_[j % L]);
            launches += s.last_launches();
        }
    }
    for (uint64_t l = 0; l < L && l < nq; ++l) {
        if (streams_[l] == st) continue;
        PLAID_CUDA(cudaEventRecord(joins_[l], streams_[l]));
        PLAID_CUDA(cudaStreamWaitEvent(st, joins_[l], 0));
    }
    last_launches_ = launches;
}

void BatchSearcher::search(const float* q, uint64_t nq, uint64_t rows, uint64_t dim, const plaid_params& p,
                           uint32_t* out_pids, float* out_scores, uint64_t* out_n) {
    const IndexView& ix = index_->view();
    for (uint64_t j = 0; j < nq; ++j) out_n[j] = 0;
    // shape checks here; the per-row norm check (types.cpp:61-72, in-order
    // fp64) runs on the device, one CTA's warp per query (at 1024 queries the
    // host loop was ~2 ms of the call), reported by sync() below
    if (nq && rows == 0) fail(PLAID_INVALID_PARAMS, "query must contain at least one token");
    if (nq && dim != ix.dim)
        fail(PLAID_DIMENSION_MISMATCH,
             "query dim " + std::to_string(dim) + " does not match index dim " + std::to_string(ix.dim));
    validate_params_host(p, ix.K);
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    if (nq == 0) return;
    DeviceGuard g(device_);
    const uint64_t nqf = nq * rows * dim, nout = nq * p.k;
    q_.ensure(nqf);
    pids_.ensure(nout);
    scores_.ensure(nout);
    n_.ensure(nq);
    if (hq_cap_ < nqf) {
        if (h_q_) cudaFreeHost(h_q_);
        h_q_ = nullptr;
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_q_), nqf * sizeof(float)));
        hq_cap_ = nqf;
    }
    if (ho_cap_ < nout + nq) {
        if (h_pids_) cudaFreeHost(h_pids_);
        if (h_scores_) cudaFreeHost(h_scores_);
        if (h_n_) cudaFreeHost(h_n_);
        h_pids_ = nullptr, h_scores_ = nullptr, h_n_ = nullptr;
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_pids_), (nout + nq) * sizeof(uint32_t)));
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_scores_), (nout + nq) * sizeof(float)));
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_n_), nq * sizeof(uint64_t)));
        ho_cap_ = nout + nq;
    }
    // staging copy into pinned memory, large batches split over host threads
    // (one core copies ~8 GB/s: 2 ms for 1024 queries); with the wave engine
    // one wave at a time, so that wave j + 1's staging and upload overlap wave
    // j on the GPU
    auto stage = [&](uint64_t b0, uint64_t bytes) {
        const uint32_t nthr =
            bytes >= (4u << 20) ? std::min<uint32_t>(8, std::max(1u, std::thread::hardware_concurrency())) : 1u;
        char* dst = reinterpret_cast<char*>(h_q_) + b0;
        const char* src = reinterpret_cast<const char*>(q) + b0;
        if (nthr == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::vector<std::thread> pool;
        const uint64_t per = (bytes / nthr + 4095) & ~uint64_t(4095);
        for (uint32_t t = 0; t < nthr; ++t) {
            const uint64_t o = uint64_t(t) * per;
            if (o >= bytes) break;
            const uint64_t len = std::min(per, bytes - o);
            pool.emplace_back([=] { std::memcpy(dst + o, src + o, len); });
        }
        for (auto& th : pool) th.join();
    };
    cudaStream_t st = streams_[0];
    const uint64_t per_q = rows * dim;
    const uint64_t chunk = wave_ && wave_->supports(p, rows, dim) && wave_->slots() ? wave_->slots() : nq;
    for (uint64_t j0 = 0; j0 < nq; j0 += chunk) {
        const uint64_t m = std::min(chunk, nq - j0);
        stage(j0 * per_q * sizeof(float), m * per_q * sizeof(float));
        PLAID_CUDA(cudaMemcpyAsync(q_.p + j0 * per_q, h_q_ + j0 * per_q, m * per_q * sizeof(float),
                                   cudaMemcpyHostToDevice, st));
        search_device_impl(q_.p + j0 * per_q, m, rows, dim, p, pids_.p + j0 * p.k, scores_.p + j0 * p.k, n_.p + j0,
                           st, true);
    }
    PLAID_CUDA(cudaMemcpyAsync(h_n_, n_.p, nq * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    PLAID_CUDA(cudaMemcpyAsync(h_pids_, pids_.p, nout * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    PLAID_CUDA(cudaMemcpyAsync(h_scores_, scores_.p, nout * sizeof(float), cudaMemcpyDeviceToHost, st));
    PLAID_CUDA(cudaStreamSynchronize(st));
    sync();
    for (uint64_t j = 0; j < nq; ++j) {
        const uint64_t m = h_n_[j];
        out_n[j] = m;
        std::memcpy(out_pids + j * p.k, h_pids_ + j * p.k, m * sizeof(uint32_t));
        std::memcpy(out_scores + j * p.k, h_scores_ + j * p.k, m * sizeof(float));
    }
}

void BatchSearcher::sync() {
    if (wave_) wave_->check_status();
    for (auto& s : lanes_) s->sync();  // also reports device-side query validation failures
}

// ---------------------------------------------------------------- sharded (single process)
ShardedSearcher::ShardedSearcher(const std::vector<DeviceIndex*>& shards, const plaid_searcher_config& cfg, int mode)
    : mode_(mode) {
    if (shards.empty() || shards.size() > launch::kMaxShards)
        fail(PLAID_INVALID_PARAMS, "shard count must be in [1, " + std::to_string(launch::kMaxShards) + "]");
    if (mode != kGlobalExact && mode != kShardLocal) fail(PLAID_INVALID_PARAMS, "unknown shard mode");
    sh_.resize(shards.size());
    for (size_t g = 0; g < shards.size(); ++g) {
        DeviceIndex* ix = shards[g];
        if (!ix) fail(PLAID_INVALID_PARAMS, "shard index is NULL");
        const IndexView& v = ix->view();
        if (g == 0) {
            dim_ = v.dim;
            K_ = v.K;
        } else if (v.dim != dim_ || v.K != K_) {
            fail(PLAID_INVALID_PARAMS, "shards must share dim and the centroid table");
        }
        N_ += v.N;
        Shard& s = sh_[g];
        s.ix = ix;
        s.dev = ix->device();
        s.s = std::make_unique<Searcher>(ix, s.dev, cfg);
        s.st = s.s->stream();
        DeviceGuard dg(s.dev);
        for (auto& e : s.ev) PLAID_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s.q.ensure(32 * 256);
        s.cnt.ensure(8);
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s.h_cnt), 8 * sizeof(uint64_t)));
    }
    // every shard's exchange kernel reads every other shard's row: peer access
    for (auto& a : sh_)
        for (auto& b : sh_) {
            if (a.dev == b.dev) continue;
            int ok = 0;
            PLAID_CUDA(cudaDeviceCanAccessPeer(&ok, a.dev, b.dev));
            if (!ok) fail(PLAID_UNSUPPORTED, "no peer access between GPUs " + std::to_string(a.dev) + " and " +
                                                std::to_string(b.dev));
            DeviceGuard dg(a.dev);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b.dev, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else PLAID_CUDA(e);
        }
    PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_q_), 32 * 256 * sizeof(float)));
}

ShardedSearcher::~ShardedSearcher() {
    for (auto& s : sh_) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(s.dev);
        if (s.st) cudaStreamSynchronize(s.st);
        for (auto& e : s.ev)
            if (e) cudaEventDestroy(e);
        if (s.h_cnt) cudaFreeHost(s.h_cnt);
        cudaSetDevice(prev);
    }
    if (h_q_) cudaFreeHost(h_q_);
    if (h_out_) cudaFreeHost(h_out_);
}

// dst's stream waits for event `which` of every shard, then gathers their
// rows (x2, x3 or result rows) into `out` on dst's device.
void ShardedSearcher::gather(Shard& dst, int which, uint64_t words, uint64_t* out) {
    launch::PeerRows src{};
    for (size_t g = 0; g < sh_.size(); ++g) {
        Shard& s = sh_[g];
        if (&s != &dst) PLAID_CUDA(cudaStreamWaitEvent(dst.st, s.ev[which], 0));
        src.p[g] = which == 0 ? s.x2.p : which == 1 ? s.x3.p : s.rows.p;
    }
    DeviceGuard dg(dst.dev);
    launch::gather_rows(src, uint32_t(sh_.size()), words, out, dst.st);
}

void ShardedSearcher::search(const float* q, uint64_t rows, uint64_t dim, const plaid_params& p, uint32_t* out_pids,
                             float* out_scores, uint64_t* out_n, plaid_trace* trace) {
    *out_n = 0;
    if (trace) std::memset(trace, 0, sizeof *trace);
    validate_query_host(q, rows, dim, dim_);  // types.cpp:61-72, then :88-99
    validate_params_host(p, K_);
    if (rows > 32) fail(PLAID_UNSUPPORTED, "engine supports |Q| <= 32 query tokens");
    const uint32_t G = uint32_t(sh_.size());
    const uint64_t k = p.k;
    // exchange strides over the GLOBAL passage count (>= every shard's width)
    const bool df = p.disable_filter != 0;
    const uint64_t s2 = mode_ == kGlobalExact && !df ? std::min<uint64_t>(p.ndocs, N_) : 0;
    const uint64_t s3 = mode_ == kGlobalExact && !df ? std::min<uint64_t>(stage3_width(p), N_) : 0;
    const uint64_t row_words = k + 1;  // [k u32 pids | k f32 scores | u64 n] as u64 words
    std::memcpy(h_q_, q, rows * dim * sizeof(float));
    uint64_t launches = 0;
    for (auto& s : sh_) {
        DeviceGuard dg(s.dev);
        s.x2.ensure(std::max<uint64_t>(s2, 1));
        s.g2.ensure(std::max<uint64_t>(G * s2, 1));
        s.x3.ensure(std::max<uint64_t>(s3, 1));
        s.g3.ensure(std::max<uint64_t>(G * s3, 1));
        s.rows.ensure(row_words);
        PLAID_CUDA(cudaMemcpyAsync(s.q.p, h_q_, rows * dim * sizeof(float), cudaMemcpyHostToDevice, s.st));
    }
    auto row_ptrs = [&](Shard& s, uint32_t*& pids, float*& scores, uint64_t*& n) {
        uint32_t* r = reinterpret_cast<uint32_t*>(s.rows.p);
        pids = r;
        scores = reinterpret_cast<float*>(r + k);
        n = reinterpret_cast<uint64_t*>(r + 2 * k);
    };
    if (mode_ == kShardLocal) {
        for (auto& s : sh_) {
            DeviceGuard dg(s.dev);
            uint32_t* pp;
            float* ps;
            uint64_t* pn;
            row_ptrs(s, pp, ps, pn);
            s.s->search_device(s.q.p, 1, rows, dim, p, pp, ps, pn, s.st);
            launches += s.s->last_launches();
        }
    } else {
        for (auto& s : sh_) {
            DeviceGuard dg(s.dev);
            s.s->shard_phase1(s.q.p, rows, dim, p, s.x2.p, s2, s.st);
            PLAID_CUDA(cudaEventRecord(s.ev[0], s.st));
        }
        for (auto& s : sh_) {
            if (s2) gather(s, 0, s2, s.g2.p);
            DeviceGuard dg(s.dev);
            s.s->shard_phase2(s.g2.p, G, s.x3.p, s3, s.st);
            PLAID_CUDA(cudaEventRecord(s.ev[1], s.st));
        }
        for (auto& s : sh_) {
            if (s3) gather(s, 1, s3, s.g3.p);
            DeviceGuard dg(s.dev);
            uint32_t* pp;
            float* ps;
            uint64_t* pn;
            row_ptrs(s, pp, ps, pn);
            s.s->shard_phase3(s.g3.p, G, pp, ps, pn, s.st);
            launches += s.s->last_launches();
        }
    }
    for (auto& s : sh_) {
        DeviceGuard dg(s.dev);
        s.s->trace_counters_device(s.cnt.p, s.st);
        PLAID_CUDA(cudaMemcpyAsync(s.h_cnt, s.cnt.p, 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s.st));
        PLAID_CUDA(cudaEventRecord(s.ev[2], s.st));
    }
    // merge on shard 0's device: gather every result row, one select
    Shard& s0 = sh_[0];
    DeviceGuard dg(s0.dev);
    grows_.ensure(G * row_words);
    gather(s0, 2, row_words, grows_.p);
    const uint64_t kk = (k + 3) / 4 * 4;
    out_.ensure(2 * kk + 2);
    if (h_out_k_ < kk) {
        if (h_out_) cudaFreeHost(h_out_);
        h_out_ = nullptr;
        PLAID_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_out_), (2 * kk + 2) * sizeof(uint32_t)));
        h_out_k_ = kk;
    }
    uint64_t* d_n = reinterpret_cast<uint64_t*>(out_.p + 2 * kk);
    s0.s->merge_topk_rows_device(reinterpret_cast<const uint32_t*>(grows_.p), G, k, out_.p,
                                 reinterpret_cast<float*>(out_.p + kk), d_n, s0.st);
    PLAID_CUDA(cudaMemcpyAsync(h_out_, out_.p, (2 * kk + 2) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s0.st));
    PLAID_CUDA(cudaStreamSynchronize(s0.st));
    for (auto& s : sh_) s.s->sync();  // device-side failures (e.g. query validation) surface here
    last_launches_ = launches + G + 1;
    const uint64_t n = *reinterpret_cast<const uint64_t*>(h_out_ + 2 * kk);
    *out_n = n;
    std::memcpy(out_pids, h_out_, n * sizeof(uint32_t));
    std::memcpy(out_scores, h_out_ + kk, n * sizeof(float));
    if (trace) {
        uint64_t c[6] = {};
        for (auto& s : sh_)
            for (int j = 0; j < 6; ++j) c[j] += s.h_cnt[j];
        trace->stage1_candidates = c[0];
        trace->centroid_matmul_count = 1;
        if (c[0] > 0) {  // pipeline.cpp:249-252
            trace->stage2_out = df ? c[0] : c[1];  // pipeline.cpp:255-258
            trace->stage3_out = df ? c[0] : c[2];
            trace->final_out = n;
            trace->stage2_rows_gathered = c[4];
            trace->stage3_rows_gathered = c[5];
            trace->decompressed_passages = trace->stage3_out;
        }
    }
}

}  // namespace plaid

// Profiling knob: stop every search after its first `cap` kernel launches
// (-1 = off); returns the previous cap.  Not part of include/plaid.h.
extern "C" long long plaid_debug_set_launch_cap(long long cap) {
    return static_cast<long long>(plaid::launch::set_launch_cap(cap));
}
