// sparse.cuh -- device CSR/CSC buffer, scratch arena, sparse kernels (see sparse.cu).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace sfdg {

// Stream-ordered bump arena over retained device chunks. reset() rewinds; callers
// only reuse memory on the same stream, so earlier kernels are ordered before reuse.
class Scratch {
  public:
    ~Scratch() { release(); }
    template <class T>
    T* take(int64_t n) {
        const size_t bytes = round_up(std::max<int64_t>(n, 1) * sizeof(T), 256);
        while (cur < chunks.size() && used + bytes > chunks[cur].size) {
            ++cur;
            used = 0;
        }
        if (cur == chunks.size()) {
            // Double the last chunk, but never with more than 1 GB of slack beyond the request:
            // plain doubling over-allocated by many GB at c5 (single takes of 1-4 GB) and ran a
            // 180 GB device out of memory; some slack keeps later, slightly larger take sequences
            // (and stream captures, which must not allocate) inside existing chunks.
            const size_t last2 = chunks.empty() ? (size_t)64 << 20 : chunks.back().size * 2;
            size_t sz = std::max<size_t>(bytes, std::min<size_t>(last2, bytes + ((size_t)1 << 30)));
            Chunk c{nullptr, sz};
            CK(cudaMalloc(&c.ptr, sz));
            chunks.push_back(c);
            used = 0;
        }
        T* p = reinterpret_cast<T*>(static_cast<char*>(chunks[cur].ptr) + used);
        used += bytes;
        if (poison()) CK(cudaMemset(p, 0xff, bytes));  // debugging aid: NaN-fill (SFDG_POISON=1)
        return p;
    }
    void reset() {
        cur = 0;
        used = 0;
    }
    // Before a stream capture (which must not cudaMalloc): make sure takes totalling up to
    // `bytes` after this point find existing chunks. The position is unchanged.
    void headroom(size_t bytes) {
        const size_t c0 = cur, u0 = used;
        take<char>((int64_t)bytes);
        cur = c0;
        used = u0;
    }
    void release() {
        for (auto& c : chunks) cudaFree(c.ptr);
        chunks.clear();
        reset();
    }

  private:
    static bool poison() {
        static const bool on = std::getenv("SFDG_POISON") && std::getenv("SFDG_POISON")[0] == '1';
        return on;
    }
    struct Chunk {
        void* ptr;
        size_t size;
    };
    std::vector<Chunk> chunks;
    size_t cur = 0, used = 0;
};

// A' on the device (sparse.hpp:19-57): CSR with int32 offsets (nnz per flush < 2^31)
// plus its stable transpose (CSC) built once per flush.
struct DevCsr {
    int m = 0, d = 0;
    int64_t nnz = 0;
    int* row_ptr = nullptr;  // m+1
    uint32_t* col = nullptr; // nnz
    double* val = nullptr;   // nnz
    int* col_ptr = nullptr;  // d+1
    int* row_idx = nullptr;  // nnz (CSC)
    double* cval = nullptr;  // nnz (CSC)
    int rows_cap = 0, d_cap = 0;
    int64_t nnz_cap = 0;
    void reserve(int m_cap, int64_t nnz_cap);
    void set_shape(int m, int d, int64_t nnz);
    void release();
    ~DevCsr() { release(); }
};

// Work plan of the gather SpMM over one CSR (or CSC) operand, built once per flush.
// Rows longer than 2*piece are cut into piece-long pieces, processed by the same launch as the
// short rows (pieces first, so their latency chains overlap the rest) and summed per row, in
// piece order, by the piece that finishes last. The short rows follow in descending length
// (`order`, a counting sort by length): with skewed row lengths (geometric / lognormal rows,
// Zipf columns) a static warp-to-row assignment in natural order leaves a tail of long rows
// on a few warps, longest-first keeps the warps even (c4 CSR: 201 -> 145 us per launch,
// tools/spmm_lab.cu). The order only changes which warp computes a row, never the row's
// arithmetic, so results do not depend on it.
// piece: 128 entries, doubled while a piece stays under half the grid's per-warp share of the
// entries (up to 512 at c3-c5), so the partial rows of very long rows stay few; for a gathered
// panel larger than L2, shortened again so the pieces in flight cover an L2-sized window of it
// (spmm_big_piece_length: c5 CSC 64). A long row's partials are summed in two levels.
constexpr int kPiece = 128;
constexpr int kPieceGroup = 64;  // pieces per first-level sum of a long row's partials
int spmm_piece_length(int64_t nnz);
// for gathered panels larger than the L2: the pieces in flight must cover an L2-sized window
int spmm_big_piece_length(int piece, int64_t nnz, int64_t in_rows, size_t panel_bytes, size_t l2_bytes);
struct SegPlan {
    int rows = 0;
    int piece = kPiece;
    int* long_rows = nullptr;
    int* long_first = nullptr;
    int* piece_beg = nullptr;
    int* piece_end = nullptr;
    int* piece_li = nullptr;  // long-row index of each piece
    int* arrive = nullptr;    // per long row: piece groups finished in the current launch (self-resetting)
    int* garrive = nullptr;   // per group of kPieceGroup pieces (at its first piece): pieces finished
    bool garrive_fresh = false;  // newly allocated: zeroed by the next build() on its stream
    int* order = nullptr;     // the short rows, longest first
    // Processing order of the pieces (null: piece order): by the first input index a piece
    // gathers (the row of a CSC piece, the column of a CSR piece) in coarse buckets, so the grid
    // works on pieces of many long rows over the same window of the input panel at a time
    int* porder = nullptr;
    bool has_porder = false;  // porder filled by the last build
    const int* piece_order() const { return has_porder ? porder : nullptr; }
    int* counts = nullptr;  // device [nlong, npieces, nshort]
    int* ticket = nullptr;  // device [next piece, warps done]: pieces by ticket (big panels)
    bool big = false;       // the gathered panel is larger than the L2 (set by build)
    int host_long = -1;     // long rows as known on the host (-1: unknown -> always run the piece path)
    int64_t host_pieces = -1;  // pieces as known on the host (-1: unknown -> worst-case partial buffer)
    // Partial rows of the pieces: a retained buffer (not scratch), so its address is fixed for
    // the sweep-block CUDA graphs; grown by ensure_partial() outside any capture.
    mutable double* partial = nullptr;
    mutable int64_t partial_cap = 0;
    void ensure_partial(int64_t doubles) const;
    int cap_rows = 0;
    int64_t cap_pieces = 0;
    // d_idx / idx_range (optional): the gathered index array and its range, for porder, which
    // is built when the gathered panel (panel_bytes) is larger than the L2
    void build(const int* d_ptr, int nrows, int64_t nnz, Scratch& scr, cudaStream_t st, const int* d_idx = nullptr,
               int idx_range = 0, size_t panel_bytes = 0);
    void reserve_pieces(int64_t need);  // piece arrays for >= need pieces
    void release();
    ~SegPlan() { release(); }
};

// The most frequent columns of a flush (per-flush frequency ranking): their input-panel rows
// are staged once per CTA in shared memory by TMA bulk copies, so every nonzero in those
// columns reads the panel row from SMEM instead of gathering it through L2. idx is the CSR
// column array relabelled for it: hot column -> its slot (< n), other column c -> n + c.
struct HotSet {
    const int* cols = nullptr;  // n column ids, device
    const int* idx = nullptr;   // relabelled CSR column indices, device
    int n = 0;
};

// Shared memory the hot rows of a panel `ncols` wide may use, and the resulting row count.
int hot_rows_capacity(int ncols);

void exclusive_scan(const int64_t* d_in, int64_t* d_out, int64_t n, Scratch& scr, cudaStream_t st);
void rebase_row_ptr(const int64_t* d_src, int64_t base, int m, int* d_dst, cudaStream_t st);
void build_transpose(DevCsr& a, Scratch& scr, cudaStream_t st);
// out (nrows x ncols, ldo) = sparse(ptr, idx, val) * in (ld), ncols even.
// in_rows / alg_cols (profiling only): rows of the input panel and the unpadded panel width,
// for the launch's declared algorithmic bytes 12 nnz + 8 (nrows + 1) + 8 alg_cols (in_rows + nrows)
// (SURVEY 8(d)); -1 = nrows / ncols.
// hot (optional): stage those input rows in shared memory (see HotSet); results are bit-identical.
void spmm(const int* d_ptr, const int* d_idx, const double* d_val, int nrows, const SegPlan& plan, int64_t nnz,
          const double* d_in, int ld, int ncols, double* d_out, int ldo, Scratch& scr, cudaStream_t st,
          int64_t in_rows = -1, int alg_cols = -1, const HotSet* hot = nullptr);
// slot (d ints) = -1 except slot[cols[i]] = i; idx2[k] = slot[col[k]] >= 0 ? slot : n + col[k].
void hot_relabel(const int* d_cols_hot, int n, const uint32_t* col, int64_t nnz, int d, int* slot, int* idx2,
                 cudaStream_t st);
// First invalid row (or -1) of a device-resident CSR batch; kind_out gets ERR_BAD_* bits.
int64_t validate_rows_device(const int64_t* d_row_ptr, int64_t nrows, const uint32_t* d_cols, const double* d_vals,
                             uint32_t d, int* kind_out, Scratch& scr, cudaStream_t st);

}  // namespace sfdg
