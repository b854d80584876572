// verify.cuh -- persistent verifier kernel arguments (see verify.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sfdg {

struct VerifyArgs {
    // A' as CSR (u = A' x) and CSC (A'^T u)
    const int* row_ptr;
    const uint32_t* col;
    const double* val;
    const int* col_ptr;
    const int* row_idx;
    const double* cval;
    int64_t m, d;
    int64_t nnz;
    // B'^T: d x ell, row stride ldb (the right half of the [B | B']^T stack)
    const double* bt;
    int64_t ldb;
    int ell;
    double scale;      // 2 / Delta
    int steps;         // ceil(c_v log2(d / delta_i))   (shrink.cpp:81-82)
    const double* x0;  // d raw normals (unit_sphere_vector draws)
    // workspace
    double* u;      // m
    double* ybuf;   // 2 d
    double* tpart;  // nblocks * ell
    double* t;      // ell
    double* part;   // nblocks
    unsigned* bar;  // 2
    int* err;
    double* out;  // [accepted, log_mag, steps_run]
    int stage_bytes;  // dynamic shared memory for the block's CSR/CSC slices (0 = read from global)
    int resident;     // 1: also keep the block's B'^T rows in shared memory for all steps
    // Columns longer than 2 kPiece (skewed data: Zipf columns) are split into pieces that every
    // warp of the grid shares (the CSC SegPlan of the SpMM), summed per column in fixed order.
    int has_long;
    int piece;              // the plan's piece length: a column is long above 2 piece entries
    const int* long_cols;   // ascending column ids
    const int* long_first;  // first piece of each long column
    const int* piece_beg;
    const int* piece_end;
    const int* counts;      // [n_long, n_pieces] (device)
    double* lpart;          // n_pieces partial sums
    const int64_t* ccost;   // d + 1 column-cost prefix (verify_column_costs) or null: equal counts
    // CSR work plan of the kernel-sequence verifier's u = A' x (the SpMM's row SegPlan): pieces of
    // the long rows, summed in piece order by the piece that finishes last, then the short rows
    // longest first. Null r_counts: every row in natural order (no pieces).
    const int* r_counts;    // [nlong, npieces, nshort] (device)
    const int* r_piece_beg;
    const int* r_piece_end;
    const int* r_piece_li;
    const int* r_long_rows;
    const int* r_long_first;
    const int* r_order;
    double* r_part;         // npieces partial sums
    int* r_arrive;          // nlong arrival counters (zero between launches: self-resetting)
    // ... and of its w = A'^T u (the CSC SegPlan: long_cols / long_first / piece_* / counts above)
    const int* c_order;     // short columns longest first (null: natural order, no pieces)
    const int* c_piece_li;  // long-column index of each piece
    int* c_arrive;          // per long column arrival counters (self-resetting)
    double* w;              // d: w = A'^T u
};

class Scratch;
// Exclusive prefix of the per-column costs that balance the persistent verifier's column ranges.
void verify_column_costs(const int* d_col_ptr, int64_t d, int ell, int piece, int64_t* d_prefix, Scratch& scr,
                         cudaStream_t st);

int verify_grid_blocks(int device, int64_t d, int lp);  // cooperative grid for this B' size
// Smallest grid (>= the streaming grid, <= one block per SM) whose blocks can hold their
// B'^T rows and CSR/CSC slices in shared memory for the whole verification; 0 = none.
int verify_resident_blocks(int device, int64_t m, int64_t d, int ell, int64_t nnz, int min_blocks);
int verify_cluster_size(int64_t d, int lp);            // > 0: one cluster of that many CTAs instead
void verify_launch(const VerifyArgs& args, int nblocks, int cluster, cudaStream_t st);

// The verifier as a kernel sequence (three kernels per power step, no persistent grid; see
// verify.cu). verify_setup writes the per-call scalars (2 / Delta, steps) into `state`
// (verify_state_bytes() of device memory); verify_sequence enqueues the steps (the caller
// captures it once per step count as a CUDA graph). tpart: nblk * ell, part: nblk. Long columns
// (has_long) are summed from their pieces (one more kernel per step).
int verify_graph_blocks(int device, int64_t d);
size_t verify_state_bytes();
void verify_setup(void* state, double scale, int steps, cudaStream_t st);
void verify_sequence(const VerifyArgs& args, void* state, int nblk, int sms, cudaStream_t st);

}  // namespace sfdg
