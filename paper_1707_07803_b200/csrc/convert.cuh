// Sparse -> MPO conversion structure (convert.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace mpob {

// Result of the single-device conversion of one nnz shard (sparse.py:234-250):
// per kept nonzero (input order) i1, j1, values and block id ti; the sorted
// unique block keys uniq (key = br + nrb * bc).
struct ConvLocal {
  DBuf<int64_t> i1, j1, ti, uniq;
  DBuf<double> values;
  int64_t nkept = 0;
  int64_t rank = 0;
  // lazy entries (fast path, no explicit zeros): i1, j1, values are derived
  // from the input on demand (ensure_entries); the input must outlive it --
  // host uploads are owned here, device inputs are the caller's
  bool lazy = false;
  const int64_t* src_row = nullptr;
  const int64_t* src_col = nullptr;
  const double* src_val = nullptr;
  int64_t I1 = 1, J1 = 1;
  DBuf<int64_t> own_row, own_col;
  DBuf<double> own_val;
};

// bucketed fast path (convert_fast.cu); false: not applicable (the caller
// takes the onesweep path), c untouched
bool convert_fast(cudaStream_t st, const int64_t* row1, const int64_t* col1, const double* val,
                  int64_t n, int64_t I1, int64_t J1, int64_t nrb, int64_t ncb, ConvLocal& c);
void ensure_entries(cudaStream_t st, ConvLocal& c);

ConvLocal convert_local(cudaStream_t st, const int64_t* row1, const int64_t* col1,
                        const double* val, int64_t n, int64_t I1, int64_t J1, int64_t nrb,
                        int64_t ncb);
void level_digits(cudaStream_t st, const int64_t* uniq, int64_t rank, int64_t nrb,
                  const std::vector<int64_t>& rf, const std::vector<int64_t>& cf, int level,
                  int64_t* rowd, int64_t* cold);
void exclusive_scan_u32(cudaStream_t st, const unsigned* in, int64_t n, int64_t* out,
                        int64_t* total_dev);
int key_bits(uint64_t max_key);
// stable LSD sort of (key, pay) on the low `bits` key bits; low_bits > 0
// lets it skip the passes below bit low_bits when the keys are found
// non-decreasing in those bits
void radix_sort_pairs(cudaStream_t st, uint64_t* key, unsigned* pay, int64_t n, int bits,
                      uint64_t* key_tmp, unsigned* pay_tmp, bool& result_in_tmp,
                      int low_bits = 0);

}  // namespace mpob

namespace mpob {
void conv_dense_core(cudaStream_t st, const ConvLocal& c, const std::vector<int64_t>& rf,
                     const std::vector<int64_t>& cf, int level, double* out);
// dense core `level` of the unit-rank terms of blocks [start, stop) (one
// chunk of the capped accumulation, sparse.py:262-271)
void conv_chunk_core(cudaStream_t st, const ConvLocal& c, const std::vector<int64_t>& rf,
                     const std::vector<int64_t>& cf, int level, int64_t start, int64_t stop,
                     double* out);
int64_t keys_unique(cudaStream_t st, const int64_t* keys, int64_t n, int64_t max_key,
                    int64_t* out);
void keys_lookup(cudaStream_t st, const int64_t* table, int64_t ntab, const int64_t* q,
                 int64_t nq, int64_t* out);
void keys_search(cudaStream_t st, const int64_t* table, int64_t ntab, const int64_t* q,
                 int64_t nq, int64_t offset, bool exact, int64_t* out);
void remap_ids(cudaStream_t st, const int64_t* map, int64_t* ti, int64_t n);
}  // namespace mpob
