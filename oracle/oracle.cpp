// oracle/oracle.cpp -- CPU oracle for the BRMerge SpGEMM hot path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load, call, link or
// execute anything under oracle/. The product path (paper_2206_06611_b200/)
// never imports it and shares no code, header, table or helper with it.
//
// Plain, slow, single-threaded, obviously correct; fp64 everywhere, compiled
// with -ffp-contract=off so every product is rounded before it is added.
// Citations are to /root/reference/PAPER.md (arxiv 2206.06611):
//   Eq. (2)  PAPER.md:95  "C_{i*} = sum_k A_ik * B_k*"  (row-wise dataflow)
//   Alg. 1   PAPER.md:165-218  BRMerge accumulation method
//   §II.B.2  PAPER.md:143  "computes the number of intermediate products
//            (n_prod) per output row"
//   Fig. 2   PAPER.md:158  "vals with duplicate cols are combined into one
//            val ... merged two by two in a tree-like hierarchy"
//
// Explicit zeros produced by cancellation are KEPT (the paper's accumulators
// merge by index only; reading R3).
//
// Pins (tests/test_oracle_pins.py): dense matmul on tiny inputs, identity and
// permutation invariants, nnz(C_i) <= n_prod_i, closed forms for the 27-point
// stencil and the 5-point-Laplacian x aggregation product, exact-integer
// agreement of both accumulation orders, Fig. 2 round count.
#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

namespace {

struct Result {
  int64_t rows = 0;
  std::vector<int64_t> rpt;
  std::vector<int32_t> col;
  std::vector<double> val;
  std::vector<int32_t> rounds;  // BRMerge only: merge rounds per output row
};

// One output row by Eq. (2), accumulating in a sorted map keyed by column.
// Products are added in k order (the order of A's row).
void gustavson_row(int64_t i, const int64_t* arpt, const int32_t* acol,
                   const double* aval, const int64_t* brpt, const int32_t* bcol,
                   const double* bval, Result& r) {
  std::map<int32_t, double> acc;
  for (int64_t p = arpt[i]; p < arpt[i + 1]; ++p) {
    const int32_t k = acol[p];
    const double a = aval[p];
    for (int64_t q = brpt[k]; q < brpt[k + 1]; ++q) {
      const double prod = a * bval[q];
      auto it = acc.find(bcol[q]);
      if (it == acc.end())
        acc.emplace(bcol[q], prod);
      else
        it->second = it->second + prod;
    }
  }
  for (const auto& kv : acc) {
    r.col.push_back(kv.first);
    r.val.push_back(kv.second);
  }
  r.rpt.push_back(static_cast<int64_t>(r.col.size()));
}

// "consume two lists and store to dst_buffer" (Alg. 1 line 25): the
// merge-sort merge of two column-sorted lists, "except that the vals with
// duplicate cols are combined into one val" (Fig. 2 caption).
int64_t merge_two(int64_t la, const int32_t* ac, const double* av, int64_t lb,
                  const int32_t* bc, const double* bv, int32_t* oc, double* ov) {
  int64_t i = 0, j = 0, n = 0;
  while (i < la && j < lb) {
    if (ac[i] < bc[j]) {
      oc[n] = ac[i]; ov[n] = av[i]; ++i;
    } else if (bc[j] < ac[i]) {
      oc[n] = bc[j]; ov[n] = bv[j]; ++j;
    } else {
      oc[n] = ac[i]; ov[n] = av[i] + bv[j]; ++i; ++j;
    }
    ++n;
  }
  while (i < la) { oc[n] = ac[i]; ov[n] = av[i]; ++i; ++n; }
  while (j < lb) { oc[n] = bc[j]; ov[n] = bv[j]; ++j; ++n; }
  return n;
}

// Algorithm 1, one output row i, step by step in the paper's order and names.
// `trace` (optional) receives the total live element count after the
// multiplying phase and after every merge round.
int brmerge_row(int64_t i, const int64_t* arpt, const int32_t* acol,
                const double* aval, const int64_t* brpt, const int32_t* bcol,
                const double* bval, std::vector<int32_t>& ping_col,
                std::vector<double>& ping_val, std::vector<int32_t>& pong_col,
                std::vector<double>& pong_val, std::vector<int64_t>& ping_list_offset,
                std::vector<int64_t>& pong_list_offset, Result& r,
                std::vector<int64_t>* trace) {
  // Lines 7-9
  int32_t* dst_col = ping_col.data();
  double* dst_val = ping_val.data();
  int64_t* dst_list_offset = ping_list_offset.data();
  int64_t buffer_incr = 0, list_incr = 0;
  dst_list_offset[0] = 0;
  // Lines 10-15: multiplying phase.
  for (int64_t p = arpt[i]; p < arpt[i + 1]; ++p) {
    const int32_t k = acol[p];
    for (int64_t q = brpt[k]; q < brpt[k + 1]; ++q) {
      dst_col[buffer_incr] = bcol[q];
      dst_val[buffer_incr] = aval[p] * bval[q];
      ++buffer_incr;
    }
    dst_list_offset[++list_incr] = buffer_incr;
  }
  if (trace) trace->push_back(buffer_incr);
  // Lines 16-20
  int64_t num_list = list_incr;
  int32_t* src_col = dst_col;
  double* src_val = dst_val;
  int64_t* src_list_offset = dst_list_offset;
  dst_col = pong_col.data();
  dst_val = pong_val.data();
  dst_list_offset = pong_list_offset.data();
  int rounds = 0;
  // Lines 21-35: accumulating phase.
  while (num_list > 1) {
    int64_t inner_num_list = num_list;
    num_list = 0;
    int64_t li = 0;  // next unconsumed source list
    dst_list_offset[0] = 0;
    int64_t out = 0;
    while (inner_num_list) {
      if (inner_num_list >= 2) {
        const int64_t a0 = src_list_offset[li], a1 = src_list_offset[li + 1],
                      b1 = src_list_offset[li + 2];
        out += merge_two(a1 - a0, src_col + a0, src_val + a0, b1 - a1, src_col + a1,
                         src_val + a1, dst_col + out, dst_val + out);
        inner_num_list -= 2;
        li += 2;
      } else if (inner_num_list == 1) {  // copy the last list to dst_buffer
        const int64_t a0 = src_list_offset[li], a1 = src_list_offset[li + 1];
        for (int64_t e = a0; e < a1; ++e) {
          dst_col[out] = src_col[e];
          dst_val[out] = src_val[e];
          ++out;
        }
        inner_num_list -= 1;
        li += 1;
      }
      dst_list_offset[++num_list] = out;
    }
    // Lines 33-34: swap roles without data movement.
    std::swap(src_col, dst_col);
    std::swap(src_val, dst_val);
    std::swap(src_list_offset, dst_list_offset);
    ++rounds;
    if (trace) trace->push_back(out);
  }
  // Line 36: store the i-th result row (it is in src after the last swap).
  const int64_t n = num_list == 0 ? 0 : src_list_offset[1];
  for (int64_t e = 0; e < n; ++e) {
    r.col.push_back(src_col[e]);
    r.val.push_back(src_val[e]);
  }
  r.rpt.push_back(static_cast<int64_t>(r.col.size()));
  return rounds;
}

}  // namespace

extern "C" {

// §II.B.2 / Alg. 1 line 1: n_prod of every output row,
// nprod[i] = sum_{k in A_i*} nnz(B_k*). Returns the total.
int64_t oracle_row_nprod(int64_t M, const int64_t* arpt, const int32_t* acol,
                         const int64_t* brpt, int64_t* nprod) {
  int64_t total = 0;
  for (int64_t i = 0; i < M; ++i) {
    int64_t s = 0;
    for (int64_t p = arpt[i]; p < arpt[i + 1]; ++p) s += brpt[acol[p] + 1] - brpt[acol[p]];
    nprod[i] = s;
    total += s;
  }
  return total;
}

// Row sizes only: nnz(C_i*) = |{ j : exists k in A_i* with j in B_k* }|, the
// pattern of Eq. (2) with structural zeros kept (reading R3),
// counted with a "last row seen" stamp per column (a plain set-membership
// array of B.cols entries) -- the definition, without the values. For the
// listed rows (all when null), out[t] = size of row rows[t].
void oracle_row_sizes(int64_t M, const int64_t* arpt, const int32_t* acol, const int64_t* brpt,
                      const int32_t* bcol, int64_t ncols, const int64_t* rows, int64_t nrows,
                      int64_t* out) {
  std::vector<int64_t> seen(ncols > 0 ? ncols : 1, -1);
  const int64_t n = rows ? nrows : M;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = rows ? rows[t] : t;
    int64_t count = 0;
    for (int64_t p = arpt[i]; p < arpt[i + 1]; ++p) {
      const int32_t k = acol[p];
      for (int64_t q = brpt[k]; q < brpt[k + 1]; ++q) {
        if (seen[bcol[q]] != t) {
          seen[bcol[q]] = t;
          ++count;
        }
      }
    }
    out[t] = count;
  }
}

// Eq. (2) with a sorted-map accumulator for the listed rows (all rows when
// rows == nullptr). Result rows appear in the order of `rows`.
void* oracle_gustavson(int64_t M, const int64_t* arpt, const int32_t* acol,
                       const double* aval, const int64_t* brpt, const int32_t* bcol,
                       const double* bval, const int64_t* rows, int64_t nrows) {
  Result* r = new Result;
  const int64_t n = rows ? nrows : M;
  r->rows = n;
  r->rpt.reserve(n + 1);
  r->rpt.push_back(0);
  for (int64_t t = 0; t < n; ++t)
    gustavson_row(rows ? rows[t] : t, arpt, acol, aval, brpt, bcol, bval, *r);
  return r;
}

// Algorithm 1 (BRMerge accumulation) for the listed rows (all when null).
// Buffers are sized once by max_row_nprod_C / max_row_nnz_A (lines 1-5) and
// reused for every row (reading R2).
void* oracle_brmerge(int64_t M, const int64_t* arpt, const int32_t* acol,
                     const double* aval, const int64_t* brpt, const int32_t* bcol,
                     const double* bval, const int64_t* rows, int64_t nrows) {
  Result* r = new Result;
  const int64_t n = rows ? nrows : M;
  r->rows = n;
  // Line 1: max_row_nprod_C, max_row_nnz_A over the rows computed.
  int64_t max_row_nprod_C = 0, max_row_nnz_A = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = rows ? rows[t] : t;
    int64_t s = 0;
    for (int64_t p = arpt[i]; p < arpt[i + 1]; ++p) s += brpt[acol[p] + 1] - brpt[acol[p]];
    if (s > max_row_nprod_C) max_row_nprod_C = s;
    if (arpt[i + 1] - arpt[i] > max_row_nnz_A) max_row_nnz_A = arpt[i + 1] - arpt[i];
  }
  // Lines 2-5.
  std::vector<int32_t> ping_col(max_row_nprod_C + 1), pong_col(max_row_nprod_C + 1);
  std::vector<double> ping_val(max_row_nprod_C + 1), pong_val(max_row_nprod_C + 1);
  std::vector<int64_t> ping_list_offset(max_row_nnz_A + 1), pong_list_offset(max_row_nnz_A + 1);
  r->rpt.reserve(n + 1);
  r->rpt.push_back(0);
  r->rounds.reserve(n);
  for (int64_t t = 0; t < n; ++t)
    r->rounds.push_back(brmerge_row(rows ? rows[t] : t, arpt, acol, aval, brpt, bcol,
                                    bval, ping_col, ping_val, pong_col, pong_val,
                                    ping_list_offset, pong_list_offset, *r, nullptr));
  return r;
}

// Live element totals of one row: after the multiplying phase, then after
// each merge round. Returns the number of entries written (rounds + 1).
int64_t oracle_brmerge_trace(const int64_t* arpt, const int32_t* acol, const double* aval,
                             const int64_t* brpt, const int32_t* bcol, const double* bval,
                             int64_t row, int64_t* totals, int64_t cap) {
  int64_t s = 0;
  for (int64_t p = arpt[row]; p < arpt[row + 1]; ++p) s += brpt[acol[p] + 1] - brpt[acol[p]];
  const int64_t la = arpt[row + 1] - arpt[row];
  std::vector<int32_t> pc(s + 1), qc(s + 1);
  std::vector<double> pv(s + 1), qv(s + 1);
  std::vector<int64_t> po(la + 1), qo(la + 1);
  Result r;
  r.rpt.push_back(0);
  std::vector<int64_t> trace;
  brmerge_row(row, arpt, acol, aval, brpt, bcol, bval, pc, pv, qc, qv, po, qo, r, &trace);
  const int64_t n = static_cast<int64_t>(trace.size()) < cap ? trace.size() : cap;
  for (int64_t e = 0; e < n; ++e) totals[e] = trace[e];
  return static_cast<int64_t>(trace.size());
}

// Fig. 2 merge of two lists, exposed for unit pins.
int64_t oracle_merge_two(int64_t la, const int32_t* ac, const double* av, int64_t lb,
                         const int32_t* bc, const double* bv, int32_t* oc, double* ov) {
  return merge_two(la, ac, av, lb, bc, bv, oc, ov);
}

int64_t oracle_result_nnz(void* h) { return static_cast<Result*>(h)->rpt.back(); }
int64_t oracle_result_rows(void* h) { return static_cast<Result*>(h)->rows; }

void oracle_result_copy(void* h, int64_t* rpt, int32_t* col, double* val, int32_t* rounds) {
  const Result* r = static_cast<Result*>(h);
  std::memcpy(rpt, r->rpt.data(), r->rpt.size() * sizeof(int64_t));
  if (!r->col.empty()) {
    std::memcpy(col, r->col.data(), r->col.size() * sizeof(int32_t));
    std::memcpy(val, r->val.data(), r->val.size() * sizeof(double));
  }
  if (rounds && !r->rounds.empty())
    std::memcpy(rounds, r->rounds.data(), r->rounds.size() * sizeof(int32_t));
}

void oracle_result_free(void* h) { delete static_cast<Result*>(h); }

}  // extern "C"
