// bm25.cu -- GPU BM25 scoring feeding K4.
//
// score[q][u] = sum over the query's terms t, in query order, of
//               idf[t] * tf[t][u] * (k1 + 1) / (tf[t][u] + norm[u])
// exactly as Bm25Index.score (retrieval.py:129-141): float64, the same
// association, no FMA contraction (__dmul_rn / __dadd_rn / __ddiv_rn are
// correctly rounded like the host's IEEE ops), terms absent from a unit
// skipped.  idf and norm come from the host (math.log on the host), so the
// scores are bit-identical to the reference's.
#include <cuda_runtime.h>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"

namespace dbsa {

// grid (ceil(n_units / 128), n_queries), 128 threads: one thread per (query, unit).
__global__ void bm25_kernel(const int32_t *__restrict__ terms, int32_t max_terms, const uint16_t *__restrict__ tf,
                            const double *__restrict__ idf, const double *__restrict__ norm, int64_t n_units,
                            double k1p1, double *__restrict__ out) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (u >= n_units) return;
  const int32_t *qt = terms + (int64_t)q * max_terms;
  const double nu = norm[u];
  double acc = 0.0;
  for (int i = 0; i < max_terms; ++i) {
    const int32_t t = qt[i];
    if (t < 0) continue;  // padding or a term absent from the index vocabulary
    const uint16_t f16 = tf[(int64_t)t * n_units + u];
    if (f16 == 0) continue;
    const double f = (double)f16;
    const double num = __dmul_rn(__dmul_rn(idf[t], f), k1p1);
    acc = __dadd_rn(acc, __ddiv_rn(num, __dadd_rn(f, nu)));
  }
  out[(int64_t)q * n_units + u] = acc;
}

}  // namespace dbsa

extern "C" int dbsa_bm25_scores(const int32_t *term_ids, int64_t n_queries, int32_t max_terms, const uint16_t *tf,
                                const double *idf, const double *norm, int64_t n_units, double k1p1, double *out,
                                void *stream) {
  using namespace dbsa;
  if (n_queries < 0 || n_units < 1 || max_terms < 0)
    return set_error(DBSA_ERR_VALIDATION, "bm25: bad sizes (queries %lld, units %lld, terms %d)",
                     (long long)n_queries, (long long)n_units, max_terms);
  if (n_queries == 0) return DBSA_OK;
  if (n_queries > 65535) return set_error(DBSA_ERR_SHAPE, "bm25: at most 65535 queries per launch");
  dim3 grid((unsigned)((n_units + 127) / 128), (unsigned)n_queries);
  bm25_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(term_ids, max_terms, tf, idf, norm, n_units,
                                                                        k1p1, out);
  return check_launch("bm25_scores");
}
