// Reference-side drop-in for the B200 path: the adapter a maintainer adds to
// tesseract-sim (proj/src/b200_backend.cpp in their tree) so that existing
// callers -- verify sweeps, train_toy, the CLI -- run on B200 through the
// C-ABI (include/tess.h, libtess.so) with the reference's own types.
//
// Each function has the signature of the reference operator it replaces,
// plus the compute precision (TESS_F32: CUDA-core fp32, within 1e-5 of the
// fp64 reference; TESS_BF16: tcgen05 tensor cores, fp32 accumulate):
//   tesseract_matmul          algorithms.hpp:54-57
//   tesseract_backward_dense  algorithms.hpp:78-80
//   summa_matmul              algorithms.hpp:37  (= Tesseract on [q,q,1])
//   megatron_1d_linear        algorithms.hpp:86-87
//   layer_run                 layers.hpp:195-197
// Results carry the reference's CommStats, rebuilt exactly from the
// library's per-rank, per-kind counters with CommStats::add_send/add_recv
// (runtime.hpp:56-59), and, when TesseractOptions::record_trace is set, the
// reference's trace (runtime.hpp:74-85). Status codes come back as the
// reference's exception classes (error.hpp:11-48).
#pragma once

#include "tess.h"
#include "tsim/algorithms.hpp"
#include "tsim/layers.hpp"

namespace tsim::b200 {

AlgoResult tesseract_matmul(const Matrix& a, const Matrix& b, const GridSpec& grid,
                            MatmulVariant variant = MatmulVariant::NN,
                            const TesseractOptions& options = {},
                            tess_dtype compute = TESS_F32);

DenseBackwardResult tesseract_backward_dense(const Matrix& c_grad, const Matrix& a,
                                             const Matrix& b, const GridSpec& grid,
                                             tess_dtype compute = TESS_F32);

AlgoResult summa_matmul(const Matrix& a, const Matrix& b, int q, tess_dtype compute = TESS_F32);

AlgoResult megatron_1d_linear(const Matrix& x, const Matrix& w1, const Matrix& w2, int p,
                              tess_dtype compute = TESS_F32);

LayerRunResult layer_run(LayerOp op, const Matrix& x, const Matrix& dy, const BlockParams& params,
                         const LayerDims& dims, const GridSpec& grid,
                         tess_dtype compute = TESS_F32);

}  // namespace tsim::b200
