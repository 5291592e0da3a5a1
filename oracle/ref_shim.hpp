// TEST INFRASTRUCTURE ONLY (oracle/_ref build). Force-included into
// oracle/ref_capi.cpp when compiling the unmodified reference headers.
//
// The reference's train.hpp:189-191 passes a bare `nullptr` to the
// `std::vector<DenseMatrix<T>>* x_grads_out` parameter of the function
// template backward_all_active (engine.hpp:177-185). Template argument
// deduction fails on nullptr_t, so no TU that includes train.hpp compiles.
// This overload accepts nullptr_t and forwards with a typed null pointer;
// the reference sources themselves are not modified.
#pragma once

#include <cstddef>
#include <vector>

#include "pathgcn/engine.hpp"

namespace pathgcn {

template <typename T>
std::vector<DenseMatrix<T>> backward_all_active(const GroupedCsr& graph,
                                                const EpochArtifacts<T>& arts,
                                                const DenseMatrix<T>& top_grad,
                                                const ModelParams<T>& params, CommitMode commit,
                                                int workers, WorkCounters& counters,
                                                std::nullptr_t, std::size_t col_chunk = 0) {
    return backward_all_active<T>(graph, arts, top_grad, params, commit, workers, counters,
                                  static_cast<std::vector<DenseMatrix<T>>*>(nullptr), col_chunk);
}

}  // namespace pathgcn
