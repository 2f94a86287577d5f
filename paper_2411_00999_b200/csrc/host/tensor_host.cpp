// tensor_host.cpp — host implementation of the drop-in gnstk::Tensor
// (include/gnstk/tensor.hpp).  Semantics follow the reference's
// proj/src/tensor.cpp: "tensor: " error prefix (:12-14), row-major strides
// (:52-56), contract's loop order — output labels row-major, then summed labels
// by first appearance with the last varying fastest, repeated labels walking
// the diagonal (:94-205) — trailing-axis broadcasting (:219-271) and
// reductions that visit the reduced axes row-major (:302-360).  The same
// visiting order gives bit-identical sums.
//
// Every loop nest here is one `Odometer`: a multi-index over `dims` with a
// per-stream stride table, advanced last axis fastest, that keeps one flat
// offset per stream.
#include <algorithm>
#include <cctype>
#include <stdexcept>
#include <string>

#include "gnstk/tensor.hpp"

namespace gnstk {
namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument("tensor: " + msg); }

Index checked_numel(const Shape& s) {
    Index n = 1;
    for (Index e : s) {
        if (e < 0) fail("negative extent");
        n *= e;
    }
    return n;
}

struct Odometer {
    std::vector<Index> dims;
    std::vector<std::vector<Index>> stride;  // [stream][axis]
    std::vector<Index> idx;
    std::vector<Index> off;                  // [stream]

    Odometer(std::vector<Index> d, std::size_t streams)
        : dims(std::move(d)), stride(streams, std::vector<Index>(dims.size(), 0)), idx(dims.size(), 0),
          off(streams, 0) {}

    /// Advance axes [lo, hi) by one (hi - 1 fastest); false when they wrap to zero.
    bool next(std::size_t lo, std::size_t hi) {
        for (std::size_t a = hi; a-- > lo;) {
            ++idx[a];
            for (std::size_t s = 0; s < off.size(); ++s) off[s] += stride[s][a];
            if (idx[a] < dims[a]) return true;
            for (std::size_t s = 0; s < off.size(); ++s) off[s] -= idx[a] * stride[s][a];
            idx[a] = 0;
        }
        return false;
    }
};

}  // namespace

// ----------------------------------------------------------------- class --
Tensor::Tensor(Shape shape) : shape_(std::move(shape)) {
    data_.assign(static_cast<std::size_t>(checked_numel(shape_)), 0.0);
    init_strides();
}

Tensor::Tensor(Shape shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (checked_numel(shape_) != static_cast<Index>(data_.size())) fail("data length does not match shape product");
    init_strides();
}

Tensor Tensor::scalar(double v) { return Tensor(Shape{}, std::vector<double>{v}); }

Tensor Tensor::full(Shape shape, double v) {
    Tensor t(std::move(shape));
    std::fill(t.data_.begin(), t.data_.end(), v);
    return t;
}

void Tensor::init_strides() {
    strides_.resize(shape_.size());
    Index s = 1;
    for (std::size_t a = shape_.size(); a-- > 0;) {
        strides_[a] = s;
        s *= shape_[a];
    }
}

double& Tensor::at(std::span<const Index> idx) {
    if (static_cast<Index>(idx.size()) != rank()) fail("index rank mismatch");
    Index flat = 0;
    for (std::size_t a = 0; a < idx.size(); ++a) {
        if (idx[a] < 0 || idx[a] >= shape_[a]) fail("index out of bounds");
        flat += idx[a] * strides_[a];
    }
    return data_[static_cast<std::size_t>(flat)];
}

double Tensor::at(std::span<const Index> idx) const { return const_cast<Tensor*>(this)->at(idx); }

double Tensor::item() const {
    if (data_.size() != 1) fail("item() requires a single-element tensor");
    return data_[0];
}

// -------------------------------------------------------------- contract --
Tensor contract(std::string_view spec, std::span<const Tensor> ops) {
    if (ops.empty()) fail("contract needs at least one operand");
    const std::size_t arrow = spec.find("->");
    if (arrow == std::string_view::npos) fail("contraction spec needs '->'");
    std::vector<std::string> in(1);
    for (char c : spec.substr(0, arrow)) {
        if (c == ',')
            in.emplace_back();
        else if (std::isalpha(static_cast<unsigned char>(c)))
            in.back().push_back(c);
        else
            fail(std::string("invalid character in spec: '") + c + "'");
    }
    std::string out_labels;
    for (char c : spec.substr(arrow + 2)) {
        if (!std::isalpha(static_cast<unsigned char>(c))) fail(std::string("invalid character in spec: '") + c + "'");
        if (out_labels.find(c) != std::string::npos) fail("repeated label in output");
        out_labels.push_back(c);
    }
    if (in.size() != ops.size()) fail("operand count does not match spec");

    // distinct labels by first appearance, with their extents
    std::string labels;
    std::vector<Index> extent;
    for (std::size_t o = 0; o < ops.size(); ++o) {
        if (static_cast<Index>(in[o].size()) != ops[o].rank()) fail("operand rank does not match spec");
        for (std::size_t a = 0; a < in[o].size(); ++a) {
            const std::size_t p = labels.find(in[o][a]);
            const Index e = ops[o].shape()[a];
            if (p == std::string::npos) {
                labels.push_back(in[o][a]);
                extent.push_back(e);
            } else if (extent[p] != e) {
                fail(std::string("extent mismatch on label '") + in[o][a] + "'");
            }
        }
    }
    for (char c : out_labels)
        if (labels.find(c) == std::string::npos) fail(std::string("output label '") + c + "' absent from inputs");

    std::string loop = out_labels;  // output axes, then summed labels by first appearance
    for (char c : labels)
        if (out_labels.find(c) == std::string::npos) loop.push_back(c);
    std::vector<Index> dims;
    for (char c : loop) dims.push_back(extent[labels.find(c)]);
    Odometer od(dims, ops.size());
    for (std::size_t o = 0; o < ops.size(); ++o)
        for (std::size_t a = 0; a < in[o].size(); ++a)
            od.stride[o][loop.find(in[o][a])] += ops[o].strides()[a];  // repeated labels: the diagonal

    const std::size_t n_out = out_labels.size();
    Tensor out(Shape(dims.begin(), dims.begin() + static_cast<std::ptrdiff_t>(n_out)));
    Index n_sum = 1;
    for (std::size_t a = n_out; a < dims.size(); ++a) n_sum *= dims[a];
    if (out.size() == 0 || n_sum == 0) return out;

    for (Index f = 0; f < out.size(); ++f) {
        double acc = 0.0;
        do {
            double term = 1.0;
            for (std::size_t o = 0; o < ops.size(); ++o) term *= ops[o].data()[od.off[o]];
            acc += term;
        } while (od.next(n_out, dims.size()));
        out[f] = acc;
        // summed axes are back at zero; step the output axes
        od.next(0, n_out);
    }
    return out;
}

Tensor contract(std::string_view spec, const Tensor& a) { return contract(spec, std::span<const Tensor>(&a, 1)); }

Tensor contract(std::string_view spec, const Tensor& a, const Tensor& b) {
    const Tensor ops[2] = {a, b};
    return contract(spec, std::span<const Tensor>(ops, 2));
}

// ----------------------------------------------------------- elementwise --
namespace {

template <typename F>
Tensor broadcast_binary(const Tensor& a, const Tensor& b, F f) {
    if (a.same_shape(b)) {
        Tensor r(a.shape());
        for (Index i = 0; i < r.size(); ++i) r[i] = f(a[i], b[i]);
        return r;
    }
    const std::size_t rank = std::max(a.shape().size(), b.shape().size());
    auto ext = [rank](const Tensor& t, std::size_t axis) -> Index {  // implied leading 1s
        const std::size_t lead = rank - t.shape().size();
        return axis < lead ? 1 : t.shape()[axis - lead];
    };
    Shape shape(rank);
    for (std::size_t i = 0; i < rank; ++i) {
        const Index ea = ext(a, i), eb = ext(b, i);
        if (ea != eb && ea != 1 && eb != 1) fail("shapes not broadcast-compatible");
        shape[i] = ea == 1 ? eb : ea;
    }
    Tensor r(shape);
    if (r.size() == 0) return r;
    Odometer od(shape, 2);
    const Tensor* t[2] = {&a, &b};
    for (std::size_t s = 0; s < 2; ++s) {
        const std::size_t lead = rank - t[s]->shape().size();
        for (std::size_t i = lead; i < rank; ++i)
            if (t[s]->shape()[i - lead] != 1) od.stride[s][i] = t[s]->strides()[i - lead];
    }
    Index i = 0;
    do {
        r[i++] = f(a.data()[od.off[0]], b.data()[od.off[1]]);
    } while (od.next(0, rank));
    return r;
}

enum class Red { Sum, Mean, Sqnorm };

Tensor reduce(const Tensor& a, std::span<const Index> axes, Red op) {
    std::vector<char> red(static_cast<std::size_t>(a.rank()), 0);
    for (Index ax : axes) {
        if (ax < 0 || ax >= a.rank()) fail("reduction axis out of range");
        if (red[static_cast<std::size_t>(ax)]) fail("duplicate reduction axis");
        red[static_cast<std::size_t>(ax)] = 1;
    }
    // kept axes first (the output, row-major), reduced axes after (row-major)
    std::vector<Index> dims, st;
    Shape kept;
    for (int pass = 0; pass < 2; ++pass)
        for (std::size_t d = 0; d < red.size(); ++d)
            if (red[d] == pass) {
                dims.push_back(a.shape()[d]);
                st.push_back(a.strides()[d]);
                if (!pass) kept.push_back(a.shape()[d]);
            }
    const std::size_t n_keep = kept.size();
    Index n_red = 1;
    for (std::size_t d = n_keep; d < dims.size(); ++d) n_red *= dims[d];
    if (op == Red::Mean && a.size() == 0) fail("mean reduction over an empty tensor");
    Tensor out(kept);
    if (out.size() == 0) return out;
    if (n_red == 0) return out;
    Odometer od(dims, 1);
    od.stride[0] = st;
    for (Index f = 0; f < out.size(); ++f) {
        double acc = 0.0;
        do {
            const double v = a.data()[od.off[0]];
            acc += op == Red::Sqnorm ? v * v : v;
        } while (od.next(n_keep, dims.size()));
        out[f] = op == Red::Mean ? acc / static_cast<double>(n_red) : acc;
        od.next(0, n_keep);
    }
    return out;
}

std::vector<Index> every_axis(const Tensor& a) {
    std::vector<Index> ax(static_cast<std::size_t>(a.rank()));
    for (std::size_t i = 0; i < ax.size(); ++i) ax[i] = static_cast<Index>(i);
    return ax;
}

}  // namespace

Tensor add(const Tensor& a, const Tensor& b) {
    return broadcast_binary(a, b, [](double x, double y) { return x + y; });
}
Tensor sub(const Tensor& a, const Tensor& b) {
    return broadcast_binary(a, b, [](double x, double y) { return x - y; });
}
Tensor mul(const Tensor& a, const Tensor& b) {
    return broadcast_binary(a, b, [](double x, double y) { return x * y; });
}
Tensor square(const Tensor& a) {
    Tensor r(a.shape());
    for (Index i = 0; i < r.size(); ++i) r[i] = a[i] * a[i];
    return r;
}
Tensor scale(const Tensor& a, double c) {
    Tensor r(a.shape());
    for (Index i = 0; i < r.size(); ++i) r[i] = a[i] * c;
    return r;
}

Tensor reduce_sum(const Tensor& a, std::span<const Index> axes) { return reduce(a, axes, Red::Sum); }
Tensor reduce_mean(const Tensor& a, std::span<const Index> axes) { return reduce(a, axes, Red::Mean); }
Tensor reduce_sqnorm(const Tensor& a, std::span<const Index> axes) { return reduce(a, axes, Red::Sqnorm); }
double sum_all(const Tensor& a) { return reduce(a, every_axis(a), Red::Sum).item(); }
double mean_all(const Tensor& a) { return reduce(a, every_axis(a), Red::Mean).item(); }
double sqnorm_all(const Tensor& a) { return reduce(a, every_axis(a), Red::Sqnorm).item(); }

}  // namespace gnstk
