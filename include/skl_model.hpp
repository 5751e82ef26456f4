/*
 * skl_model.hpp -- model files (the reference's JSON manifest + 'PNTR' blob)
 * in C++, for Linear / SKLinear / ReLU chains: model_load -> skl::Model whose
 * forward() is model_forward on the device.
 *
 * Reference (/root/reference/proj/src/nn_model.cpp):
 *   model_load                          :448-531 (guards :453-466)
 *   sk_linear_from_json (descriptors)   :290-311
 *   blob layout, Linear w then b         :405-407, 473-481
 *   model_forward                        :111-122
 * SKLinear sketches are re-realised on the GPU from their (dist, rows, cols,
 * seed) descriptors -- bit-identical to SketchOp::realized -- under the same
 * rng_algorithm guard.  Errors are skl::load_error (rnla::nn::load_error,
 * errors.hpp:40-45) and skl::shape_error for a layer that is not part of a
 * Linear/ReLU chain.
 *
 * Needs nlohmann/json.hpp on the include path (the reference's own JSON
 * library; this image ships a copy with cudnn_frontend).
 */
#ifndef SKL_MODEL_HPP_
#define SKL_MODEL_HPP_

#include <nlohmann/json.hpp>

#include <cstring>
#include <fstream>
#include <iterator>

#include "skl_chain.hpp"

namespace skl {

struct load_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Model {
    std::string dtype;               // file precision: "f32" / "f64"
    std::vector<std::string> names;  // layer names, file order
    std::unique_ptr<Chain> chain;    // the Linear / SKLinear / ReLU layers on the device

    // model_forward (nn_model.cpp:111-122): x [T, d_in] -> y [T, d_out] (internal buffer).
    const void* forward(const void* x, int64_t T, cudaStream_t st = nullptr) {
        return chain->forward(x, T, st, /*train=*/false);
    }
};

namespace detail {
class BlobReader {  // nn_model.cpp:196-246
  public:
    BlobReader(const std::vector<unsigned char>& b, bool f32, size_t pos) : b_(b), f32_(f32), pos_(pos) {}
    std::vector<double> read(size_t n) {
        const size_t w = f32_ ? 4 : 8;
        if (pos_ + n * w > b_.size()) throw load_error("model blob too short for declared layers");
        std::vector<double> out(n);
        for (size_t i = 0; i < n; ++i) {
            if (f32_) {
                float f;
                std::memcpy(&f, b_.data() + pos_ + 4 * i, 4);
                out[i] = f;
            } else {
                std::memcpy(&out[i], b_.data() + pos_ + 8 * i, 8);
            }
        }
        pos_ += n * w;
        return out;
    }
    size_t pos() const { return pos_; }

  private:
    const std::vector<unsigned char>& b_;
    bool f32_;
    size_t pos_;
};
}  // namespace detail

// model_load(path) on the device in element type `dtype`.
inline Model model_load(const std::string& path, skl_dtype dtype = SKL_BF16) {
    using nlohmann::json;
    std::ifstream in(path, std::ios::binary);
    if (!in) throw load_error("model_load: cannot open " + path);
    const std::string manifest((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    json root;
    try {
        root = json::parse(manifest);
    } catch (const json::exception& e) {
        throw load_error(std::string("model_load: malformed manifest: ") + e.what());
    }
    Model m;
    std::vector<Chain::Layer> layers;
    try {
        if (root.at("format_version").get<int>() != 1) throw load_error("model_load: unsupported format_version");
        if (root.at("rng_algorithm").get<std::string>() != skl_rng_algorithm())
            throw load_error("model_load: manifest uses an unknown rng_algorithm");
        m.dtype = root.at("dtype").get<std::string>();
        if (m.dtype != "f64" && m.dtype != "f32") throw load_error("model_load: unsupported dtype " + m.dtype);
        std::ifstream bin(path + ".bin", std::ios::binary);  // blob_path_for, nn_model.cpp:392
        if (!bin) throw load_error("model_load: cannot open " + path + ".bin");
        const std::vector<unsigned char> blob((std::istreambuf_iterator<char>(bin)), std::istreambuf_iterator<char>());
        if (blob.size() < 5 || std::memcmp(blob.data(), "PNTR", 4) != 0) throw load_error("model_load: bad blob magic");
        if (blob[4] != 1) throw load_error("model_load: unsupported blob version");
        detail::BlobReader rd(blob, m.dtype == "f32", 5);
        for (const json& j : root.at("layers")) {
            const std::string name = j.at("name").get<std::string>(), type = j.at("type").get<std::string>();
            for (const auto& n : m.names)
                if (n == name) throw load_error("model_load: duplicate layer name " + name);
            if (type == "SKLinear") {
                const int64_t d_in = j.at("d_in"), d_out = j.at("d_out"), l = j.at("num_terms"),
                              k = j.at("low_rank");
                std::vector<SkLinear::SketchDesc> descs;
                for (const json& s : j.at("sketches")) {
                    const std::string dist = s.at("dist").get<std::string>();
                    if (dist != "gaussian" && dist != "rademacher")
                        throw parameter_error("SKLinear: sketch distribution " + dist + " is not on this path");
                    descs.push_back({dist == "gaussian" ? SKL_DIST_GAUSSIAN : SKL_DIST_RADEMACHER,
                                     s.at("rows").get<int64_t>(), s.at("cols").get<int64_t>(),
                                     s.at("seed").get<uint64_t>()});
                }
                if ((int64_t)descs.size() != 2 * l) throw load_error("SKLinear manifest: expected 2*num_terms sketches");
                std::vector<double> u1((size_t)(l * k * d_in)), u2((size_t)(l * d_out * k));
                for (int64_t i = 0; i < l; ++i) {  // blob: u1_0, u2_0, u1_1, u2_1, ..., bias
                    const auto a = rd.read((size_t)(k * d_in));
                    std::copy(a.begin(), a.end(), u1.begin() + i * k * d_in);
                    const auto b = rd.read((size_t)(d_out * k));
                    std::copy(b.begin(), b.end(), u2.begin() + i * d_out * k);
                }
                const auto bias = rd.read((size_t)d_out);
                layers.emplace_back(
                    SkLinear::from_parts(d_in, d_out, l, k, dtype, descs, u1.data(), u2.data(), bias.data()));
            } else if (type == "Linear") {
                const int64_t d_in = j.at("d_in"), d_out = j.at("d_out");
                const auto w = rd.read((size_t)(d_out * d_in));
                const auto b = rd.read((size_t)d_out);
                layers.emplace_back(DenseLinear::from_parts(d_in, d_out, dtype, w.data(), b.data()));
            } else if (type == "ReLU") {
                layers.emplace_back(Relu{});
            } else {
                // Conv2d / SKConv2d / attention: loadable in the reference, but not part of a
                // Linear/ReLU chain (model_forward throws shape_error for them, nn_model.cpp:117-119)
                throw shape_error("model_load: layer '" + name + "' (" + type +
                                  ") is not part of a Linear/ReLU chain");
            }
            m.names.push_back(name);
        }
        if (rd.pos() != blob.size()) throw load_error("model_load: blob length does not match manifest");
    } catch (const json::exception& e) {
        throw load_error(std::string("model_load: malformed manifest: ") + e.what());
    }
    m.chain = std::make_unique<Chain>(std::move(layers));
    return m;
}

}  // namespace skl

#endif  // SKL_MODEL_HPP_
