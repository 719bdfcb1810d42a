// SAAPTNS1 artifact I/O: the reference CLI's partition,
// IVF and Q-model files, read straight into device partitions / Q-models.
//
// Format (tensor_io.hpp:14-16, tensor_io.cpp:12-152): magic "SAAPTNS" + version
// '1', u32 dtype (0 f32, 1 u64), u32 ndim (<= 8), ndim x u64 dims, row-major
// little-endian payload, nothing after it.  Error kinds and messages follow
// IoError (tensor_io.hpp:18-38); validation failures that the reference
// reports as std::invalid_argument (non-finite entries, non-unit centroids,
// an offset table that is not a prefix sum) return SAAP_ERR_INVALID_ARGUMENT.
// Host code only: no device work except the uploads of the loaded artifacts.
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "common.cuh"

namespace {

using saap_b200::set_error;

thread_local int g_io_kind = -1;

struct IoFail {
    int kind;
    std::string msg;
};
struct ArgFail {
    std::string msg;
};

enum : int { OpenFailed = 0, BadMagic, BadVersion, BadDtype, BadShape, Truncated };

template <typename F>
int io_guard(F&& f) {
    g_io_kind = -1;
    try {
        f();
        return SAAP_OK;
    } catch (const IoFail& e) {
        g_io_kind = e.kind;
        set_error(e.msg);
        return SAAP_ERR_IO;
    } catch (const ArgFail& e) {
        set_error(e.msg);
        return SAAP_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return SAAP_ERR_CUDA;
    }
}

constexpr char kMagic[7] = {'S', 'A', 'A', 'P', 'T', 'N', 'S'};
constexpr char kVersion = '1';
constexpr uint32_t kF32 = 0, kU64 = 1;

struct File {
    std::FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : path(p ? p : "") {
        if (!p) throw ArgFail{"artifact path: null argument"};
        f = std::fopen(p, mode);
        if (!f) throw IoFail{OpenFailed, "cannot open " + path + " (mode " + mode + ")"};
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void write(const void* p, size_t n) {
        if (n > 0 && std::fwrite(p, 1, n, f) != n) throw IoFail{OpenFailed, "short write to " + path};
    }
    void read(void* p, size_t n, const char* what) {
        if (n > 0 && std::fread(p, 1, n, f) != n)
            throw IoFail{Truncated, path + ": truncated while reading " + what};
    }
};

void write_header(File& f, uint32_t dtype, const std::vector<uint64_t>& dims) {
    f.write(kMagic, 7);
    f.write(&kVersion, 1);
    f.write(&dtype, 4);
    const uint32_t nd = (uint32_t)dims.size();
    f.write(&nd, 4);
    for (uint64_t d : dims) f.write(&d, 8);
}

std::vector<uint64_t> read_header(File& f, uint32_t expect) {
    char m[7];
    f.read(m, 7, "magic");
    if (std::memcmp(m, kMagic, 7) != 0) throw IoFail{BadMagic, f.path + ": bad magic bytes"};
    char v = 0;
    f.read(&v, 1, "version");
    if (v != kVersion)
        throw IoFail{BadVersion, f.path + ": unsupported format version '" + std::string(1, v) + "'"};
    uint32_t dt = 0;
    f.read(&dt, 4, "dtype");
    if (dt != expect)
        throw IoFail{BadDtype, f.path + ": dtype " + std::to_string(dt) + ", expected " +
                                       std::to_string(expect)};
    uint32_t nd = 0;
    f.read(&nd, 4, "ndim");
    if (nd > 8) throw IoFail{BadShape, f.path + ": implausible ndim " + std::to_string(nd)};
    std::vector<uint64_t> dims(nd);
    for (auto& d : dims) f.read(&d, 8, "dims");
    return dims;
}

void check_eof(File& f) {
    unsigned char c;
    if (std::fread(&c, 1, 1, f.f) == 1) throw IoFail{BadShape, f.path + ": trailing bytes after payload"};
}

std::string shape_str(uint64_t r, uint64_t c) {
    return std::to_string(r) + "x" + std::to_string(c);
}

// tensor_read (tensor_io.cpp:117-133) incl. TensorBlock::validate (tensor.cpp:20-30)
std::vector<float> read_f32(const char* path, uint64_t& rows, uint64_t& dim) {
    File f(path, "rb");
    auto dims = read_header(f, kF32);
    if (dims.size() != 2)
        throw IoFail{BadShape, f.path + ": expected 2-d tensor, got ndim " + std::to_string(dims.size())};
    rows = dims[0];
    dim = dims[1];
    std::vector<float> v(rows * dim);
    f.read(v.data(), v.size() * 4, "payload");
    check_eof(f);
    for (float x : v)
        if (!std::isfinite(x)) throw ArgFail{f.path + ": non-finite entry"};
    return v;
}

std::vector<uint64_t> read_u64(const char* path) {
    File f(path, "rb");
    auto dims = read_header(f, kU64);
    if (dims.size() != 1)
        throw IoFail{BadShape, f.path + ": expected 1-d sequence, got ndim " + std::to_string(dims.size())};
    std::vector<uint64_t> v(dims[0]);
    f.read(v.data(), v.size() * 8, "payload");
    check_eof(f);
    return v;
}

void write_f32(const char* path, const float* data, uint64_t rows, uint64_t dim) {
    if (rows * dim && !data) throw ArgFail{"tensor_write: null data"};
    File f(path, "wb");
    write_header(f, kF32, {rows, dim});
    f.write(data, rows * dim * 4);
}

void write_u64(const char* path, const uint64_t* v, uint64_t n) {
    if (n && !v) throw ArgFail{"u64_write: null data"};
    File f(path, "wb");
    write_header(f, kU64, {n});
    f.write(v, n * 8);
}

template <typename T>
void put(const std::vector<T>& v, T* out, uint64_t cap, const char* what) {
    if (!out) return;
    if (cap < v.size()) throw ArgFail{std::string(what) + ": output buffer too small"};
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
}

const char* const kQmNames[8] = {"w1", "b1", "bn_gamma", "bn_beta",
                                 "bn_run_mean", "bn_run_var", "w2", "b2"};

}  // namespace

extern "C" {

int saap_last_io_kind(void) { return g_io_kind; }

int saap_tensor_write(const char* path, const float* data, uint64_t rows, uint64_t dim) {
    return io_guard([&] { write_f32(path, data, rows, dim); });
}

int saap_tensor_read(const char* path, float* out, uint64_t cap, uint64_t* rows, uint64_t* dim) {
    return io_guard([&] {
        uint64_t r = 0, d = 0;
        auto v = read_f32(path, r, d);
        put(v, out, cap, "tensor_read");
        if (rows) *rows = r;
        if (dim) *dim = d;
    });
}

int saap_u64_write(const char* path, const uint64_t* v, uint64_t n) {
    return io_guard([&] { write_u64(path, v, n); });
}

int saap_u64_read(const char* path, uint64_t* out, uint64_t cap, uint64_t* n) {
    return io_guard([&] {
        auto v = read_u64(path);
        put(v, out, cap, "u64_read");
        if (n) *n = v.size();
    });
}

// partition_load (partition.cpp:265-276): f32 [C x d], every row unit norm
// within 1e-5 (norm in fp64, index order), then uploaded as a device partition.
int saap_partition_load(saap_ctx* ctx, const char* path, saap_partition** out) {
    std::vector<float> v;
    uint64_t C = 0, d = 0;
    int rc = io_guard([&] {
        if (!out) throw ArgFail{"partition_load: null argument"};
        v = read_f32(path, C, d);
        for (uint64_t c = 0; c < C; ++c) {
            double s = 0.0;
            for (uint64_t j = 0; j < d; ++j) s += (double)v[c * d + j] * (double)v[c * d + j];
            const double n = std::sqrt(s);
            if (std::abs(n - 1.0) > 1e-5)
                throw ArgFail{"partition_load: centroid " + std::to_string(c) +
                              " is not unit norm (" + std::to_string(n) + ")"};
        }
    });
    if (rc != SAAP_OK) return rc;
    return saap_partition_create(ctx, v.data(), C, d, out);
}

// ivf_load (partition.cpp:285-295).  off/idx may be NULL to query sizes.
int saap_ivf_load(const char* off_path, const char* idx_path, uint64_t* off, uint64_t off_cap,
                  uint64_t* n_off, uint64_t* idx, uint64_t idx_cap, uint64_t* n_idx) {
    return io_guard([&] {
        auto o = read_u64(off_path);
        auto i = read_u64(idx_path);
        bool sorted = true;
        for (size_t k = 1; k < o.size(); ++k) sorted &= o[k - 1] <= o[k];
        if (o.empty() || o.front() != 0 || o.back() != i.size() || !sorted)
            throw ArgFail{"ivf_load: offset table is not a valid prefix sum"};
        put(o, off, off_cap, "ivf_load");
        put(i, idx, idx_cap, "ivf_load");
        if (n_off) *n_off = o.size();
        if (n_idx) *n_idx = i.size();
    });
}

// qmodel_save / qmodel_load (qmodel.cpp:530-589): manifest.txt ("name rows
// cols" per line, checkpoint order) + one f32 tensor per parameter; the f32
// payload widens to fp64 on load (mat_from_tensor, qmodel.cpp:21-27).
int saap_qmodel_save(const char* dir, uint64_t d, uint64_t h, uint64_t C,
                     const double* const* params) {
    return io_guard([&] {
        if (!dir || !params) throw ArgFail{"qmodel_save: null argument"};
        ::mkdir(dir, 0777);  // create_directories for one level; existing is fine
        const std::string base(dir);
        const uint64_t shp[8][2] = {{d, h}, {1, h}, {1, h}, {1, h}, {1, h}, {1, h}, {h, C}, {1, C}};
        std::ofstream man(base + "/manifest.txt");
        if (!man) throw IoFail{OpenFailed, "cannot write " + base + "/manifest.txt"};
        for (int k = 0; k < 8; ++k) {
            if (!params[k]) throw ArgFail{"qmodel_save: null parameter"};
            man << kQmNames[k] << ' ' << shp[k][0] << ' ' << shp[k][1] << '\n';
            std::vector<float> t(shp[k][0] * shp[k][1]);
            for (size_t e = 0; e < t.size(); ++e) t[e] = (float)params[k][e];
            write_f32((base + "/" + kQmNames[k] + ".tensor").c_str(), t.data(), shp[k][0], shp[k][1]);
        }
        if (!man.flush()) throw IoFail{OpenFailed, "short write to " + base + "/manifest.txt"};
    });
}

// dims[3] = (d, h, C); params[8] receive the fp64 parameters in checkpoint
// order when non-NULL (caps are the element counts dims imply: pass NULL
// first to query dims).
int saap_qmodel_read(const char* dir, uint64_t* dims, double* const* params) {
    return io_guard([&] {
        if (!dir || !dims) throw ArgFail{"qmodel_load: null argument"};
        const std::string base(dir);
        std::ifstream man(base + "/manifest.txt");
        if (!man) throw IoFail{OpenFailed, "cannot read " + base + "/manifest.txt"};
        std::vector<std::vector<float>> t(8);
        uint64_t r[8] = {}, c[8] = {};
        std::string line;
        size_t slot = 0;
        while (std::getline(man, line)) {
            if (line.empty()) continue;
            std::istringstream ls(line);
            std::string name;
            uint64_t rows = 0, cols = 0;
            if (!(ls >> name >> rows >> cols)) throw IoFail{BadShape, "malformed manifest line: " + line};
            if (slot >= 8 || name != kQmNames[slot])
                throw IoFail{BadShape, "unexpected checkpoint entry '" + name + "' at slot " +
                                               std::to_string(slot)};
            t[slot] = read_f32((base + "/" + name + ".tensor").c_str(), r[slot], c[slot]);
            if (r[slot] != rows || c[slot] != cols)
                throw IoFail{BadShape, "manifest shape " + shape_str(rows, cols) +
                                               " disagrees with tensor " + shape_str(r[slot], c[slot]) +
                                               " for " + name};
            ++slot;
        }
        if (slot != 8)
            throw IoFail{Truncated, "checkpoint manifest lists " + std::to_string(slot) + " of 8 tensors"};
        // w1 [d x h], b1 [1 x h], w2 [h x C], b2 [1 x C]
        if (c[0] != c[1] || c[0] != r[6] || c[6] != c[7])
            throw IoFail{BadShape, "checkpoint tensor shapes are inconsistent"};
        dims[0] = r[0];
        dims[1] = c[0];
        dims[2] = c[6];
        if (params)
            for (int k = 0; k < 8; ++k)
                if (params[k])
                    for (size_t e = 0; e < t[k].size(); ++e) params[k][e] = (double)t[k][e];
    });
}

int saap_qmodel_load(saap_ctx* ctx, const char* dir, saap_qmodel** out) {
    uint64_t dims[3] = {};
    int rc = saap_qmodel_read(dir, dims, nullptr);
    if (rc != SAAP_OK) return rc;
    const uint64_t d = dims[0], h = dims[1], C = dims[2];
    std::vector<double> w1(d * h), w2(h * C), b2(C), v[5];
    for (auto& x : v) x.resize(h);
    double* const ps[8] = {w1.data(), v[0].data(), v[1].data(), v[2].data(),
                           v[3].data(), v[4].data(), w2.data(), b2.data()};
    rc = saap_qmodel_read(dir, dims, ps);
    if (rc != SAAP_OK) return rc;
    return saap_qmodel_create(ctx, d, h, C, ps[0], ps[1], ps[2], ps[3], ps[4], ps[5], ps[6], ps[7],
                              out);
}

}  // extern "C"
