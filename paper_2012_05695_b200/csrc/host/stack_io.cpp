// Frame stacks and frame sources (ingest boundary). Behaviour follows the reference
// `proj/core/src/image_stack.cpp:162-247` (raw_stack) and `frame_source.cpp:15-102`.
#include "ddm/errors.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/image_stack.hpp"
#include "json_lite.hpp"

#include <algorithm>
#include <cstdio>
#include <cctype>
#include <cstring>
#include <fstream>

#include <fcntl.h>
#include <unistd.h>

namespace fs = std::filesystem;

namespace ddm {

void ImageStack::validate() const {
    if (width < 1 || height < 1 || frames < 1)
        throw InputError("image stack: dimensions must be positive");
    if (pixels.size() != std::size_t(pixels_per_frame()) * std::size_t(frames))
        throw InputError("image stack: payload size does not match dimensions");
}

StackFormat parse_stack_format(const std::string& name) {
    if (name == "pgm_dir") return StackFormat::PgmDir;
    if (name == "raw_stack") return StackFormat::RawStack;
    throw InputError("unknown stack format '" + name + "'");
}

std::string to_string(StackFormat format) {
    return format == StackFormat::PgmDir ? "pgm_dir" : "raw_stack";
}

namespace {

struct RawHeader {
    int width = 0, height = 0, frames = 0;
    double frame_interval = 1.0;
    std::int64_t payload_offset = 0;
};

RawHeader read_raw_header(std::ifstream& in, const fs::path& path) {
    std::string line;
    if (!std::getline(in, line)) throw InputError("raw_stack " + path.string() + ": missing header line");
    RawHeader h;
    h.payload_offset = std::int64_t(line.size()) + 1;
    try {
        const json::Value j = json::parse(line);
        h.width = int(j.at("width").as_int());
        h.height = int(j.at("height").as_int());
        h.frames = int(j.at("frames").as_int());
        if (j.at("dtype").as_string() != "u16le")
            throw InputError("raw_stack " + path.string() + ": unsupported dtype");
        if (j.has("frame_interval")) h.frame_interval = j.at("frame_interval").as_double();
    } catch (const InputError&) {
        throw;
    } catch (const std::exception& e) {
        throw InputError("raw_stack " + path.string() + ": bad header: " + e.what());
    }
    if (h.width < 1 || h.height < 1 || h.frames < 1)
        throw InputError("raw_stack " + path.string() + ": dimensions must be positive");
    return h;
}

}  // namespace

ImageStack load_stack(const fs::path& path, StackFormat format) {
    if (format == StackFormat::PgmDir) {
        const PgmDirSource src(path);
        ImageStack st;
        st.width = src.width();
        st.height = src.height();
        st.frames = src.frames();
        st.pixels.resize(std::size_t(st.width) * st.height * st.frames);
        for (int n = 0; n < st.frames; ++n) src.read_frame(n, st.frame(n));
        return st;
    }
    if (!fs::exists(path)) throw IoError("path does not exist: " + path.string());
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path.string());
    const RawHeader h = read_raw_header(in, path);
    ImageStack st;
    st.width = h.width;
    st.height = h.height;
    st.frames = h.frames;
    st.frame_interval = h.frame_interval;
    st.pixels.resize(std::size_t(h.width) * h.height * h.frames);
    const std::int64_t bytes = std::int64_t(st.pixels.size()) * 2;
    std::vector<unsigned char> raw(static_cast<std::size_t>(bytes));
    in.read(reinterpret_cast<char*>(raw.data()), bytes);
    if (in.gcount() != bytes) throw InputError("raw_stack " + path.string() + ": truncated payload");
    for (std::size_t i = 0; i < st.pixels.size(); ++i)
        st.pixels[i] = std::uint16_t(raw[2 * i] | (raw[2 * i + 1] << 8));
    return st;
}

void write_pgm(std::span<const std::uint16_t> frame, int width, int height, const fs::path& path) {
    if (width < 1 || height < 1 || std::size_t(width) * std::size_t(height) != frame.size())
        throw InputError("write_pgm: frame size does not match dimensions");
    char head[64];
    const int hn = std::snprintf(head, sizeof head, "P5\n%d %d\n65535\n", width, height);
    std::vector<unsigned char> bytes(std::size_t(hn) + 2 * frame.size());
    std::memcpy(bytes.data(), head, std::size_t(hn));
    unsigned char* px = bytes.data() + hn;
    for (const std::uint16_t v : frame) {   // big-endian samples (maxval > 255)
        *px++ = static_cast<unsigned char>(v >> 8);
        *px++ = static_cast<unsigned char>(v & 0xFFu);
    }
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot create " + path.string());
    out.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
    if (!out) throw IoError("short write to " + path.string());
}

void write_raw_stack(const ImageStack& stack, const fs::path& path) {
    // one JSON header line, then the samples as u16 little-endian (`image_stack.cpp:223-247`)
    stack.validate();
    json::Value h = json::Value::object();
    h.obj["width"] = json::Value::integer(stack.width);
    h.obj["height"] = json::Value::integer(stack.height);
    h.obj["frames"] = json::Value::integer(stack.frames);
    h.obj["dtype"] = json::Value::string("u16le");
    h.obj["frame_interval"] = json::Value::number(stack.frame_interval);
    std::string bytes = json::dump(h);
    bytes.push_back('\n');
    const std::size_t head = bytes.size();
    bytes.resize(head + 2 * stack.pixels.size());
    unsigned char* dst = reinterpret_cast<unsigned char*>(bytes.data()) + head;
    for (const std::uint16_t px : stack.pixels) {   // explicit LE, whatever the host order
        *dst++ = static_cast<unsigned char>(px);
        *dst++ = static_cast<unsigned char>(px >> 8);
    }
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path.string() + " for writing");
    const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    if (std::fclose(f) != 0 || !ok) throw IoError("write failed for " + path.string());
}

MemoryFrameSource::MemoryFrameSource(ImageStack stack) : stack_(std::move(stack)) {
    stack_.validate();
}

void MemoryFrameSource::read_frame(int n, std::span<std::uint16_t> out) const {
    const auto f = stack_.frame(n);
    std::memcpy(out.data(), f.data(), f.size_bytes());
}

ViewFrameSource::ViewFrameSource(const std::uint16_t* pixels, int width, int height, int frames,
                                 double frame_interval)
    : px_(pixels), w_(width), h_(height), n_(frames), dt_(frame_interval) {
    if (!pixels || width < 1 || height < 1 || frames < 1)
        throw InputError("frame view: dimensions must be positive and pixels non-null");
}

void ViewFrameSource::read_frame(int n, std::span<std::uint16_t> out) const {
    std::memcpy(out.data(), px_ + std::size_t(n) * std::size_t(pixels_per_frame()),
                std::size_t(pixels_per_frame()) * 2);
}

RawStackFileSource::RawStackFileSource(const fs::path& path) : path_(path) {
    if (!fs::exists(path)) throw IoError("path does not exist: " + path.string());
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path.string());
    const RawHeader h = read_raw_header(in, path);
    width_ = h.width;
    height_ = h.height;
    frames_ = h.frames;
    frame_interval_ = h.frame_interval;
    payload_offset_ = h.payload_offset;
    const std::int64_t size = std::int64_t(fs::file_size(path));
    if (size < payload_offset_ + 2 * pixels_per_frame() * frames_)
        throw InputError("raw_stack " + path.string() + ": truncated payload");
    fd_ = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd_ < 0) throw IoError("cannot open " + path.string());
}

RawStackFileSource::~RawStackFileSource() {
    if (fd_ >= 0) ::close(fd_);
}

void RawStackFileSource::read_frames(int first, int count, std::uint16_t* out) const {
    // one positioned read: no shared file offset, so concurrent calls need no lock (the
    // reference serialises seek + read behind a mutex, `frame_source.cpp:64-78`)
    const std::int64_t bytes = 2 * pixels_per_frame() * count;
    std::int64_t done = 0;
    auto* dst = reinterpret_cast<char*>(out);
    while (done < bytes) {
        const ssize_t r = ::pread(fd_, dst + done, std::size_t(bytes - done),
                                  off_t(payload_offset_ + std::int64_t(first) * 2 * pixels_per_frame() + done));
        if (r <= 0) throw IoError("raw_stack " + path_.string() + ": short read");
        done += r;
    }
    // payload is little endian; this build targets little-endian hosts (as the reference)
}

void RawStackFileSource::read_frame(int n, std::span<std::uint16_t> out) const {
    read_frames(n, 1, out.data());
}

namespace {

// PGM header token: whitespace and '#' comments skipped (`image_stack.cpp:20-39`)
std::string pgm_token(std::istream& in) {
    int c = in.get();
    while (c != EOF) {
        if (c == '#') {
            while (c != EOF && c != '\n') c = in.get();
        } else if (!std::isspace(c)) {
            break;
        }
        c = in.get();
    }
    std::string tok;
    while (c != EOF && !std::isspace(c)) {
        tok.push_back(char(c));
        c = in.get();
    }
    return tok;
}

int pgm_int(const std::string& tok, const char* what, const fs::path& f) {
    std::size_t pos = 0;
    long v = 0;
    try {
        v = std::stol(tok, &pos);
    } catch (const std::exception&) {
        pos = 0;
    }
    if (pos != tok.size() || tok.empty() || v < 1)
        throw InputError("pgm " + f.string() + ": bad " + what + " '" + tok + "'");
    return int(v);
}

// reads one P5 / maxval 65535 frame (big-endian samples) into out (or only the size)
void read_pgm(const fs::path& f, int& w, int& h, std::uint16_t* out, std::size_t capacity) {
    std::ifstream in(f, std::ios::binary);
    if (!in) throw IoError("cannot open " + f.string());
    const std::string magic = pgm_token(in);
    if (magic != "P5") throw InputError("pgm " + f.string() + ": not a binary PGM (magic '" + magic + "')");
    w = pgm_int(pgm_token(in), "width", f);
    h = pgm_int(pgm_token(in), "height", f);
    const std::string maxval = pgm_token(in);
    if (maxval != "65535") throw InputError("pgm " + f.string() + ": maxval must be 65535, got '" + maxval + "'");
    if (!out) return;
    const std::size_t count = std::size_t(w) * std::size_t(h);
    if (count > capacity) throw InputError("pgm " + f.string() + ": frame dimensions differ from the first frame");
    in.read(reinterpret_cast<char*>(out), std::streamsize(count * 2));
    if (std::size_t(in.gcount()) != count * 2) throw InputError("pgm " + f.string() + ": truncated payload");
    for (std::size_t i = 0; i < count; ++i) out[i] = std::uint16_t((out[i] >> 8) | (out[i] << 8));
}

std::vector<fs::path> pgm_files(const fs::path& dir) {
    if (!fs::exists(dir)) throw IoError("path does not exist: " + dir.string());
    if (!fs::is_directory(dir)) throw InputError("pgm_dir input is not a directory: " + dir.string());
    std::vector<fs::path> files;
    for (const auto& e : fs::directory_iterator(dir))
        if (e.is_regular_file() && e.path().extension() == ".pgm") files.push_back(e.path());
    if (files.empty()) throw InputError("no *.pgm files in " + dir.string());
    std::sort(files.begin(), files.end(),
              [](const fs::path& a, const fs::path& b) { return a.filename().string() < b.filename().string(); });
    return files;
}

}  // namespace

PgmDirSource::PgmDirSource(const fs::path& dir) : files_(pgm_files(dir)) {
    read_pgm(files_.front(), width_, height_, nullptr, 0);
}

void PgmDirSource::read_frame(int n, std::span<std::uint16_t> out) const {
    int w = 0, h = 0;
    read_pgm(files_[std::size_t(n)], w, h, out.data(), out.size());
    if (w != width_ || h != height_)
        throw InputError("pgm " + files_[std::size_t(n)].string() + ": frame dimensions differ from the first frame");
}

std::unique_ptr<FrameSource> open_frame_source(const fs::path& path, StackFormat format) {
    if (format == StackFormat::PgmDir) return std::make_unique<PgmDirSource>(path);
    return std::make_unique<RawStackFileSource>(path);
}

}  // namespace ddm
