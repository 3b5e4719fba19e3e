// Frame stacks and frame sources (ingest boundary). Behaviour follows the reference
// `proj/core/src/image_stack.cpp:162-247` (raw_stack) and `frame_source.cpp:15-102`.
#include "ddm/errors.hpp"
#include "ddm/frame_source.hpp"
#include "ddm/image_stack.hpp"
#include "json_lite.hpp"

#include <cstring>
#include <fstream>

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
    if (format != StackFormat::RawStack)
        throw InputError("pgm_dir stacks are not supported by the b200 build; convert to raw_stack");
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

void write_raw_stack(const ImageStack& stack, const fs::path& path) {
    stack.validate();
    json::Value h = json::Value::object();
    h.obj["width"] = json::Value::integer(stack.width);
    h.obj["height"] = json::Value::integer(stack.height);
    h.obj["frames"] = json::Value::integer(stack.frames);
    h.obj["dtype"] = json::Value::string("u16le");
    h.obj["frame_interval"] = json::Value::number(stack.frame_interval);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot open " + path.string() + " for writing");
    out << json::dump(h) << '\n';
    std::vector<unsigned char> raw(stack.pixels.size() * 2);
    for (std::size_t i = 0; i < stack.pixels.size(); ++i) {
        raw[2 * i] = (unsigned char)(stack.pixels[i] & 0xFF);
        raw[2 * i + 1] = (unsigned char)(stack.pixels[i] >> 8);
    }
    out.write(reinterpret_cast<const char*>(raw.data()), std::streamsize(raw.size()));
    if (!out) throw IoError("write failed for " + path.string());
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
    file_.open(path, std::ios::binary);
    if (!file_) throw IoError("cannot open " + path.string());
    const RawHeader h = read_raw_header(file_, path);
    width_ = h.width;
    height_ = h.height;
    frames_ = h.frames;
    frame_interval_ = h.frame_interval;
    payload_offset_ = h.payload_offset;
    file_.seekg(0, std::ios::end);
    const std::int64_t size = std::int64_t(file_.tellg());
    if (size < payload_offset_ + 2 * pixels_per_frame() * frames_)
        throw InputError("raw_stack " + path.string() + ": truncated payload");
}

void RawStackFileSource::read_frames(int first, int count, std::uint16_t* out) const {
    const std::int64_t bytes = 2 * pixels_per_frame() * count;
    {
        std::lock_guard<std::mutex> lock(mutex_);
        file_.clear();
        file_.seekg(payload_offset_ + std::int64_t(first) * 2 * pixels_per_frame());
        file_.read(reinterpret_cast<char*>(out), bytes);
        if (file_.gcount() != bytes) throw IoError("raw_stack " + path_.string() + ": short read");
    }
    // payload is little endian; this build targets little-endian hosts (as the reference)
}

void RawStackFileSource::read_frame(int n, std::span<std::uint16_t> out) const {
    read_frames(n, 1, out.data());
}

std::unique_ptr<FrameSource> open_frame_source(const fs::path& path, StackFormat format) {
    if (format == StackFormat::PgmDir)
        throw InputError("pgm_dir stacks are not supported by the b200 build; convert to raw_stack");
    return std::make_unique<RawStackFileSource>(path);
}

}  // namespace ddm
