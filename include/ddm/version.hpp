// ddm-b200: library and on-disk format versions, same names as the reference
// (`proj/core/include/ddm/version.hpp`). The on-disk formats (raw stack, map files,
// partials, manifests) are the reference's, byte for byte, so kFormatVersion matches it.
#ifndef DDM_VERSION_HPP
#define DDM_VERSION_HPP

namespace ddm {

inline constexpr const char* kVersion = "0.1.0";
inline constexpr int kFormatVersion = 1;

}  // namespace ddm

#endif
