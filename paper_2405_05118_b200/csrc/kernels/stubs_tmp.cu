#include "../plan.hpp"
namespace mdhb {
std::unique_ptr<Routine> make_prl(const Problem&, const Config*, Config*) { return nullptr; }


}
